# ncu capture of the persistent kernel (short C5 run) + launch list of bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python scripts/profile_run.py --config ${CFG:-C5} --iters ${ITERS:-2}"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bl_layout_kernel -c 1 \
    -o gpurun_out/prof_${TAG:-r1} $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
if [ "${LAUNCHES:-1}" = "1" ]; then
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
fi
