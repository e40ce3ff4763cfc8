# Round-end evidence: build, smoke, full GPU tests, default bench line,
# every config, ncu launch list + full capture of the bench-shaped C5 launch.
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final/build.log 2>&1; echo build rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke rc=$?
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/final/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/final/bench_main.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final/bench_ref.log 2>&1; echo ref rc=$?
for c in C1 C2 C3b64 C3b256 C3b1024 C4 C6; do
  timeout -s KILL 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final/bench_$c.log 2>&1; echo "$c rc=$?"
done
timeout -s KILL 300 python bench.py --r -2 --steps 3 --warmup 3 --no-cpu-baseline --no-bh > gpurun_out/final/bench_C5_r-2.log 2>&1; echo r2 rc=$?
python scripts/profile_run.py --config C5 --iters 50 > gpurun_out/final/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bl_layout_kernel -c 1 \
    -o gpurun_out/final/prof_C5_50it -f python scripts/profile_run.py --config C5 --iters 50 > gpurun_out/final/ncu_full.log 2>&1; echo ncu rc=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final/ncu_launch.log 2>&1; echo launches rc=$?
