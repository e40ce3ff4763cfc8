# ncu --set full of one layout launch (default: the bench's C5 50-iteration
# launch), after the same command has exited 0 without ncu.
mkdir -p gpurun_out
CMD="python scripts/profile_run.py --config ${CFG:-C5} --iters ${ITERS:-50}"
$CMD > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bl_layout_kernel -c 1 \
    -o gpurun_out/prof_${TAG:-r1} $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
