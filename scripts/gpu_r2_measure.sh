#!/bin/bash
# Round-2 measurement call: smoke, pytest -m gpu (parity margins logged),
# the default bench line, the ncu launch list of the same bench command and
# one ncu --set full capture of the C5 bench-shaped layout launch.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2m
O=gpurun_out/r2m
rm -f $O/parity_margins.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
if [ "${SKIP_TESTS:-0}" != "1" ]; then
BL_PARITY_LOG=$PWD/$O/parity_margins.jsonl timeout 2400 python -m pytest tests -m gpu -q \
  --timeout 900 ${PYTEST_ARGS:-} > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest_gpu.log
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > $O/bench.log 2>&1; rc=$?; echo bench rc=$rc
tail -c 1500 $O/bench.log
if [ $rc = 0 ] && [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --cpu-seconds 1 > $O/ncu_launches.log 2>&1; echo ncu-launch rc=$?
  CMD="python scripts/profile_run.py --config C5 --iters 50"
  $CMD > $O/plain_full.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bl_layout_kernel -c 1 \
      -o $O/prof_C5 $CMD > $O/ncu_full.log 2>&1; echo ncu-full rc=$?
fi
