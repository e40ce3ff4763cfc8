#!/bin/bash
# Round-2 GPU-box check (libbl.so is built here and travels with the snapshot):
# smoke, pytest -m gpu with the parity-margin log, the default bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/parity_margins.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
if [ "${SKIP_TESTS:-0}" != "1" ]; then
BL_PARITY_LOG=$PWD/gpurun_out/parity_margins.jsonl timeout 1500 python -m pytest tests -m gpu -q \
  --timeout 900 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
fi
if [ "${SKIP_BENCH:-0}" != "1" ]; then
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -c 3000 gpurun_out/bench.log
fi
