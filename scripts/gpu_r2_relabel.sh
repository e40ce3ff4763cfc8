#!/bin/bash
# Batch randomisation by relabelling: parity tests of both modes, the checked
# build, and the cost of the two modes per config.
cd "$(dirname "$0")/.."
O=gpurun_out/r2rl; mkdir -p $O
timeout 1500 python -m pytest ${PYTEST_FILES:-tests/test_gpu_shuffle.py tests/test_gpu_checked.py} -m gpu -q --timeout 900 -s ${PYTEST_ARGS:-} > $O/pytest.log 2>&1; echo pytest rc=$?
grep -a "iteration .: median\|passed\|failed\|FAILED" $O/pytest.log | tail -15
if [ "${SKIP_COST:-0}" != "1" ]; then
timeout 900 python scripts/shuffle_cost.py ${COST_CONFIGS:-} > $O/shuffle_cost.jsonl 2> $O/shuffle_cost.err; echo cost rc=$?
cat $O/shuffle_cost.jsonl; tail -5 $O/shuffle_cost.err
fi
