#!/bin/bash
# Cooperative long-row walk of the latency driver: parity / checked tests, then A/B.
cd "$(dirname "$0")/.."
O=gpurun_out/r2lc; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py tests/test_gpu_shuffle.py -m gpu -q --timeout 900 > $O/pytest.log 2>&1; echo pytest rc=$?
grep -a "passed\|failed\|FAILED" $O/pytest.log | tail -8
for m in 1 0; do
  echo "BL_LCOOP=$m"
  BL_LCOOP=$m timeout 600 python scripts/shuffle_cost.py C2 C4 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config'], 'seq ms/iter %.4f' % d['ms_per_iter_sequential'], 'relabel %.4f' % d['ms_per_iter_relabel'])"
done
