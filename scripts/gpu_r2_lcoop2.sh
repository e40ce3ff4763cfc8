#!/bin/bash
cd "$(dirname "$0")/.."
for c in ${CFGS:-C2 C3b256 C4}; do
  for m in ${MODES:-auto 0 1}; do
    if [ $m = auto ]; then unset BL_LCOOP; else export BL_LCOOP=$m; fi
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-bh --no-shuffle --no-metrics --no-cpu-baseline --latency-configs "" 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$c BL_LCOOP=$m', 'it/s %.1f' % d['iters_per_sec'], 'ms/step %.3f' % d['ms_per_step'])"
  done
done
