#!/bin/bash
# BatchLayoutBH with the batch inputs prefetched across the grid barrier:
# BH tests, then it/s with / without (BL_BH_PRE2) per config.
cd "$(dirname "$0")/.."
O=gpurun_out/r2bh; mkdir -p $O
timeout -s KILL 1200 python -m pytest tests/test_gpu_bh.py -m gpu -q > $O/t_bh.log 2>&1; echo t=$?; tail -4 $O/t_bh.log
for c in ${CFGS:-C5 C4 C2 C3b256}; do
  for m in 1 0; do
    BL_BH_PRE2=$m timeout -s KILL 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-shuffle --no-metrics > $O/${c}_pre2_$m.log 2>&1
  done
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/r2bh/*_pre2_*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); b = d.get("bh", {})
            print(f"{f.split('/')[-1][:-4]:16s} exact it/s {d['iters_per_sec']:.1f}  BH it/s {b.get('iters_per_sec',0):.1f} x{b.get('speedup_vs_exact',0):.2f} ms/step {b.get('ms_per_step')}")
PY
BL_PROFILE=1 timeout 300 python scripts/profile_bh.py --config C5 > $O/profile_C5.json 2>&1; tail -3 $O/profile_C5.json
