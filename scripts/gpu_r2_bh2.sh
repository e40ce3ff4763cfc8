#!/bin/bash
# BatchLayoutBH leaf-list capacity A/B (libbl_lcap*.so built with -DBH_LCAP=...)
cd "$(dirname "$0")/.."
O=gpurun_out/r2bh2; mkdir -p $O
for L in ${LIBS:-libbl libbl_lcap64 libbl_lcap128}; do
  for c in ${CFGS:-C5 C4 C3b256}; do
    BL_LIBRARY=$PWD/paper_2002_08233_b200/$L.so timeout -s KILL 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-shuffle --no-metrics --latency-configs "" > $O/${c}_$L.log 2>&1
  done
  BL_LIBRARY=$PWD/paper_2002_08233_b200/$L.so BL_PROFILE=1 timeout 300 python scripts/profile_bh.py --config C5 > $O/profile_C5_$L.json 2>&1; tail -1 $O/profile_C5_$L.json
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/r2bh2/C*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); b = d.get("bh", {})
            print(f"{f.split('/')[-1][:-4]:24s} BH it/s {b.get('iters_per_sec',0):.1f} x{b.get('speedup_vs_exact',0):.2f} ms/step {b.get('ms_per_step')}")
PY
