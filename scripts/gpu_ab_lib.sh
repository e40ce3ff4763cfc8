# Same-box A/B of two builds of libbl (BL_LIBRARY=libbl_A.so vs the in-tree
# libbl.so), interleaved, bench.py per config.  No rebuild on the box.
mkdir -p gpurun_out/ablib
A=$(pwd)/paper_2002_08233_b200/libbl_A.so
for rep in ${AB_REPS:-1 2}; do
  for c in ${AB_CONFIGS:-C2 C4 C3b256 C5}; do
    BL_LIBRARY=$A timeout -s KILL 300 python bench.py --config $c --steps ${AB_STEPS:-2} --warmup 3 --no-cpu-baseline --no-bh ${AB_ARGS:-} > gpurun_out/ablib/${c}_A_$rep.log 2>&1
    timeout -s KILL 300 python bench.py --config $c --steps ${AB_STEPS:-2} --warmup 3 --no-cpu-baseline --no-bh ${AB_ARGS:-} > gpurun_out/ablib/${c}_B_$rep.log 2>&1
  done
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/ablib/*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); r = d["roofline"]
            print(f"{f.split('/')[-1][:-4]:16s} {d['value']:.4e} frac {r['frac']:.4f} it/s {d['iters_per_sec']:.1f} {r.get('driver')}")
PY
