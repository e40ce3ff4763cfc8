# Same-box A/B of two libbl builds on the BatchLayoutBH secondary line
mkdir -p gpurun_out/abbh
A=$(pwd)/paper_2002_08233_b200/libbl_A.so
timeout -s KILL 900 python -m pytest tests/test_gpu_bh.py -m gpu -q -x > gpurun_out/abbh/t_bh.log 2>&1; echo t=$?; tail -1 gpurun_out/abbh/t_bh.log
for c in ${CFGS:-C5 C4 C2}; do
  BL_LIBRARY=$A timeout -s KILL 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/abbh/${c}_A.log 2>&1
  timeout -s KILL 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/abbh/${c}_B.log 2>&1
done
timeout 300 python scripts/profile_bh.py --config C5 --iters 3 > gpurun_out/abbh/profile_bh_C5.json 2>&1
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/abbh/*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); b = d.get("bh", {})
            print(f"{f.split('/')[-1][:-4]:10s} BH it/s {b.get('iters_per_sec',0):.1f} x{b.get('speedup_vs_exact',0):.2f}")
PY
cat gpurun_out/abbh/profile_bh_C5.json
