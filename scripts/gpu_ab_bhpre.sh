# BH per-iteration precomputation: GPU BH tests, then bench with / without
mkdir -p gpurun_out/bhpre
timeout -s KILL 900 python -m pytest tests/test_gpu_bh.py -m gpu -q -x > gpurun_out/bhpre/t_bh.log 2>&1; echo t=$?; tail -2 gpurun_out/bhpre/t_bh.log
for c in ${CFGS:-C5 C4 C2 C3b256 C6}; do
  timeout -s KILL 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bhpre/${c}_pre.log 2>&1
  BL_BH_PRE=0 timeout -s KILL 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bhpre/${c}_old.log 2>&1
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/bhpre/*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); b = d.get("bh", {})
            print(f"{f.split('/')[-1][:-4]:16s} exact it/s {d['iters_per_sec']:.1f}  BH it/s {b.get('iters_per_sec',0):.1f} x{b.get('speedup_vs_exact',0):.2f} visits/step {b.get('visits_per_step')}")
PY
