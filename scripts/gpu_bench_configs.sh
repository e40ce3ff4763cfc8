python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_models.py -m gpu -q -x > gpurun_out/t_b8.log 2>&1; echo t=$?; tail -2 gpurun_out/t_b8.log
mkdir -p gpurun_out/variants
for c in C5 C4 C2 C3b256 C3b1024; do
  timeout -s KILL 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-bh > gpurun_out/variants/${c}_b8.log 2>&1
done
timeout 300 python scripts/batch_times.py --config C4 > gpurun_out/bt_C4_b8.json 2>&1
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/variants/*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); r = d["roofline"]
            print(f"{f.split('/')[-1][:-4]:20s} {d['value']:.4e} frac {r['frac']:.4f} it/s {d['iters_per_sec']:.1f} {r.get('driver')}")
PY
