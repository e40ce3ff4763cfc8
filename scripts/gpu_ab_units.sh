python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "async or drivers or C5" > gpurun_out/t_async.log 2>&1; echo t=$?; tail -1 gpurun_out/t_async.log
mkdir -p gpurun_out/variants
for rep in 1 2; do
for c in C5 C6; do
  timeout -s KILL 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-bh > gpurun_out/variants/${c}_new_$rep.log 2>&1
  BL_RED_CAP=16384 BL_NSUB=6 BL_GUIDED=1 timeout -s KILL 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-bh > gpurun_out/variants/${c}_old_$rep.log 2>&1
done
timeout -s KILL 300 python bench.py --config C5 --r -2 --steps 2 --warmup 3 --no-cpu-baseline --no-bh > gpurun_out/variants/C5r2_new_$rep.log 2>&1
BL_RED_CAP=16384 BL_NSUB=6 BL_GUIDED=1 timeout -s KILL 300 python bench.py --config C5 --r -2 --steps 2 --warmup 3 --no-cpu-baseline --no-bh > gpurun_out/variants/C5r2_old_$rep.log 2>&1
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/variants/*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); r = d["roofline"]
            print(f"{f.split('/')[-1][:-4]:20s} {d['value']:.4e} frac {r['frac']:.4f} {r['kernel'].split(' ')[0]} {r.get('driver')}")
PY
