# bench.py C5 under a list of env variants (comma-separated VAR=val), one line each
mkdir -p gpurun_out/variants
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
for v in ${VARIANTS:-default}; do
  e=$(echo $v | tr ',' ' '); [ "$v" = "default" ] && e=""
  env $e timeout -s KILL 300 python bench.py --config ${CFG:-C5} --steps ${STEPS:-2} --warmup 3 --no-cpu-baseline --no-bh > gpurun_out/variants/$v.log 2>&1; echo "$v rc=$?"
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/variants/*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); r = d["roofline"]
            print(f"{f.split('/')[-1][:-4]:40s} {d['value']:.4e} frac {r['frac']:.4f} {r['kernel'].split(' ')[0]} {r.get('driver')}")
PY
