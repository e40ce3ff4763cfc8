# A/B of an env-selected kernel option on the GPU box: build, a guarded parity
# subset, then bench.py with and without the option, interleaved.
#   AB_ENV="BL_ASYNC=0" AB_CONFIGS="C5 C4" AB_K="drivers or async" bash scripts/gpu_ab.sh
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
if [ -n "${AB_K:-}" ]; then
  timeout -s KILL ${AB_TEST_TIMEOUT:-600} python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$AB_K" > gpurun_out/ab_tests.log 2>&1
  rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/ab_tests.log
  [ $rc -ne 0 ] && exit 1
fi
for c in ${AB_CONFIGS:-C5}; do
  for rep in ${AB_REPS:-1 2}; do
    timeout -s KILL 300 python bench.py --config $c --steps ${AB_STEPS:-3} --warmup 3 --no-cpu-baseline --no-bh ${AB_ARGS:-} > gpurun_out/ab_${c}_new_$rep.log 2>&1; echo "$c new rc=$?"
    env $AB_ENV timeout -s KILL 300 python bench.py --config $c --steps ${AB_STEPS:-3} --warmup 3 --no-cpu-baseline --no-bh ${AB_ARGS:-} > gpurun_out/ab_${c}_old_$rep.log 2>&1; echo "$c old rc=$?"
  done
done
python - <<'PY'
import glob, json, re
for f in sorted(glob.glob("gpurun_out/ab_*_*_*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            print(f, d.get("value"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), d.get("iters_per_sec"))
PY
