# GPU-box check: build, microbench, smoke, gpu tests, bench (+ variants).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 120 python -c "import paper_2002_08233_b200 as bl, json; print(json.dumps(bl.bl_microbench()))" > gpurun_out/microbench.log 2>&1; echo mb rc=$?
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
fi
if [ "${SKIP_BENCH:-0}" != "1" ]; then
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 10 --prof > gpurun_out/bench.log 2>&1; echo bench rc=$?
fi
for v in ${BENCH_VARIANTS:-}; do
  env $(echo $v | tr ',' ' ') timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --prof > gpurun_out/bench_$v.log 2>&1; echo "bench $v rc=$?"
done
