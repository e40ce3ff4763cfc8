# bench.py on every config (parity configs too), one JSON line each
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in ${CONFIGS:-C1 C2 C3b64 C3b256 C3b1024 C4 C5}; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_cfg_$c.log 2>&1; echo "$c rc=$?"
done
