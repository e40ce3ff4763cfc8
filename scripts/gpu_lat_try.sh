mkdir -p gpurun_out/lat
timeout 300 python scripts/latency_sweep.py --configs C2,C3b256,C3b1024,C4 --variants ";LAT=1" --iters 20 > gpurun_out/lat/sweep.jsonl 2>gpurun_out/lat/err.txt; echo rc=$?
python -c "
import json
for l in open('gpurun_out/lat/sweep.jsonl'):
    d=json.loads(l); print(d['config'], d['driver'], round(d['us_per_batch'],3), d.get('vs_default_1it'))"
tail -3 gpurun_out/lat/err.txt
for c in C2:200 C4:50; do cfg=${c%%:*}; it=${c##*:}
BL_LAT=1 BL_PROFILE=1 BL_LIBRARY=$PWD/paper_2002_08233_b200/libbl_ts.so timeout 120 python scripts/async_profile.py --config $cfg --iters $it > gpurun_out/lat/ts_$cfg.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/lat/ts_$cfg.json')); print('$cfg', json.dumps(d.get('cta0_timeline_us_per_batch')))" 2>&1 | tail -2
done
BL_LAT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "one_iteration or one_batch or max_batches or tol or fuzz_shapes_one" > gpurun_out/lat/pytest.log 2>&1; tail -4 gpurun_out/lat/pytest.log
