set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 120 python -c "
import paper_2002_08233_b200 as bl, json
print(json.dumps(bl.bl_microbench()))
" > gpurun_out/microbench.log 2>&1; echo mb rc=$?
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/*.log
