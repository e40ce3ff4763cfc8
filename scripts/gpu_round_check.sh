mkdir -p gpurun_out
SKIP_BENCH=1 bash scripts/gpu_check.sh
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_main.log 2>&1; echo bench rc=$?
AB_ENV="BL_ASYNC=0" AB_CONFIGS="C6" AB_REPS="1" bash scripts/gpu_ab.sh
mkdir -p gpurun_out/r2; AB_ENV="BL_ASYNC=0" AB_CONFIGS="C5" AB_REPS="1" AB_ARGS="--r -2" bash scripts/gpu_ab.sh > gpurun_out/r2/ab.txt; cat gpurun_out/r2/ab.txt | tail -3
