#!/bin/bash
# Round-2 GPU call E: fence / poll A/B (same box), the update-task overlap,
# the new standalone a5 kernel, gpu tests, bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2e
L=paper_2002_08233_b200
CF=C2,C3b256,C4,C3b1024
for lib in libbl libbl_f1 libbl_f2 libbl_a; do
  BL_LIBRARY=$PWD/$L/$lib.so timeout 300 python scripts/latency_sweep.py --configs $CF --variants "" --iters 100 > gpurun_out/r2e/lat_$lib.jsonl 2>&1
done
BL_LIBRARY=$PWD/$L/libbl_a.so timeout 300 python scripts/latency_sweep.py --configs C2,C3b256,C4 --variants "T=2,TP=1,MU=4,ASYNC=1" --iters 100 > gpurun_out/r2e/lat_libbl_a_small.jsonl 2>&1
for c in C2 C4; do
  BL_PROFILE=1 BL_LIBRARY=$PWD/$L/libbl_ts.so timeout 120 python scripts/async_profile.py --config $c --iters 100 > gpurun_out/r2e/ts_$c.json 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum --clock-control none --csv python scripts/metrics_run.py --what attr,eu > gpurun_out/r2e/ncu_attr_eu_launches.csv 2>&1; echo ncu rc=$?
bash scripts/gpu_r2.sh
