#!/bin/bash
# Round-2 GPU call D: same-box latency A/B (before: libbl_a.so = the build
# before the fence/poll change; r1: round-1 library; after: libbl.so), the
# per-hop timelines (-DBL_PHASE_TS builds), ncu of step a5 and EU, gpu tests.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2d
L=paper_2002_08233_b200
CF=C2,C3b256,C4,C3b1024
timeout 300 python scripts/latency_sweep.py --configs $CF --variants "T=8,TP=2;T=2,TP=1,MU=4;T=4,TP=1,MU=4" --iters 100 > gpurun_out/r2d/lat_after.jsonl 2>&1; echo after rc=$?
BL_LIBRARY=$PWD/$L/libbl_a.so timeout 300 python scripts/latency_sweep.py --configs $CF --variants "T=2,TP=1,MU=4,ASYNC=1" --iters 100 > gpurun_out/r2d/lat_before_fence.jsonl 2>&1; echo before rc=$?
BL_LIBRARY=$PWD/$L/libbl_r1.so timeout 300 python scripts/latency_sweep.py --configs $CF --variants "" --iters 100 > gpurun_out/r2d/lat_r1.jsonl 2>&1; echo r1 rc=$?
for c in C2 C3b256 C4; do
  BL_PROFILE=1 BL_LIBRARY=$PWD/$L/libbl_ts.so timeout 120 python scripts/async_profile.py --config $c --iters 20 > gpurun_out/r2d/ts_after_$c.json 2>&1
  BL_PROFILE=1 BL_LIBRARY=$PWD/$L/libbl_r1_ts.so timeout 120 python scripts/async_profile.py --config $c --iters 20 > gpurun_out/r2d/ts_r1_$c.json 2>&1
  BL_LIBRARY=$PWD/$L/libbl_r1_ts.so timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-bh --no-shuffle --no-metrics --latency-configs "" --prof > gpurun_out/r2d/prof_r1_$c.log 2>&1
done
echo ts done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum --clock-control none --csv python scripts/metrics_run.py --what attr,eu > gpurun_out/r2d/ncu_attr_eu_launches.csv 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bla_items|blm_eu_pass" -c 3 -o gpurun_out/r2d/attr_eu python scripts/metrics_run.py --what attr,eu > gpurun_out/r2d/ncu_full.log 2>&1; echo ncu2 rc=$?
SKIP_BENCH=1 bash scripts/gpu_r2.sh
