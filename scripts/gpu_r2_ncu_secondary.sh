#!/bin/bash
# ncu --set full of the secondary kernels of round 2 (each after its plain run
# exited 0): the latency driver at C4 (20 iterations), BatchLayoutBH at C5 (2
# iterations), the relabel kernel at C5.
cd "$(dirname "$0")/.."
O=gpurun_out/r2ncu; mkdir -p $O
run() {  # tag, kernel regex, command...
  local tag=$1 rx=$2; shift 2
  "$@" > $O/plain_$tag.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -c 1 -o $O/$tag "$@" > $O/ncu_$tag.log 2>&1
  echo "$tag rc=$?"
}
run lat_C4 bl_layout_kernel python scripts/profile_run.py --config C4 --iters 20
run bh_C5 bl_bh_kernel python scripts/profile_run.py --config C5 --iters 2 --algo 1
run relabel_C5 bl_relabel_kernel python scripts/shuffle_cost.py C5
