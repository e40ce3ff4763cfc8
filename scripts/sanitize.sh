#!/bin/bash
# compute-sanitizer evidence for the hand-rolled memory ordering of libbl's
# layout kernels: memcheck, racecheck and synccheck on
# every batch driver, through a torch-free host program (scripts/san_driver).
# Logs: gpurun_out/sanitizer/<case>_<tool>.log, summary in
# gpurun_out/sanitizer/summary.txt.
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitizer
mkdir -p $OUT
SAN=/usr/local/cuda/bin/compute-sanitizer
g++ -O2 -std=c++17 -o scripts/san_driver scripts/san_driver.cpp \
  -Lpaper_2002_08233_b200 -lbl -Wl,-rpath,$PWD/paper_2002_08233_b200 \
  -L/usr/local/cuda/lib64 -lcudart || { echo "build failed"; exit 1; }
$SAN --version | head -2 > $OUT/summary.txt
# case name | env | driver args
CASES=(
  "C1grid_cluster||grid 32 256 2"
  "tri_pipelined|BL_CLUSTER=0 BL_ASYNC=0|tri 24 64 2"
  "tri_async|BL_CLUSTER=0 BL_ASYNC=1|tri 24 64 2"
  "rand2048_async|BL_CLUSTER=0 BL_ASYNC=1|rand 2048 256 2"
  "rand2048_twobarrier|BL_CLUSTER=0 BL_PIPELINE=0|rand 2048 256 2"
  "rand2048_pipelined|BL_CLUSTER=0 BL_ASYNC=0|rand 2048 256 2"
  "rand2048_bh||rand 2048 256 2 bh"
)
TOOLS=${TOOLS:-"memcheck racecheck synccheck"}
for c in "${CASES[@]}"; do
  IFS='|' read -r name envs args <<< "$c"
  for tool in $TOOLS; do
    log=$OUT/${name}_${tool}.log
    extra=""
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    env $envs timeout ${SAN_TIMEOUT:-900} $SAN --tool $tool $extra --print-limit 50 \
      ./scripts/san_driver $args > $log 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Target application returned" $log | tr '\n' ' ')
    echo "$name $tool rc=$rc $summ" | tee -a $OUT/summary.txt
  done
done
