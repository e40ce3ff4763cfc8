#!/bin/bash
# Round-2 GPU call: latency sweep (new vs round-1 library), gpu tests, bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/gpu_r2_lat.sh
BL_LIBRARY=$PWD/paper_2002_08233_b200/libbl_r1.so timeout 300 python scripts/latency_sweep.py --configs C2,C3b256,C4 --variants "" --iters 100 > gpurun_out/latency_r1.jsonl 2>&1; echo r1 rc=$?
cat gpurun_out/latency_r1.jsonl | cut -c1-200
bash scripts/gpu_r2.sh
