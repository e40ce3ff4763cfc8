#!/bin/bash
# Round-2 latency sweep on the GPU box (no rebuild: the .so files travel).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
V="T=4,TP=1;T=4,TP=2;T=2,TP=1;T=1,TP=1;T=2,TP=1,MU=4;T=2,TP=1,MU=8;T=4,TP=2,MU=8;T=2,TP=1,ASYNC=1;T=2,TP=1,ASYNC=0;T=2,TP=1,MU=4,ASYNC=1;T=2,TP=1,SPIN=128;T=2,TP=1,MU=4,ASYNC=1,SPIN=128;T=1,TP=1,MU=4,ASYNC=1"
timeout 900 python scripts/latency_sweep.py --configs ${LAT_CONFIGS:-C2,C3b256,C4} --variants "${LAT_VARIANTS:-$V}" --iters 100 > gpurun_out/latency_sweep.jsonl 2> gpurun_out/latency_sweep.err
echo sweep rc=$?
python - <<'PY'
import json
for l in open("gpurun_out/latency_sweep.jsonl"):
    r = json.loads(l)
    if "error" in r:
        print(r["config"], r["env"], "ERROR", r["error"][:80]); continue
    print(f'{r["config"]:8s} {r["us_per_batch"]:7.2f} us  {r["driver"]:10s} {r["kernel"]:28s} {r["env"]} {r.get("vs_default_1it", "")}')
PY
