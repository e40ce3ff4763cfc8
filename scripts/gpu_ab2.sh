#!/bin/bash
# Same-box interleaved A/B of builds (BL_LIBRARY) with scripts/latency_sweep.py:
# us per dependent batch per config.  AB_LIBS = space-separated .so names in
# paper_2002_08233_b200/ (first = baseline).
cd "$(dirname "$0")/.."
O=gpurun_out/${AB_TAG:-ab2}; mkdir -p $O; rm -f $O/*.jsonl
for rep in ${AB_REPS:-1 2}; do
  for lib in ${AB_LIBS:-libbl_base.so libbl.so}; do
    BL_LIBRARY=$PWD/paper_2002_08233_b200/$lib timeout 600 python scripts/latency_sweep.py \
      --configs ${AB_CONFIGS:-C2,C3b256,C4,C5} --variants "${AB_VARIANTS:-}" --iters ${AB_ITERS:-20} \
      > $O/${lib%.so}_$rep.jsonl 2> $O/${lib%.so}_$rep.err
  done
done
python - "$O" <<'PY'
import glob, json, sys, collections
r = collections.defaultdict(list)
for f in sorted(glob.glob(sys.argv[1] + "/*.jsonl")):
    lib = f.split("/")[-1].rsplit("_", 1)[0]
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            if "us_per_batch" in d:
                r[(d["config"], json.dumps(d["env"]), lib)].append(d["us_per_batch"])
for k in sorted(r):
    print(f"{k[0]:8s} {k[1]:30s} {k[2]:14s} " + " ".join(f"{x:8.3f}" for x in r[k]))
PY
