#!/bin/bash
# Round-2: async-driver warp-time breakdown and CTA-0 per-hop timeline
# (profiling build libbl_ts.so = -DBL_PHASE_TS), per config.
cd "$(dirname "$0")/.."
O=gpurun_out/${TS_TAG:-ts}; mkdir -p $O
L=$PWD/paper_2002_08233_b200/${TS_LIB:-libbl_ts.so}
for c in ${TS_CONFIGS:-C5:5 C4:50 C3b256:100 C2:200}; do
  cfg=${c%%:*}; it=${c##*:}
  BL_PROFILE=1 BL_LIBRARY=$L timeout 300 python scripts/async_profile.py --config $cfg --iters $it > $O/ts_$cfg.json 2>&1
  echo "$cfg rc=$?"; python -c "import json; d=json.load(open('$O/ts_$cfg.json')); print(json.dumps(d.get('warp_time_fraction'))); print(json.dumps(d.get('cta0_timeline_us_per_batch'))); print(json.dumps(d.get('cta_busy_rel')))" 2>&1 | cut -c1-400
done
