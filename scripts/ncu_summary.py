"""Summarise an `ncu --set full` capture of the bench-shaped layout launch
(`ncu -i X.ncu-rep --page raw --csv`) into the files bench.py reads:
profiles/traffic.json (DRAM bytes per launch) and profiles/pipes.json (XU,
FMA, FMA-heavy, ALU pipe and issue utilisation, L2 sectors, instructions).

  ncu -i gpurun_out/r2m/prof_C5.ncu-rep --page raw --csv > profiles/r2/ncu_full_C5_50it.csv
  python scripts/ncu_summary.py profiles/r2/ncu_full_C5_50it.csv --workload C5 --kernel 'bl_layout_kernel<512,8,2>'
"""
import argparse
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "l2_sectors": "lts__t_sectors.sum",
    "inst_executed": "smsp__inst_executed.sum",
    "xu": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fma": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "fmaheavy": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "alu": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm_cycles": "sm__cycles_elapsed.avg",
}
SCALE = {"ms": 1e6, "us": 1e3, "ns": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e3, "msecond": 1e6,
         "nsecond": 1.0, "second": 1e9}


def read(path):
    rows = list(csv.reader(open(path)))
    h, u, v = rows[0], rows[1], rows[2]
    out = {}
    for name, key in KEYS.items():
        if key in h:
            i = h.index(key)
            x = float(v[i].replace(",", ""))
            out[name] = x * SCALE.get(u[i], 1.0)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--kernel", default="bl_layout_kernel<512,8,1>")
    a = ap.parse_args()
    m = read(a.csv)
    src = (f"ncu --set full --clock-control none of scripts/profile_run.py --config {a.workload} "
           f"--iters 50 (one bench-shaped launch); {os.path.relpath(a.csv, ROOT)}")
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    tr = json.load(open(tr_path)) if os.path.exists(tr_path) else {}
    tr[a.workload] = {"kernel": a.kernel, "bytes_per_launch": m["dram_read"] + m["dram_write"],
                      "dram_read_bytes": m["dram_read"], "dram_write_bytes": m["dram_write"],
                      "l2_sectors_per_launch": m.get("l2_sectors"), "source": src}
    json.dump(tr, open(tr_path, "w"), indent=1)
    pp_path = os.path.join(ROOT, "profiles", "pipes.json")
    pp = json.load(open(pp_path)) if os.path.exists(pp_path) else {}
    pp[a.workload] = {"kernel": a.kernel, "xu": m["xu"] / 100, "fma": m["fma"] / 100,
                      "fmaheavy": m.get("fmaheavy", 0) / 100, "alu": m.get("alu", 0) / 100,
                      "issue": m["issue"] / 100, "inst_executed": m.get("inst_executed"),
                      "l2_sectors": m.get("l2_sectors"), "duration_ms": m["duration_ns"] / 1e6,
                      "basis": "fraction of peak sustained (active cycles) over the whole launch",
                      "source": src}
    json.dump(pp, open(pp_path, "w"), indent=1)
    print(json.dumps({"traffic": tr[a.workload], "pipes": pp[a.workload]}, indent=1))


if __name__ == "__main__":
    main()
