"""Summarise one kernel of an ncu --set full capture into profiles/ JSON.

    python tools/ncu_summary.py REP.ncu-rep --kernel k_diffuse --sweeps 200 \
        --workload "C3 ..." --out profiles/r1_diffuse_ncu.json [--traffic profiles/diffusion_traffic.json]

The traffic file is what bench.py reads for roofline.traffic (DRAM bytes per
sweep of the diffusion kernel).
"""
from __future__ import annotations

import argparse
import csv
import json
import subprocess

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel", default="k_diffuse")
    ap.add_argument("--sweeps", type=int, default=200)
    ap.add_argument("--algorithmic-bytes-per-sweep", type=float, default=838860800.0)
    ap.add_argument("--workload", default="C3 torus4096x2048 face, 1000 sweeps, 10 ADMM iters")
    ap.add_argument("--capture", default="ncu --set full --clock-control none --import-source on, "
                                          "tools/profile_diffusion.py 3 200 (one launch of 200 sweeps)")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    ik = hdr.index("Kernel Name")
    data = [r for r in rows[2:] if len(r) > ik and a.kernel in r[ik]]
    if not data:
        raise SystemExit(f"no {a.kernel} launch in {a.rep}")
    r = data[0]
    m = {}
    val = {}
    for name in METRICS:
        if name in hdr:
            i = hdr.index(name)
            m[name] = f"{r[i]} {units[i]}".strip()
            try:
                val[name] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
            except ValueError:
                pass
    dur = val["gpu__time_duration.sum"]
    dram = val["dram__bytes_read.sum"] + val["dram__bytes_write.sum"]
    per_sweep = dram / a.sweeps
    out = {"metrics": m, "workload": a.workload, "kernel": r[ik].split("(")[0], "capture": a.capture,
           "dram_bytes_per_sweep": per_sweep, "algorithmic_bytes_per_sweep": a.algorithmic_bytes_per_sweep,
           "dram_over_algorithmic": per_sweep / a.algorithmic_bytes_per_sweep, "duration_s": dur,
           "dram_GBps": dram / dur / 1e9, "source": a.rep}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    if a.traffic:
        t = {k: out[k] for k in ("workload", "capture", "dram_bytes_per_sweep", "algorithmic_bytes_per_sweep",
                                 "dram_over_algorithmic", "duration_s", "dram_GBps")}
        t["kernel"] = "k_diffuse_tma"
        t["source"] = f"{a.out} (from {a.rep})"
        with open(a.traffic, "w") as f:
            json.dump(t, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
