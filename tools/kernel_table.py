"""Per-kernel DRAM throughput of an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv:
launches, time, DRAM bytes and achieved GB/s per kernel against the measured
HBM peak (MEASURED_PEAKS.json hbm_gbs). ncu serialises launches and replays
each with cold caches, so times are per-kernel, not the pipelined run's.

    python tools/kernel_table.py K.csv --out profiles/r1_kernel_table.json [--workload ...]
"""
import argparse
import collections
import csv
import json
import os

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out")
    ap.add_argument("--workload", default="C3 torus4096x2048 face, 1000 sweeps, 10 ADMM iters (one gh_distance_host call)")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ik, iid, im, iv, iu = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.defaultdict(dict)
    names = {}
    for r in data:
        if len(r) <= iv:
            continue
        per[r[iid]][r[im]] = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        names[r[iid]] = r[ik].split("(")[0].replace("<unnamed>::", "").replace("void ", "")[:60]
    peak = None
    pk = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peak = json.load(open(pk)).get("hbm_gbs")
    agg = collections.OrderedDict()
    for k, m in per.items():
        n = names[k]
        e = agg.setdefault(n, {"launches": 0, "time_s": 0.0, "dram_bytes": 0.0})
        e["launches"] += 1
        e["time_s"] += m.get("gpu__time_duration.sum", 0.0)
        e["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    total = sum(e["time_s"] for e in agg.values())
    out = []
    for n, e in sorted(agg.items(), key=lambda kv: -kv[1]["time_s"]):
        gbs = e["dram_bytes"] / e["time_s"] / 1e9 if e["time_s"] > 0 else 0.0
        out.append({"kernel": n, "launches": e["launches"], "time_ms": 1e3 * e["time_s"],
                    "share": e["time_s"] / total if total else 0.0, "dram_GB": e["dram_bytes"] / 1e9,
                    "dram_GBps": gbs, "frac_of_peak": gbs / peak if peak else None})
    print(f"{len(per)} launches, {1e3 * total:.3f} ms (ncu: serialised, cold caches); peak {peak} GB/s")
    print(f"{'share':>6} {'ms':>9} {'n':>4} {'GB':>8} {'GB/s':>7} {'frac':>5}  kernel")
    for e in out:
        fr = f"{e['frac_of_peak']:.2f}" if e["frac_of_peak"] is not None else "-"
        print(f"{100 * e['share']:5.1f}% {e['time_ms']:9.3f} {e['launches']:4d} {e['dram_GB']:8.3f} "
              f"{e['dram_GBps']:7.0f} {fr:>5}  {e['kernel']}")
    if a.out:
        json.dump({"workload": a.workload, "peak_GBps": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                   "total_ms": 1e3 * total, "kernels": out}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
