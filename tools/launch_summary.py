"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
agg, cnt, tot = collections.Counter(), collections.Counter(), 0.0
for r in data:
    if len(r) <= iv:
        continue
    us = float(r[iv].replace(",", "")) * scale[r[iu]]
    name = r[ik].split("(")[0].replace("<unnamed>::", "").replace("void ", "")[:70]
    agg[name] += us
    cnt[name] += 1
    tot += us
print(f"{len(data)} launches, {tot/1e3:.3f} ms total (ncu: serialised, cold caches; compare shares)")
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{100*v/tot:6.2f}%  {v/1e3:10.3f} ms  x{cnt[k]:4d}  {k}")
