"""Summarise an ncu report's source page per CUDA source line (stall samples)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[2]
i_line, i_src, i_s = 0, 1, hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
per_line = {}
cur = None
for r in rows[3:]:
    if len(r) <= i_s:
        continue
    if r[i_line].strip():
        cur = (r[i_line], r[i_src][:90])
    try:
        s = int(r[i_s])
    except ValueError:
        continue
    d = per_line.setdefault(cur, [0, {}])
    d[0] += s
    for i in stall_cols:
        try:
            v = int(r[i])
        except ValueError:
            continue
        if v:
            d[1][hdr[i]] = d[1].get(hdr[i], 0) + v
total = sum(v[0] for v in per_line.values())
print("total samples", total)
for k, (s, st) in sorted(per_line.items(), key=lambda x: -x[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    top = sorted(st.items(), key=lambda x: -x[1])[:3]
    print(f"{100*s/total:5.1f}% L{k[0]:>4} {k[1]!r} " + " ".join(f"{n[6:]}={100*v/total:.1f}" for n, v in top))
