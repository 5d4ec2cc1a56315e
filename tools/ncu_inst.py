"""Instructions executed per CUDA source line from an ncu report."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[2]
i_e = hdr.index("Instructions Executed")
per, cur = {}, None
for r in rows[3:]:
    if len(r) <= i_e:
        continue
    if r[0].strip():
        cur = (r[0], r[1][:90])
    try:
        per[cur] = per.get(cur, 0) + int(r[i_e])
    except ValueError:
        pass
tot = sum(per.values())
print("total warp instructions", tot)
for k, v in sorted(per.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100*v/tot:5.1f}% L{k[0]:>4} {k[1]!r}")
