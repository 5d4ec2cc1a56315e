"""SASS instruction summary of the hot kernels (evidence for the profiles/).

Disassembles lib/libgeoheat_b200.so (cuobjdump -sass, no GPU needed) and counts,
per kernel, the mnemonics that show how it moves data: UBLKCP (cp.async.bulk
into shared memory), SYNCS.* (mbarrier), LDG/STG (global loads/stores, with
their cache qualifiers), LDS/STS, CCTL (L1 invalidation after an acquire),
MEMBAR/FENCE, ATOM/RED, DMUL/DADD/DFMA, and the register count.

    python tools/sass_summary.py [--kernels regex] [--out profiles/r2_sass_summary.txt]
"""
from __future__ import annotations

import argparse
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1812_06060_b200", "lib", "libgeoheat_b200.so")
GROUPS = ["UBLKCP", "SYNCS", "LDG", "STG", "LDS", "STS", "LD", "ST", "CCTL", "MEMBAR", "FENCE", "ATOM", "ATOMG", "RED",
          "DMUL", "DADD", "DFMA", "MUFU", "BAR", "NANOSLEEP", "SHFL", "UTMALDG", "UTMASTG", "UTCHMMA", "HMMA"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return out[:len(names)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernels", default="k_diffuse_tma|k_face_g|k_face_lambda_pair|k_edge_x|k_edge_lambda_w|k_bfs|k_chain")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    regs = {}
    for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+)", res):
        regs[m.group(1)] = int(m.group(2))
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    mangled = [f.split("\n", 1)[0].strip() for f in funcs]
    names = demangle(mangled)
    lines = []
    pat = re.compile(a.kernels)
    for mg, name, body in zip(mangled, names, funcs):
        if not pat.search(name):
            continue
        counts = collections.Counter()
        detail = collections.Counter()
        n = 0
        for ins in re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", body):
            n += 1
            op = ins.split(".")[0]
            counts[op] += 1
            if op in ("LDG", "STG", "SYNCS", "UBLKCP", "CCTL", "ATOMG", "RED", "MEMBAR", "FENCE", "LD", "ST"):
                detail[ins] += 1
        short = re.sub(r"\(anonymous namespace\)::", "", name)
        short = re.sub(r"\(.*\)$", "", short) if "TmaArgs" not in short else short.split("(")[0]
        row = f"{short:<40} regs {regs.get(mg, '?'):>4}  instructions {n:>6}  " + "  ".join(
            f"{g} {counts[g]}" for g in GROUPS if counts[g])
        lines.append(row)
        lines.append("    " + ", ".join(f"{k} x{v}" for k, v in sorted(detail.items())))
    text = "\n".join(lines) + "\n"
    sys.stdout.write(text)
    if a.out:
        with open(a.out, "w") as f:
            f.write(f"# cuobjdump -sass {os.path.relpath(LIB, ROOT)} (sm_100a), tools/sass_summary.py\n" + text)


if __name__ == "__main__":
    main()
