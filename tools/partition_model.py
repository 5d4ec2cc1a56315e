"""Model of the multi-GPU speed-up of the two diffusion partitions.

Per step tau of the sweep pipeline (levels L = tau - 2s active, 0 <= s < S),
a GPU's step time is t(R) = a + c + b R for its R active rows: a = the step
floor (dependency round trip, ~3 us measured), c = NVLink
exchange latency (2 us assumed), b = 1 / (70 G rows/s) the per-row cost of one
B200. One GPU: sum_tau (a + b R_tau). BFS bands (gh::plan_bands): every band
on its own GPU, the step waits for the busiest band. Slices: every GPU 1/N of
every step's rows. Also the bands emulated on one GPU (each band 1/N of the
SMs). Ring sizes from the device BFS of the seeded config.

    python tools/partition_model.py [--configs 3,4,5] [--sweeps 1000] [--out profiles/r2_partition_model.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1812_06060_b200 import bands  # noqa: E402


def active_rows(sizes, lo, hi, S, nsteps):
    out = np.zeros(nsteps)
    for L in range(lo, hi):
        out[L:L + 2 * S:2] += sizes[L]
    return out


def model(sizes, S=1000, a=3e-6, c=2e-6, b=1 / 70e9):
    nlev = len(sizes)
    nsteps = nlev + 2 * S - 1
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    tot = active_rows(sizes, 0, nlev, S, nsteps)
    single = float(np.sum(a + b * tot))
    res = {"levels": nlev, "one_gpu_s": single, "rows_per_step_mean": float(tot.mean())}
    for N in (2, 4, 8):
        cut = bands.plan_bands(off.astype(np.int32), N)
        parts = [active_rows(sizes, cut[r], cut[r + 1], S, nsteps) for r in range(N)]
        frac = [sizes[cut[r]:cut[r + 1]].sum() / sizes.sum() for r in range(N)]
        emu = float(np.sum(a + np.max([p * b / f for p, f in zip(parts, frac)], axis=0)))
        real_b = float(np.sum(a + c + np.max([p * b for p in parts], axis=0)))
        real_s = float(np.sum(a + c + tot * b / N))
        res[str(N)] = {"bands_speedup": single / real_b, "slices_speedup": single / real_s,
                  "bands_emulated_over_one": emu / single}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,4,5")
    ap.add_argument("--sweeps", type=int, default=1000)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import paper_1812_06060_b200 as gh
    from paper_1812_06060_b200 import meshgen
    out = []
    for k in [int(x) for x in a.configs.split(",")]:
        w = meshgen.config(k)
        mesh = gh.build_mesh(w.positions, w.faces)
        lv = gh.bfs_levels(mesh, w.sources)
        sizes = np.diff(lv.offsets.astype(np.int64)).astype(np.float64)
        del mesh, lv, w
        r = dict(config=k, **model(sizes, a.sweeps))
        out.append(r)
        print(json.dumps(r), flush=True)
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
