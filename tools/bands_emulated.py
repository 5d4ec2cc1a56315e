"""The multi-GPU partitions emulated on one GPU: gs_diffuse split into 1, 2, 4,
8 BFS bands or sector slices, all parts in one cooperative launch (the links
between parts are same-device pointers; the kernel code path is the
multi-GPU one). Reports the launch time per part count and checks every
result bit-identical to the single-part solve (gh_gs_diffuse).

On one GPU the parts share the SMs (blocks in proportion to rows), so the
emulated time measures the partition's overhead — idle parts, ghost-row
exports, per-source dependency checks — not a speed-up: ideal is the
single-part time.

    python tools/bands_emulated.py [configs] [sweeps] [--partitions bands,slices] --out profiles/...json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1812_06060_b200 as gh  # noqa: E402
from paper_1812_06060_b200 import bands, meshgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="?", default="3,4")
ap.add_argument("sweeps", nargs="?", type=int, default=1000)
ap.add_argument("--partitions", default="bands,slices")
ap.add_argument("--parts", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--out")
a = ap.parse_args()
rows = []
for cfg in [int(x) for x in a.configs.split(",")]:
    w = meshgen.config(cfg)
    mesh = gh.build_mesh(w.positions, w.faces)
    lv = gh.bfs_levels(mesh, w.sources)
    t = w.t if w.t is not None else gh.diffusion_time(mesh, w.m)
    reach = mesh.vertex_count() - lv.unreachable_count
    times = []
    for _ in range(a.reps):
        rep = gh.SolverReport()
        ref = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=a.sweeps), rep)
        times.append(rep.device_ms)
    base = float(np.median(times))
    rows.append({"config": cfg, "name": w.name, "partition": "none", "parts": 1, "sweeps": a.sweeps,
                 "levels": lv.level_count(), "launch_ms": base, "vertex_updates_per_s": reach * a.sweeps / (base * 1e-3)})
    print(json.dumps(rows[-1]), flush=True)
    for part in a.partitions.split(","):
        for nb in [int(x) for x in a.parts.split(",")]:
            times = []
            for _ in range(a.reps):
                rep = gh.SolverReport()
                u = bands.gs_diffuse_bands(mesh, lv, nb, t, a.sweeps, report=rep, partition=part)
                times.append(rep.device_ms)
            same = bool(np.array_equal(u.view(np.uint64), ref.view(np.uint64)))
            ms = float(np.median(times))
            row = {"config": cfg, "name": w.name, "partition": part, "parts": nb, "sweeps": a.sweeps,
                   "launch_ms": ms, "over_single": ms / base,
                   "vertex_updates_per_s": reach * a.sweeps / (ms * 1e-3), "bitwise_equal_to_single": same}
            rows.append(row)
            print(json.dumps(row), flush=True)
    del mesh, lv
if a.out:
    json.dump({"what": "partitioned diffusion emulated on one GPU (all parts in one launch)", "rows": rows},
              open(a.out, "w"), indent=1)
