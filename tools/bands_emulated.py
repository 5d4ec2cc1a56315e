"""The multi-GPU band schedule emulated on one GPU: gs_diffuse split into 1, 2,
4, 8 BFS bands, all in one cooperative launch (the neighbour links are
same-device pointers; the kernel code path is the multi-GPU one). Reports the
launch time per band count and checks every result bit-identical to 1 band.

    python tools/bands_emulated.py [configs] [sweeps] --out profiles/r1_bands_emulated.json
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
ap.add_argument("--out")
a = ap.parse_args()
rows = []
for cfg in [int(x) for x in a.configs.split(",")]:
    w = meshgen.config(cfg)
    mesh = gh.build_mesh(w.positions, w.faces)
    lv = gh.bfs_levels(mesh, w.sources)
    t = w.t if w.t is not None else gh.diffusion_time(mesh, w.m)
    reach = mesh.vertex_count() - lv.unreachable_count
    ref = None
    for nb in (1, 2, 4, 8):
        times = []
        for _ in range(3):
            rep = gh.SolverReport()
            u = bands.gs_diffuse_bands(mesh, lv, nb, t, a.sweeps, report=rep)
            times.append(rep.device_ms)
        if ref is None:
            ref = u
        same = bool(np.array_equal(u.view(np.uint64), ref.view(np.uint64)))
        ms = float(np.median(times))
        row = {"config": cfg, "name": w.name, "bands": nb, "sweeps": a.sweeps, "launch_ms": ms,
               "vertex_updates_per_s": reach * a.sweeps / (ms * 1e-3), "bitwise_equal_to_1_band": same}
        rows.append(row)
        print(json.dumps(row), flush=True)
if a.out:
    json.dump({"what": "band-sharded diffusion emulated on one GPU (all bands in one launch)", "rows": rows},
              open(a.out, "w"), indent=1)
