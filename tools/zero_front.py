"""How far the nonzero heat reaches: per sweep count, the largest BFS level holding a
nonzero u (any bit set) and the share of reachable vertices at or below it.

    python tools/zero_front.py CONFIG SWEEPS[,SWEEPS...]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06060_b200 as gh  # noqa: E402
from paper_1812_06060_b200 import meshgen  # noqa: E402

cfg = int(sys.argv[1])
counts = [int(x) for x in sys.argv[2].split(",")]
w = meshgen.config(cfg)
mesh = gh.build_mesh(w.positions, w.faces)
lv = gh.bfs_levels(mesh, w.sources)
t = w.t if w.t is not None else gh.diffusion_time(mesh, w.m)
level = lv.level_of_vertex
offs = lv.offsets
nlev = lv.level_count()
for s in counts:
    rep = gh.SolverReport()
    u = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=s), rep)
    nz = u.view(np.uint64) != 0
    lmax = int(level[nz].max())
    print(json.dumps({"config": cfg, "sweeps": s, "levels": nlev, "max_nonzero_level": lmax,
                      "negative_zero": int((u.view(np.uint64) == 1 << 63).sum()),
                      "rows_at_or_below": int(offs[lmax + 1]), "reachable": int(offs[-1]),
                      "share": float(offs[lmax + 1] / offs[-1]), "device_ms": rep.device_ms}), flush=True)
