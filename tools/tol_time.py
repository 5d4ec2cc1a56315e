"""Cost of the E1 early-stop path (gs_diffuse with residual_tolerance) per sweep
against the plain pipelined solve, and of one exact left-to-right E1 sum.

    python tools/tol_time.py [config] [sweeps]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06060_b200 as gh  # noqa: E402
from paper_1812_06060_b200 import meshgen  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = meshgen.config(cfg)
mesh = gh.build_mesh(w.positions, w.faces)
lv = gh.bfs_levels(mesh, w.sources)
t = w.t if w.t is not None else gh.diffusion_time(mesh, w.m)
out = {"config": cfg, "sweeps": sweeps}
for rep_i in range(2):
    r = gh.SolverReport()
    t0 = time.perf_counter()
    u = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=sweeps), r)
    out["plain_wall_ms"] = 1e3 * (time.perf_counter() - t0)
    out["plain_device_ms"] = r.device_ms
for rep_i in range(2):
    r = gh.SolverReport()
    t0 = time.perf_counter()
    u2 = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=sweeps, residual_tolerance=1e-300), r)
    out["tol_wall_ms"] = 1e3 * (time.perf_counter() - t0)
out["bitwise"] = bool(np.array_equal(u.view(np.uint64), u2.view(np.uint64)))
out["tol_per_sweep_ms"] = out["tol_wall_ms"] / sweeps
sq = np.random.RandomState(1).standard_normal(mesh.vertex_count()) ** 2 * 10.0 ** np.random.RandomState(2).uniform(-300, 0, mesh.vertex_count())
for rep_i in range(3):
    t0 = time.perf_counter()
    s = gh.geoheat.deterministic_sum(sq)
    out["exact_sum_wall_ms_incl_h2d"] = 1e3 * (time.perf_counter() - t0)
out["exact_sum_ok"] = s == float(np.cumsum(sq)[-1])
for rep_i in range(3):
    t0 = time.perf_counter()
    e1 = gh.diffusion_residual(mesh, u, t, w.sources, levels=lv)
    out["diffusion_residual_wall_ms"] = 1e3 * (time.perf_counter() - t0)
print(json.dumps(out))
