"""A small workload that launches every kernel family once (a quick GPU check, and the
input for compute-sanitizer where the pool allows it):
mesh load (binary PLY on the device), build, BFS, diffusion (single band and
2-band emulation), normalisation, both ADMMs, integration, CG heat method,
exact sums, Dijkstra, subdivision.

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_06060_b200 import bands as GB, geoheat as g, meshgen  # noqa: E402

P, F = meshgen.torus(48, 24, 2.0, 0.7)[:2]
mesh = g.build_mesh(P, F)
data = g.serialize_mesh(mesh, g.MeshFormat.PLY)
mesh2 = g.load_mesh(data, g.MeshFormat.PLY)
assert np.array_equal(mesh2.download("positions"), mesh.download("positions"))
lv = g.bfs_levels(mesh, [0, 100])
t = g.diffusion_time(mesh, 1.0)
u = g.gs_diffuse(mesh, lv, t, g.DiffusionConfig(sweeps=20))
u2 = GB.gs_diffuse_bands(mesh, lv, 2, t, 20)
assert np.array_equal(np.asarray(u2), u)
nt = g.normalized_target_gradients(mesh, u)
fr = g.admm_face_optimize(mesh, nt.field, g.AdmmConfig(max_iterations=3))
er = g.admm_edge_optimize(mesh, nt.field, g.AdmmConfig(max_iterations=3))
d1 = g.integrate_face_gradients(mesh, lv, fr.gradients)
d2 = g.integrate_edge_differences(mesh, lv, er.differences)
dp, _ = g.poisson_heat_method(mesh, [0, 100], t, 1e-6)
s = g.deterministic_sum(np.abs(np.random.RandomState(0).normal(size=300_000)))
dj = g.dijkstra_edge_distance(mesh, [0])
fine = g.midpoint_subdivide(mesh, 1)
e1 = g.diffusion_residual(mesh, u, t, [0, 100], lv)
print("sanitize smoke ok", float(d1.max()), float(d2.max()), float(dp.max()), s, float(dj.max()), fine.vertex_count(), e1)
