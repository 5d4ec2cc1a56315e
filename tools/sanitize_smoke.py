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

# exact-zero skipping: a 1400-ring ribbon with a small partial layout, a small
# first cap and margin, so the truncated launches, the redo path, the layout extension with a
# carried state and the ADMM active sets (flag screening included) all run
os.environ.update(GH_PARTIAL_LEVELS="300", GH_ZERO_LEVELS_FIRST="128", GH_ZERO_LEVELS_MARGIN="8")
g.set_zero_level_truncation(True)  # opt-in
nx, ny = 1400, 6
x, y = np.meshgrid(np.arange(nx, dtype=np.float64), np.arange(ny, dtype=np.float64), indexing="ij")
Pr = np.stack([x, y, 0.05 * np.sin(0.3 * x) * np.cos(0.4 * y)], -1).reshape(-1, 3)
i, j = np.meshgrid(np.arange(nx - 1), np.arange(ny - 1), indexing="ij")
a = (i * ny + j).ravel()
Fr = np.concatenate([np.stack([a, a + ny, a + ny + 1], 1), np.stack([a, a + ny + 1, a + 1], 1)]).astype(np.int32)
rm = g.build_mesh(Pr, Fr)
rl = g.bfs_levels(rm, [0])
tr = g.diffusion_time(rm, 1.0)
ur = g.gs_diffuse(rm, rl, tr, g.DiffusionConfig(sweeps=40))
st = rl.diffusion_stats
g.set_zero_level_truncation(False)
rl2 = g.bfs_levels(rm, [0])
ur2 = g.gs_diffuse(rm, rl2, tr, g.DiffusionConfig(sweeps=40))
g.set_zero_level_truncation(True)
assert np.array_equal(ur.view(np.uint64), ur2.view(np.uint64)), "truncated diffusion differs"
for method in ("face", "edge"):
    da, _ = g.distance(rl, method, 40, tr)
    g.set_zero_level_truncation(False)
    db, _ = g.distance(rl2, method, 40, tr)
    g.set_zero_level_truncation(True)
    assert np.array_equal(da.view(np.uint64), db.view(np.uint64)), method
g.set_zero_level_truncation(False)
print("zero skipping ok", st, rl.layout_levels)
