"""Run the diffusion solve on a BASELINE config for ncu captures.

    python tools/profile_diffusion.py [config] [sweeps] [repeats]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06060_b200 as gh  # noqa: E402
from paper_1812_06060_b200 import meshgen  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
repeats = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = meshgen.config(cfg)
mesh = gh.build_mesh(w.positions, w.faces)
lv = gh.bfs_levels(mesh, w.sources)
t = w.t if w.t is not None else gh.diffusion_time(mesh, w.m)
for _ in range(repeats):
    rep = gh.SolverReport()
    gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=sweeps), rep, keep_on_device=True)
    print(f"config {cfg} {w.name}: {sweeps} sweeps in {rep.device_ms:.3f} ms "
          f"({(mesh.vertex_count() - lv.unreachable_count) * sweeps / rep.device_ms / 1e6:.3f} G vu/s)", flush=True)
