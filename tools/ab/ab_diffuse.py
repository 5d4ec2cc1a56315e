"""A/B of two builds of the library on the diffusion solve (same box, alternating processes).
    python tools/ab/ab_diffuse.py LIB CONFIG SWEEPS REPEATS"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1812_06060_b200 import _lib
if sys.argv[1] == "general":
    os.environ["GH_DIFFUSE_GENERAL"] = "1"
elif sys.argv[1] != "default":
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
import paper_1812_06060_b200 as gh
from paper_1812_06060_b200 import meshgen
cfg, sweeps, rep = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
w = meshgen.config(cfg)
mesh = gh.build_mesh(w.positions, w.faces)
lv = gh.bfs_levels(mesh, w.sources)
t = w.t if w.t is not None else gh.diffusion_time(mesh, w.m)
gh.set_zero_level_truncation(False)
ms = []
for _ in range(rep):
    r = gh.SolverReport()
    gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=sweeps), r, keep_on_device=True)
    ms.append(round(r.device_ms, 2))
print(sys.argv[1], cfg, ms, flush=True)
