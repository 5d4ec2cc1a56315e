"""Wall time of bfs_levels (BFS, parents, ring order, diffusion layout) on BASELINE configs.

    python tools/bfs_time.py
"""
import sys, time
sys.path.insert(0, '.')
import paper_1812_06060_b200 as gh
from paper_1812_06060_b200 import meshgen
for cfg in (3, 4, 2):
    w = meshgen.config(cfg)
    mesh = gh.build_mesh(w.positions, w.faces)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        lv = gh.bfs_levels(mesh, w.sources)
        ts.append(time.perf_counter() - t0)
        del lv  # one level set alive at a time (no pool growth)
    print(cfg, "bfs_levels (BFS + parents + diffusion layout) ms", [round(1e3 * x, 2) for x in ts], flush=True)
