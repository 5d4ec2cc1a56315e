"""Time normalisation + face/edge ADMM + integration on a BASELINE config (device-resident u)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06060_b200 as gh  # noqa: E402
from paper_1812_06060_b200 import meshgen  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
w = meshgen.config(cfg)
mesh = gh.build_mesh(w.positions, w.faces)
lv = gh.bfs_levels(mesh, w.sources)
for method in ("face", "edge"):
    for _ in range(3):
        d, r = gh.distance(lv, method, sweeps, w.t, w.m)
    print(f"config {cfg} {method}: normalize {r.normalize_ms:.3f} ms, ADMM {r.admm_iterations} it {r.optimization_ms:.3f} ms "
          f"({r.optimization_ms / max(r.admm_iterations, 1):.3f} ms/it), integrate {r.integration_ms:.3f} ms", flush=True)
