"""Build a BASELINE config's mesh on the device (for launch lists of the build kernels).

    python tools/profile_build.py [config] [repeats]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06060_b200 as gh  # noqa: E402
from paper_1812_06060_b200 import meshgen  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
repeats = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = meshgen.config(cfg)
for _ in range(repeats):
    t0 = time.perf_counter()
    mesh = gh.build_mesh(w.positions, w.faces)
    t1 = time.perf_counter()
    print(f"config {cfg} {w.name}: build_mesh {1e3 * (t1 - t0):.1f} ms", flush=True)
    del mesh
