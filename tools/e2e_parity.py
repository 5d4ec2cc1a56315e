"""The headline workload end to end against the compiled reference, bit for bit.

Runs the bench's end-to-end call (gh_distance_host: host arrays in, distances
out, t = m h^2 computed on the device) and the reference's own chain
(build_mesh, diffusion_time, bfs_levels, gs_diffuse, normalized_target_
gradients, admm_*_optimize, integrate_*; oracle/_ref, OpenMP on all host
cores) on the same BASELINE config, and records whether the distance fields
are identical (field_hash, report.hpp:145-153).

    python tools/e2e_parity.py [--configs 2,3] [--out gpurun_out/e2e_parity.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, run_pipeline  # noqa: E402
from paper_1812_06060_b200 import geoheat as g  # noqa: E402
from paper_1812_06060_b200 import meshgen  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "e2e_parity.json"))
    args = ap.parse_args()
    ref = Oracle("reference")
    ref.set_threads(os.cpu_count() or 1)
    out = []
    for k in [int(x) for x in args.configs.split(",")]:
        w = meshgen.config(k)
        t0 = time.perf_counter()
        d, rep = g.distance_host(w.positions, w.faces, w.sources, method=w.method, sweeps=w.sweeps, t=w.t, m=w.m,
                                 admm=g.AdmmConfig(max_iterations=w.admm_iters))
        t1 = time.perf_counter()
        r = run_pipeline(ref, w.positions, w.faces, w.sources, m=w.m, t=w.t, sweeps=w.sweeps,
                         admm_iters=w.admm_iters, method=w.method)
        t2 = time.perf_counter()
        d_ref = r["d"]
        rec = {"config": k, "name": w.name, "method": w.method, "vertices": int(w.positions.shape[0]),
               "sweeps": w.sweeps, "t_device": rep.t, "t_reference": r["t"], "t_identical": rep.t == r["t"],
               "admm_iterations": [rep.admm_iterations, r["report"].iterations],
               "hash_device": f"{g.field_hash(d):016x}", "hash_reference": f"{ref.field_hash(d_ref):016x}",
               "bitwise_identical": bool(np.array_equal(d, d_ref)),
               "max_abs_diff": float(np.max(np.abs(d - d_ref))) if d.size else 0.0,
               "device_e2e_s": t1 - t0, "reference_chain_s": t2 - t1, "reference_threads": os.cpu_count()}
        out.append(rec)
        print(json.dumps(rec), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
