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

from oracle.oracle import Oracle  # noqa: E402
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
        for _ in range(2):  # warm-up: module load, pool growth to this config's size
            g.distance_host(w.positions, w.faces, w.sources, method=w.method, sweeps=w.sweeps, t=w.t, m=w.m,
                            admm=g.AdmmConfig(max_iterations=w.admm_iters))
        t0 = time.perf_counter()
        d, rep = g.distance_host(w.positions, w.faces, w.sources, method=w.method, sweeps=w.sweeps, t=w.t, m=w.m,
                                 admm=g.AdmmConfig(max_iterations=w.admm_iters))
        t_dev = time.perf_counter() - t0
        # the reference chain stage by stage (run_pipeline, tools/geoheat.cpp:71-143)
        ref_ms = {}
        c0 = time.perf_counter()
        om = ref.build_mesh(w.positions, w.faces)
        c1 = time.perf_counter()
        t_ref = w.t if w.t is not None else om.diffusion_time(w.m)
        lv = om.bfs(w.sources)
        c2 = time.perf_counter()
        u, _ = om.gs_diffuse(lv, t_ref, w.sweeps)
        c3 = time.perf_counter()
        H, zc = om.normalized_target_gradients(u)
        c4 = time.perf_counter()
        if w.method == "face":
            G, orep = om.admm_face(H, w.admm_iters)
            c5 = time.perf_counter()
            d_ref = om.integrate_face(lv, G)
        else:
            X, orep = om.admm_edge(H, w.admm_iters)
            c5 = time.perf_counter()
            d_ref = om.integrate_edge(lv, X)
        c6 = time.perf_counter()
        t2 = c6
        ref_ms = {"build_mesh": 1e3 * (c1 - c0), "h_t_bfs": 1e3 * (c2 - c1), "gs_diffuse": 1e3 * (c3 - c2),
                  "normalize": 1e3 * (c4 - c3), "admm": 1e3 * (c5 - c4), "integrate": 1e3 * (c6 - c5)}
        r = {"t": t_ref, "report": orep}
        rec = {"config": k, "name": w.name, "method": w.method, "vertices": int(w.positions.shape[0]),
               "sweeps": w.sweeps, "t_device": rep.t, "t_reference": r["t"], "t_identical": rep.t == r["t"],
               "admm_iterations": [rep.admm_iterations, r["report"].iterations],
               "hash_device": f"{g.field_hash(d):016x}", "hash_reference": f"{ref.field_hash(d_ref):016x}",
               "bitwise_identical": bool(np.array_equal(d, d_ref)),
               "max_abs_diff": float(np.max(np.abs(d - d_ref))) if d.size else 0.0,
               "device_e2e_s": t_dev, "device_stages_ms": {"build": rep.build_ms, "bfs_layout": rep.bfs_ms,
                                                             "diffusion": rep.diffusion_ms,
                                                             "normalize": rep.normalize_ms,
                                                             "admm": rep.optimization_ms,
                                                             "integrate": rep.integration_ms},
               "reference_chain_s": t2 - c0, "reference_stages_ms": ref_ms, "reference_threads": os.cpu_count()}
        out.append(rec)
        print(json.dumps(rec), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
