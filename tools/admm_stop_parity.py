"""ADMM stop-decision parity at BASELINE scale (same iteration
counts). The device diffusion result (bit-identical to the reference's) is
normalised on both sides (bitwise) and handed to the device ADMM and to the
compiled reference's admm_face_optimize / admm_edge_optimize. The residual
norms are the only values summed in a different order (tree vs left-to-right),
so the record is: iteration counts and converged flags (must match), and the
largest relative difference between the two residual histories — how close a
residual would have to land to its threshold for the stop decision to flip.

    python tools/admm_stop_parity.py [--configs 2,3] [--iters 10,100]
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


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3")
    ap.add_argument("--iters", default="10,100")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "admm_stop_parity.json"))
    args = ap.parse_args()
    ref = Oracle("reference")
    out = []
    for k in [int(x) for x in args.configs.split(",")]:
        w = meshgen.config(k)
        mesh = g.build_mesh(w.positions, w.faces)
        lv = g.bfs_levels(mesh, w.sources)
        t = w.t if w.t is not None else g.diffusion_time(mesh, w.m)
        u = g.gs_diffuse(mesh, lv, t, g.DiffusionConfig(sweeps=w.sweeps))
        nt = g.normalized_target_gradients(mesh, u)
        om = ref.build_mesh(w.positions, w.faces)
        H_ref, zc_ref = om.normalized_target_gradients(u)
        assert np.array_equal(nt.field, H_ref) and nt.zero_count == zc_ref
        for method in ("face", "edge"):
            for iters in [int(x) for x in args.iters.split(",")]:
                cfg = g.AdmmConfig(max_iterations=iters)
                t0 = time.perf_counter()
                if method == "face":
                    res = g.admm_face_optimize(mesh, nt.field, cfg)
                    ours_out = res.gradients
                else:
                    res = g.admm_edge_optimize(mesh, nt.field, cfg)
                    ours_out = res.differences
                t1 = time.perf_counter()
                fn = om.admm_face if method == "face" else om.admm_edge
                r_out, rr = fn(H_ref, iters)
                t2 = time.perf_counter()
                rec = {
                    "config": k, "name": w.name, "method": method, "max_iterations": iters,
                    "iterations": [res.report.iterations, rr.iterations],
                    "converged": [res.report.converged, rr.converged],
                    "same_decision": res.report.iterations == rr.iterations and res.report.converged == rr.converged,
                    "primal_hist_max_rel_diff": rel(res.report.primal_history, rr.primal_history),
                    "dual_hist_max_rel_diff": rel(res.report.dual_history, rr.dual_history),
                    "final_primal": [res.report.final_primal, rr.final_primal],
                    "final_dual": [res.report.final_dual, rr.final_dual],
                    "output_max_rel_diff": rel(np.ravel(ours_out), np.ravel(r_out)),
                    "output_bitwise": bool(np.array_equal(np.ravel(ours_out), np.ravel(r_out))),
                    "device_s": t1 - t0, "reference_s": t2 - t1,
                }
                out.append(rec)
                print(json.dumps(rec), flush=True)
        del om, mesh, lv
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
