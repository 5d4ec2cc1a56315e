"""The E1 early stop (gs_diffuse with residual_tolerance, diffusion.hpp:110-117)
at full BASELINE size against the compiled reference.

The device runs `sweeps` sweeps with a vanishing tolerance to get the E1
history, the tolerance is set to the history's value at sweep `stop` (so the
reference and the device must both stop exactly there: the rule is E1 <= tol),
and both sides run with it: stop sweep, converged flag, u and the whole E1
history must be bit-identical. Timing of the device path per sweep beside the
plain pipelined solve.

    python tools/tol_parity.py [--configs 3] [--sweeps 80] [--stop 60] [--out gpurun_out/tol_parity.json]
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
import paper_1812_06060_b200 as gh  # noqa: E402
from paper_1812_06060_b200 import meshgen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3")
    ap.add_argument("--sweeps", type=int, default=80)
    ap.add_argument("--stop", type=int, default=60)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "tol_parity.json"))
    a = ap.parse_args()
    ref = Oracle("reference")
    ref.set_threads(os.cpu_count() or 1)
    rows = []
    for k in [int(x) for x in a.configs.split(",")]:
        w = meshgen.config(k)
        mesh = gh.build_mesh(w.positions, w.faces)
        lv = gh.bfs_levels(mesh, w.sources)
        t = w.t if w.t is not None else gh.diffusion_time(mesh, w.m)
        rep = gh.SolverReport()
        gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=a.sweeps, residual_tolerance=0.0), rep)
        hist = list(rep.residual_history)
        tol = hist[a.stop - 1]
        cfg = gh.DiffusionConfig(sweeps=a.sweeps, residual_tolerance=tol)
        times = []
        for _ in range(3):
            r = gh.SolverReport()
            t0 = time.perf_counter()
            u = gh.gs_diffuse(mesh, lv, t, cfg, r)
            times.append(time.perf_counter() - t0)
        plain = []
        for _ in range(3):
            r2 = gh.SolverReport()
            t0 = time.perf_counter()
            gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=r.iterations), r2)
            plain.append(time.perf_counter() - t0)
        om = ref.build_mesh(w.positions, w.faces)
        ol = om.bfs(w.sources)
        t_ref = om.diffusion_time(w.m) if w.t is None else w.t
        c0 = time.perf_counter()
        u_ref, orep = om.gs_diffuse_tol(ol, t_ref, a.sweeps, tol)
        ref_s = time.perf_counter() - c0
        hd, hr = np.asarray(r.residual_history), np.asarray(orep.primal_history)
        row = {"config": k, "name": w.name, "vertices": int(w.positions.shape[0]), "sweeps": a.sweeps,
               "tolerance": tol, "t_identical": t == t_ref,
               "iterations": [r.iterations, orep.iterations], "converged": [r.converged, orep.converged],
               "u_bitwise": bool(np.array_equal(u.view(np.uint64), u_ref.view(np.uint64))),
               "e1_history_bitwise": bool(hd.size == hr.size and np.array_equal(hd.view(np.uint64), hr.view(np.uint64))),
               "e1_final": [float(hd[-1]), float(hr[-1])], "u_hash": f"{gh.field_hash(u):016x}",
               "device_tol_s": float(np.median(times)), "device_plain_same_sweeps_s": float(np.median(plain)),
               "device_tol_over_plain": float(np.median(times) / np.median(plain)),
               "reference_tol_s": ref_s, "reference_threads": os.cpu_count()}
        rows.append(row)
        print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(rows, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
