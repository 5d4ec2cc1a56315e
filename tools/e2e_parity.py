"""The headline workload end to end against the compiled reference, bit for bit.

Runs the bench's end-to-end call (gh_distance_host: host arrays in, distances
out, t = m h^2 computed on the device) and the reference's own chain
(build_mesh, diffusion_time, bfs_levels, gs_diffuse, normalized_target_
gradients, admm_*_optimize, integrate_*; oracle/_ref, OpenMP on all host
cores) on the same BASELINE config, and records whether the distance fields
are identical (field_hash, report.hpp:145-153), the ADMM iteration counts,
converged flags and residual histories of both sides, and each ADMM
iteration's residual/threshold ratios (the stop rule grad_face.hpp:175-177,
grad_edge.hpp:168-170; the edge method's early stop is live
on large meshes).

    python tools/e2e_parity.py [--cases 2,3,3:edge,5:edge] [--sweeps N]
                               [--out gpurun_out/e2e_parity.json]

A case is `config[:method]` (the config's own method by default). The JSON
is rewritten after every case, so a run cut short keeps what it finished.
Config 5 needs ~150 GB of host memory for the reference chain.
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_1812_06060_b200 import geoheat as g  # noqa: E402
from paper_1812_06060_b200 import meshgen  # noqa: E402


def rss_gb() -> float:
    try:
        with open("/proc/self/status") as f:
            for line in f:
                if line.startswith("VmHWM:"):
                    return int(line.split()[1]) / 2**20
    except OSError:
        pass
    return -1.0


def run_case(ref: Oracle, k: int, method: str, sweeps: int, warm: int) -> dict:
    w = meshgen.config(k)
    if method:
        w.method = method
    if sweeps:
        w.sweeps = sweeps
    admm = g.AdmmConfig(max_iterations=w.admm_iters)
    nv, nf = int(w.positions.shape[0]), int(w.faces.shape[0])
    for _ in range(warm):  # module load, pool growth to this config's size
        g.distance_host(w.positions, w.faces, w.sources, method=w.method, sweeps=w.sweeps, t=w.t, m=w.m, admm=admm)
    t0 = time.perf_counter()
    d, rep = g.distance_host(w.positions, w.faces, w.sources, method=w.method, sweeps=w.sweeps, t=w.t, m=w.m,
                             admm=admm)
    t_dev = time.perf_counter() - t0
    hash_dev = f"{g.field_hash(d):016x}"
    dev = {"t": rep.t, "admm_iterations": rep.admm_iterations, "converged": rep.converged,
           "final_primal": rep.final_primal, "final_dual": rep.final_dual, "zero_count": rep.zero_count,
           "e2e_s": t_dev, "stages_ms": {"build": rep.build_ms, "bfs_layout": rep.bfs_ms,
                                         "diffusion": rep.diffusion_ms, "normalize": rep.normalize_ms,
                                         "admm": rep.optimization_ms, "integrate": rep.integration_ms}}
    print(json.dumps({"config": k, "method": w.method, "device": dev, "hash_device": hash_dev}), flush=True)

    # the reference chain stage by stage (run_pipeline, tools/geoheat.cpp:71-143)
    c0 = time.perf_counter()
    om = ref.build_mesh(w.positions, w.faces)
    sources = w.sources
    w.positions = w.faces = None  # config 5: the reference's own TriMesh is ~95 GB
    gc.collect()
    c1 = time.perf_counter()
    t_ref = w.t if w.t is not None else om.diffusion_time(w.m)
    lv = om.bfs(sources)
    nlev = lv.nlev
    c2 = time.perf_counter()
    u, _ = om.gs_diffuse(lv, t_ref, w.sweeps)
    c3 = time.perf_counter()
    H, zc = om.normalized_target_gradients(u)
    del u
    c4 = time.perf_counter()
    if w.method == "face":
        sol, orep = om.admm_face(H, w.admm_iters)
        scale = float("nan")  # the face threshold sqrt(sum (A1 + A2)) is not recomputed here
    else:
        sol, orep = om.admm_edge(H, w.admm_iters)
        scale = math.sqrt(3.0 * nf)  # grad_edge.hpp:82
    del H
    c5 = time.perf_counter()
    d_ref = om.integrate_face(lv, sol) if w.method == "face" else om.integrate_edge(lv, sol)
    c6 = time.perf_counter()
    del sol
    hash_ref = f"{ref.field_hash(d_ref):016x}"
    same = bool(np.array_equal(d.view(np.uint64), d_ref.view(np.uint64)))
    fin = np.isfinite(d) & np.isfinite(d_ref)
    rel = float(np.max(np.abs(d[fin] - d_ref[fin]) / np.maximum(np.abs(d_ref[fin]), 1e-300))) if fin.any() else 0.0
    thr = scale * 1e-5
    return {"config": k, "name": w.name, "method": w.method, "vertices": nv, "faces": nf, "levels": nlev,
            "sweeps": w.sweeps, "admm_max_iterations": w.admm_iters,
            "t_device": rep.t, "t_reference": t_ref, "t_identical": rep.t == t_ref,
            "zero_count": [rep.zero_count, zc],
            "admm_iterations": [rep.admm_iterations, orep.iterations],
            "converged": [bool(rep.converged), bool(orep.converged)],
            "final_primal": [rep.final_primal, orep.final_primal], "final_dual": [rep.final_dual, orep.final_dual],
            "reference_primal_over_threshold": [p / thr for p in orep.primal_history] if w.method == "edge" else None,
            "reference_dual_over_threshold": [x / thr for x in orep.dual_history] if w.method == "edge" else None,
            "hash_device": hash_dev, "hash_reference": hash_ref, "bitwise_identical": same,
            "max_rel_diff_finite": rel, "inf_positions_identical": bool(np.array_equal(np.isinf(d), np.isinf(d_ref))),
            "device_e2e_s": t_dev, "device_stages_ms": dev["stages_ms"],
            "reference_chain_s": c6 - c0,
            "reference_stages_ms": {"build_mesh": 1e3 * (c1 - c0), "h_t_bfs": 1e3 * (c2 - c1),
                                    "gs_diffuse": 1e3 * (c3 - c2), "normalize": 1e3 * (c4 - c3),
                                    "admm": 1e3 * (c5 - c4), "integrate": 1e3 * (c6 - c5)},
            "reference_threads": os.cpu_count(), "host_peak_rss_gb": rss_gb()}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", "--configs", dest="cases", default="2,3")
    ap.add_argument("--sweeps", type=int, default=0, help="0 = the config's own (1000)")
    ap.add_argument("--warm", type=int, default=2)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "e2e_parity.json"))
    args = ap.parse_args()
    ref = Oracle("reference")
    ref.set_threads(os.cpu_count() or 1)
    out = []
    for case in args.cases.split(","):
        k, _, method = case.partition(":")
        rec = run_case(ref, int(k), method, args.sweeps, args.warm)
        out.append(rec)
        print(json.dumps(rec), flush=True)
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
        gc.collect()


if __name__ == "__main__":
    main()
