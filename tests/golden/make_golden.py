"""Generate the golden fixtures in tests/golden/ from the reference itself.

Runs the UNMODIFIED reference headers (oracle/_ref/libgeoheat_ref.so, built by
oracle/build_ref.sh from /root/reference with the Eigen shim) on the
reference's own test meshes (proj/tests/test_meshes.hpp generators) and
records every stage of the solver loop. Needs /root/reference, so it runs in
the build container only; the .npz outputs are committed and travel.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import ARRAYS, Oracle, OracleMeshError  # noqa: E402

# (name, generator, params, sources, m or t, sweeps, admm iterations, extra)
CASES = [
    ("unit_square", "unit_square", (), [0], dict(t=1.0), 200, 10),
    ("hex_disk12_two_sources", "hex_disk", (12,), [0, 7], dict(m=1.0), 60, 10),
    ("icosphere3", "icosphere", (3,), [0], dict(m=1.0), 100, 10),
    ("icosphere5_config1", "icosphere", (5,), [0], dict(m=1.0), 1000, 10),
    ("torus60x30_three_sources", "torus", (60, 30), [0, 1, 30], dict(m=1.0), 301, 10),
    ("grid64x40_two_sources", "grid", (64, 40), [0, 2624], dict(m=1.0), 50, 10),
    ("two_disjoint_triangles", "two_disjoint_triangles", (), [0], dict(m=1.0), 7, 10),
    ("strip40_column_sources", "strip", (40,), [0, 41], dict(m=1.0), 4000, 10),
    ("ladder10", "ladder", (10,), [3], dict(m=1.0), 40, 3),
    ("polar_disk6x12", "polar_disk", (6, 12), [0], dict(m=4.0), 80, 10),
    ("uv_sphere8x16_all_iters", "uv_sphere", (8, 16), [0, 0, 5], dict(m=1.0), 30, 25),
    ("icosphere3_zero_sweeps", "icosphere", (3,), [5], dict(m=1.0), 0, 0),
    ("hex_disk5_converges", "hex_disk", (5,), [0], dict(m=1.0), 300, 400),
]

# DiffusionConfig::residual_tolerance early stop (diffusion.hpp:110-117); the first
# mirrors test_diffusion.cpp:140-154 (hex_disk_mesh(6), 10000 sweeps, 1e-8)
TOL_CASES = [
    ("tol_hex_disk6", "hex_disk", (6,), [0], 1.0, 10000, 1e-8),
    ("tol_icosphere3", "icosphere", (3,), [0, 100], 1.0, 3000, 1e-6),
    ("tol_torus24x12_never", "torus", (24, 12), [5], 1.0, 40, 1e-30),
]

# build_mesh rejection cases (mesh.hpp:133-183), from test_mesh.cpp:48-75
ERROR_CASES = [
    ("repeated_vertex", [[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 1]]),
    ("zero_area", [[0, 0, 0], [1, 0, 0], [2, 0, 0]], [[0, 1, 2]]),
    ("index_out_of_range", [[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 6]]),
    ("non_manifold", [[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1]], [[0, 1, 2], [1, 0, 3], [0, 1, 4]]),
    ("winding", [[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], [[0, 1, 2], [0, 3, 2]]),
    ("second_face_degenerate", [[0, 0, 0], [1, 0, 0], [0, 1, 0], [3, 3, 0]], [[0, 1, 2], [1, 1, 3]]),
]


def run_case(o: Oracle, name, gen, params, sources, tm, sweeps, iters):
    P, F = o.test_mesh(gen, *params)
    mesh = o.build_mesh(P, F)
    lv = mesh.bfs(sources)
    t = tm["t"] if "t" in tm else mesh.diffusion_time(tm["m"])
    u, _ = mesh.gs_diffuse(lv, t, sweeps)
    H, zc = mesh.normalized_target_gradients(u)
    G, fr = mesh.admm_face(H, iters)
    X, er = mesh.admm_edge(H, iters)
    d_face = mesh.integrate_face(lv, G)
    d_edge = mesh.integrate_edge(lv, X)
    out = dict(positions=P, faces=F, sources=np.asarray(sources, np.int32), t=np.float64(t),
               sweeps=np.int32(sweeps), admm_iters=np.int32(iters), avg_edge_length=np.float64(mesh.average_edge_length()),
               level_of_vertex=lv.level_of_vertex, parent_of_vertex=lv.parent_of_vertex, order=lv.order,
               offsets=lv.offsets, unreachable=np.int32(lv.unreachable), u=u, H=H, zero_count=np.int32(zc), G=G, X=X,
               d_face=d_face, d_edge=d_edge)
    for arr, _ in ARRAYS:
        out["mesh_" + arr] = mesh.array(arr)
    for tag, r in (("face", fr), ("edge", er)):
        out[f"{tag}_iterations"] = np.int32(r.iterations)
        out[f"{tag}_converged"] = np.int32(r.converged)
        out[f"{tag}_primal"] = np.asarray(r.primal_history)
        out[f"{tag}_dual"] = np.asarray(r.dual_history)
        out[f"{tag}_state_bytes_formula"] = np.uint64(r.state_bytes_formula)
    # warm start: `initial` (diffusion.hpp:71), 3 more sweeps from the result
    if sweeps > 0:
        u2, _ = mesh.gs_diffuse(lv, t, 3, initial=u)
        out["u_warm3"] = u2
    out["hash_d_face"] = np.uint64(o.field_hash(d_face))
    out["hash_d_edge"] = np.uint64(o.field_hash(d_edge))
    out["e1"] = np.float64(mesh.diffusion_residual(u, t, sources))
    return out


def main():
    o = Oracle("reference")
    o.set_threads(1)
    index = {}
    for name, gen, params, sources, tm, sweeps, iters in CASES:
        out = run_case(o, name, gen, params, sources, tm, sweeps, iters)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        index[name] = dict(generator=gen, params=list(params), sources=sources, sweeps=sweeps, admm_iters=iters,
                           hash_d_face=f"{int(out['hash_d_face']):016x}", hash_d_edge=f"{int(out['hash_d_edge']):016x}",
                           zero_count=int(out["zero_count"]), face_iterations=int(out["face_iterations"]),
                           edge_iterations=int(out["edge_iterations"]), face_converged=int(out["face_converged"]),
                           edge_converged=int(out["edge_converged"]))
        print(name, index[name])
    tol_index = {}
    for name, gen, params, sources, m, sweeps, tol in TOL_CASES:
        P, F = o.test_mesh(gen, *params)
        mesh = o.build_mesh(P, F)
        lv = mesh.bfs(sources)
        t = mesh.diffusion_time(m)
        u, rep = mesh.gs_diffuse_tol(lv, t, sweeps, tol)
        np.savez_compressed(os.path.join(HERE, "tol", f"{name}.npz"), positions=P, faces=F,
                            sources=np.asarray(sources, np.int32), t=np.float64(t), sweeps=np.int32(sweeps),
                            tolerance=np.float64(tol), u=u, iterations=np.int32(rep.iterations),
                            converged=np.int32(rep.converged), residual_history=np.asarray(rep.primal_history))
        tol_index[name] = dict(iterations=rep.iterations, converged=rep.converged,
                               last_e1=rep.primal_history[-1] if rep.primal_history else None)
        print(name, tol_index[name])
    errors = {}
    for name, P, F in ERROR_CASES:
        try:
            o.build_mesh(np.asarray(P, float), np.asarray(F, np.int32))
            errors[name] = None
        except OracleMeshError as e:
            errors[name] = str(e)
        except ValueError as e:
            errors[name] = "invalid: " + str(e)
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump({"cases": index, "tolerance_cases": tol_index, "errors": {n: dict(positions=P, faces=F, message=errors[n])
                                              for n, P, F in ERROR_CASES},
                   "generated_by": "tests/golden/make_golden.py with oracle/_ref/libgeoheat_ref.so"}, f, indent=1)
    print(json.dumps(errors, indent=1))


if __name__ == "__main__":
    main()
