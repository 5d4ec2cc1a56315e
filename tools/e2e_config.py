"""End-to-end solve of a BASELINE config through gh_distance_host (host arrays in,
host distances out), twice, with stage timings and a determinism check.

    python tools/e2e_config.py CONFIG [SWEEPS [REPEATS [skip]]]   # "skip": the opt-in exact-zero skipping on
"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1812_06060_b200 import geoheat as G, meshgen  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
repeats = int(sys.argv[3]) if len(sys.argv) > 3 else 2
skip = len(sys.argv) > 4 and sys.argv[4] == "skip"
G.set_zero_level_truncation(skip)
t0 = time.time()
w = meshgen.config(cfg)
gen_s = time.time() - t0
L = G._lib.load()
P = np.ascontiguousarray(w.positions)
F = np.ascontiguousarray(w.faces, dtype=np.int32)
S = np.ascontiguousarray(w.sources, dtype=np.int32)
pp, pf, pd = C.c_void_p(), C.c_void_p(), C.c_void_p()
for ptr, nb in ((pp, P.nbytes), (pf, F.nbytes), (pd, 8 * P.shape[0])):
    G._check(L.gh_host_alloc(nb, C.byref(ptr)))
C.memmove(pp, P.ctypes.data, P.nbytes)
C.memmove(pf, F.ctypes.data, F.nbytes)
pcfg = G._pipeline_config(w.method, sweeps, w.t, w.m, G.AdmmConfig())
hashes = []
for it in range(repeats):
    rr = G.gh_run_report()
    t1 = time.perf_counter()
    G._check(L.gh_distance_host(pp, P.shape[0], pf, F.shape[0], S.ctypes.data_as(C.c_void_p), S.size, C.byref(pcfg),
                                pd, C.byref(rr)))
    wall = time.perf_counter() - t1
    d = np.ctypeslib.as_array((C.c_double * P.shape[0]).from_address(pd.value))
    hashes.append(G.field_hash(d))
    fin = np.isfinite(d)
    out = dict(zero_skipping=skip, config=cfg, name=w.name, method=w.method, vertices=int(P.shape[0]), faces=int(F.shape[0]), sweeps=sweeps,
               iteration=it, wall_s=wall, t=rr.t, build_ms=rr.build_ms, bfs_ms=rr.bfs_ms, diffusion_ms=rr.diffusion_ms,
               normalize_ms=rr.normalize_ms, admm_ms=rr.optimization_ms, integrate_ms=rr.integration_ms,
               admm_iterations=rr.admm_iterations, converged=bool(rr.converged), zero_count=rr.zero_count,
               vertex_updates_per_s=int(rr.diffusion_row_updates) / (rr.diffusion_ms * 1e-3),  # executed
               row_updates_executed=int(rr.diffusion_row_updates), row_updates_nominal=int(P.shape[0]) * sweeps,
               diffusion_active_levels=int(rr.diffusion_active_levels), diffusion_launches=int(rr.diffusion_launches),
               finite=int(fin.sum()), d_max=float(d[fin].max()), hash=f"{hashes[-1]:016x}", meshgen_s=gen_s)
    print(json.dumps(out), flush=True)
print(json.dumps({"deterministic": len(set(hashes)) == 1}))
