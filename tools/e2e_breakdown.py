"""Wall-clock breakdown of one end-to-end solve through the C ABI (config 3)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1812_06060_b200 as gh  # noqa: E402
from paper_1812_06060_b200 import geoheat as G, meshgen  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = meshgen.config(cfg)
L = G._lib.load()
P = np.ascontiguousarray(w.positions)
F = np.ascontiguousarray(w.faces, dtype=np.int32)
S = np.ascontiguousarray(w.sources, dtype=np.int32)
pp, pf, pd = C.c_void_p(), C.c_void_p(), C.c_void_p()
for ptr, nb in ((pp, P.nbytes), (pf, F.nbytes), (pd, 8 * P.shape[0])):
    G._check(L.gh_host_alloc(nb, C.byref(ptr)))
C.memmove(pp, P.ctypes.data, P.nbytes)
C.memmove(pf, F.ctypes.data, F.nbytes)
pcfg = G._pipeline_config(w.method, w.sweeps, w.t, w.m, G.AdmmConfig())
try:  # the default memory pool's reserved / used bytes (stream-ordered allocations)
    _rt = C.CDLL("/usr/local/cuda/lib64/libcudart.so.12")
except OSError:
    _rt = None


def pool_gb():
    if _rt is None:
        return ""
    pool = C.c_void_p()
    _rt.cudaDeviceGetDefaultMemPool(C.byref(pool), 0)
    out = []
    for attr in (5, 7):  # cudaMemPoolAttrReservedMemCurrent, cudaMemPoolAttrUsedMemCurrent
        v = C.c_uint64()
        _rt.cudaMemPoolGetAttribute(pool, attr, C.byref(v))
        out.append(v.value / 1e9)
    return f" pool reserved {out[0]:.2f} GB used {out[1]:.2f} GB"
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    t0 = time.perf_counter()
    m = C.c_void_p()
    G._check(L.gh_mesh_create(pp, P.shape[0], pf, F.shape[0], C.byref(m)))
    t1 = time.perf_counter()
    lv = C.c_void_p()
    G._check(L.gh_bfs_create(m, S.ctypes.data_as(C.c_void_p), S.size, C.byref(lv)))
    t2 = time.perf_counter()
    rr = G.gh_run_report()
    G._check(L.gh_distance(lv, C.byref(pcfg), pd, C.byref(rr)))
    t3 = time.perf_counter()
    L.gh_bfs_destroy(lv)
    t4 = time.perf_counter()
    L.gh_mesh_destroy(m)
    t5 = time.perf_counter()
    print(f"iter {it}: create {1e3*(t1-t0):.1f} bfs {1e3*(t2-t1):.1f} distance {1e3*(t3-t2):.1f} "
          f"(diff {rr.diffusion_ms:.1f} norm {rr.normalize_ms:.1f} admm {rr.optimization_ms:.1f} int {rr.integration_ms:.1f} "
          f"total_ev {rr.total_ms:.1f}) destroy_lv {1e3*(t4-t3):.1f} destroy_mesh {1e3*(t5-t4):.1f} "
          f"all {1e3*(t5-t0):.1f} ms", flush=True)
    t0 = time.perf_counter()
    rr = G.gh_run_report()
    G._check(L.gh_distance_host(pp, P.shape[0], pf, F.shape[0], S.ctypes.data_as(C.c_void_p), S.size, C.byref(pcfg),
                                pd, C.byref(rr)))
    print(f"   distance_host {1e3*(time.perf_counter()-t0):.1f} ms (report total {rr.total_ms:.1f}, "
          f"admm {rr.optimization_ms:.1f}){pool_gb()}", flush=True)
