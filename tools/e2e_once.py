"""One end-to-end solve of a BASELINE config through gh_distance_host (host
arrays in, distances out) — the command the per-kernel ncu table is taken on:

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file K.csv python tools/e2e_once.py 3
    python tools/kernel_table.py K.csv --out profiles/r1_kernel_table.json
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1812_06060_b200 import geoheat as G, meshgen  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = meshgen.config(cfg)
L = G._lib.load()
P = np.ascontiguousarray(w.positions)
F = np.ascontiguousarray(w.faces, dtype=np.int32)
S = np.ascontiguousarray(w.sources, dtype=np.int32)
d = np.zeros(P.shape[0])
pcfg = G._pipeline_config(w.method, w.sweeps, w.t, w.m, G.AdmmConfig())
rr = G.gh_run_report()
G._check(L.gh_distance_host(P.ctypes.data_as(C.c_void_p), P.shape[0], F.ctypes.data_as(C.c_void_p), F.shape[0],
                            S.ctypes.data_as(C.c_void_p), S.size, C.byref(pcfg), d.ctypes.data_as(C.c_void_p),
                            C.byref(rr)))
print(f"config {cfg}: {rr.kernel_launches} kernel launches, hash {G.field_hash(d):016x}")
