"""Seeded synthetic meshes for BASELINE.json configs 1-5 (host C, workloads/meshgen.c).

The reference measures no public dataset; these generators stand in for the
paper's scanned models with the shapes, sizes and value distributions
BASELINE.json names. Both the GPU path and the CPU oracle consume the same
arrays. Formulas and seeds: DESIGN.md §5.

The generator library is lib/libgh_meshgen.so by default; the CPU reference
arm of bench.py calls use_library() with its own build of the same source
(oracle/_ref/libgh_meshgen.so), so that process maps nothing of the product.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _build

SEEDS = {k: 1812060600 + k for k in range(1, 6)}

_lib = None
_lib_path = None


def use_library(path: str) -> None:
    """Load the generators from `path` (a build of workloads/meshgen.c) instead."""
    global _lib, _lib_path
    if _lib is not None and _lib_path != path:
        raise RuntimeError("meshgen: a generator library is already loaded")
    _lib_path = path


def _load():
    global _lib, _lib_path
    if _lib is None:
        if _lib_path is None:
            if not os.path.exists(_build.MESHGEN_LIB):
                _build.build_meshgen()
            _lib_path = _build.MESHGEN_LIB
        L = C.CDLL(_lib_path)
        PP = C.POINTER(C.POINTER(C.c_double))
        PI = C.POINTER(C.POINTER(C.c_int32))
        i32p = C.POINTER(C.c_int32)
        L.gh_gen_icosphere.argtypes = [C.c_int32, C.c_double, PP, i32p, PI, i32p]
        L.gh_gen_torus.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_int32,
                                   i32p, PP, i32p, PI, i32p]
        L.gh_gen_grid.argtypes = [C.c_int32, C.c_double, C.c_double, C.c_uint64, PP, i32p, PI, i32p]
        L.gh_gen_sh_displace.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_double, C.c_uint64]
        L.gh_gen_free.argtypes = [C.c_void_p]
        L.gh_gen_mt64_first.argtypes = [C.c_uint64]
        L.gh_gen_mt64_first.restype = C.c_uint64
        _lib = L
    return _lib


def _take(pos, nv, faces, nf):
    L = _load()
    P = np.ctypeslib.as_array(pos, shape=(nv.value, 3)).copy()
    Fc = np.ctypeslib.as_array(faces, shape=(nf.value, 3)).copy()
    L.gh_gen_free(pos)
    L.gh_gen_free(faces)
    return P, Fc


def icosphere(subdivisions: int, radius: float = 1.0):
    """icosphere_mesh (reference tests/test_meshes.hpp:94-129), identical vertex order."""
    pos, faces = C.POINTER(C.c_double)(), C.POINTER(C.c_int32)()
    nv, nf = C.c_int32(), C.c_int32()
    rc = _load().gh_gen_icosphere(subdivisions, radius, C.byref(pos), C.byref(nv), C.byref(faces), C.byref(nf))
    if rc:
        raise MemoryError(f"icosphere({subdivisions}): rc={rc}")
    return _take(pos, nv, faces, nf)


def torus(nu: int, nv_: int, big_radius: float = 2.0, tube_radius: float = 0.7, sigma: float = 0.0, seed: int = 0,
          nsources: int = 0):
    """torus_mesh (test_meshes.hpp:132-153) + seeded tube-normal noise and sources."""
    pos, faces = C.POINTER(C.c_double)(), C.POINTER(C.c_int32)()
    nv, nf = C.c_int32(), C.c_int32()
    src = np.zeros(max(nsources, 1), np.int32)
    rc = _load().gh_gen_torus(nu, nv_, big_radius, tube_radius, sigma, seed, nsources,
                              src.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(pos), C.byref(nv), C.byref(faces),
                              C.byref(nf))
    if rc:
        raise MemoryError(f"torus({nu},{nv_}): rc={rc}")
    P, Fc = _take(pos, nv, faces, nf)
    return P, Fc, src[:nsources]


def grid(n: int, jitter: float = 0.0, amp: float = 0.0, seed: int = 0):
    """n x n jittered grid with alternating diagonals (config 2)."""
    pos, faces = C.POINTER(C.c_double)(), C.POINTER(C.c_int32)()
    nv, nf = C.c_int32(), C.c_int32()
    rc = _load().gh_gen_grid(n, jitter, amp, seed, C.byref(pos), C.byref(nv), C.byref(faces), C.byref(nf))
    if rc:
        raise MemoryError(f"grid({n}): rc={rc}")
    return _take(pos, nv, faces, nf)


def sh_displace(P: np.ndarray, lmax: int = 8, amplitude: float = 0.05, seed: int = 0) -> np.ndarray:
    P = np.ascontiguousarray(P, dtype=np.float64)
    rc = _load().gh_gen_sh_displace(P.ctypes.data_as(C.c_void_p), P.shape[0], lmax, amplitude, seed)
    if rc:
        raise ValueError(f"sh_displace rc={rc}")
    return P


@dataclass
class Workload:
    name: str
    positions: np.ndarray
    faces: np.ndarray
    sources: np.ndarray
    t: Optional[float]     # None: t = m * (mean edge)^2 computed from the mesh
    m: float
    method: str
    sweeps: int = 1000
    admm_iters: int = 10


def config(k: int, scale: int = 1) -> Workload:
    """BASELINE.json configs[k-1]; `scale` > 1 shrinks the grid/torus linearly
    (same topology, fewer vertices) for fast parity tests."""
    seed = SEEDS[k]
    if k == 1:
        P, Fc = icosphere(5)
        return Workload("icosphere5", P, Fc, np.array([0], np.int32), None, 1.0, "face")
    if k == 2:
        n = (1024 // scale) + 1
        P, Fc = grid(n, jitter=0.2, amp=0.02, seed=seed)
        h = 1.0 / (n - 1)
        centre = (n // 2) * n + n // 2
        return Workload(f"grid{n}", P, Fc, np.array([centre], np.int32), h * h, 1.0, "face")
    if k == 3:
        nu, nvv = 4096 // scale, 2048 // scale
        P, Fc, S = torus(nu, nvv, 1.0, 0.3, 1e-3 * 0.3, seed, 4)
        return Workload(f"torus{nu}x{nvv}", P, Fc, S, None, 1.0, "face")
    if k == 4:
        level = 11
        while scale > 1 and level > 3:
            scale //= 2
            level -= 1
        P, Fc = icosphere(level)
        P = sh_displace(P, 8, 0.05, seed)
        return Workload(f"icosphere{level}_sh", P, Fc, np.array([0], np.int32), None, 1.0, "face")
    if k == 5:
        nu, nvv = 16384 // scale, 12288 // scale
        P, Fc, S = torus(nu, nvv, 1.0, 0.3, 1e-4 * 0.3, seed, 1)
        return Workload(f"torus{nu}x{nvv}", P, Fc, S, None, 1.0, "edge")
    raise KeyError(k)
