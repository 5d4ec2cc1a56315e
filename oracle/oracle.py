"""TEST INFRASTRUCTURE ONLY — ctypes front end for the CPU parity oracles.

Loads either oracle/_ref/libgeoheat_ref.so (the unmodified reference headers,
built by oracle/build_ref.sh) or oracle/_ref/libgeoheat_port.so (the plain-C
restatement oracle/geoheat_oracle.c). Both export the API of
oracle/geoheat_oracle.h. Only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline legs may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

ARRAYS = [
    ("positions", np.float64), ("faces", np.int32), ("halfedge_twin", np.int32),
    ("halfedge_edge", np.int32), ("edge_vertices", np.int32), ("edge_halfedges", np.int32),
    ("interior_edges", np.int32), ("interior_edge_index", np.int32), ("vertex_on_boundary", np.uint8),
    ("face_area", np.float64), ("face_normal", np.float64), ("vertex_area", np.float64),
    ("halfedge_cot", np.float64), ("edge_weight", np.float64), ("vertex_weight_sum", np.float64),
    ("vv_offset", np.int32), ("vv_index", np.int32), ("vv_edge", np.int32), ("vv_weight", np.float64),
    ("vc_offset", np.int32), ("vc_corner", np.int32),
]
ARRAY_ID = {name: i for i, (name, _) in enumerate(ARRAYS)}


class OracleMeshError(RuntimeError):
    pass


class _Report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("converged", C.c_int32), ("final_primal", C.c_double),
        ("final_dual", C.c_double), ("primal_history", C.POINTER(C.c_double)),
        ("dual_history", C.POINTER(C.c_double)), ("history_capacity", C.c_int32),
        ("state_bytes_formula", C.c_uint64), ("state_bytes_allocated", C.c_uint64),
        ("wall_seconds", C.c_double),
    ]


@dataclass
class OracleReport:
    iterations: int = 0
    converged: bool = False
    final_primal: float = 0.0
    final_dual: float = 0.0
    primal_history: list = field(default_factory=list)
    dual_history: list = field(default_factory=list)
    state_bytes_formula: int = 0
    state_bytes_allocated: int = 0
    wall_seconds: float = 0.0


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def build(quiet: bool = True) -> None:
    """Compile the oracle libraries (oracle/build_ref.sh)."""
    subprocess.run(["bash", os.path.join(HERE, "build_ref.sh")], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def lib_path(kind: str) -> str:
    return os.path.join(REF_DIR, "libgeoheat_ref.so" if kind == "reference" else "libgeoheat_port.so")


def available(kind: str) -> bool:
    return os.path.exists(lib_path(kind))


class Oracle:
    """One loaded oracle library: kind 'reference' (oracle/_ref) or 'port'."""

    def __init__(self, kind: str = "port"):
        path = lib_path(kind)
        if not os.path.exists(path):
            if kind == "port" or os.path.isdir("/root/reference/proj/include"):
                build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.kind = kind
        self.lib = L = C.CDLL(path)
        vp, i32, f64 = C.c_void_p, C.c_int32, C.c_double
        L.gho_build_mesh.argtypes = [vp, i32, vp, i32, C.POINTER(vp), C.c_char_p, i32]
        L.gho_mesh_free.argtypes = [vp]
        L.gho_mesh_counts.argtypes = [vp, vp]
        L.gho_mesh_array.argtypes = [vp, i32, C.POINTER(C.c_int64)]
        L.gho_mesh_array.restype = vp
        L.gho_average_edge_length.argtypes = [vp]
        L.gho_average_edge_length.restype = f64
        L.gho_triangulation_quality.argtypes = [vp]
        L.gho_triangulation_quality.restype = f64
        L.gho_bfs.argtypes = [vp, vp, i32, C.POINTER(vp), C.c_char_p, i32]
        L.gho_levels_free.argtypes = [vp]
        L.gho_levels_info.argtypes = [vp, vp]
        L.gho_levels_get.argtypes = [vp, vp, vp, vp, vp]
        L.gho_set_threads.argtypes = [i32]
        L.gho_gs_diffuse.argtypes = [vp, vp, f64, i32, vp, vp, C.POINTER(_Report)]
        L.gho_gs_diffuse_tol.argtypes = [vp, vp, f64, i32, f64, vp, vp, C.POINTER(_Report)]
        L.gho_diffusion_residual.argtypes = [vp, vp, f64, vp, i32]
        L.gho_diffusion_residual.restype = f64
        L.gho_face_gradient.argtypes = [vp, vp, vp]
        L.gho_normalized_target_gradients.argtypes = [vp, vp, vp]
        L.gho_normalized_target_gradients.restype = i32
        for fn in (L.gho_admm_face, L.gho_admm_edge):
            fn.argtypes = [vp, vp, i32, f64, f64, f64, vp, C.POINTER(_Report)]
        L.gho_integrate_face.argtypes = [vp, vp, vp, vp]
        L.gho_integrate_edge.argtypes = [vp, vp, vp, vp]
        L.gho_field_hash.argtypes = [vp, C.c_int64]
        L.gho_field_hash.restype = C.c_uint64
        if kind == "reference":
            L.gho_ref_test_mesh.argtypes = [C.c_char_p, vp, i32, C.POINTER(C.POINTER(C.c_double)),
                                            C.POINTER(i32), C.POINTER(C.POINTER(C.c_int32)), C.POINTER(i32)]
            L.gho_ref_free.argtypes = [vp]
            L.gho_ref_analytic.argtypes = [vp, i32, vp, i32, vp]
            L.gho_ref_mean_relative_error.argtypes = [vp, vp, C.c_int64, vp, i32]
            L.gho_ref_mean_relative_error.restype = f64
            L.gho_ref_load_mesh.argtypes = [C.c_char_p, C.c_int64, i32, C.POINTER(vp), C.c_char_p, i32]
            L.gho_ref_save_mesh.argtypes = [vp, i32, vp, C.POINTER(C.c_int64)]
            L.gho_ref_save_mesh.restype = C.POINTER(C.c_char)
            L.gho_ref_write_distances.argtypes = [vp, C.c_int64, i32, C.POINTER(C.c_int64)]
            L.gho_ref_write_distances.restype = C.POINTER(C.c_char)
            L.gho_ref_poisson.argtypes = [vp, vp, i32, f64, f64, vp, vp, vp, C.c_char_p, i32]
            L.gho_ref_dijkstra.argtypes = [vp, vp, i32, vp]
            L.gho_ref_subdivide.argtypes = [vp, i32]
            L.gho_ref_subdivide.restype = vp
            L.gho_ref_recovery_error.argtypes = [vp, vp, C.c_int64]
            L.gho_ref_recovery_error.restype = f64
            L.gho_ref_mre_excluded.argtypes = [vp, vp, C.c_int64, vp, i32]
            L.gho_ref_mre_excluded.restype = i32

    # ---- mesh
    def build_mesh(self, positions, faces) -> "OMesh":
        pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        fc = np.ascontiguousarray(faces, dtype=np.int32).reshape(-1, 3)
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = self.lib.gho_build_mesh(_p(pos), pos.shape[0], _p(fc), fc.shape[0], C.byref(h), err, 512)
        if rc == 1:
            raise OracleMeshError(err.value.decode())
        if rc != 0:
            raise ValueError(err.value.decode())
        return OMesh(self, h)

    def set_threads(self, n: int) -> None:
        self.lib.gho_set_threads(int(n))

    def field_hash(self, values) -> int:
        v = np.ascontiguousarray(values, dtype=np.float64)
        return int(self.lib.gho_field_hash(_p(v), v.size))

    # ---- reference-only extras
    def test_mesh(self, name: str, *params):
        assert self.kind == "reference"
        pr = np.asarray(params, dtype=np.float64)
        pos = C.POINTER(C.c_double)()
        fcs = C.POINTER(C.c_int32)()
        nv, nf = C.c_int32(), C.c_int32()
        rc = self.lib.gho_ref_test_mesh(name.encode(), _p(pr) if pr.size else None, pr.size, C.byref(pos),
                                        C.byref(nv), C.byref(fcs), C.byref(nf))
        if rc != 0:
            raise ValueError(f"test mesh {name}: rc={rc}")
        P = np.ctypeslib.as_array(pos, shape=(nv.value, 3)).copy()
        Fa = np.ctypeslib.as_array(fcs, shape=(nf.value, 3)).copy()
        self.lib.gho_ref_free(pos)
        self.lib.gho_ref_free(fcs)
        return P, Fa


    def load_mesh(self, data: bytes, fmt: int) -> "OMesh":
        """load_mesh(istream, format) of the reference (0 OBJ, 1 PLY); raises
        OracleMeshError with the reference's exception text."""
        assert self.kind == "reference"
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = self.lib.gho_ref_load_mesh(data, len(data), int(fmt), C.byref(h), err, 1024)
        if rc != 0:
            raise OracleMeshError(err.value.decode(errors="replace"))
        return OMesh(self, h)

    def _take(self, ptr, n) -> bytes:
        out = C.string_at(ptr, n.value)
        self.lib.gho_ref_free(ptr)
        return out

    def save_mesh(self, mesh: "OMesh", fmt: int, quality=None) -> bytes:
        assert self.kind == "reference"
        q = None if quality is None else np.ascontiguousarray(quality, dtype=np.float64)
        n = C.c_int64()
        ptr = self.lib.gho_ref_save_mesh(mesh.h, int(fmt), _p(q) if q is not None else None, C.byref(n))
        return self._take(ptr, n)

    def poisson(self, mesh: "OMesh", sources, t: float, tol: float):
        """poisson_heat_method -> (d, (heat_it, poisson_it), (heat_res, poisson_res))."""
        assert self.kind == "reference"
        S = np.ascontiguousarray(sources, dtype=np.int32)
        d = np.empty(mesh.nv, np.float64)
        it = np.zeros(2, np.int32)
        res = np.zeros(2, np.float64)
        err = C.create_string_buffer(512)
        if self.lib.gho_ref_poisson(mesh.h, _p(S), S.size, float(t), float(tol), _p(d), _p(it), _p(res), err, 512):
            raise OracleMeshError(err.value.decode())
        return d, (int(it[0]), int(it[1])), (float(res[0]), float(res[1]))

    def dijkstra(self, mesh: "OMesh", sources) -> np.ndarray:
        assert self.kind == "reference"
        S = np.ascontiguousarray(sources, dtype=np.int32)
        d = np.empty(mesh.nv, np.float64)
        self.lib.gho_ref_dijkstra(mesh.h, _p(S), S.size, _p(d))
        return d

    def subdivide(self, mesh: "OMesh", levels: int) -> "OMesh":
        assert self.kind == "reference"
        return OMesh(self, C.c_void_p(self.lib.gho_ref_subdivide(mesh.h, int(levels))))

    def recovery_error(self, d, d_ref) -> float:
        a, b = np.ascontiguousarray(d, np.float64), np.ascontiguousarray(d_ref, np.float64)
        return float(self.lib.gho_ref_recovery_error(_p(a), _p(b), a.size))

    def mre_excluded(self, d, d_ref, sources) -> int:
        a, b = np.ascontiguousarray(d, np.float64), np.ascontiguousarray(d_ref, np.float64)
        S = np.ascontiguousarray(sources, dtype=np.int32)
        return int(self.lib.gho_ref_mre_excluded(_p(a), _p(b), a.size, _p(S), S.size))

    def write_distances(self, d, csv: bool) -> bytes:
        assert self.kind == "reference"
        v = np.ascontiguousarray(d, dtype=np.float64)
        n = C.c_int64()
        ptr = self.lib.gho_ref_write_distances(_p(v), v.size, 1 if csv else 0, C.byref(n))
        return self._take(ptr, n)


class OMesh:
    def __init__(self, oracle: Oracle, handle):
        self.o, self.h, self.L = oracle, handle, oracle.lib
        c = np.zeros(4, np.int32)
        self.L.gho_mesh_counts(self.h, _p(c))
        self.nv, self.nf, self.ne, self.ni = (int(x) for x in c)

    def __del__(self):
        try:
            self.L.gho_mesh_free(self.h)
        except Exception:
            pass

    def array(self, name: str) -> np.ndarray:
        n = C.c_int64()
        ptr = self.L.gho_mesh_array(self.h, ARRAY_ID[name], C.byref(n))
        dt = dict(ARRAYS)[name]
        if n.value == 0:
            return np.zeros(0, dt)
        buf = (C.c_char * (n.value * np.dtype(dt).itemsize)).from_address(ptr)
        return np.frombuffer(buf, dtype=dt).copy()

    def average_edge_length(self) -> float:
        return float(self.L.gho_average_edge_length(self.h))

    def triangulation_quality(self) -> float:
        return float(self.L.gho_triangulation_quality(self.h))

    def diffusion_time(self, m: float = 1.0) -> float:
        h = self.average_edge_length()
        return m * h * h

    def bfs(self, sources) -> "OLevels":
        s = np.ascontiguousarray(sources, dtype=np.int32)
        h = C.c_void_p()
        err = C.create_string_buffer(256)
        rc = self.L.gho_bfs(self.h, _p(s) if s.size else None, s.size, C.byref(h), err, 256)
        if rc != 0:
            raise ValueError(err.value.decode())
        return OLevels(self, h)

    def gs_diffuse(self, levels: "OLevels", t: float, sweeps: int, initial=None):
        u = np.zeros(self.nv, np.float64)
        init = None if initial is None else np.ascontiguousarray(initial, dtype=np.float64)
        rep = _Report()
        rc = self.L.gho_gs_diffuse(self.h, levels.h, float(t), int(sweeps), _p(init), _p(u), C.byref(rep))
        if rc != 0:
            raise ValueError("gs_diffuse: invalid argument")
        return u, OracleReport(iterations=rep.iterations, wall_seconds=rep.wall_seconds)

    def gs_diffuse_tol(self, levels: "OLevels", t: float, sweeps: int, tolerance: float, initial=None):
        """gs_diffuse with DiffusionConfig::residual_tolerance; returns (u, report with E1 history)."""
        u = np.zeros(self.nv, np.float64)
        init = None if initial is None else np.ascontiguousarray(initial, dtype=np.float64)
        hist = np.zeros(max(int(sweeps), 1))
        rep = _Report()
        rep.primal_history = hist.ctypes.data_as(C.POINTER(C.c_double))
        rep.history_capacity = hist.size
        rc = self.L.gho_gs_diffuse_tol(self.h, levels.h, float(t), int(sweeps), float(tolerance), _p(init), _p(u),
                                       C.byref(rep))
        if rc != 0:
            raise ValueError("gs_diffuse: invalid argument")
        return u, OracleReport(iterations=rep.iterations, converged=bool(rep.converged),
                               primal_history=hist[:rep.iterations].tolist(), wall_seconds=rep.wall_seconds)

    def diffusion_residual(self, u, t, sources) -> float:
        u = np.ascontiguousarray(u, dtype=np.float64)
        s = np.ascontiguousarray(sources, dtype=np.int32)
        return float(self.L.gho_diffusion_residual(self.h, _p(u), float(t), _p(s), s.size))

    def face_gradient(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        g = np.zeros((self.nf, 3), np.float64)
        self.L.gho_face_gradient(self.h, _p(u), _p(g))
        return g

    def normalized_target_gradients(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        H = np.zeros((self.nf, 3), np.float64)
        z = self.L.gho_normalized_target_gradients(self.h, _p(u), _p(H))
        return H, int(z)

    def _admm(self, fn, H, n_out, max_iterations, eps1, eps2, mu):
        H = np.ascontiguousarray(H, dtype=np.float64)
        out = np.zeros(n_out, np.float64)
        cap = max(int(max_iterations), 1)
        ph, dh = np.zeros(cap), np.zeros(cap)
        rep = _Report()
        rep.primal_history = ph.ctypes.data_as(C.POINTER(C.c_double))
        rep.dual_history = dh.ctypes.data_as(C.POINTER(C.c_double))
        rep.history_capacity = cap
        rc = fn(self.h, _p(H), int(max_iterations), float(eps1), float(eps2), float(mu), _p(out), C.byref(rep))
        if rc != 0:
            raise ValueError("admm: invalid config")
        r = OracleReport(rep.iterations, bool(rep.converged), rep.final_primal, rep.final_dual,
                         ph[:rep.iterations].tolist(), dh[:rep.iterations].tolist(), rep.state_bytes_formula,
                         rep.state_bytes_allocated, rep.wall_seconds)
        return out, r

    def admm_face(self, H, max_iterations=10, eps1=1e-5, eps2=1e-5, mu=100.0):
        g, r = self._admm(self.L.gho_admm_face, H, 3 * self.nf, max_iterations, eps1, eps2, mu)
        return g.reshape(-1, 3), r

    def admm_edge(self, H, max_iterations=10, eps1=1e-5, eps2=1e-5, mu=100.0):
        return self._admm(self.L.gho_admm_edge, H, self.ne, max_iterations, eps1, eps2, mu)

    def integrate_face(self, levels, G):
        G = np.ascontiguousarray(G, dtype=np.float64)
        d = np.zeros(self.nv, np.float64)
        self.L.gho_integrate_face(self.h, levels.h, _p(G), _p(d))
        return d

    def integrate_edge(self, levels, X):
        X = np.ascontiguousarray(X, dtype=np.float64)
        d = np.zeros(self.nv, np.float64)
        self.L.gho_integrate_edge(self.h, levels.h, _p(X), _p(d))
        return d

    # reference-only
    def analytic(self, kind: int, sources):
        s = np.ascontiguousarray(sources, dtype=np.int32)
        d = np.zeros(self.nv, np.float64)
        rc = self.L.gho_ref_analytic(self.h, int(kind), _p(s), s.size, _p(d))
        if rc != 0:
            raise ValueError("analytic oracle rejected the mesh")
        return d

    def mean_relative_error(self, d, d_ref, sources) -> float:
        d = np.ascontiguousarray(d, dtype=np.float64)
        r = np.ascontiguousarray(d_ref, dtype=np.float64)
        s = np.ascontiguousarray(sources, dtype=np.int32)
        return float(self.L.gho_ref_mean_relative_error(_p(d), _p(r), d.size, _p(s), s.size))


class OLevels:
    def __init__(self, mesh: OMesh, handle):
        self.m, self.h, self.L = mesh, handle, mesh.L
        info = np.zeros(2, np.int32)
        self.L.gho_levels_info(self.h, _p(info))
        self.nlev, self.unreachable = int(info[0]), int(info[1])
        nv = mesh.nv
        self.level_of_vertex = np.zeros(nv, np.int32)
        self.parent_of_vertex = np.zeros(nv, np.int32)
        self.order = np.zeros(nv - self.unreachable, np.int32)
        self.offsets = np.zeros(self.nlev + 1, np.int32)
        self.L.gho_levels_get(self.h, _p(self.level_of_vertex), _p(self.parent_of_vertex), _p(self.order),
                              _p(self.offsets))

    def __del__(self):
        try:
            self.L.gho_levels_free(self.h)
        except Exception:
            pass


def run_pipeline(o: Oracle, positions, faces, sources, *, m=1.0, t=None, sweeps=1000, admm_iters=10, mu=100.0,
                 eps=1e-5, method="face"):
    """The library chain of run_pipeline (tools/geoheat.cpp:71-161) without I/O."""
    mesh = o.build_mesh(positions, faces)
    if t is None:
        t = mesh.diffusion_time(m)
    lv = mesh.bfs(sources)
    u, _ = mesh.gs_diffuse(lv, t, sweeps)
    H, zc = mesh.normalized_target_gradients(u)
    if method == "face":
        G, rep = mesh.admm_face(H, admm_iters, eps, eps, mu)
        d = mesh.integrate_face(lv, G)
        X = None
    else:
        X, rep = mesh.admm_edge(H, admm_iters, eps, eps, mu)
        d = mesh.integrate_edge(lv, X)
        G = None
    return dict(mesh=mesh, levels=lv, t=t, u=u, H=H, zero_count=zc, G=G, X=X, d=d, report=rep)
