"""Python mirror of the reference's `geoheat` solver-loop API, on the B200 path.

Same names, argument meaning and error behaviour as the reference C++ API
(reference/proj/include/geoheat/*.hpp), so parity tests read like the
reference's own tests. Every call goes through the C ABI of
include/geoheat_b200.h (lib/libgeoheat_b200.so); nothing here computes the
solver loop on the CPU. Exceptions:
  MeshError      <- GH_ERR_MESH     (geoheat::MeshError, common.hpp:30-32)
  ValueError     <- GH_ERR_INVALID  (std::invalid_argument)
  SolverError    <- GH_ERR_SOLVER   (geoheat::SolverError, common.hpp:35-37)
  GeoheatCudaError <- GH_ERR_CUDA / no device
"""
from __future__ import annotations

import atexit
import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import gh_admm_config, gh_levels_info, gh_mesh_info, gh_pipeline_config, gh_run_report, gh_solver_report


_SHUTTING_DOWN = [False]


@atexit.register
def _mark_shutdown() -> None:
    # handles still alive at interpreter exit are left to process teardown
    _SHUTTING_DOWN[0] = True


class MeshError(RuntimeError):
    pass


class SolverError(RuntimeError):
    pass


class GeoheatCudaError(RuntimeError):
    pass


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = _lib.load().gh_last_error().decode()
    if rc == 1:
        raise MeshError(msg)
    if rc == 2:
        raise ValueError(msg)
    if rc == 3:
        raise SolverError(msg)
    raise GeoheatCudaError(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


MESH_ARRAYS = [
    ("positions", np.float64, 3, "V"), ("faces", np.int32, 3, "F"), ("halfedge_twin", np.int32, 1, "H"),
    ("halfedge_edge", np.int32, 1, "H"), ("edge_vertices", np.int32, 2, "E"), ("edge_halfedges", np.int32, 2, "E"),
    ("interior_edges", np.int32, 1, "I"), ("interior_edge_index", np.int32, 1, "E"),
    ("vertex_on_boundary", np.uint8, 1, "V"), ("face_area", np.float64, 1, "F"), ("face_normal", np.float64, 3, "F"),
    ("vertex_area", np.float64, 1, "V"), ("halfedge_cot", np.float64, 1, "H"), ("edge_weight", np.float64, 1, "E"),
    ("vertex_weight_sum", np.float64, 1, "V"), ("vv_offset", np.int32, 1, "V+1"), ("vv_index", np.int32, 1, "2E"),
    ("vv_edge", np.int32, 1, "2E"), ("vv_weight", np.float64, 1, "2E"), ("vc_offset", np.int32, 1, "V+1"),
    ("vc_corner", np.int32, 1, "H"),
]


# ---------------------------------------------------------------- configs / reports
@dataclass
class DiffusionConfig:
    """DiffusionConfig (diffusion.hpp:16-25)."""
    m: float = 1.0
    sweeps: int = 1000
    residual_tolerance: Optional[float] = None

    def validate(self) -> None:
        if not self.m > 0.0:
            raise ValueError("DiffusionConfig: m must be positive")
        if self.sweeps < 0:
            raise ValueError("DiffusionConfig: sweeps must be >= 0")


@dataclass
class AdmmConfig:
    """AdmmConfig (grad_face.hpp:15-26)."""
    max_iterations: int = 10
    eps1: float = 1e-5
    eps2: float = 1e-5
    mu: float = 100.0

    def validate(self) -> None:
        if self.max_iterations < 0:
            raise ValueError("AdmmConfig: max_iterations must be >= 0")
        if not (self.eps1 > 0.0 and self.eps2 > 0.0):
            raise ValueError("AdmmConfig: eps must be positive")
        if not self.mu > 0.0:
            raise ValueError("AdmmConfig: mu must be positive")

    def _c(self) -> gh_admm_config:
        return gh_admm_config(int(self.max_iterations), float(self.eps1), float(self.eps2), float(self.mu))


@dataclass
class SolverReport:
    """SolverReport (report.hpp:16-27) plus device timing."""
    iterations: int = 0
    converged: bool = False
    final_primal: float = 0.0
    final_dual: float = 0.0
    primal_history: list = field(default_factory=list)
    dual_history: list = field(default_factory=list)
    residual_history: list = field(default_factory=list)
    wall_seconds: float = 0.0
    state_bytes_formula: int = 0
    state_bytes_allocated: int = 0
    device_ms: float = 0.0
    kernel_launches: int = 0


class OptimizerKind(enum.IntEnum):
    Face = 0
    Edge = 1


# ---------------------------------------------------------------- mesh
class TriMesh:
    """Device-resident TriMesh (mesh.hpp:21-94) behind a gh_mesh handle."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        self._lib = _lib.load()
        info = gh_mesh_info()
        _check(self._lib.gh_mesh_get_info(self._h, C.byref(info)))
        self._nv, self._nf, self._ne, self._ni = info.vertices, info.faces, info.edges, info.interior_edges
        self.boundary_vertex_count = info.boundary_vertices
        self.device_bytes = info.device_bytes

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and not _SHUTTING_DOWN[0]:
            self._lib.gh_mesh_destroy(h)
            self._h = None

    def vertex_count(self) -> int:
        return self._nv

    def face_count(self) -> int:
        return self._nf

    def edge_count(self) -> int:
        return self._ne

    def halfedge_count(self) -> int:
        return 3 * self._nf

    def interior_edge_count(self) -> int:
        return self._ni

    def download(self, name: str) -> np.ndarray:
        """Copy one TriMesh field to the host (parity checks)."""
        for i, (n, dt, width, size) in enumerate(MESH_ARRAYS):
            if n == name:
                count = {"V": self._nv, "F": self._nf, "H": 3 * self._nf, "E": self._ne, "I": self._ni,
                         "V+1": self._nv + 1, "2E": 2 * self._ne}[size]
                total = count * width
                out = np.empty(total, dtype=dt)
                _check(self._lib.gh_mesh_download(self._h, i, _ptr(out), total))
                return out.reshape(-1, width) if width > 1 else out
        raise KeyError(name)

    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        for n, *_ in MESH_ARRAYS:
            if n == name:
                return self.download(name)
        raise AttributeError(name)


def build_mesh(positions, faces) -> TriMesh:
    """build_mesh (mesh.hpp:113-286) on the device; raises MeshError like the reference."""
    P = _f64(positions).reshape(-1, 3)
    Fc = np.ascontiguousarray(faces, dtype=np.int32).reshape(-1, 3)
    h = C.c_void_p()
    _check(_lib.load().gh_mesh_create(_ptr(P), P.shape[0], _ptr(Fc), Fc.shape[0], C.byref(h)))
    return TriMesh(h)


# ---- mesh I/O (mesh_io.hpp)
class MeshFormat(enum.IntEnum):
    OBJ = 0
    PLY = 1


@dataclass
class LoadReport:
    format: int
    binary: bool
    device_decoded: bool
    host_threads: int
    bytes: int
    read_ms: float
    parse_ms: float
    build_ms: float
    total_ms: float
    kernel_launches: int


def _load_report(r) -> LoadReport:
    return LoadReport(r.format, bool(r.binary), bool(r.device_decoded), r.host_threads, r.bytes, r.read_ms,
                      r.parse_ms, r.build_ms, r.total_ms, r.kernel_launches)


def format_from_path(path: str) -> MeshFormat:
    """format_from_path (mesh_io.hpp:271-278)."""
    f = C.c_int32()
    _check(_lib.load().gh_mesh_format_from_path(os.fsencode(path), C.byref(f)))
    return MeshFormat(f.value)


def load_mesh(source, format: Optional[MeshFormat] = None, with_report: bool = False):
    """load_mesh (mesh_io.hpp:267-285): a path (format from its extension) or
    bytes plus a MeshFormat; returns the device TriMesh (and a LoadReport)."""
    h = C.c_void_p()
    rep = _lib.gh_load_report()
    if isinstance(source, (bytes, bytearray, memoryview)):
        if format is None:
            raise ValueError("load_mesh(bytes) needs a format")
        data = bytes(source)
        _check(_lib.load().gh_mesh_load_memory(data, len(data), int(format), C.byref(h), C.byref(rep)))
    else:
        _check(_lib.load().gh_mesh_load(os.fsencode(os.fspath(source)), C.byref(h), C.byref(rep)))
    mesh = TriMesh(h)
    return (mesh, _load_report(rep)) if with_report else mesh


def parse_mesh_text(data: bytes, format: MeshFormat, threads: int = 0):
    """Host tokeniser of the text formats: (positions [V,3], faces [F,3]) as the
    reference hands them to build_mesh."""
    L = _lib.load()
    pp, fp = C.POINTER(C.c_double)(), C.POINTER(C.c_int32)()
    nv, nf = C.c_int64(), C.c_int64()
    _check(L.gh_mesh_parse_text(bytes(data), len(data), int(format), int(threads), C.byref(pp), C.byref(nv),
                                C.byref(fp), C.byref(nf)))
    try:
        P = np.ctypeslib.as_array(pp, shape=(max(nv.value, 1) * 3,))[:3 * nv.value].copy().reshape(-1, 3)
        Fc = np.ctypeslib.as_array(fp, shape=(max(nf.value, 1) * 3,))[:3 * nf.value].copy().reshape(-1, 3)
    finally:
        L.gh_free(C.cast(pp, C.c_void_p))
        L.gh_free(C.cast(fp, C.c_void_p))
    return P, Fc


def _take_bytes(ptr: C.c_void_p, n: C.c_uint64) -> bytes:
    try:
        return C.string_at(ptr, n.value)
    finally:
        _lib.load().gh_free(ptr)


def serialize_mesh(mesh: TriMesh, format: MeshFormat, quality=None) -> bytes:
    """save_obj / save_ply (mesh_io.hpp:287-319) to bytes."""
    q = None if quality is None else _f64(quality)
    ptr, n = C.c_void_p(), C.c_uint64()
    _check(_lib.load().gh_mesh_serialize(mesh._h, int(format), _ptr(q), C.byref(ptr), C.byref(n)))
    return _take_bytes(ptr, n)


def save_mesh(path: str, mesh: TriMesh, quality=None) -> None:
    """save_mesh (mesh_io.hpp:321-326); quality adds save_ply's per-vertex property."""
    q = None if quality is None else _f64(quality)
    _check(_lib.load().gh_mesh_save(mesh._h, os.fsencode(os.fspath(path)), _ptr(q)))


def format_distances(d, csv: bool = False) -> bytes:
    """write_distances_txt / write_distances_csv (mesh_io.hpp:329-344) to bytes."""
    v = _f64(d)
    ptr, n = C.c_void_p(), C.c_uint64()
    _check(_lib.load().gh_format_distances(_ptr(v), v.size, 1 if csv else 0, C.byref(ptr), C.byref(n)))
    return _take_bytes(ptr, n)


def write_distances(path: str, d, csv: bool = False) -> None:
    v = _f64(d)
    _check(_lib.load().gh_write_distances(os.fsencode(os.fspath(path)), _ptr(v), v.size, 1 if csv else 0))


def average_edge_length(mesh: TriMesh) -> float:
    """average_edge_length (mesh.hpp:289-293); deterministic tree sum on the device."""
    h = C.c_double()
    _check(mesh._lib.gh_average_edge_length(mesh._h, C.byref(h)))
    return h.value


def diffusion_time(mesh: TriMesh, m: float) -> float:
    """diffusion_time (diffusion.hpp:28-32): t = m * h^2."""
    t = C.c_double()
    _check(mesh._lib.gh_diffusion_time(mesh._h, float(m), C.byref(t)))
    return t.value


def face_gradient(mesh: TriMesh, u) -> np.ndarray:
    """face_gradient (mesh.hpp:314-327)."""
    u = _f64(u)
    g = np.empty((mesh.face_count(), 3), np.float64)
    _check(mesh._lib.gh_face_gradient(mesh._h, _ptr(u), _ptr(g)))
    return g


# ---------------------------------------------------------------- BFS
class BfsLevels:
    """BfsLevels (bfs.hpp:15-22) behind a gh_levels handle (borrows its mesh)."""

    def __init__(self, mesh: TriMesh, handle: C.c_void_p):
        self.mesh = mesh
        self._h = handle
        self._lib = mesh._lib
        info = gh_levels_info()
        _check(self._lib.gh_bfs_get_info(self._h, C.byref(info)))
        self._nlev = info.level_count
        self.unreachable_count = info.unreachable_count
        self.max_level_width = info.max_level_width
        self._cache = None

    @property
    def column_bits(self) -> int:
        """Column width (16 or 32) the last diffusion on these levels streamed; 0 before one ran."""
        info = gh_levels_info()
        _check(self._lib.gh_bfs_get_info(self._h, C.byref(info)))
        return info.column_bits

    @property
    def diffusion_stats(self) -> dict:
        """The last gs_diffuse on these levels: levels its last launch updated, launches, launches
        redone after a too-tight truncation, vertex updates executed."""
        info = gh_levels_info()
        _check(self._lib.gh_bfs_get_info(self._h, C.byref(info)))
        return {"active_levels": info.active_levels, "launches": info.diffusion_launches,
                "retries": info.diffusion_retries, "row_updates": info.row_updates}

    @property
    def layout_levels(self) -> int:
        """Levels the diffusion layout covers (all of them, or the first rings of a mesh the heat cannot cross)."""
        info = gh_levels_info()
        _check(self._lib.gh_bfs_get_info(self._h, C.byref(info)))
        return info.layout_levels

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and not _SHUTTING_DOWN[0]:
            self._lib.gh_bfs_destroy(h)
            self._h = None

    def level_count(self) -> int:
        return self._nlev

    def u_device(self):
        """The device buffer of the diffusion result u [V] as a torch tensor (no copy)."""
        import torch
        p, n = C.c_void_p(), C.c_int64()
        _check(self._lib.gh_levels_u_device(self._h, C.byref(p), C.byref(n)))

        class _View:
            __cuda_array_interface__ = {"shape": (n.value,), "typestr": "<f8", "data": (p.value, False),
                                        "version": 3}
        return torch.as_tensor(_View(), device=f"cuda:{torch.cuda.current_device()}")

    def _arrays(self):
        if self._cache is None:
            nv = self.mesh.vertex_count()
            lv = np.empty(nv, np.int32)
            par = np.empty(nv, np.int32)
            order = np.empty(nv - self.unreachable_count, np.int32)
            off = np.empty(self._nlev + 1, np.int32)
            _check(self._lib.gh_bfs_download(self._h, _ptr(lv), _ptr(par), _ptr(order), _ptr(off)))
            self._cache = (lv, par, order, off)
        return self._cache

    @property
    def level_of_vertex(self) -> np.ndarray:
        return self._arrays()[0]

    @property
    def parent_of_vertex(self) -> np.ndarray:
        return self._arrays()[1]

    @property
    def order(self) -> np.ndarray:
        return self._arrays()[2]

    @property
    def offsets(self) -> np.ndarray:
        return self._arrays()[3]

    @property
    def levels(self):
        _, _, order, off = self._arrays()
        return [order[off[i]:off[i + 1]] for i in range(self._nlev)]


def bfs_levels(mesh: TriMesh, sources: Sequence[int]) -> BfsLevels:
    """bfs_levels (bfs.hpp:26-72); ValueError on empty / out-of-range sources."""
    s = np.ascontiguousarray(sources, dtype=np.int32)
    h = C.c_void_p()
    _check(mesh._lib.gh_bfs_create(mesh._h, _ptr(s) if s.size else None, s.size, C.byref(h)))
    return BfsLevels(mesh, h)


# ---------------------------------------------------------------- diffusion
def gs_diffuse(mesh: TriMesh, levels: BfsLevels, t: float, config: DiffusionConfig = DiffusionConfig(),
               report: Optional[SolverReport] = None, initial=None, keep_on_device: bool = False):
    """gs_diffuse (diffusion.hpp:57-124): BFS-ordered Gauss-Seidel, sweep-pipelined on the GPU.

    Returns u [V] (None with keep_on_device=True: the result stays in HBM,
    used by bench.py to time the device-resident solve)."""
    if levels.mesh is not mesh:
        raise ValueError("gs_diffuse: levels were built on a different mesh")
    config.validate()
    init = None if initial is None else _f64(initial)
    if init is not None and init.size != mesh.vertex_count():
        raise ValueError("gs_diffuse: initial has the wrong length")
    u = None if keep_on_device else np.empty(mesh.vertex_count(), np.float64)
    rep = gh_solver_report()
    if config.residual_tolerance is None:
        _check(mesh._lib.gh_gs_diffuse(levels._h, float(t), int(config.sweeps), _ptr(init), _ptr(u), C.byref(rep)))
        hist = []
    else:
        rh = np.zeros(max(int(config.sweeps), 1))
        rep.residual_history = rh.ctypes.data_as(C.POINTER(C.c_double))
        rep.history_capacity = rh.size
        _check(mesh._lib.gh_gs_diffuse_tol(levels._h, float(t), int(config.sweeps), float(config.residual_tolerance),
                                           _ptr(init), _ptr(u), C.byref(rep)))
        hist = rh[:rep.iterations].tolist()
    if report is not None:
        report.iterations = rep.iterations
        report.converged = bool(rep.converged)
        report.residual_history = hist
        report.wall_seconds = rep.wall_seconds
        report.device_ms = rep.device_ms
        report.kernel_launches = rep.kernel_launches
        report.state_bytes_allocated = rep.state_bytes_allocated
    return u


def diffusion_residual(mesh: TriMesh, u, t: float, sources: Sequence[int], levels: Optional[BfsLevels] = None) -> float:
    """diffusion_residual (diffusion.hpp:35-49): E1 = ||(A - t Lc) u - u0||."""
    if levels is None or not np.array_equal(np.unique(np.asarray(sources)), levels.levels[0]):
        levels = bfs_levels(mesh, sources)
    u = _f64(u)
    e1 = C.c_double()
    _check(mesh._lib.gh_diffusion_residual(levels._h, _ptr(u), float(t), C.byref(e1)))
    return e1.value


@dataclass
class NormalizedGradients:
    field: np.ndarray
    zero_count: int = 0


def normalized_target_gradients(mesh: TriMesh, u) -> NormalizedGradients:
    """normalized_target_gradients (diffusion.hpp:132-145)."""
    u = _f64(u)
    H = np.empty((mesh.face_count(), 3), np.float64)
    z = C.c_int32()
    _check(mesh._lib.gh_normalized_target_gradients(mesh._h, _ptr(u), _ptr(H), C.byref(z)))
    return NormalizedGradients(H, z.value)


# ---------------------------------------------------------------- ADMM
@dataclass
class FaceAdmmResult:
    gradients: np.ndarray
    report: SolverReport


@dataclass
class EdgeAdmmResult:
    differences: np.ndarray
    report: SolverReport


def _report(rep: gh_solver_report, ph, dh) -> SolverReport:
    n = rep.iterations
    return SolverReport(n, bool(rep.converged), rep.final_primal, rep.final_dual, ph[:n].tolist(), dh[:n].tolist(), [],
                        rep.wall_seconds, rep.state_bytes_formula, rep.state_bytes_allocated, rep.device_ms,
                        rep.kernel_launches)


def _solver_report_struct(cap):
    ph, dh = np.zeros(max(cap, 1)), np.zeros(max(cap, 1))
    rep = gh_solver_report()
    rep.primal_history = ph.ctypes.data_as(C.POINTER(C.c_double))
    rep.dual_history = dh.ctypes.data_as(C.POINTER(C.c_double))
    rep.history_capacity = max(cap, 1)
    return rep, ph, dh


def admm_face_optimize(mesh: TriMesh, targets, config: AdmmConfig = AdmmConfig()) -> FaceAdmmResult:
    """admm_face_optimize (grad_face.hpp:228-237)."""
    config.validate()
    H = _f64(targets).reshape(-1, 3)
    G = np.empty_like(H)
    rep, ph, dh = _solver_report_struct(config.max_iterations)
    cfg = config._c()
    _check(mesh._lib.gh_admm_face_optimize(mesh._h, _ptr(H), C.byref(cfg), _ptr(G), C.byref(rep)))
    return FaceAdmmResult(G, _report(rep, ph, dh))


def admm_edge_optimize(mesh: TriMesh, targets, config: AdmmConfig = AdmmConfig()) -> EdgeAdmmResult:
    """admm_edge_optimize (grad_edge.hpp:207-216)."""
    config.validate()
    H = _f64(targets).reshape(-1, 3)
    X = np.empty(mesh.edge_count(), np.float64)
    rep, ph, dh = _solver_report_struct(config.max_iterations)
    cfg = config._c()
    _check(mesh._lib.gh_admm_edge_optimize(mesh._h, _ptr(H), C.byref(cfg), _ptr(X), C.byref(rep)))
    return EdgeAdmmResult(X, _report(rep, ph, dh))


def solver_state_bytes(mesh: TriMesh, kind: OptimizerKind) -> int:
    """solver_state_bytes (grad_face.hpp:217-223)."""
    b = C.c_uint64()
    _check(mesh._lib.gh_solver_state_bytes(mesh._h, int(kind), C.byref(b)))
    return b.value


# ---------------------------------------------------------------- integration
def integrate_face_gradients(mesh: TriMesh, levels: BfsLevels, gradients) -> np.ndarray:
    """integrate_face_gradients (integrate.hpp:40-59)."""
    G = _f64(gradients).reshape(-1, 3)
    d = np.empty(mesh.vertex_count(), np.float64)
    _check(mesh._lib.gh_integrate_face_gradients(levels._h, _ptr(G), _ptr(d)))
    return d


def integrate_edge_differences(mesh: TriMesh, levels: BfsLevels, differences) -> np.ndarray:
    """integrate_edge_differences (integrate.hpp:64-75)."""
    X = _f64(differences)
    d = np.empty(mesh.vertex_count(), np.float64)
    _check(mesh._lib.gh_integrate_edge_differences(levels._h, _ptr(X), _ptr(d)))
    return d


# ---------------------------------------------------------------- fused pipeline
@dataclass
class RunReport:
    """Subset of RunReport (report.hpp:50-90) filled by the fused device pipeline."""
    t: float = 0.0
    gs_iterations: int = 0
    admm_iterations: int = 0
    converged: bool = False
    zero_count: int = 0
    final_primal: float = 0.0
    final_dual: float = 0.0
    build_ms: float = 0.0
    bfs_ms: float = 0.0
    diffusion_ms: float = 0.0
    normalize_ms: float = 0.0
    optimization_ms: float = 0.0
    integration_ms: float = 0.0
    d2h_ms: float = 0.0
    total_ms: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    solver_state_bytes: int = 0
    kernel_launches: int = 0
    cg_iterations: int = 0
    diffusion_e1: float = -1.0
    poisson_residual: float = 0.0
    state_bytes_allocated: int = 0
    diffusion_row_updates: int = 0
    diffusion_active_levels: int = 0
    diffusion_launches: int = 0


_METHODS = {"face": 0, "edge": 1, "poisson": 2}


def _pipeline_config(method, sweeps, t, m, admm: AdmmConfig, cg_tol: float = 1e-5,
                     diffusion_e1: bool = False, u_ready: bool = False) -> gh_pipeline_config:
    meth = _METHODS[method] if isinstance(method, str) else int(method)
    flags = (1 if diffusion_e1 else 0) | (2 if u_ready else 0)
    return gh_pipeline_config(meth, int(sweeps), float(t if t is not None else 0.0), float(m), admm._c(),
                              float(cg_tol), flags, 0)


def _run_report(r: gh_run_report) -> RunReport:
    return RunReport(**{f.name: (bool(getattr(r, f.name)) if f.name == "converged" else getattr(r, f.name))
                        for f in RunReport.__dataclass_fields__.values()})


def distance(levels: BfsLevels, method: str = "face", sweeps: int = 1000, t: Optional[float] = None, m: float = 1.0,
             admm: AdmmConfig = AdmmConfig(), cg_tol: float = 1e-5, diffusion_e1: bool = False,
             u_ready: bool = False):
    """The solver chain of run_pipeline (tools/geoheat.cpp:96-143), device-resident between stages;
    method "face" | "edge" | "poisson" (the CG heat method, cg_tol = the CLI's --eps). u_ready: the
    levels' device u (u_device()) already holds the diffusion result, e.g. a partitioned solve
    merged across ranks on the device; the diffusion is skipped."""
    d = np.empty(levels.mesh.vertex_count(), np.float64)
    cfg = _pipeline_config(method, sweeps, t, m, admm, cg_tol, diffusion_e1, u_ready)
    rep = gh_run_report()
    _check(levels._lib.gh_distance(levels._h, C.byref(cfg), _ptr(d), C.byref(rep)))
    return d, _run_report(rep)


def distance_host(positions, faces, sources, method: str = "face", sweeps: int = 1000, t: Optional[float] = None,
                  m: float = 1.0, admm: AdmmConfig = AdmmConfig(), out: Optional[np.ndarray] = None):
    """Host arrays in, host distances out: H2D, build, BFS, solve, D2H in one call."""
    P = _f64(positions).reshape(-1, 3)
    Fc = np.ascontiguousarray(faces, dtype=np.int32).reshape(-1, 3)
    S = np.ascontiguousarray(sources, dtype=np.int32)
    if out is not None and not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.ndim == 1
                                and out.size == P.shape[0] and out.flags.c_contiguous and out.flags.writeable):
        raise ValueError(f"distance_host: out must be a writeable C-contiguous float64 array of {P.shape[0]} values")
    d = out if out is not None else np.empty(P.shape[0], np.float64)
    cfg = _pipeline_config(method, sweeps, t, m, admm)
    rep = gh_run_report()
    _check(_lib.load().gh_distance_host(_ptr(P), P.shape[0], _ptr(Fc), Fc.shape[0], _ptr(S), S.size, C.byref(cfg),
                                        _ptr(d), C.byref(rep)))
    return d, _run_report(rep)


@dataclass
class PoissonReport:
    """PoissonReport (reference.hpp:163-170)."""
    heat_iterations: int
    poisson_iterations: int
    heat_residual: float
    poisson_residual: float
    heat_seconds: float
    poisson_seconds: float
    kernel_launches: int


def poisson_heat_method(mesh: TriMesh, sources: Sequence[int], t: float, cg_tol: float,
                        levels: Optional[BfsLevels] = None):
    """poisson_heat_method (reference.hpp:175-216) on the device -> (d, PoissonReport)."""
    lv = levels if levels is not None else bfs_levels(mesh, sources)
    d = np.empty(mesh.vertex_count(), np.float64)
    rep = _lib.gh_poisson_report()
    _check(lv._lib.gh_poisson_heat_method(lv._h, float(t), float(cg_tol), _ptr(d), C.byref(rep)))
    return d, PoissonReport(rep.heat_iterations, rep.poisson_iterations, rep.heat_residual, rep.poisson_residual,
                            rep.heat_seconds, rep.poisson_seconds, rep.kernel_launches)


def triangulation_quality(mesh: TriMesh) -> float:
    """triangulation_quality (mesh.hpp:297-310)."""
    v = C.c_double()
    _check(mesh._lib.gh_triangulation_quality(mesh._h, C.byref(v)))
    return v.value


def midpoint_subdivide(mesh: TriMesh, levels: int) -> TriMesh:
    """midpoint_subdivide (subdivide.hpp:14-44) on the device."""
    h = C.c_void_p()
    _check(mesh._lib.gh_mesh_subdivide(mesh._h, int(levels), C.byref(h)))
    return TriMesh(h)


class AnalyticSurface(enum.IntEnum):
    PlaneEuclidean = 0
    SphereGreatCircle = 1


def analytic_oracle(kind: AnalyticSurface, mesh: TriMesh, sources: Sequence[int]) -> np.ndarray:
    """analytic_oracle (reference.hpp:283-321); ValueError off the surface."""
    S = np.ascontiguousarray(sources, dtype=np.int32)
    d = np.empty(mesh.vertex_count(), np.float64)
    _check(mesh._lib.gh_analytic_distance(mesh._h, int(kind), _ptr(S), S.size, _ptr(d)))
    return d


def dijkstra_edge_distance(mesh: TriMesh, sources: Sequence[int]) -> np.ndarray:
    """dijkstra_edge_distance (reference.hpp:220-245)."""
    S = np.ascontiguousarray(sources, dtype=np.int32)
    d = np.empty(mesh.vertex_count(), np.float64)
    _check(mesh._lib.gh_dijkstra_distance(mesh._h, _ptr(S), S.size, _ptr(d)))
    return d


def error_metrics(d, d_ref, sources: Sequence[int]):
    """(mean_relative_error, excluded, recovery_error) (reference.hpp:250-276)."""
    a, b = _f64(d), _f64(d_ref)
    S = np.ascontiguousarray(sources, dtype=np.int32)
    mre, e2, exc = C.c_double(), C.c_double(), C.c_int32()
    _check(_lib.load().gh_error_metrics(_ptr(a), _ptr(b), a.size, _ptr(S), S.size, C.byref(mre), C.byref(exc),
                                        C.byref(e2)))
    return mre.value, exc.value, e2.value


def deterministic_sum(terms) -> float:
    """deterministic_sum (parallel.hpp:50-54): the left-to-right sum, bit for bit, on the device."""
    v = _f64(terms)
    out = C.c_double()
    _check(_lib.load().gh_deterministic_sum(_ptr(v), v.size, C.byref(out)))
    return out.value


def deterministic_sums(terms) -> np.ndarray:
    """One deterministic_sum per row of a 2-D array (parallel.hpp:50-54), bit for bit, one device block per row."""
    v = np.ascontiguousarray(terms, dtype=np.float64)
    if v.ndim != 2:
        raise ValueError("deterministic_sums: terms must be a 2-D array (one sum per row)")
    out = np.empty(v.shape[0], dtype=np.float64)
    _check(_lib.load().gh_deterministic_sums(_ptr(v), v.shape[1], v.shape[0], _ptr(out)))
    return out


def field_hash(values) -> int:
    """field_hash (report.hpp:145-153)."""
    v = _f64(values)
    return int(_lib.load().gh_field_hash(_ptr(v), v.size))


def device_count() -> int:
    n = C.c_int32()
    _check(_lib.load().gh_device_count(C.byref(n)))
    return n.value


def set_zero_level_truncation(on: bool) -> None:
    """Opt-in exact-zero skipping: gs_diffuse updates only the BFS levels the heat can reach before it
    underflows to +0 (verified in the kernel) and the fused chain's ADMM skips elements that provably
    stay +0 — bit-identical results (include/geoheat_b200.h). Off by default."""
    _check(_lib.load().gh_set_zero_level_truncation(1 if on else 0))


def release_cached_memory() -> None:
    """Hand the library's cached device memory (block cache + pool free blocks) back to the driver."""
    _check(_lib.load().gh_release_cached_memory())
