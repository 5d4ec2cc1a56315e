"""ctypes binding of the C ABI in include/geoheat_b200.h.

Loads the in-tree lib/libgeoheat_b200.so. There is no fallback: if the
library is missing or no CUDA device is present, calls fail loudly
(GeoheatCudaError), exactly as the ABI does.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _build

LIB_PATH = _build.CUDA_LIB


class gh_mesh_info(C.Structure):
    _fields_ = [("vertices", C.c_int32), ("faces", C.c_int32), ("edges", C.c_int32),
                ("interior_edges", C.c_int32), ("boundary_vertices", C.c_int32), ("device_bytes", C.c_uint64)]


class gh_levels_info(C.Structure):
    _fields_ = [("level_count", C.c_int32), ("unreachable_count", C.c_int32), ("max_level_width", C.c_int32),
                ("column_bits", C.c_int32), ("active_levels", C.c_int32), ("diffusion_launches", C.c_int32),
                ("diffusion_retries", C.c_int32), ("layout_levels", C.c_int32), ("row_updates", C.c_uint64)]


class gh_admm_config(C.Structure):
    _fields_ = [("max_iterations", C.c_int32), ("eps1", C.c_double), ("eps2", C.c_double), ("mu", C.c_double)]


class gh_solver_report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("final_primal", C.c_double),
                ("final_dual", C.c_double), ("primal_history", C.POINTER(C.c_double)),
                ("dual_history", C.POINTER(C.c_double)), ("residual_history", C.POINTER(C.c_double)),
                ("history_capacity", C.c_int32), ("state_bytes_formula", C.c_uint64),
                ("state_bytes_allocated", C.c_uint64), ("wall_seconds", C.c_double), ("device_ms", C.c_double),
                ("kernel_launches", C.c_int32)]


class gh_pipeline_config(C.Structure):
    _fields_ = [("method", C.c_int32), ("sweeps", C.c_int32), ("t", C.c_double), ("m", C.c_double),
                ("admm", gh_admm_config), ("cg_tol", C.c_double), ("flags", C.c_int32), ("reserved", C.c_int32)]


class gh_run_report(C.Structure):
    _fields_ = [("t", C.c_double), ("gs_iterations", C.c_int32), ("admm_iterations", C.c_int32),
                ("converged", C.c_int32), ("zero_count", C.c_int32), ("final_primal", C.c_double),
                ("final_dual", C.c_double), ("build_ms", C.c_double), ("bfs_ms", C.c_double),
                ("diffusion_ms", C.c_double), ("normalize_ms", C.c_double), ("optimization_ms", C.c_double),
                ("integration_ms", C.c_double), ("h2d_ms", C.c_double), ("d2h_ms", C.c_double),
                ("total_ms", C.c_double), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("solver_state_bytes", C.c_uint64), ("kernel_launches", C.c_int32), ("cg_iterations", C.c_int32),
                ("diffusion_e1", C.c_double), ("poisson_residual", C.c_double),
                ("state_bytes_allocated", C.c_uint64), ("diffusion_row_updates", C.c_uint64),
                ("diffusion_active_levels", C.c_int32), ("diffusion_launches", C.c_int32)]


class gh_poisson_report(C.Structure):
    _fields_ = [("heat_iterations", C.c_int32), ("poisson_iterations", C.c_int32), ("heat_residual", C.c_double),
                ("poisson_residual", C.c_double), ("heat_seconds", C.c_double), ("poisson_seconds", C.c_double),
                ("kernel_launches", C.c_int32), ("reserved", C.c_int32)]


class gh_load_report(C.Structure):
    _fields_ = [("format", C.c_int32), ("binary", C.c_int32), ("device_decoded", C.c_int32),
                ("host_threads", C.c_int32), ("bytes", C.c_uint64), ("read_ms", C.c_double),
                ("parse_ms", C.c_double), ("build_ms", C.c_double), ("total_ms", C.c_double),
                ("kernel_launches", C.c_int32), ("reserved", C.c_int32)]


# (name, restype, argtypes) for every exported symbol of include/geoheat_b200.h
vp, i32, i64, f64, st = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_int
SIGNATURES = [
    ("gh_last_error", C.c_char_p, []),
    ("gh_version", C.c_char_p, []),
    ("gh_set_device", st, [i32]),
    ("gh_device_count", st, [C.POINTER(i32)]),
    ("gh_host_alloc", st, [C.c_size_t, C.POINTER(vp)]),
    ("gh_host_free", st, [vp]),
    ("gh_release_cached_memory", st, []),
    ("gh_set_zero_level_truncation", st, [C.c_int32]),
    ("gh_mesh_create", st, [vp, i32, vp, i32, C.POINTER(vp)]),
    ("gh_mesh_destroy", st, [vp]),
    ("gh_mesh_get_info", st, [vp, C.POINTER(gh_mesh_info)]),
    ("gh_mesh_download", st, [vp, i32, vp, i64]),
    ("gh_average_edge_length", st, [vp, C.POINTER(f64)]),
    ("gh_diffusion_time", st, [vp, f64, C.POINTER(f64)]),
    ("gh_face_gradient", st, [vp, vp, vp]),
    ("gh_mesh_format_from_path", st, [C.c_char_p, C.POINTER(i32)]),
    ("gh_mesh_load", st, [C.c_char_p, C.POINTER(vp), C.POINTER(gh_load_report)]),
    ("gh_mesh_load_memory", st, [C.c_char_p, C.c_uint64, i32, C.POINTER(vp), C.POINTER(gh_load_report)]),
    ("gh_mesh_parse_text", st, [C.c_char_p, C.c_uint64, i32, i32, C.POINTER(C.POINTER(f64)), C.POINTER(i64),
                                C.POINTER(C.POINTER(C.c_int32)), C.POINTER(i64)]),
    ("gh_mesh_serialize", st, [vp, i32, vp, C.POINTER(vp), C.POINTER(C.c_uint64)]),
    ("gh_mesh_save", st, [vp, C.c_char_p, vp]),
    ("gh_format_distances", st, [vp, i64, i32, C.POINTER(vp), C.POINTER(C.c_uint64)]),
    ("gh_write_distances", st, [C.c_char_p, vp, i64, i32]),
    ("gh_free", None, [vp]),
    ("gh_bfs_create", st, [vp, vp, i32, C.POINTER(vp)]),
    ("gh_bfs_destroy", st, [vp]),
    ("gh_bfs_get_info", st, [vp, C.POINTER(gh_levels_info)]),
    ("gh_bfs_download", st, [vp, vp, vp, vp, vp]),
    ("gh_gs_diffuse", st, [vp, f64, i32, vp, vp, C.POINTER(gh_solver_report)]),
    ("gh_gs_diffuse_tol", st, [vp, f64, i32, f64, vp, vp, C.POINTER(gh_solver_report)]),
    ("gh_diffusion_residual", st, [vp, vp, f64, C.POINTER(f64)]),
    ("gh_normalized_target_gradients", st, [vp, vp, vp, C.POINTER(i32)]),
    ("gh_admm_face_optimize", st, [vp, vp, C.POINTER(gh_admm_config), vp, C.POINTER(gh_solver_report)]),
    ("gh_admm_edge_optimize", st, [vp, vp, C.POINTER(gh_admm_config), vp, C.POINTER(gh_solver_report)]),
    ("gh_solver_state_bytes", st, [vp, i32, C.POINTER(C.c_uint64)]),
    ("gh_integrate_face_gradients", st, [vp, vp, vp]),
    ("gh_integrate_edge_differences", st, [vp, vp, vp]),
    ("gh_distance", st, [vp, C.POINTER(gh_pipeline_config), vp, C.POINTER(gh_run_report)]),
    ("gh_distance_host", st, [vp, i32, vp, i32, vp, i32, C.POINTER(gh_pipeline_config), vp, C.POINTER(gh_run_report)]),
    ("gh_plan_bands", st, [vp, i32, i32, vp]),
    ("gh_gs_diffuse_bands", st, [vp, i32, f64, i32, vp, vp, C.POINTER(gh_solver_report)]),
    ("gh_band_create", st, [vp, i32, i32, C.POINTER(vp)]),
    ("gh_gs_diffuse_partitioned", st, [vp, i32, i32, f64, i32, vp, vp, C.POINTER(gh_solver_report)]),
    ("gh_band_create_partitioned", st, [vp, i32, i32, i32, C.POINTER(vp)]),
    ("gh_band_connect_all", st, [vp, C.POINTER(C.c_char_p), i32]),
    ("gh_band_adopt", st, [vp, vp]),
    ("gh_band_launch_group", st, [vp, i32, f64, i32, vp, vp, vp]),
    ("gh_band_download", st, [vp, i32, vp]),
    ("gh_band_own_mask", st, [vp, vp]),
    ("gh_levels_u_device", st, [vp, C.POINTER(vp), C.POINTER(i64)]),
    ("gh_band_destroy", st, [vp]),
    ("gh_band_info", st, [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
    ("gh_band_export", st, [vp, vp, i32, C.POINTER(i32)]),
    ("gh_band_connect", st, [vp, vp, vp]),
    ("gh_band_prepare", st, [vp, f64, vp]),
    ("gh_band_launch", st, [vp, f64, i32, vp, C.POINTER(gh_solver_report)]),
    ("gh_poisson_heat_method", st, [vp, f64, f64, vp, C.POINTER(gh_poisson_report)]),
    ("gh_triangulation_quality", st, [vp, C.POINTER(f64)]),
    ("gh_mesh_subdivide", st, [vp, i32, C.POINTER(vp)]),
    ("gh_analytic_distance", st, [vp, i32, vp, i32, vp]),
    ("gh_dijkstra_distance", st, [vp, vp, i32, vp]),
    ("gh_error_metrics", st, [vp, vp, i64, vp, i32, C.POINTER(f64), C.POINTER(i32), C.POINTER(f64)]),
    ("gh_deterministic_sum", st, [vp, i64, C.POINTER(f64)]),
    ("gh_deterministic_sums", st, [vp, i64, i32, vp]),
    ("gh_field_hash", C.c_uint64, [vp, i64]),
]

_lib = None


def load() -> C.CDLL:
    """Load (once) the CUDA library; raise if it was never built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (the CUDA path has no fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
