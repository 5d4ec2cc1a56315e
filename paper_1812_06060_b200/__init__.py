"""geoheat on B200: the solver loop of the parallel heat method (arXiv 1812.06060)
as hand-written sm_100a CUDA behind a C ABI (include/geoheat_b200.h).

`geoheat` mirrors the reference C++ API (reference/proj/include/geoheat);
`meshgen` builds the seeded BASELINE meshes. See DESIGN.md.
"""
from . import geoheat, meshgen  # noqa: F401
from .geoheat import (AdmmConfig, BfsLevels, DiffusionConfig, EdgeAdmmResult, FaceAdmmResult,  # noqa: F401
                      GeoheatCudaError, MeshError, NormalizedGradients, OptimizerKind, SolverError, SolverReport,
                      TriMesh, admm_edge_optimize, admm_face_optimize, average_edge_length, bfs_levels, build_mesh,
                      diffusion_residual, diffusion_time, distance, distance_host, face_gradient, field_hash,
                      gs_diffuse, integrate_edge_differences, integrate_face_gradients, normalized_target_gradients,
                      release_cached_memory, set_zero_level_truncation, solver_state_bytes)
from .geoheat import (AnalyticSurface, LoadReport, MeshFormat, PoissonReport, analytic_oracle,  # noqa: F401
                      dijkstra_edge_distance, error_metrics, format_distances, format_from_path, load_mesh,
                      midpoint_subdivide, parse_mesh_text, poisson_heat_method, save_mesh, serialize_mesh,
                      triangulation_quality, write_distances)
