/* geoheat_b200 — C ABI of the B200 (sm_100a) solver loop for the parallel heat
 * method (arXiv 1812.06060). Plain pointers and sizes only; no C++ or torch
 * types cross this boundary; no exception escapes it.
 *
 * The reference exposes the path as inline C++ free functions in
 * namespace geoheat (reference/proj/include/geoheat/). Each entry point below
 * names the reference function it replaces; include/geoheat_b200.hpp wraps
 * them back into the reference's exact C++ signatures and exception types so
 * run_pipeline (tools/geoheat.cpp:71-161) switches backend with a one-line
 * change.
 *
 * Conventions
 *   - int32 indices, fp64 values, arrays laid out like the reference's
 *     std::vector<Vec3> (xyz interleaved) / std::array<Index,3>.
 *   - every function returns a gh_status; gh_last_error() gives the message
 *     of the last failure on the calling thread.
 *   - handles own device memory on the device that was current (or chosen by
 *     gh_set_device) at creation, and one CUDA stream each. Thread-safe: calls
 *     on one mesh (or on levels / bands built on it) from several host threads
 *     are serialised by a per-mesh lock (the reference's functions are pure on
 *     const objects, so concurrent calls must not corrupt each other); calls on
 *     different meshes run concurrently. Every call restores the calling
 *     thread's current CUDA device before it returns.
 *   - host buffers are caller-owned; outputs are written before return.
 */
#ifndef GEOHEAT_B200_H
#define GEOHEAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GH_OK = 0,
  GH_ERR_MESH = 1,     /* geoheat::MeshError      (common.hpp:30-32)  */
  GH_ERR_INVALID = 2,  /* std::invalid_argument                       */
  GH_ERR_SOLVER = 3,   /* geoheat::SolverError    (common.hpp:35-37)  */
  GH_ERR_CUDA = 4,     /* CUDA runtime / no device / out of memory    */
  GH_ERR_INTERNAL = 5
} gh_status;

/* Opaque device-resident TriMesh (mesh.hpp:21-94). */
typedef struct gh_mesh gh_mesh;
/* Opaque device-resident BfsLevels (bfs.hpp:15-22) plus the BFS-renumbered
 * diffusion layout derived from it. Borrows its gh_mesh; handles may be
 * destroyed in any order (a mesh destroyed while levels are alive is freed
 * with its last gh_levels). */
typedef struct gh_levels gh_levels;

/* Array ids for gh_mesh_download: the fields of TriMesh in declaration order
 * (mesh.hpp:22-49); element type and length in the comment. */
typedef enum {
  GH_POSITIONS = 0,           /* f64 [3V]  */
  GH_FACES = 1,               /* i32 [3F]  */
  GH_HALFEDGE_TWIN = 2,       /* i32 [3F]  */
  GH_HALFEDGE_EDGE = 3,       /* i32 [3F]  */
  GH_EDGE_VERTICES = 4,       /* i32 [2E]  */
  GH_EDGE_HALFEDGES = 5,      /* i32 [2E]  */
  GH_INTERIOR_EDGES = 6,      /* i32 [Eint]*/
  GH_INTERIOR_EDGE_INDEX = 7, /* i32 [E]   */
  GH_VERTEX_ON_BOUNDARY = 8,  /* u8  [V]   */
  GH_FACE_AREA = 9,           /* f64 [F]   */
  GH_FACE_NORMAL = 10,        /* f64 [3F]  */
  GH_VERTEX_AREA = 11,        /* f64 [V]   */
  GH_HALFEDGE_COT = 12,       /* f64 [3F]  */
  GH_EDGE_WEIGHT = 13,        /* f64 [E]   */
  GH_VERTEX_WEIGHT_SUM = 14,  /* f64 [V]   */
  GH_VV_OFFSET = 15,          /* i32 [V+1] */
  GH_VV_INDEX = 16,           /* i32 [2E]  */
  GH_VV_EDGE = 17,            /* i32 [2E]  */
  GH_VV_WEIGHT = 18,          /* f64 [2E]  */
  GH_VC_OFFSET = 19,          /* i32 [V+1] */
  GH_VC_CORNER = 20,          /* i32 [3F]  */
  GH_NUM_MESH_ARRAYS = 21
} gh_mesh_array;

typedef struct {
  int32_t vertices, faces, edges, interior_edges, boundary_vertices;
  uint64_t device_bytes; /* device memory held by the handle */
} gh_mesh_info;

typedef struct {
  int32_t level_count;       /* BfsLevels::level_count()        */
  int32_t unreachable_count; /* BfsLevels::unreachable_count    */
  int32_t max_level_width;   /* widest ring                     */
  int32_t column_bits;       /* columns the last gs_diffuse streamed: 16 or 32 (0 before the first) */
  /* zero-level truncation of the last gs_diffuse (gh_set_zero_level_truncation): */
  int32_t active_levels;      /* levels its last launch updated; level_count when nothing was truncated */
  int32_t diffusion_launches; /* pipelined launches it ran (1 without truncation) */
  int32_t diffusion_retries;  /* launches redone with a larger cap */
  int32_t layout_levels;      /* levels the diffusion layout covers (the first rings only on meshes the heat cannot cross; grows on demand) */
  uint64_t row_updates;       /* vertex updates executed (reachable x sweeps without truncation) */
} gh_levels_info;

/* AdmmConfig (grad_face.hpp:15-26). */
typedef struct {
  int32_t max_iterations; /* default 10  */
  double eps1;            /* default 1e-5 */
  double eps2;            /* default 1e-5 */
  double mu;              /* default 100  */
} gh_admm_config;

/* SolverReport (report.hpp:16-27) plus device timing. History buffers are
 * caller-owned and may be NULL; history_capacity entries are written. */
typedef struct {
  int32_t iterations;
  int32_t converged;
  double final_primal;
  double final_dual;
  double* primal_history;
  double* dual_history;
  double* residual_history; /* E1 per sweep (gh_gs_diffuse_tol), may be NULL */
  int32_t history_capacity;
  uint64_t state_bytes_formula;   /* solver_state_bytes (grad_face.hpp:217-223) */
  uint64_t state_bytes_allocated; /* device bytes the solver state occupies     */
  double wall_seconds;            /* host wall time of the call                 */
  double device_ms;               /* CUDA-event time of the solver kernels      */
  int32_t kernel_launches;        /* kernels this call launched                 */
} gh_solver_report;

/* Pipeline selection (PipelineOptions, tools/geoheat.cpp:27-38). */
typedef enum { GH_METHOD_FACE = 0, GH_METHOD_EDGE = 1, GH_METHOD_POISSON = 2 } gh_method;
/* gh_pipeline_config.flags */
enum {
  GH_PIPE_DIFFUSION_E1 = 1, /* also compute diffusion_residual of u (geoheat.cpp:117) */
  GH_PIPE_U_READY = 2       /* u is already the levels' diffusion result (gh_levels_u_device, e.g. a
                               partitioned solve merged across ranks on the device): skip the diffusion */
};

typedef struct {
  int32_t method;   /* gh_method */
  int32_t sweeps;   /* Gauss-Seidel sweeps (gs_iters), default 1000 */
  double t;         /* diffusion time; <= 0 means m * h^2 from the mesh */
  double m;         /* smoothing factor used when t <= 0 */
  gh_admm_config admm;
  double cg_tol;    /* GH_METHOD_POISSON: CG tolerance (the CLI's --eps) */
  int32_t flags;    /* GH_PIPE_* */
  int32_t reserved;
} gh_pipeline_config;

/* Per-stage record of gh_distance (RunReport, report.hpp:50-90). */
typedef struct {
  double t;
  int32_t gs_iterations;
  int32_t admm_iterations;
  int32_t converged;
  int32_t zero_count; /* faces whose heat gradient underflowed (diffusion.hpp:128) */
  double final_primal;
  double final_dual;
  double build_ms;      /* device mesh build (gh_distance_host only) */
  double bfs_ms;        /* BFS + layout      (gh_distance_host only) */
  double diffusion_ms;
  double normalize_ms;
  double optimization_ms;
  double integration_ms;
  double h2d_ms, d2h_ms;
  double total_ms;      /* CUDA-event time of the whole call */
  uint64_t h2d_bytes, d2h_bytes;
  uint64_t solver_state_bytes;
  int32_t kernel_launches;
  int32_t cg_iterations;  /* GH_METHOD_POISSON: heat + Poisson CG iterations */
  double diffusion_e1;    /* GH_PIPE_DIFFUSION_E1, else -1 */
  double poisson_residual;/* GH_METHOD_POISSON: final relative residual (reported as final_primal) */
  uint64_t state_bytes_allocated; /* device bytes of the optimiser state (SolverReport field) */
  /* zero-level truncation of the diffusion (gh_set_zero_level_truncation; gh_levels_info has the same): */
  uint64_t diffusion_row_updates;   /* vertex updates executed (reachable x sweeps without truncation) */
  int32_t diffusion_active_levels;  /* levels the last diffusion launch updated */
  int32_t diffusion_launches;       /* pipelined launches (1 without truncation) */
} gh_run_report;

/* ---- runtime */
const char* gh_last_error(void);
const char* gh_version(void);
gh_status gh_set_device(int32_t device);
gh_status gh_device_count(int32_t* count);
/* Pinned host memory for staging (cudaMallocHost / cudaFreeHost). */
gh_status gh_host_alloc(size_t bytes, void** out);
gh_status gh_host_free(void* p);
/* Return the device memory this library keeps cached for reuse (its exact-size
   block cache and the stream-ordered pool's free blocks) to the driver, on every
   device it has used. Handles stay valid. Call it before other processes need
   the memory (the pool otherwise keeps what a large solve grew to). */
gh_status gh_release_cached_memory(void);
/* Exact-zero skipping (opt-in: off by default, so that every update the
   reference executes is executed; GH_ZERO_LEVELS=1 in the environment also
   turns it on). With t ~ h^2 the heat underflows to exactly
   +0 a few hundred rings from the sources; levels beyond that front provably
   stay +0, and the solve updates only the levels below a cap that the kernel
   verifies (a nonzero bit at the cap's top level redoes the launch with a
   larger cap); the fused chain's ADMM likewise skips faces and edges that
   provably stay +0. The results are the reference's bit for bit (diffusion.hpp:
   73-108 evaluated on the levels that can differ from zero); process-wide. */
gh_status gh_set_zero_level_truncation(int32_t on);

/* ---- mesh: build_mesh (mesh.hpp:113-286), device preprocessing */
gh_status gh_mesh_create(const double* positions, int32_t nv, const int32_t* faces, int32_t nf, gh_mesh** out);
gh_status gh_mesh_destroy(gh_mesh* mesh);
gh_status gh_mesh_get_info(const gh_mesh* mesh, gh_mesh_info* info);
/* Copy one TriMesh array to host (`count` elements of the array's type). */
gh_status gh_mesh_download(const gh_mesh* mesh, int32_t which, void* host_out, int64_t count);
/* average_edge_length (mesh.hpp:289-293): the edge-order sum, bit-identical. */
gh_status gh_average_edge_length(gh_mesh* mesh, double* h_out);
/* diffusion_time (diffusion.hpp:28-32): t = m * h * h. */
gh_status gh_diffusion_time(gh_mesh* mesh, double m, double* t_out);
/* face_gradient (mesh.hpp:314-327): u [V] -> grad [3F]. */
gh_status gh_face_gradient(gh_mesh* mesh, const double* u, double* grad_out);

/* ---- mesh I/O: load_mesh / save_mesh / distance writers (mesh_io.hpp)
 * Same accepted inputs, values and error messages (status GH_ERR_MESH) as
 * the reference loader. Binary little-endian PLY records are decoded on the
 * device straight into the mesh arrays; OBJ and ASCII PLY are tokenised by
 * host threads with std::istream >> double semantics. */
typedef enum { GH_FORMAT_OBJ = 0, GH_FORMAT_PLY = 1 } gh_mesh_format;   /* MeshFormat (mesh_io.hpp:18) */
typedef enum { GH_DISTANCES_TXT = 0, GH_DISTANCES_CSV = 1 } gh_distance_format;

typedef struct {
  int32_t format;          /* gh_mesh_format */
  int32_t binary;          /* PLY body is binary_little_endian */
  int32_t device_decoded;  /* binary records were decoded on the device */
  int32_t host_threads;    /* threads that read / tokenised the input */
  uint64_t bytes;          /* input size */
  double read_ms;          /* map the file, stream binary records to the device */
  double parse_ms;         /* header, tokenising or device record decode */
  double build_ms;         /* build_mesh on the device (text formats) */
  double total_ms;
  int32_t kernel_launches;
  int32_t reserved;
} gh_load_report;

/* format_from_path (mesh_io.hpp:271-278): ".obj" / ".ply", case-insensitive. */
gh_status gh_mesh_format_from_path(const char* path, int32_t* format_out);
/* load_mesh(path) (mesh_io.hpp:280-285) -> device mesh. report may be NULL. */
gh_status gh_mesh_load(const char* path, gh_mesh** out, gh_load_report* report);
/* load_mesh(istream, format) (mesh_io.hpp:267-269) over a host buffer. */
gh_status gh_mesh_load_memory(const void* data, uint64_t bytes, int32_t format, gh_mesh** out,
                              gh_load_report* report);
/* The host tokeniser alone for the text formats (OBJ, ASCII PLY): positions
 * [3V] and faces [3F] as load_obj / load_ply hand them to build_mesh. Arrays
 * are malloc'd, released with gh_free. Binary PLY is rejected (its records
 * are decoded on the device by gh_mesh_load*). threads <= 0: automatic. */
gh_status gh_mesh_parse_text(const void* data, uint64_t bytes, int32_t format, int32_t threads, double** positions,
                             int64_t* nv, int32_t** faces, int64_t* nf);
/* save_obj / save_ply (mesh_io.hpp:287-319) into a malloc'd buffer (gh_free).
 * quality (host [V]) adds the per-vertex "quality" property; PLY only. */
gh_status gh_mesh_serialize(gh_mesh* mesh, int32_t format, const double* quality, void** data, uint64_t* bytes);
/* save_mesh (mesh_io.hpp:321-326) with save_ply's optional quality. */
gh_status gh_mesh_save(gh_mesh* mesh, const char* path, const double* quality);
/* write_distances_txt / write_distances_csv (mesh_io.hpp:329-344). */
gh_status gh_format_distances(const double* d, int64_t n, int32_t format, void** data, uint64_t* bytes);
gh_status gh_write_distances(const char* path, const double* d, int64_t n, int32_t format);
void gh_free(void* p);

/* ---- BFS: bfs_levels (bfs.hpp:26-72) */
gh_status gh_bfs_create(gh_mesh* mesh, const int32_t* sources, int32_t ns, gh_levels** out);
gh_status gh_bfs_destroy(gh_levels* levels);
gh_status gh_bfs_get_info(const gh_levels* levels, gh_levels_info* info);
/* Any output may be NULL. order: rings concatenated (V - unreachable
 * entries); offsets: level_count + 1 ring boundaries. */
gh_status gh_bfs_download(const gh_levels* levels, int32_t* level_of_vertex, int32_t* parent_of_vertex,
                          int32_t* order, int32_t* offsets);

/* ---- diffusion: gs_diffuse (diffusion.hpp:57-124) */
/* initial: NULL (u = u0) or a host warm start [V]. u_out: host [V], or NULL to
 * keep the result on the device only (benchmarking; see gh_levels_u_device). */
gh_status gh_gs_diffuse(gh_levels* levels, double t, int32_t sweeps, const double* initial, double* u_out,
                        gh_solver_report* report);
/* gs_diffuse with DiffusionConfig::residual_tolerance (diffusion.hpp:19,
 * 110-117): after every sweep E1 is computed and the iteration stops once
 * E1 <= tolerance; report->residual_history receives E1 per sweep. */
gh_status gh_gs_diffuse_tol(gh_levels* levels, double t, int32_t sweeps, double tolerance, const double* initial,
                            double* u_out, gh_solver_report* report);
/* diffusion_residual (diffusion.hpp:35-49), E1 of a host u. */
gh_status gh_diffusion_residual(gh_levels* levels, const double* u, double t, double* e1_out);

/* ---- normalisation: normalized_target_gradients (diffusion.hpp:132-145) */
gh_status gh_normalized_target_gradients(gh_mesh* mesh, const double* u, double* h_out, int32_t* zero_count);

/* ---- integrability optimisation */
/* admm_face_optimize (grad_face.hpp:228-237): H [3F] -> G [3F]. */
gh_status gh_admm_face_optimize(gh_mesh* mesh, const double* h, const gh_admm_config* config, double* g_out,
                                 gh_solver_report* report);
/* admm_edge_optimize (grad_edge.hpp:207-216): H [3F] -> X [E]. */
gh_status gh_admm_edge_optimize(gh_mesh* mesh, const double* h, const gh_admm_config* config, double* x_out,
                                gh_solver_report* report);
/* solver_state_bytes (grad_face.hpp:217-223); method is gh_method. */
gh_status gh_solver_state_bytes(const gh_mesh* mesh, int32_t method, uint64_t* bytes_out);

/* ---- distance recovery */
/* integrate_face_gradients (integrate.hpp:40-59): G [3F] -> d [V]. */
gh_status gh_integrate_face_gradients(gh_levels* levels, const double* g, double* d_out);
/* integrate_edge_differences (integrate.hpp:64-75): X [E] -> d [V]. */
gh_status gh_integrate_edge_differences(gh_levels* levels, const double* x, double* d_out);

/* ---- fused solver loop, device-resident between stages
 * (the chain of run_pipeline, tools/geoheat.cpp:108-143). d_out host [V]. */
gh_status gh_distance(gh_levels* levels, const gh_pipeline_config* config, double* d_out, gh_run_report* report);
/* Host arrays in -> host distances out, everything on the device in between:
 * H2D, build_mesh, bfs_levels, gh_distance, D2H (the end-to-end path). */
gh_status gh_distance_host(const double* positions, int32_t nv, const int32_t* faces, int32_t nf,
                           const int32_t* sources, int32_t ns, const gh_pipeline_config* config, double* d_out,
                           gh_run_report* report);

/* ---- classic heat method on CG: poisson_heat_method (reference.hpp:175-216)
 * Jacobi-preconditioned CG (cg_solve, reference.hpp:35-84) on the heat
 * operator, normalised gradients, integrated divergence, CG on the reduced
 * Poisson operator; sources are the levels' ring 0. GH_ERR_SOLVER on a CG
 * breakdown. d_out: host [V] (inf for unreachable vertices). */
typedef struct {
  int32_t heat_iterations, poisson_iterations;
  double heat_residual, poisson_residual; /* relative residuals */
  double heat_seconds, poisson_seconds;
  int32_t kernel_launches, reserved;
} gh_poisson_report;
gh_status gh_poisson_heat_method(gh_levels* levels, double t, double cg_tol, double* d_out, gh_poisson_report* report);

/* ---- evaluation layer of the CLI */
/* triangulation_quality (mesh.hpp:297-310): the face-order sum, bit-identical. */
gh_status gh_triangulation_quality(gh_mesh* mesh, double* tau_out);
/* midpoint_subdivide (subdivide.hpp:14-44) -> a new device mesh. */
gh_status gh_mesh_subdivide(gh_mesh* mesh, int32_t levels, gh_mesh** out);
typedef enum { GH_SURFACE_PLANE = 0, GH_SURFACE_SPHERE = 1 } gh_analytic_surface; /* AnalyticSurface */
/* analytic_oracle (reference.hpp:283-321); GH_ERR_INVALID off the surface. */
gh_status gh_analytic_distance(gh_mesh* mesh, int32_t kind, const int32_t* sources, int32_t ns, double* d_out);
/* dijkstra_edge_distance (reference.hpp:220-245). */
gh_status gh_dijkstra_distance(gh_mesh* mesh, const int32_t* sources, int32_t ns, double* d_out);
/* mean_relative_error (reference.hpp:250-266) and recovery_error (268-276)
 * of two host fields, on the current device. */
gh_status gh_error_metrics(const double* d, const double* d_ref, int64_t n, const int32_t* sources, int32_t ns,
                           double* mean_rel_error, int32_t* excluded, double* e2);

/* ---- BFS-band sharding of the diffusion
 * Levels are cut into nbands contiguous bands of about equal rows; band r
 * computes its own levels and keeps ghost copies of levels lb-1 and le, which
 * the neighbours write directly (peer stores + per-level counters) while
 * the single dataflow kernel runs. Results are bit-identical to gh_gs_diffuse. */
typedef struct gh_band gh_band;
/* The band plan: cut_out[nbands + 1] level boundaries for ring offsets[nlev + 1]
 * (host only; the same plan every rank computes). */
gh_status gh_plan_bands(const int32_t* offsets, int32_t nlev, int32_t nbands, int32_t* cut_out);
/* All bands in one process on the current device (one launch): the
 * single-GPU emulation of the multi-GPU schedule. nbands <= 8. */
gh_status gh_gs_diffuse_bands(gh_levels* levels, int32_t nbands, double t, int32_t sweeps, const double* initial,
                              double* u_out, gh_solver_report* report);
/* One band per process/GPU: create, export its IPC blob, connect to the
 * neighbours' blobs, prepare (all ranks) -> barrier -> launch (all ranks). */
gh_status gh_band_create(gh_levels* levels, int32_t rank, int32_t nranks, gh_band** out);
gh_status gh_band_destroy(gh_band* band);
gh_status gh_band_info(const gh_band* band, int32_t* lb, int32_t* le, int32_t* own_rows);
/* blob NULL: *size receives the blob size. */
gh_status gh_band_export(const gh_band* band, void* blob, int32_t capacity, int32_t* size);
/* lower_blob / upper_blob NULL for the first / last band. */
gh_status gh_band_connect(gh_band* band, const void* lower_blob, const void* upper_blob);
/* Every rank prepares before any rank launches (a barrier between), and no rank
   prepares the next solve until every rank's gh_band_launch of the previous one
   has returned (a barrier after the launch): the upper neighbour's last sweep
   writes into this band's ghost rows and counters after this band's own kernel
   may have finished, and prepare re-initialises both. */
gh_status gh_band_prepare(gh_band* band, double t, const double* initial);
/* u_out (host [V], may be NULL): this band's vertices hold the result. */
gh_status gh_band_launch(gh_band* band, double t, int32_t sweeps, double* u_out, gh_solver_report* report);

/* One process driving parts whose buffers live in other processes (more
 * parts than GPUs, or tests on one GPU): gh_band_adopt maps the mutable
 * buffers (u, per-level counters, per-source ghost counters) of the same part
 * exported by another process (its gh_band_export blob) through CUDA IPC and
 * uses them in place of the band's own; gh_band_launch_group runs parts
 * 0..n-1 of one partition (in order) in ONE cooperative launch on this device,
 * linked to each other through their current buffers (system-scope releases
 * and polls when any is adopted), and returns u; gh_band_download writes this
 * part's own rows of u after `sweeps` sweeps into u_out (vertex order; other
 * entries kept). */
gh_status gh_band_adopt(gh_band* band, const void* blob);
gh_status gh_band_launch_group(gh_band* const* bands, int32_t n, double t, int32_t sweeps, const double* initial,
                               double* u_out, gh_solver_report* report);
gh_status gh_band_download(const gh_band* band, int32_t sweeps, double* u_out);

/* ---- Sector slices: every slice owns a contiguous 1/nslices
 * of every BFS ring (in the diffusion layout's ring order), so every slice
 * has work at every step of the sweep pipeline, however the level count
 * compares with the sweep count. Foreign neighbours of a slice's rows are
 * ghost rows the owners write (peer stores + per-(source, level) counters)
 * from inside the one dataflow kernel. Results are bit-identical to
 * gh_gs_diffuse. GH_PARTITION_BANDS selects the BFS bands above. */
typedef enum { GH_PARTITION_BANDS = 0, GH_PARTITION_SLICES = 1 } gh_partition;
/* All parts in one process on the current device (one launch), nparts <= 8. */
gh_status gh_gs_diffuse_partitioned(gh_levels* levels, int32_t nparts, int32_t partition, double t, int32_t sweeps,
                                    const double* initial, double* u_out, gh_solver_report* report);
/* One part per process/GPU (bands: as gh_band_create). Slices connect to
 * every other rank: blobs[nranks] from gh_band_export of each rank (its own
 * entry is ignored). Prepare/launch and their barriers as for bands. */
gh_status gh_band_create_partitioned(gh_levels* levels, int32_t rank, int32_t nranks, int32_t partition,
                                     gh_band** out);
gh_status gh_band_connect_all(gh_band* band, const void* const* blobs, int32_t nranks);
/* The device buffer holding the levels' diffusion result u [V] (original
 * vertex order): written by gh_gs_diffuse*, gh_band_launch (this part's
 * vertices), read by gh_distance with GH_PIPE_U_READY. Valid while the
 * levels live; for device-side merges (e.g. an NCCL all-reduce). */
gh_status gh_levels_u_device(gh_levels* levels, double** u_dev, int64_t* n);
/* mask_out[V] (host): 1 for the vertices whose u this part computes. */
gh_status gh_band_own_mask(const gh_band* band, uint8_t* mask_out);

/* deterministic_sum (parallel.hpp:50-54): the left-to-right sum of n host
 * doubles, bit-identical. Non-negative terms take the parallel exact path
 * (the library uses it for average_edge_length); any negative term falls
 * back to one device thread adding in order. */
gh_status gh_deterministic_sum(const double* terms, int64_t n, double* sum_out);
/* count independent deterministic_sums at once: sums_out[i] = the left-to-right
 * sum of terms[i*n .. i*n+n), bit-identical, one device block per sum (the
 * engine behind the E1 history of gh_gs_diffuse_tol). Any signs. */
gh_status gh_deterministic_sums(const double* terms, int64_t n, int32_t count, double* sums_out);

/* field_hash (report.hpp:145-153): FNV-1a over the bytes of n doubles. */
uint64_t gh_field_hash(const double* values, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* GEOHEAT_B200_H */
