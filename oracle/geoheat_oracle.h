/* TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
 *
 * C-callable oracle API for the parallel heat-method solver loop of
 * arXiv 1812.06060, as implemented by the reference `geoheat` headers
 * (/root/reference/proj/include/geoheat). Two libraries export exactly these
 * symbols:
 *
 *   oracle/_ref/libgeoheat_ref.so    the UNMODIFIED reference headers compiled
 *                                    against oracle/eigen_shim (ref_driver.cpp)
 *   oracle/_ref/libgeoheat_port.so   the plain-C restatement geoheat_oracle.c
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load them. The product path
 * (paper_1812_06060_b200) never does.
 *
 * Mesh array ids follow the order of the fields of `TriMesh`
 * (reference mesh.hpp:21-94) and match gh_mesh_array in include/geoheat_b200.h.
 */
#ifndef GEOHEAT_ORACLE_H
#define GEOHEAT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GHO_POSITIONS = 0,         /* f64 [3V]   */
  GHO_FACES = 1,             /* i32 [3F]   */
  GHO_HALFEDGE_TWIN = 2,     /* i32 [3F]   */
  GHO_HALFEDGE_EDGE = 3,     /* i32 [3F]   */
  GHO_EDGE_VERTICES = 4,     /* i32 [2E]   */
  GHO_EDGE_HALFEDGES = 5,    /* i32 [2E]   */
  GHO_INTERIOR_EDGES = 6,    /* i32 [Eint] */
  GHO_INTERIOR_EDGE_INDEX = 7, /* i32 [E]  */
  GHO_VERTEX_ON_BOUNDARY = 8, /* u8 [V]    */
  GHO_FACE_AREA = 9,         /* f64 [F]    */
  GHO_FACE_NORMAL = 10,      /* f64 [3F]   */
  GHO_VERTEX_AREA = 11,      /* f64 [V]    */
  GHO_HALFEDGE_COT = 12,     /* f64 [3F]   */
  GHO_EDGE_WEIGHT = 13,      /* f64 [E]    */
  GHO_VERTEX_WEIGHT_SUM = 14, /* f64 [V]   */
  GHO_VV_OFFSET = 15,        /* i32 [V+1]  */
  GHO_VV_INDEX = 16,         /* i32 [2E]   */
  GHO_VV_EDGE = 17,          /* i32 [2E]   */
  GHO_VV_WEIGHT = 18,        /* f64 [2E]   */
  GHO_VC_OFFSET = 19,        /* i32 [V+1]  */
  GHO_VC_CORNER = 20,        /* i32 [3F]   */
  GHO_NUM_ARRAYS = 21
};

typedef struct gho_mesh gho_mesh;
typedef struct gho_levels gho_levels;

/* SolverReport (reference report.hpp:16-27); histories are caller buffers. */
typedef struct {
  int32_t iterations;
  int32_t converged;
  double final_primal;
  double final_dual;
  double* primal_history; /* capacity entries, may be NULL */
  double* dual_history;   /* capacity entries, may be NULL */
  int32_t history_capacity;
  uint64_t state_bytes_formula;
  uint64_t state_bytes_allocated;
  double wall_seconds;
} gho_report;

/* return codes: 0 ok, 1 MeshError, 2 std::invalid_argument, 3 SolverError */
int gho_build_mesh(const double* positions, int32_t nv, const int32_t* faces, int32_t nf,
                   gho_mesh** out, char* err, int32_t errlen);
void gho_mesh_free(gho_mesh* mesh);
void gho_mesh_counts(const gho_mesh* mesh, int32_t counts[4]); /* V, F, E, E_int */
const void* gho_mesh_array(const gho_mesh* mesh, int32_t which, int64_t* count);
double gho_average_edge_length(const gho_mesh* mesh);
double gho_triangulation_quality(const gho_mesh* mesh);

int gho_bfs(const gho_mesh* mesh, const int32_t* sources, int32_t ns, gho_levels** out, char* err,
            int32_t errlen);
void gho_levels_free(gho_levels* levels);
void gho_levels_info(const gho_levels* levels, int32_t info[2]); /* nlev, unreachable */
/* order: the rings D_0, D_1, ... concatenated (reachable vertices);
 * offsets: nlev + 1 ring boundaries into order. Any pointer may be NULL. */
void gho_levels_get(const gho_levels* levels, int32_t* level_of_vertex, int32_t* parent_of_vertex,
                    int32_t* order, int32_t* offsets);

void gho_set_threads(int32_t threads);
int gho_gs_diffuse(const gho_mesh* mesh, const gho_levels* levels, double t, int32_t sweeps,
                   const double* initial, double* u_out, gho_report* report);
/* gs_diffuse with DiffusionConfig::residual_tolerance (diffusion.hpp:110-117);
 * report->primal_history receives E1 per sweep (capacity entries). */
int gho_gs_diffuse_tol(const gho_mesh* mesh, const gho_levels* levels, double t, int32_t sweeps, double tolerance,
                       const double* initial, double* u_out, gho_report* report);
double gho_diffusion_residual(const gho_mesh* mesh, const double* u, double t, const int32_t* sources,
                              int32_t ns);
void gho_face_gradient(const gho_mesh* mesh, const double* u, double* grad_out);
int32_t gho_normalized_target_gradients(const gho_mesh* mesh, const double* u, double* h_out);
int gho_admm_face(const gho_mesh* mesh, const double* h, int32_t max_iterations, double eps1, double eps2,
                  double mu, double* g_out, gho_report* report);
int gho_admm_edge(const gho_mesh* mesh, const double* h, int32_t max_iterations, double eps1, double eps2,
                  double mu, double* x_out, gho_report* report);
void gho_integrate_face(const gho_mesh* mesh, const gho_levels* levels, const double* g, double* d_out);
void gho_integrate_edge(const gho_mesh* mesh, const gho_levels* levels, const double* x, double* d_out);
uint64_t gho_field_hash(const double* values, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
