// TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
//
// Adapts the UNMODIFIED reference headers (/root/reference/proj/include/geoheat,
// compiled in place, never copied) to the C oracle API of geoheat_oracle.h.
// Built by oracle/build_ref.sh into oracle/_ref/libgeoheat_ref.so with the
// reference's own flags (-std=gnu++20 -O2 -DNDEBUG -fopenmp, no -march, so no
// FMA) against oracle/eigen_shim. Every entry point forwards to the reference
// function named in its comment; nothing here re-implements solver arithmetic.

#include "geoheat/bfs.hpp"
#include "geoheat/diffusion.hpp"
#include "geoheat/grad_edge.hpp"
#include "geoheat/grad_face.hpp"
#include "geoheat/integrate.hpp"
#include "geoheat/mesh.hpp"
#include "geoheat/mesh_io.hpp"
#include "geoheat/parallel.hpp"
#include "geoheat/reference.hpp"
#include "geoheat/report.hpp"
#include "geoheat/subdivide.hpp"
#include "test_meshes.hpp"  // reference tests/test_meshes.hpp (generators only)

#include "geoheat_oracle.h"

#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

using namespace geoheat;

struct gho_mesh {
  TriMesh m;
};
struct gho_levels {
  BfsLevels l;
  std::vector<Index> order, offsets;
};

namespace {
void put_err(char* err, int32_t errlen, const char* what) {
  if (err && errlen > 0) {
    std::strncpy(err, what, static_cast<size_t>(errlen) - 1);
    err[errlen - 1] = 0;
  }
}
void fill_report(const SolverReport& r, gho_report* out) {
  if (!out) return;
  out->iterations = r.iterations;
  out->converged = r.converged ? 1 : 0;
  out->final_primal = r.final_primal;
  out->final_dual = r.final_dual;
  for (int i = 0; i < out->history_capacity; ++i) {
    if (out->primal_history && i < static_cast<int>(r.primal_history.size())) out->primal_history[i] = r.primal_history[i];
    if (out->dual_history && i < static_cast<int>(r.dual_history.size())) out->dual_history[i] = r.dual_history[i];
  }
  out->state_bytes_formula = r.state_bytes_formula;
  out->state_bytes_allocated = r.state_bytes_allocated;
  out->wall_seconds = r.wall_seconds;
}
FaceField to_field(const double* v, Index n) {
  FaceField f(n);
  for (Index i = 0; i < n; ++i) f[i] = Vec3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  return f;
}
void from_field(const FaceField& f, double* out) {
  for (size_t i = 0; i < f.size(); ++i)
    for (int k = 0; k < 3; ++k) out[3 * i + k] = f[i][k];
}
}  // namespace

extern "C" {

// build_mesh (mesh.hpp:113-286)
int gho_build_mesh(const double* positions, int32_t nv, const int32_t* faces, int32_t nf, gho_mesh** out,
                   char* err, int32_t errlen) {
  std::vector<Vec3> p(nv);
  for (int32_t i = 0; i < nv; ++i) p[i] = Vec3(positions[3 * i], positions[3 * i + 1], positions[3 * i + 2]);
  std::vector<std::array<Index, 3>> f(nf);
  for (int32_t i = 0; i < nf; ++i) f[i] = {faces[3 * i], faces[3 * i + 1], faces[3 * i + 2]};
  try {
    auto* h = new gho_mesh{build_mesh(std::move(p), std::move(f))};
    *out = h;
    return 0;
  } catch (const MeshError& e) {
    put_err(err, errlen, e.what());
    return 1;
  } catch (const std::invalid_argument& e) {
    put_err(err, errlen, e.what());
    return 2;
  }
}

void gho_mesh_free(gho_mesh* mesh) { delete mesh; }

void gho_mesh_counts(const gho_mesh* mesh, int32_t counts[4]) {
  counts[0] = mesh->m.vertex_count();
  counts[1] = mesh->m.face_count();
  counts[2] = mesh->m.edge_count();
  counts[3] = mesh->m.interior_edge_count();
}

const void* gho_mesh_array(const gho_mesh* mesh, int32_t which, int64_t* count) {
  const TriMesh& m = mesh->m;
  switch (which) {
    case GHO_POSITIONS: *count = 3 * (int64_t)m.positions.size(); return m.positions.data();
    case GHO_FACES: *count = 3 * (int64_t)m.faces.size(); return m.faces.data();
    case GHO_HALFEDGE_TWIN: *count = m.halfedge_twin.size(); return m.halfedge_twin.data();
    case GHO_HALFEDGE_EDGE: *count = m.halfedge_edge.size(); return m.halfedge_edge.data();
    case GHO_EDGE_VERTICES: *count = 2 * (int64_t)m.edge_vertices.size(); return m.edge_vertices.data();
    case GHO_EDGE_HALFEDGES: *count = 2 * (int64_t)m.edge_halfedges.size(); return m.edge_halfedges.data();
    case GHO_INTERIOR_EDGES: *count = m.interior_edges.size(); return m.interior_edges.data();
    case GHO_INTERIOR_EDGE_INDEX: *count = m.interior_edge_index.size(); return m.interior_edge_index.data();
    case GHO_VERTEX_ON_BOUNDARY: *count = m.vertex_on_boundary.size(); return m.vertex_on_boundary.data();
    case GHO_FACE_AREA: *count = m.face_area.size(); return m.face_area.data();
    case GHO_FACE_NORMAL: *count = 3 * (int64_t)m.face_normal.size(); return m.face_normal.data();
    case GHO_VERTEX_AREA: *count = m.vertex_area.size(); return m.vertex_area.data();
    case GHO_HALFEDGE_COT: *count = m.halfedge_cot.size(); return m.halfedge_cot.data();
    case GHO_EDGE_WEIGHT: *count = m.edge_weight.size(); return m.edge_weight.data();
    case GHO_VERTEX_WEIGHT_SUM: *count = m.vertex_weight_sum.size(); return m.vertex_weight_sum.data();
    case GHO_VV_OFFSET: *count = m.vv_offset.size(); return m.vv_offset.data();
    case GHO_VV_INDEX: *count = m.vv_index.size(); return m.vv_index.data();
    case GHO_VV_EDGE: *count = m.vv_edge.size(); return m.vv_edge.data();
    case GHO_VV_WEIGHT: *count = m.vv_weight.size(); return m.vv_weight.data();
    case GHO_VC_OFFSET: *count = m.vc_offset.size(); return m.vc_offset.data();
    case GHO_VC_CORNER: *count = m.vc_corner.size(); return m.vc_corner.data();
    default: *count = 0; return nullptr;
  }
}

// average_edge_length (mesh.hpp:289-293)
double gho_average_edge_length(const gho_mesh* mesh) { return average_edge_length(mesh->m); }
// triangulation_quality (mesh.hpp:297-310)
double gho_triangulation_quality(const gho_mesh* mesh) { return triangulation_quality(mesh->m); }

// bfs_levels (bfs.hpp:26-72)
int gho_bfs(const gho_mesh* mesh, const int32_t* sources, int32_t ns, gho_levels** out, char* err,
            int32_t errlen) {
  try {
    auto* h = new gho_levels{bfs_levels(mesh->m, std::span<const Index>(sources, ns)), {}, {}};
    h->offsets.push_back(0);
    for (const auto& ring : h->l.levels) {
      h->order.insert(h->order.end(), ring.begin(), ring.end());
      h->offsets.push_back(static_cast<Index>(h->order.size()));
    }
    *out = h;
    return 0;
  } catch (const std::invalid_argument& e) {
    put_err(err, errlen, e.what());
    return 2;
  }
}

void gho_levels_free(gho_levels* levels) { delete levels; }

void gho_levels_info(const gho_levels* levels, int32_t info[2]) {
  info[0] = levels->l.level_count();
  info[1] = levels->l.unreachable_count;
}

void gho_levels_get(const gho_levels* levels, int32_t* level_of_vertex, int32_t* parent_of_vertex,
                    int32_t* order, int32_t* offsets) {
  const auto& l = levels->l;
  if (level_of_vertex) std::memcpy(level_of_vertex, l.level_of_vertex.data(), l.level_of_vertex.size() * 4);
  if (parent_of_vertex) std::memcpy(parent_of_vertex, l.parent_of_vertex.data(), l.parent_of_vertex.size() * 4);
  if (order) std::memcpy(order, levels->order.data(), levels->order.size() * 4);
  if (offsets) std::memcpy(offsets, levels->offsets.data(), levels->offsets.size() * 4);
}

// set_thread_count (parallel.hpp:25)
void gho_set_threads(int32_t threads) { set_thread_count(threads); }

// gs_diffuse (diffusion.hpp:57-124)
int gho_gs_diffuse(const gho_mesh* mesh, const gho_levels* levels, double t, int32_t sweeps,
                   const double* initial, double* u_out, gho_report* report) {
  DiffusionConfig cfg;
  cfg.sweeps = sweeps;
  SolverReport rep;
  try {
    VertexScalarField u;
    if (initial) {
      VertexScalarField init(initial, initial + mesh->m.vertex_count());
      u = gs_diffuse(mesh->m, levels->l, t, cfg, &rep, &init);
    } else {
      u = gs_diffuse(mesh->m, levels->l, t, cfg, &rep);
    }
    std::memcpy(u_out, u.data(), u.size() * sizeof(double));
  } catch (const std::invalid_argument&) {
    return 2;
  }
  fill_report(rep, report);
  return 0;
}

// gs_diffuse with residual_tolerance (diffusion.hpp:110-117)
int gho_gs_diffuse_tol(const gho_mesh* mesh, const gho_levels* levels, double t, int32_t sweeps, double tolerance,
                       const double* initial, double* u_out, gho_report* report) {
  DiffusionConfig cfg;
  cfg.sweeps = sweeps;
  cfg.residual_tolerance = tolerance;
  SolverReport rep;
  try {
    VertexScalarField u;
    if (initial) {
      VertexScalarField init(initial, initial + mesh->m.vertex_count());
      u = gs_diffuse(mesh->m, levels->l, t, cfg, &rep, &init);
    } else {
      u = gs_diffuse(mesh->m, levels->l, t, cfg, &rep);
    }
    std::memcpy(u_out, u.data(), u.size() * sizeof(double));
  } catch (const std::invalid_argument&) {
    return 2;
  }
  rep.primal_history = rep.residual_history;
  fill_report(rep, report);
  return 0;
}

// diffusion_residual (diffusion.hpp:35-49)
double gho_diffusion_residual(const gho_mesh* mesh, const double* u, double t, const int32_t* sources,
                              int32_t ns) {
  VertexScalarField uu(u, u + mesh->m.vertex_count());
  return diffusion_residual(mesh->m, uu, t, std::span<const Index>(sources, ns));
}

// face_gradient (mesh.hpp:314-327)
void gho_face_gradient(const gho_mesh* mesh, const double* u, double* grad_out) {
  VertexScalarField uu(u, u + mesh->m.vertex_count());
  from_field(face_gradient(mesh->m, uu), grad_out);
}

// normalized_target_gradients (diffusion.hpp:132-145)
int32_t gho_normalized_target_gradients(const gho_mesh* mesh, const double* u, double* h_out) {
  VertexScalarField uu(u, u + mesh->m.vertex_count());
  NormalizedGradients n = normalized_target_gradients(mesh->m, uu);
  from_field(n.field, h_out);
  return n.zero_count;
}

// admm_face_optimize (grad_face.hpp:228-237)
int gho_admm_face(const gho_mesh* mesh, const double* h, int32_t max_iterations, double eps1, double eps2,
                  double mu, double* g_out, gho_report* report) {
  AdmmConfig cfg;
  cfg.max_iterations = max_iterations;
  cfg.eps1 = eps1;
  cfg.eps2 = eps2;
  cfg.mu = mu;
  try {
    FaceField targets = to_field(h, mesh->m.face_count());
    FaceAdmmResult r = admm_face_optimize(mesh->m, targets, cfg);
    from_field(r.gradients, g_out);
    fill_report(r.report, report);
  } catch (const std::invalid_argument&) {
    return 2;
  }
  return 0;
}

// admm_edge_optimize (grad_edge.hpp:207-216)
int gho_admm_edge(const gho_mesh* mesh, const double* h, int32_t max_iterations, double eps1, double eps2,
                  double mu, double* x_out, gho_report* report) {
  AdmmConfig cfg;
  cfg.max_iterations = max_iterations;
  cfg.eps1 = eps1;
  cfg.eps2 = eps2;
  cfg.mu = mu;
  try {
    FaceField targets = to_field(h, mesh->m.face_count());
    EdgeAdmmResult r = admm_edge_optimize(mesh->m, targets, cfg);
    std::memcpy(x_out, r.differences.data(), r.differences.size() * sizeof(double));
    fill_report(r.report, report);
  } catch (const std::invalid_argument&) {
    return 2;
  }
  return 0;
}

// integrate_face_gradients (integrate.hpp:40-59)
void gho_integrate_face(const gho_mesh* mesh, const gho_levels* levels, const double* g, double* d_out) {
  FaceField gg = to_field(g, mesh->m.face_count());
  VertexScalarField d = integrate_face_gradients(mesh->m, levels->l, gg);
  std::memcpy(d_out, d.data(), d.size() * sizeof(double));
}

// integrate_edge_differences (integrate.hpp:64-75)
void gho_integrate_edge(const gho_mesh* mesh, const gho_levels* levels, const double* x, double* d_out) {
  EdgeDiffField xx(x, x + mesh->m.edge_count());
  VertexScalarField d = integrate_edge_differences(mesh->m, levels->l, xx);
  std::memcpy(d_out, d.data(), d.size() * sizeof(double));
}

// field_hash (report.hpp:145-153)
uint64_t gho_field_hash(const double* values, int64_t n) {
  VertexScalarField v(values, values + n);
  return field_hash(v);
}

// ---- reference-only extras: the reference's own test-mesh generators
// (tests/test_meshes.hpp) and analytic oracle (reference.hpp:283-321), used
// to produce golden fixtures and to pin the repo's mesh generators.
int gho_ref_test_mesh(const char* name, const double* params, int32_t nparams, double** pos_out, int32_t* nv,
                      int32_t** faces_out, int32_t* nf) {
  using namespace geoheat::testing;
  std::string n(name);
  auto P = [&](int i, double dflt) { return i < nparams ? params[i] : dflt; };
  TriMesh m;
  try {
    if (n == "unit_square") m = unit_square_mesh();
    else if (n == "equilateral_triangle") m = equilateral_triangle_mesh(P(0, 1.0));
    else if (n == "right_triangle") m = right_triangle_mesh();
    else if (n == "two_disjoint_triangles") m = two_disjoint_triangles_mesh();
    else if (n == "grid") m = grid_mesh((int)P(0, 4), (int)P(1, 4), P(2, 1.0), P(3, 1.0));
    else if (n == "strip") m = strip_mesh((int)P(0, 4));
    else if (n == "hex_disk") m = hex_disk_mesh((int)P(0, 4), P(1, 1.0));
    else if (n == "icosphere") m = icosphere_mesh((int)P(0, 2), P(1, 1.0));
    else if (n == "torus") m = torus_mesh((int)P(0, 24), (int)P(1, 12), P(2, 2.0), P(3, 0.7));
    else if (n == "polar_disk") m = polar_disk_mesh((int)P(0, 4), (int)P(1, 8), P(2, 1.0));
    else if (n == "uv_sphere") m = uv_sphere_mesh((int)P(0, 8), (int)P(1, 16), P(2, 1.0));
    else if (n == "ladder") m = ladder_mesh((int)P(0, 4));
    else return 2;
  } catch (const MeshError&) {
    return 1;
  }
  *nv = m.vertex_count();
  *nf = m.face_count();
  *pos_out = static_cast<double*>(std::malloc(sizeof(double) * 3 * (*nv)));
  *faces_out = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * 3 * (*nf)));
  for (Index i = 0; i < *nv; ++i)
    for (int k = 0; k < 3; ++k) (*pos_out)[3 * i + k] = m.positions[i][k];
  for (Index i = 0; i < *nf; ++i)
    for (int k = 0; k < 3; ++k) (*faces_out)[3 * i + k] = m.faces[i][k];
  return 0;
}

void gho_ref_free(void* p) { std::free(p); }

// analytic_oracle (reference.hpp:283-321): kind 0 plane, 1 sphere
int gho_ref_analytic(const gho_mesh* mesh, int32_t kind, const int32_t* sources, int32_t ns, double* d_out) {
  try {
    VertexScalarField d = analytic_oracle(kind == 0 ? AnalyticSurface::PlaneEuclidean : AnalyticSurface::SphereGreatCircle,
                                          mesh->m, std::span<const Index>(sources, ns));
    std::memcpy(d_out, d.data(), d.size() * sizeof(double));
  } catch (const std::invalid_argument&) {
    return 2;
  }
  return 0;
}

// mean_relative_error (reference.hpp:250-266)
double gho_ref_mean_relative_error(const double* d, const double* d_ref, int64_t n, const int32_t* sources,
                                   int32_t ns) {
  VertexScalarField a(d, d + n), b(d_ref, d_ref + n);
  return mean_relative_error(a, b, std::span<const Index>(sources, ns));
}

// ---- reference mesh I/O (mesh_io.hpp), the checker for gh_mesh_load* and
// the writers. load: rc 0 ok, 1 with the exception text in err.
int gho_ref_load_mesh(const char* data, int64_t n, int32_t format, gho_mesh** out, char* err, int32_t errlen) {
  try {
    std::istringstream in(std::string(data, static_cast<size_t>(n)), std::ios::in | std::ios::binary);
    TriMesh m = load_mesh(in, format == 0 ? MeshFormat::OBJ : MeshFormat::PLY);
    *out = new gho_mesh{std::move(m)};
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

// save_obj / save_ply (quality may be NULL) and the distance writers; the
// bytes are malloc'd (gho_ref_free).
static char* dup_bytes(const std::string& s, int64_t* n) {
  char* p = static_cast<char*>(std::malloc(s.size() ? s.size() : 1));
  std::memcpy(p, s.data(), s.size());
  *n = static_cast<int64_t>(s.size());
  return p;
}

char* gho_ref_save_mesh(const gho_mesh* mesh, int32_t format, const double* quality, int64_t* n) {
  std::ostringstream os(std::ios::out | std::ios::binary);
  if (format == 0) {
    save_obj(os, mesh->m);
  } else if (quality) {
    VertexScalarField q(quality, quality + mesh->m.vertex_count());
    save_ply(os, mesh->m, &q);
  } else {
    save_ply(os, mesh->m);
  }
  return dup_bytes(os.str(), n);
}

char* gho_ref_write_distances(const double* d, int64_t count, int32_t csv, int64_t* n) {
  VertexScalarField v(d, d + count);
  std::ostringstream os(std::ios::out | std::ios::binary);
  if (csv) write_distances_csv(os, v);
  else write_distances_txt(os, v);
  return dup_bytes(os.str(), n);
}

// ---- the evaluation layer and the CG heat method (reference.hpp,
// subdivide.hpp), checkers for gh_poisson_heat_method, gh_dijkstra_distance,
// gh_mesh_subdivide and gh_error_metrics.
int gho_ref_poisson(const gho_mesh* mesh, const int32_t* sources, int32_t ns, double t, double tol, double* d_out,
                    int32_t* iters, double* residuals, char* err, int32_t errlen) {
  try {
    PoissonReport rep;
    VertexScalarField d = poisson_heat_method(mesh->m, std::span<const Index>(sources, ns), t, tol, &rep);
    std::memcpy(d_out, d.data(), d.size() * sizeof(double));
    iters[0] = rep.heat_iterations;
    iters[1] = rep.poisson_iterations;
    residuals[0] = rep.heat_residual;
    residuals[1] = rep.poisson_residual;
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

void gho_ref_dijkstra(const gho_mesh* mesh, const int32_t* sources, int32_t ns, double* d_out) {
  VertexScalarField d = dijkstra_edge_distance(mesh->m, std::span<const Index>(sources, ns));
  std::memcpy(d_out, d.data(), d.size() * sizeof(double));
}

gho_mesh* gho_ref_subdivide(const gho_mesh* mesh, int32_t levels) {
  return new gho_mesh{midpoint_subdivide(mesh->m, levels)};
}

double gho_ref_recovery_error(const double* d, const double* d_ref, int64_t n) {
  VertexScalarField a(d, d + n), b(d_ref, d_ref + n);
  return recovery_error(a, b);
}

int32_t gho_ref_mre_excluded(const double* d, const double* d_ref, int64_t n, const int32_t* sources, int32_t ns) {
  VertexScalarField a(d, d + n), b(d_ref, d_ref + n);
  Index excluded = 0;
  mean_relative_error(a, b, std::span<const Index>(sources, ns), &excluded);
  return excluded;
}

}  // extern "C"
