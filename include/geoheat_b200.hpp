// geoheat_b200.hpp — the reference's C++ solver-loop API on the B200 path.
//
// Header-only C++20 wrapper over the C ABI (geoheat_b200.h). It re-exposes
// the exact signatures of the reference's inline functions
// (reference/proj/include/geoheat/*.hpp) in namespace geoheat::b200 and turns
// gh_status codes back into the reference's exception types, so a caller such
// as run_pipeline (tools/geoheat.cpp:71-161) switches backend by qualifying
// its calls with b200::.
//
// Types. Define GEOHEAT_B200_REFERENCE_TYPES after including the reference's
// <geoheat/geoheat.hpp> to reuse its Vec3 (Eigen::Vector3d), MeshError,
// SolverError, SolverReport, DiffusionConfig and AdmmConfig. Without it the
// header declares layout-compatible stand-ins, so it also builds alone.
#pragma once

#include <array>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <istream>
#include <optional>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "geoheat_b200.h"

#ifdef GEOHEAT_B200_REFERENCE_TYPES
namespace geoheat::b200 {
using ::geoheat::AdmmConfig;
using ::geoheat::AnalyticSurface;
using ::geoheat::DiffusionConfig;
using ::geoheat::MeshFormat;
using ::geoheat::PoissonReport;
using ::geoheat::Index;
using ::geoheat::MeshError;
using ::geoheat::SolverError;
using ::geoheat::SolverReport;
using ::geoheat::Vec3;
}  // namespace geoheat::b200
#else
namespace geoheat::b200 {
using Index = std::int32_t;
struct Vec3 {  // layout of Eigen::Vector3d: three contiguous doubles
  double v[3] = {0.0, 0.0, 0.0};
  Vec3() = default;
  Vec3(double x, double y, double z) : v{x, y, z} {}
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
};
class MeshError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
class SolverError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SolverReport {  // report.hpp:16-27
  int iterations = 0;
  bool converged = false;
  double final_primal = 0.0;
  double final_dual = 0.0;
  std::vector<double> primal_history;
  std::vector<double> dual_history;
  std::vector<double> residual_history;
  double wall_seconds = 0.0;
  std::uint64_t state_bytes_formula = 0;
  std::uint64_t state_bytes_allocated = 0;
};
struct DiffusionConfig {  // diffusion.hpp:16-25
  double m = 1.0;
  int sweeps = 1000;
  std::optional<double> residual_tolerance;
  void validate() const {
    if (!(m > 0.0)) throw std::invalid_argument("DiffusionConfig: m must be positive");
    if (sweeps < 0) throw std::invalid_argument("DiffusionConfig: sweeps must be >= 0");
  }
};
enum class MeshFormat { OBJ, PLY };                            // mesh_io.hpp:18
enum class AnalyticSurface { PlaneEuclidean, SphereGreatCircle };  // reference.hpp:278
struct PoissonReport {                                             // reference.hpp:163-170
  int heat_iterations = 0;
  int poisson_iterations = 0;
  double heat_residual = 0.0;
  double poisson_residual = 0.0;
  double heat_seconds = 0.0;
  double poisson_seconds = 0.0;
};
struct AdmmConfig {  // grad_face.hpp:15-26
  int max_iterations = 10;
  double eps1 = 1e-5;
  double eps2 = 1e-5;
  double mu = 100.0;
  void validate() const {
    if (max_iterations < 0) throw std::invalid_argument("AdmmConfig: max_iterations must be >= 0");
    if (!(eps1 > 0.0) || !(eps2 > 0.0)) throw std::invalid_argument("AdmmConfig: eps must be positive");
    if (!(mu > 0.0)) throw std::invalid_argument("AdmmConfig: mu must be positive");
  }
};
}  // namespace geoheat::b200
#endif

namespace geoheat::b200 {

static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be three packed doubles");

using FaceField = std::vector<Vec3>;
using EdgeDiffField = std::vector<double>;
using VertexScalarField = std::vector<double>;

/// Device failure (no GPU, out of memory, launch error): the B200 path has no CPU fallback.
class DeviceError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(gh_status s) {
  switch (s) {
    case GH_OK: return;
    case GH_ERR_MESH: throw MeshError(gh_last_error());
    case GH_ERR_INVALID: throw std::invalid_argument(gh_last_error());
    case GH_ERR_SOLVER: throw SolverError(gh_last_error());
    default: throw DeviceError(gh_last_error());
  }
}
inline const double* flat(const std::vector<Vec3>& v) { return reinterpret_cast<const double*>(v.data()); }
inline double* flat(std::vector<Vec3>& v) { return reinterpret_cast<double*>(v.data()); }
inline gh_admm_config to_c(const AdmmConfig& c) { return gh_admm_config{c.max_iterations, c.eps1, c.eps2, c.mu}; }
inline void to_report(const gh_solver_report& r, const std::vector<double>& ph, const std::vector<double>& dh,
                      SolverReport& out) {
  out.iterations = r.iterations;
  out.converged = r.converged != 0;
  out.final_primal = r.final_primal;
  out.final_dual = r.final_dual;
  out.primal_history.assign(ph.begin(), ph.begin() + r.iterations);
  out.dual_history.assign(dh.begin(), dh.begin() + r.iterations);
  out.wall_seconds = r.wall_seconds;
  out.state_bytes_formula = r.state_bytes_formula;
  out.state_bytes_allocated = r.state_bytes_allocated;
}
}  // namespace detail

/// No reference counterpart: the exact-zero skipping (DESIGN.md §3.7 — the
/// diffusion updates only the BFS levels the heat reaches before it underflows
/// to +0, the ADMM skips faces and edges that provably stay +0) changes no
/// result bit; it is opt-in (off by default: every update the reference runs
/// is run). This switches it process-wide.
inline void set_zero_level_truncation(bool on) { detail::check(gh_set_zero_level_truncation(on ? 1 : 0)); }

/// Device-resident TriMesh (mesh.hpp:21-94): move-only owner of a gh_mesh.
class TriMesh {
 public:
  TriMesh() = default;
  explicit TriMesh(gh_mesh* h) : h_(h) { detail::check(gh_mesh_get_info(h_, &info_)); }
  TriMesh(TriMesh&& o) noexcept : h_(std::exchange(o.h_, nullptr)), info_(o.info_) {}
  TriMesh& operator=(TriMesh&& o) noexcept {
    if (this != &o) {
      reset();
      h_ = std::exchange(o.h_, nullptr);
      info_ = o.info_;
    }
    return *this;
  }
  TriMesh(const TriMesh&) = delete;
  TriMesh& operator=(const TriMesh&) = delete;
  ~TriMesh() { reset(); }

  Index vertex_count() const { return info_.vertices; }
  Index face_count() const { return info_.faces; }
  Index edge_count() const { return info_.edges; }
  Index halfedge_count() const { return 3 * info_.faces; }
  Index interior_edge_count() const { return info_.interior_edges; }
  gh_mesh* handle() const { return h_; }

  /// Copy one TriMesh field to the host (T must match gh_mesh_array's element type).
  template <class T>
  std::vector<T> download(gh_mesh_array which, std::int64_t count) const {
    std::vector<T> out(static_cast<std::size_t>(count));
    detail::check(gh_mesh_download(h_, which, out.data(), count));
    return out;
  }

 private:
  void reset() {
    if (h_) gh_mesh_destroy(h_);
    h_ = nullptr;
  }
  gh_mesh* h_ = nullptr;
  gh_mesh_info info_{};
};

/// BfsLevels (bfs.hpp:15-22): the level arrays on the host plus the device handle.
struct BfsLevels {
  std::vector<Index> level_of_vertex;
  std::vector<std::vector<Index>> levels;
  std::vector<Index> parent_of_vertex;
  Index unreachable_count = 0;
  Index level_count() const { return static_cast<Index>(levels.size()); }

  BfsLevels() = default;
  BfsLevels(BfsLevels&& o) noexcept { *this = std::move(o); }
  BfsLevels& operator=(BfsLevels&& o) noexcept {
    if (this != &o) {
      if (h_) gh_bfs_destroy(h_);
      level_of_vertex = std::move(o.level_of_vertex);
      levels = std::move(o.levels);
      parent_of_vertex = std::move(o.parent_of_vertex);
      unreachable_count = o.unreachable_count;
      h_ = std::exchange(o.h_, nullptr);
      mesh_ = std::exchange(o.mesh_, nullptr);
    }
    return *this;
  }
  BfsLevels(const BfsLevels&) = delete;
  BfsLevels& operator=(const BfsLevels&) = delete;
  ~BfsLevels() {
    if (h_) gh_bfs_destroy(h_);
  }
  gh_levels* handle() const { return h_; }
  /// The levels' device layout belongs to the mesh they were built on; the
  /// solvers reject another mesh (the Python mirror raises the same way).
  void require_mesh(const TriMesh& mesh, const char* fn) const {
    if (mesh.handle() != mesh_)
      throw std::invalid_argument(std::string(fn) + ": levels were built on a different mesh");
  }

 private:
  friend BfsLevels bfs_levels(const TriMesh&, std::span<const Index>);
  gh_levels* h_ = nullptr;
  gh_mesh* mesh_ = nullptr;
};

/// build_mesh (mesh.hpp:113-286) with device preprocessing.
inline TriMesh build_mesh(std::vector<Vec3> positions, std::vector<std::array<Index, 3>> face_list) {
  gh_mesh* h = nullptr;
  detail::check(gh_mesh_create(detail::flat(positions), static_cast<std::int32_t>(positions.size()),
                               reinterpret_cast<const std::int32_t*>(face_list.data()),
                               static_cast<std::int32_t>(face_list.size()), &h));
  return TriMesh(h);
}

/// average_edge_length (mesh.hpp:289-293).
inline double average_edge_length(const TriMesh& mesh) {
  double h = 0.0;
  detail::check(gh_average_edge_length(mesh.handle(), &h));
  return h;
}

/// diffusion_time (diffusion.hpp:28-32).
inline double diffusion_time(const TriMesh& mesh, double m) {
  double t = 0.0;
  detail::check(gh_diffusion_time(mesh.handle(), m, &t));
  return t;
}

/// face_gradient (mesh.hpp:314-327).
inline FaceField face_gradient(const TriMesh& mesh, const VertexScalarField& u) {
  FaceField g(static_cast<std::size_t>(mesh.face_count()));
  detail::check(gh_face_gradient(mesh.handle(), u.data(), detail::flat(g)));
  return g;
}

/// bfs_levels (bfs.hpp:26-72).
inline BfsLevels bfs_levels(const TriMesh& mesh, std::span<const Index> sources) {
  BfsLevels out;
  detail::check(gh_bfs_create(mesh.handle(), sources.data(), static_cast<std::int32_t>(sources.size()), &out.h_));
  out.mesh_ = mesh.handle();
  gh_levels_info info{};
  detail::check(gh_bfs_get_info(out.h_, &info));
  const std::size_t nv = static_cast<std::size_t>(mesh.vertex_count());
  out.level_of_vertex.resize(nv);
  out.parent_of_vertex.resize(nv);
  std::vector<Index> order(nv - static_cast<std::size_t>(info.unreachable_count));
  std::vector<Index> offsets(static_cast<std::size_t>(info.level_count) + 1);
  detail::check(gh_bfs_download(out.h_, out.level_of_vertex.data(), out.parent_of_vertex.data(), order.data(),
                                offsets.data()));
  out.levels.resize(static_cast<std::size_t>(info.level_count));
  for (std::size_t l = 0; l < out.levels.size(); ++l)
    out.levels[l].assign(order.begin() + offsets[l], order.begin() + offsets[l + 1]);
  out.unreachable_count = info.unreachable_count;
  return out;
}

/// gs_diffuse (diffusion.hpp:57-124): sweep-pipelined on the device, bit-identical result.
inline VertexScalarField gs_diffuse(const TriMesh& mesh, const BfsLevels& levels, double t,
                                    const DiffusionConfig& config, SolverReport* report = nullptr,
                                    const VertexScalarField* initial = nullptr) {
  config.validate();
  levels.require_mesh(mesh, "gs_diffuse");
  VertexScalarField u(static_cast<std::size_t>(mesh.vertex_count()));
  gh_solver_report r{};
  std::vector<double> hist(static_cast<std::size_t>(config.sweeps > 0 ? config.sweeps : 1));
  if (config.residual_tolerance) {
    r.residual_history = hist.data();
    r.history_capacity = static_cast<std::int32_t>(hist.size());
    detail::check(gh_gs_diffuse_tol(levels.handle(), t, config.sweeps, *config.residual_tolerance,
                                    initial ? initial->data() : nullptr, u.data(), &r));
  } else {
    detail::check(gh_gs_diffuse(levels.handle(), t, config.sweeps, initial ? initial->data() : nullptr, u.data(), &r));
  }
  if (report) {
    report->iterations = r.iterations;
    report->converged = r.converged != 0;
    if (config.residual_tolerance) report->residual_history.assign(hist.begin(), hist.begin() + r.iterations);
    report->wall_seconds = r.wall_seconds;
  }
  return u;
}

/// diffusion_residual (diffusion.hpp:35-49); `levels` must be the BFS of `sources`.
inline double diffusion_residual(const TriMesh& mesh, const VertexScalarField& u, double t,
                                 const BfsLevels& levels) {
  levels.require_mesh(mesh, "diffusion_residual");
  double e1 = 0.0;
  detail::check(gh_diffusion_residual(levels.handle(), u.data(), t, &e1));
  return e1;
}

/// diffusion_residual (diffusion.hpp:35-49) with the reference's signature.
inline double diffusion_residual(const TriMesh& mesh, const VertexScalarField& u, double t,
                                 std::span<const Index> sources) {
  BfsLevels levels = bfs_levels(mesh, sources);
  return diffusion_residual(mesh, u, t, levels);
}

struct NormalizedGradients {  // diffusion.hpp:126-129
  FaceField field;
  Index zero_count = 0;
};

/// normalized_target_gradients (diffusion.hpp:132-145).
inline NormalizedGradients normalized_target_gradients(const TriMesh& mesh, const VertexScalarField& u) {
  NormalizedGradients out;
  out.field.resize(static_cast<std::size_t>(mesh.face_count()));
  detail::check(gh_normalized_target_gradients(mesh.handle(), u.data(), detail::flat(out.field), &out.zero_count));
  return out;
}

struct FaceAdmmResult {  // grad_face.hpp:208-211
  FaceField gradients;
  SolverReport report;
};
struct EdgeAdmmResult {  // grad_edge.hpp:200-203
  EdgeDiffField differences;
  SolverReport report;
};

/// admm_face_optimize (grad_face.hpp:228-237).
inline FaceAdmmResult admm_face_optimize(const TriMesh& mesh, const FaceField& targets, const AdmmConfig& config) {
  config.validate();
  FaceAdmmResult out;
  out.gradients.resize(static_cast<std::size_t>(mesh.face_count()));
  std::vector<double> ph(static_cast<std::size_t>(config.max_iterations) + 1), dh(ph.size());
  gh_solver_report r{};
  r.primal_history = ph.data();
  r.dual_history = dh.data();
  r.history_capacity = static_cast<std::int32_t>(ph.size());
  const gh_admm_config c = detail::to_c(config);
  detail::check(gh_admm_face_optimize(mesh.handle(), detail::flat(targets), &c, detail::flat(out.gradients), &r));
  detail::to_report(r, ph, dh, out.report);
  return out;
}

/// admm_edge_optimize (grad_edge.hpp:207-216).
inline EdgeAdmmResult admm_edge_optimize(const TriMesh& mesh, const FaceField& targets, const AdmmConfig& config) {
  config.validate();
  EdgeAdmmResult out;
  out.differences.resize(static_cast<std::size_t>(mesh.edge_count()));
  std::vector<double> ph(static_cast<std::size_t>(config.max_iterations) + 1), dh(ph.size());
  gh_solver_report r{};
  r.primal_history = ph.data();
  r.dual_history = dh.data();
  r.history_capacity = static_cast<std::int32_t>(ph.size());
  const gh_admm_config c = detail::to_c(config);
  detail::check(gh_admm_edge_optimize(mesh.handle(), detail::flat(targets), &c, out.differences.data(), &r));
  detail::to_report(r, ph, dh, out.report);
  return out;
}

/// integrate_face_gradients (integrate.hpp:40-59).
inline VertexScalarField integrate_face_gradients(const TriMesh& mesh, const BfsLevels& levels,
                                                  const FaceField& gradients) {
  levels.require_mesh(mesh, "integrate_face_gradients");
  VertexScalarField d(static_cast<std::size_t>(mesh.vertex_count()));
  detail::check(gh_integrate_face_gradients(levels.handle(), detail::flat(gradients), d.data()));
  return d;
}

/// integrate_edge_differences (integrate.hpp:64-75).
inline VertexScalarField integrate_edge_differences(const TriMesh& mesh, const BfsLevels& levels,
                                                    const EdgeDiffField& differences) {
  levels.require_mesh(mesh, "integrate_edge_differences");
  VertexScalarField d(static_cast<std::size_t>(mesh.vertex_count()));
  detail::check(gh_integrate_edge_differences(levels.handle(), differences.data(), d.data()));
  return d;
}

/// field_hash (report.hpp:145-153).
inline std::uint64_t field_hash(const VertexScalarField& values) {
  return gh_field_hash(values.data(), static_cast<std::int64_t>(values.size()));
}

// ---- mesh I/O (mesh_io.hpp): binary PLY decoded on the device, text
// formats tokenised by host threads; same messages as the reference.

/// format_from_path (mesh_io.hpp:271-278).
inline MeshFormat format_from_path(const std::string& path) {
  std::int32_t f = 0;
  detail::check(gh_mesh_format_from_path(path.c_str(), &f));
  return f == GH_FORMAT_OBJ ? MeshFormat::OBJ : MeshFormat::PLY;
}

/// load_mesh(path) (mesh_io.hpp:280-285).
inline TriMesh load_mesh(const std::string& path) {
  gh_mesh* h = nullptr;
  detail::check(gh_mesh_load(path.c_str(), &h, nullptr));
  return TriMesh(h);
}

/// load_mesh(istream, format) (mesh_io.hpp:267-269).
inline TriMesh load_mesh(std::istream& in, MeshFormat format) {
  const std::string data((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  gh_mesh* h = nullptr;
  detail::check(gh_mesh_load_memory(data.data(), data.size(), format == MeshFormat::OBJ ? GH_FORMAT_OBJ : GH_FORMAT_PLY,
                                    &h, nullptr));
  return TriMesh(h);
}

namespace detail {
struct Bytes {  // a gh_free'd buffer
  void* p = nullptr;
  std::uint64_t n = 0;
  ~Bytes() { gh_free(p); }
};
}  // namespace detail

/// save_obj (mesh_io.hpp:287-295).
inline void save_obj(std::ostream& os, const TriMesh& mesh) {
  detail::Bytes b;
  detail::check(gh_mesh_serialize(mesh.handle(), GH_FORMAT_OBJ, nullptr, &b.p, &b.n));
  os.write(static_cast<const char*>(b.p), static_cast<std::streamsize>(b.n));
}

/// save_ply (mesh_io.hpp:297-319): binary little-endian, optional per-vertex quality.
inline void save_ply(std::ostream& os, const TriMesh& mesh, const VertexScalarField* quality = nullptr) {
  detail::Bytes b;
  detail::check(gh_mesh_serialize(mesh.handle(), GH_FORMAT_PLY, quality ? quality->data() : nullptr, &b.p, &b.n));
  os.write(static_cast<const char*>(b.p), static_cast<std::streamsize>(b.n));
}

/// save_mesh (mesh_io.hpp:321-326).
inline void save_mesh(const std::string& path, const TriMesh& mesh) {
  detail::check(gh_mesh_save(mesh.handle(), path.c_str(), nullptr));
}

/// write_distances_txt / write_distances_csv (mesh_io.hpp:329-344).
inline void write_distances_txt(std::ostream& os, const VertexScalarField& d) {
  detail::Bytes b;
  detail::check(gh_format_distances(d.data(), static_cast<std::int64_t>(d.size()), GH_DISTANCES_TXT, &b.p, &b.n));
  os.write(static_cast<const char*>(b.p), static_cast<std::streamsize>(b.n));
}
inline void write_distances_csv(std::ostream& os, const VertexScalarField& d) {
  detail::Bytes b;
  detail::check(gh_format_distances(d.data(), static_cast<std::int64_t>(d.size()), GH_DISTANCES_CSV, &b.p, &b.n));
  os.write(static_cast<const char*>(b.p), static_cast<std::streamsize>(b.n));
}

// ---- the classic heat method and the evaluation layer (reference.hpp,
// subdivide.hpp, mesh.hpp:297-310)

/// poisson_heat_method (reference.hpp:175-216) on device CG.
inline VertexScalarField poisson_heat_method(const TriMesh& mesh, std::span<const Index> sources, double t,
                                             double cg_tol, PoissonReport* report = nullptr) {
  BfsLevels levels = bfs_levels(mesh, sources);
  VertexScalarField d(static_cast<std::size_t>(mesh.vertex_count()));
  gh_poisson_report r{};
  detail::check(gh_poisson_heat_method(levels.handle(), t, cg_tol, d.data(), &r));
  if (report) {
    report->heat_iterations = r.heat_iterations;
    report->poisson_iterations = r.poisson_iterations;
    report->heat_residual = r.heat_residual;
    report->poisson_residual = r.poisson_residual;
    report->heat_seconds = r.heat_seconds;
    report->poisson_seconds = r.poisson_seconds;
  }
  return d;
}

/// dijkstra_edge_distance (reference.hpp:220-245).
inline VertexScalarField dijkstra_edge_distance(const TriMesh& mesh, std::span<const Index> sources) {
  VertexScalarField d(static_cast<std::size_t>(mesh.vertex_count()));
  detail::check(gh_dijkstra_distance(mesh.handle(), sources.data(), static_cast<std::int32_t>(sources.size()), d.data()));
  return d;
}

/// analytic_oracle (reference.hpp:283-321).
inline VertexScalarField analytic_oracle(AnalyticSurface kind, const TriMesh& mesh, std::span<const Index> sources) {
  VertexScalarField d(static_cast<std::size_t>(mesh.vertex_count()));
  detail::check(gh_analytic_distance(mesh.handle(),
                                     kind == AnalyticSurface::PlaneEuclidean ? GH_SURFACE_PLANE : GH_SURFACE_SPHERE,
                                     sources.data(), static_cast<std::int32_t>(sources.size()), d.data()));
  return d;
}

/// mean_relative_error (reference.hpp:250-266).
inline double mean_relative_error(const VertexScalarField& d, const VertexScalarField& d_ref,
                                  std::span<const Index> sources, Index* excluded = nullptr) {
  double mre = 0.0, e2 = 0.0;
  std::int32_t exc = 0;
  detail::check(gh_error_metrics(d.data(), d_ref.data(), static_cast<std::int64_t>(d.size()), sources.data(),
                                 static_cast<std::int32_t>(sources.size()), &mre, &exc, &e2));
  if (excluded) *excluded = exc;
  return mre;
}

/// recovery_error (reference.hpp:269-276).
inline double recovery_error(const VertexScalarField& d, const VertexScalarField& d_ref) {
  double mre = 0.0, e2 = 0.0;
  std::int32_t exc = 0;
  detail::check(gh_error_metrics(d.data(), d_ref.data(), static_cast<std::int64_t>(d.size()), nullptr, 0, &mre, &exc,
                                 &e2));
  return e2;
}

/// midpoint_subdivide (subdivide.hpp:14-44).
inline TriMesh midpoint_subdivide(const TriMesh& mesh, int levels) {
  gh_mesh* h = nullptr;
  detail::check(gh_mesh_subdivide(mesh.handle(), levels, &h));
  return TriMesh(h);
}

/// deterministic_sum (parallel.hpp:50-54): left-to-right, bit-identical, on the device.
inline double deterministic_sum(const std::vector<double>& terms) {
  double out = 0.0;
  detail::check(gh_deterministic_sum(terms.data(), static_cast<std::int64_t>(terms.size()), &out));
  return out;
}

/// triangulation_quality (mesh.hpp:297-310).
inline double triangulation_quality(const TriMesh& mesh) {
  double tau = 0.0;
  detail::check(gh_triangulation_quality(mesh.handle(), &tau));
  return tau;
}

}  // namespace geoheat::b200
