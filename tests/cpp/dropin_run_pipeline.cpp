// TEST INFRASTRUCTURE: the drop-in in one program. run_pipeline's solver chain
// (reference tools/geoheat.cpp:108-143) is written once as a template over the
// backend namespace and instantiated twice: with the reference's own inline
// functions (namespace geoheat, CPU) and with include/geoheat_b200.hpp
// (namespace geoheat::b200, B200) using the reference's own types
// (GEOHEAT_B200_REFERENCE_TYPES: Eigen::Vector3d, DiffusionConfig, ...).
// Built in the build container against /root/reference (Eigen shim from
// oracle/); run on the GPU: exit 0 iff both backends give bit-identical
// distances for config 1 (face and edge).
#include <geoheat/geoheat.hpp>
#define GEOHEAT_B200_REFERENCE_TYPES
#include "geoheat_b200.hpp"
#include "test_meshes.hpp"

#include <cmath>
#include <cstdio>
#include <sstream>

namespace ref {
using namespace geoheat;
}
namespace gpu {
using namespace geoheat::b200;
}

template <class Mesh, class Levels, class Build, class Bfs, class Diffuse, class Targets, class Face, class Edge,
          class IntF, class IntE>
geoheat::VertexScalarField chain(const geoheat::TriMesh& src, bool edge, Build build, Bfs bfs, Diffuse diffuse,
                                 Targets targets, Face face, Edge edgeopt, IntF intf, IntE inte) {
  Mesh mesh = build(src.positions, src.faces);
  std::vector<geoheat::Index> sources{0};
  Levels levels = bfs(mesh, sources);
  const double t = geoheat::diffusion_time(src, 1.0);  // the reference's t for both backends
  geoheat::DiffusionConfig dc;
  dc.sweeps = 1000;
  geoheat::SolverReport rep;
  geoheat::VertexScalarField u = diffuse(mesh, levels, t, dc, &rep);
  auto h = targets(mesh, u);
  geoheat::AdmmConfig admm;
  if (edge) return inte(mesh, levels, edgeopt(mesh, h.field, admm).differences);
  return intf(mesh, levels, face(mesh, h.field, admm).gradients);
}

int main() {
  geoheat::TriMesh src = geoheat::testing::icosphere_mesh(5);
  int bad = 0;
  for (bool edge : {false, true}) {
    auto cpu = chain<geoheat::TriMesh, geoheat::BfsLevels>(
        src, edge, [](auto p, auto f) { return geoheat::build_mesh(p, f); },
        [](const auto& m, auto s) { return geoheat::bfs_levels(m, s); },
        [](const auto& m, const auto& l, double t, const auto& c, auto* r) { return geoheat::gs_diffuse(m, l, t, c, r); },
        [](const auto& m, const auto& u) { return geoheat::normalized_target_gradients(m, u); },
        [](const auto& m, const auto& h, const auto& c) { return geoheat::admm_face_optimize(m, h, c); },
        [](const auto& m, const auto& h, const auto& c) { return geoheat::admm_edge_optimize(m, h, c); },
        [](const auto& m, const auto& l, const auto& g) { return geoheat::integrate_face_gradients(m, l, g); },
        [](const auto& m, const auto& l, const auto& x) { return geoheat::integrate_edge_differences(m, l, x); });
    auto dev = chain<geoheat::b200::TriMesh, geoheat::b200::BfsLevels>(
        src, edge, [](auto p, auto f) { return geoheat::b200::build_mesh(p, f); },
        [](const auto& m, auto s) { return geoheat::b200::bfs_levels(m, s); },
        [](const auto& m, const auto& l, double t, const auto& c, auto* r) { return geoheat::b200::gs_diffuse(m, l, t, c, r); },
        [](const auto& m, const auto& u) { return geoheat::b200::normalized_target_gradients(m, u); },
        [](const auto& m, const auto& h, const auto& c) { return geoheat::b200::admm_face_optimize(m, h, c); },
        [](const auto& m, const auto& h, const auto& c) { return geoheat::b200::admm_edge_optimize(m, h, c); },
        [](const auto& m, const auto& l, const auto& g) { return geoheat::b200::integrate_face_gradients(m, l, g); },
        [](const auto& m, const auto& l, const auto& x) { return geoheat::b200::integrate_edge_differences(m, l, x); });
    const auto hc = geoheat::field_hash(cpu), hd = geoheat::field_hash(dev);
    std::printf("%s: reference %016llx  b200 %016llx  %s\n", edge ? "edge" : "face", (unsigned long long)hc,
                (unsigned long long)hd, hc == hd ? "identical" : "DIFFERENT");
    bad += hc != hd;
  }
  // the rest of the reference surface the CLI uses, on the same types
  namespace G = geoheat;
  namespace B = geoheat::b200;
  auto report = [&](const char* what, bool ok) {
    std::printf("%s: %s\n", what, ok ? "identical" : "DIFFERENT");
    bad += !ok;
  };
  geoheat::TriMesh disk = geoheat::testing::hex_disk_mesh(8);
  std::vector<geoheat::Index> src2{0, 11};
  {  // mesh_io: save with the reference, load on the device; save on the device, compare bytes
    std::stringstream obj, ply;
    G::save_obj(obj, disk);
    G::save_ply(ply, disk);
    B::TriMesh a = B::load_mesh(obj, G::MeshFormat::OBJ);
    B::TriMesh b = B::load_mesh(ply, G::MeshFormat::PLY);
    auto pa = a.download<double>(GH_POSITIONS, 3 * (std::int64_t)a.vertex_count());
    auto pb = b.download<double>(GH_POSITIONS, 3 * (std::int64_t)b.vertex_count());
    bool same = pa.size() == 3 * disk.positions.size() && pa == pb;
    for (std::size_t v = 0; same && v < disk.positions.size(); ++v)
      for (int k = 0; k < 3; ++k) same = same && pa[3 * v + k] == disk.positions[v][k];
    std::stringstream back;
    B::save_ply(back, b);
    report("load_mesh obj/ply + save_ply", same && back.str() == ply.str());
  }
  {
    B::TriMesh m = B::build_mesh(disk.positions, disk.faces);
    report("dijkstra_edge_distance", B::dijkstra_edge_distance(m, src2) == G::dijkstra_edge_distance(disk, src2));
    report("analytic_oracle plane", B::analytic_oracle(G::AnalyticSurface::PlaneEuclidean, m, src2) ==
                                        G::analytic_oracle(G::AnalyticSurface::PlaneEuclidean, disk, src2));
    B::TriMesh fine = B::midpoint_subdivide(m, 2);
    G::TriMesh rfine = G::midpoint_subdivide(disk, 2);
    auto fp = fine.download<double>(GH_POSITIONS, 3 * (std::int64_t)fine.vertex_count());
    bool sub = fine.vertex_count() == rfine.vertex_count() && fine.face_count() == rfine.face_count();
    for (std::size_t v = 0; sub && v < rfine.positions.size(); ++v)
      for (int k = 0; k < 3; ++k) sub = sub && fp[3 * v + k] == rfine.positions[v][k];
    report("midpoint_subdivide", sub);
    const double t = G::diffusion_time(disk, 1.0);
    G::PoissonReport pr, br;
    auto dr = G::poisson_heat_method(disk, src2, t, 1e-8, &pr);
    auto db = B::poisson_heat_method(m, src2, t, 1e-8, &br);
    double worst = 0.0;
    for (std::size_t v = 0; v < dr.size(); ++v) worst = std::fmax(worst, std::fabs(dr[v] - db[v]));
    std::printf("poisson_heat_method: iterations %d+%d vs %d+%d, max |diff| %.3g\n", pr.heat_iterations,
                pr.poisson_iterations, br.heat_iterations, br.poisson_iterations, worst);
    bad += !(worst <= 1e-9 && pr.heat_iterations == br.heat_iterations &&
             pr.poisson_iterations == br.poisson_iterations);
  }
  return bad;
}
