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

#include <cstdio>

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
  return bad;
}
