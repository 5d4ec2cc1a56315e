// C++ drop-in check: the reference's library chain (tests/acceptance.cpp:49-68,
// run_pipelines) written against geoheat::b200 instead of geoheat, on config 1
// (icosphere_mesh(5), source 0). argv[1] = t as a C99 hex float (the
// reference's t, from tests/golden). Exit 0 iff both distance hashes equal the
// reference's, a malformed mesh throws MeshError, levels
// of another mesh are rejected, and four host threads solving on the one mesh
// at once all get the single-thread result (the per-mesh lock of the C ABI).
#include "geoheat_b200.hpp"

#include <cstdio>
#include <cstdlib>
#include <thread>

extern "C" int gh_gen_icosphere(int32_t, double, double**, int32_t*, int32_t**, int32_t*);
extern "C" void gh_gen_free(void*);

namespace b200 = geoheat::b200;

int main(int argc, char** argv) {
  const double t = argc > 1 ? std::strtod(argv[1], nullptr) : 0.0;
  double* P = nullptr;
  int32_t* F = nullptr;
  int32_t nv = 0, nf = 0;
  if (gh_gen_icosphere(5, 1.0, &P, &nv, &F, &nf) != 0) return 10;
  std::vector<b200::Vec3> positions(nv);
  for (int32_t i = 0; i < nv; ++i) positions[i] = b200::Vec3(P[3 * i], P[3 * i + 1], P[3 * i + 2]);
  std::vector<std::array<b200::Index, 3>> faces(nf);
  for (int32_t i = 0; i < nf; ++i) faces[i] = {F[3 * i], F[3 * i + 1], F[3 * i + 2]};
  gh_gen_free(P);
  gh_gen_free(F);

  b200::TriMesh mesh = b200::build_mesh(positions, faces);
  std::vector<b200::Index> sources{0};
  b200::BfsLevels levels = b200::bfs_levels(mesh, sources);
  b200::DiffusionConfig dc;
  dc.sweeps = 1000;
  b200::VertexScalarField u = b200::gs_diffuse(mesh, levels, t, dc);
  b200::NormalizedGradients h = b200::normalized_target_gradients(mesh, u);
  b200::AdmmConfig admm;
  b200::FaceAdmmResult face = b200::admm_face_optimize(mesh, h.field, admm);
  b200::EdgeAdmmResult edge = b200::admm_edge_optimize(mesh, h.field, admm);
  const auto hf = b200::field_hash(b200::integrate_face_gradients(mesh, levels, face.gradients));
  const auto he = b200::field_hash(b200::integrate_edge_differences(mesh, levels, edge.differences));
  std::printf("zero_count %d face %016llx edge %016llx iters %d %d\n", h.zero_count, (unsigned long long)hf,
              (unsigned long long)he, face.report.iterations, edge.report.iterations);
  bool threw = false;
  try {
    std::vector<b200::Vec3> p = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}};
    b200::build_mesh(p, {{0, 1, 2}, {1, 0, 3}, {0, 1, 4}});
  } catch (const b200::MeshError& e) {
    threw = std::string(e.what()) == "non-manifold edge (0,1): 3 incident faces";
  }
  // levels built on another mesh: std::invalid_argument, as the Python mirror
  bool mismatch = false;
  {
    b200::TriMesh other = b200::build_mesh(positions, faces);
    try {
      b200::gs_diffuse(other, levels, t, dc);
    } catch (const std::invalid_argument& e) {
      mismatch = std::string(e.what()) == "gs_diffuse: levels were built on a different mesh";
    }
  }
  // concurrent solves on one mesh + levels from four threads
  std::vector<std::uint64_t> got(4, 0);
  {
    std::vector<std::thread> th;
    for (int i = 0; i < 4; ++i)
      th.emplace_back([&, i] {
        try {
          b200::DiffusionConfig c;
          c.sweeps = 300 + 100 * (i & 1);
          got[i] = b200::field_hash(b200::gs_diffuse(mesh, levels, t, c));
        } catch (...) {
          got[i] = 1;
        }
      });
    for (auto& x : th) x.join();
  }
  bool threads_ok = true;
  for (int i = 0; i < 4; ++i) {
    b200::DiffusionConfig c;
    c.sweeps = 300 + 100 * (i & 1);
    threads_ok = threads_ok && got[i] == b200::field_hash(b200::gs_diffuse(mesh, levels, t, c));
  }
  std::printf("mismatch rejected %d, threads %d\n", (int)mismatch, (int)threads_ok);
  const bool ok = hf == 0xcca540701b66bfd5ull && he == 0xa8e56e8b98582eb9ull && h.zero_count == 5560 && threw &&
                  mismatch && threads_ok;
  std::printf("%s\n", ok ? "PASS" : "FAIL");
  return ok ? 0 : 1;
}
