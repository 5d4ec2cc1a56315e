// Breadth-first distance recovery (reference integrate.hpp:19-75).
//
// The reference's step is d(v) = d(parent) + inc(v), with inc(v) computed
// before the addition (integrate.hpp:56, 72). inc depends only on the
// optimised field and the geometry, so it is computed for every vertex in one
// fully parallel gather kernel. The chain d(v) = d(parent) + inc(v) is then
// evaluated in BFS order by a co-resident kernel whose threads wait on their
// parent's published value (no per-level barrier), which reproduces the
// reference's additions exactly.

#include <algorithm>
#include <cmath>

#include "gh_internal.cuh"

using namespace ghd;

namespace {

constexpr int B = gh::kBlock;

// inc(v) for the face method (integrate.hpp:45-56), indexed by BFS position;
// e = edge_between(parent, v) (mesh.hpp:87-93) is the edge the BFS recorded
// with the parent
__global__ void k_inc_face(const int32_t* __restrict__ order, const int32_t* __restrict__ parent,
                           const int32_t* __restrict__ parent_edge, int64_t b, int64_t e,
                           const int32_t* __restrict__ edge_he, const double* __restrict__ pos,
                           const double* __restrict__ g, double* __restrict__ inc) {
  for (int64_t i = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = order[i], p = parent[v];
    const int32_t ed = parent_edge[v];
    const v3 step = sub(ld3(pos, v), ld3(pos, p));
    double sum = 0.0;
    int count = 0;
    for (int s = 0; s < 2; ++s) {
      const int32_t h = edge_he[2 * ed + s];
      if (h < 0) continue;
      sum += dot(ld3(g, h / 3), step);
      ++count;
    }
    inc[i] = ddiv(sum, (double)count);
  }
}

// inc(v) for the edge method (integrate.hpp:67-72)
__global__ void k_inc_edge(const int32_t* __restrict__ order, const int32_t* __restrict__ parent,
                           const int32_t* __restrict__ parent_edge, int64_t b, int64_t e,
                           const int32_t* __restrict__ edge_v, const double* __restrict__ x,
                           double* __restrict__ inc) {
  for (int64_t i = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = order[i], p = parent[v];
    const int32_t ed = parent_edge[v];
    const double sigma = edge_v[2 * ed] == p ? 1.0 : -1.0;
    inc[i] = sigma * x[ed];
  }
}

// d = 0 on D_0, +inf on unreachable vertices (integrate.hpp:20, 52), and a
// "pending" NaN payload no arithmetic produces on every vertex still to come.
constexpr unsigned long long kPending = 0x7FF4DEADBEEF0001ull;

__global__ void k_dist_init(const int32_t* __restrict__ level, int64_t nv, double* __restrict__ d) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x)
    d[v] = level[v] == 0 ? 0.0 : (level[v] < 0 ? INFINITY : __longlong_as_double((long long)kPending));
}

// d(v) = d(parent) + inc(v) in BFS order (run_levels, integrate.hpp:19-36):
// each thread walks its positions in increasing BFS order and waits until its
// parent's distance is published. Parents precede children in BFS order and
// every thread handles its positions in increasing order, so with all blocks
// co-resident the smallest pending position can always proceed. The additions
// are the reference's, hence bitwise; no per-level grid barrier.
__global__ void __launch_bounds__(B) k_chain(const int32_t* __restrict__ order, const int32_t* __restrict__ parent,
                                             int64_t b, int64_t e, const double* __restrict__ inc,
                                             double* __restrict__ d) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += stride) {
    const int32_t v = order[i];
    const int32_t p = parent[v];
    const double step = inc[i];
    unsigned long long x;
    unsigned ns = 0;
    for (;;) {
      asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(x) : "l"(d + p) : "memory");
      if (x != kPending) break;
      __nanosleep(ns);
      ns = ns < 256 ? ns + 32 : 256;
    }
    const double dv = __longlong_as_double((long long)x) + step;
    asm volatile("st.volatile.global.f64 [%0], %1;" ::"l"(d + v), "d"(dv) : "memory");
  }
}

void run_chain(gh_levels* L, const double* inc, double* d) {
  gh_mesh* m = L->mesh;
  cudaStream_t s = m->stream;
  k_dist_init<<<gh::grid_for(m->nv), B, 0, s>>>(L->level.p, m->nv, d);
  GH_LAUNCH_CHECK();
  m->launches++;
  const int64_t b = L->h_offsets.size() > 1 ? L->h_offsets[1] : 0, e = L->nreach;
  if (e <= b) return;
  int nsm = 0, per_sm = 0;
  GH_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device));
  GH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chain, B, 0));
  const int64_t want = (e - b + B - 1) / B;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * std::max(1, per_sm), want));
  const int32_t* order = L->order.p;
  const int32_t* parent = L->parent.p;
  void* args[] = {&order, &parent, (void*)&b, (void*)&e, &inc, &d};
  GH_CUDA(cudaLaunchCooperativeKernel((void*)k_chain, grid, B, args, 0, s));
  GH_LAUNCH_CHECK();
  m->launches++;
}

}  // namespace

namespace gh {

void integrate_face_dev(gh_levels* L, const double* d_g, double* d_d) {
  gh_mesh* m = L->mesh;
  Scratch<double> inc(L->nreach + 1, m->stream);
  const int64_t b = L->h_offsets.size() > 1 ? L->h_offsets[1] : 0, e = L->nreach;
  if (e > b) {
    k_inc_face<<<grid_for(e - b), B, 0, m->stream>>>(L->order.p, L->parent.p, L->parent_edge.p, b, e, m->edge_he.p,
                                                     m->pos.p, d_g, inc.p);
    GH_LAUNCH_CHECK();
    m->launches++;
  }
  run_chain(L, inc.p, d_d);
}

void integrate_edge_dev(gh_levels* L, const double* d_x, double* d_d) {
  gh_mesh* m = L->mesh;
  Scratch<double> inc(L->nreach + 1, m->stream);
  const int64_t b = L->h_offsets.size() > 1 ? L->h_offsets[1] : 0, e = L->nreach;
  if (e > b) {
    k_inc_edge<<<grid_for(e - b), B, 0, m->stream>>>(L->order.p, L->parent.p, L->parent_edge.p, b, e, m->edge_v.p,
                                                     d_x, inc.p);
    GH_LAUNCH_CHECK();
    m->launches++;
  }
  run_chain(L, inc.p, d_d);
}

}  // namespace gh
