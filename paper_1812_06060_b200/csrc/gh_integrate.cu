// Breadth-first distance recovery (reference integrate.hpp:19-75).
//
// The reference's step is d(v) = d(parent) + inc(v), with inc(v) computed
// before the addition (integrate.hpp:56, 72). inc depends only on the
// optimised field and the geometry, so it is computed for every vertex in one
// fully parallel gather kernel. The chain d(v) = d(parent) + inc(v) is then
// evaluated along paths of the BFS tree: every vertex continues the path of
// its parent if it is the parent's smallest-index child, else it starts a
// path of its own. One thread walks a path with d in a register (one
// dependent load per four steps, through skip records of the next four
// vertices); a path's first vertex waits for its parent's published value.
// On BFS trees of meshes the paths are long rays (config-5-like tori: a few
// thousand paths for ~10^6 vertices, at most 3 path changes on any
// root-to-leaf walk), so the chain costs about (levels / 4) dependent loads
// instead of one cross-SM publish-and-poll per level. The additions are the
// reference's, in its order: bitwise.

#include <algorithm>
#include <cmath>

#include <cub/device/device_select.cuh>

#include "gh_internal.cuh"

using namespace ghd;

namespace {

constexpr int B = gh::kBlock;

// edge_between (mesh.hpp:87-93): lower_bound in a's ascending row
__device__ __forceinline__ int32_t edge_between(const int32_t* __restrict__ off, const int32_t* __restrict__ idx,
                                                const int32_t* __restrict__ eid, int32_t a, int32_t b) {
  int32_t lo = off[a], hi = off[a + 1];
  const int32_t end = hi;
  while (lo < hi) {
    const int32_t mid = lo + ((hi - lo) >> 1);
    if (idx[mid] < b) lo = mid + 1;
    else hi = mid;
  }
  return (lo == end || idx[lo] != b) ? -1 : eid[lo];
}

// inc(v) for the face method (integrate.hpp:45-56), indexed by vertex
__global__ void k_inc_face(const int32_t* __restrict__ order, const int32_t* __restrict__ parent, int64_t b,
                           int64_t e, const int32_t* __restrict__ off, const int32_t* __restrict__ idx,
                           const int32_t* __restrict__ eid, const int32_t* __restrict__ edge_he,
                           const double* __restrict__ pos, const double* __restrict__ g, double* __restrict__ inc) {
  for (int64_t i = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = order[i], p = parent[v];
    const int32_t ed = edge_between(off, idx, eid, p, v);
    const v3 step = sub(ld3(pos, v), ld3(pos, p));
    double sum = 0.0;
    int count = 0;
    for (int s = 0; s < 2; ++s) {
      const int32_t h = edge_he[2 * ed + s];
      if (h < 0) continue;
      sum += dot(ld3(g, h / 3), step);
      ++count;
    }
    inc[v] = ddiv(sum, (double)count);
  }
}

// inc(v) for the edge method (integrate.hpp:67-72)
__global__ void k_inc_edge(const int32_t* __restrict__ order, const int32_t* __restrict__ parent, int64_t b,
                           int64_t e, const int32_t* __restrict__ off, const int32_t* __restrict__ idx,
                           const int32_t* __restrict__ eid, const int32_t* __restrict__ edge_v,
                           const double* __restrict__ x, double* __restrict__ inc) {
  for (int64_t i = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = order[i], p = parent[v];
    const int32_t ed = edge_between(off, idx, eid, p, v);
    const double sigma = edge_v[2 * ed] == p ? 1.0 : -1.0;
    inc[v] = sigma * x[ed];
  }
}

// d = 0 on D_0, +inf on unreachable vertices (integrate.hpp:20, 52), and a
// "pending" NaN payload no arithmetic produces on every vertex still to come.
constexpr unsigned long long kPending = 0x7FF4DEADBEEF0001ull;

__global__ void k_dist_init(const int32_t* __restrict__ level, int64_t nv, double* __restrict__ d) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x)
    d[v] = level[v] == 0 ? 0.0 : (level[v] < 0 ? INFINITY : __longlong_as_double((long long)kPending));
}

// path structure: dchild[v] = smallest-index child of v (>= nv: none)
__global__ void k_dchild(const int32_t* __restrict__ order, const int32_t* __restrict__ parent, int64_t b, int64_t e,
                         int32_t* __restrict__ dchild) {
  for (int64_t i = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = order[i];
    atomicMin(dchild + parent[v], v);
  }
}

// the next four vertices of v's path and their increments (-1: path ends)
constexpr int kSkip = 4;
struct __align__(16) PathNode {
  int32_t next[kSkip];
  double inc[kSkip];
};
__global__ void k_path_nodes(const int32_t* __restrict__ dchild, const double* __restrict__ inc, int64_t nv,
                             PathNode* __restrict__ node) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    PathNode n;
    int32_t c = (int32_t)v;
#pragma unroll
    for (int k = 0; k < kSkip; ++k) {
      const int32_t x = c >= 0 ? dchild[c] : -1;
      c = (x < 0 || x >= nv) ? -1 : x;  // >= nv: the memset "none" (atomicMin only lowers it to a vertex)
      n.next[k] = c;
      n.inc[k] = c >= 0 ? inc[c] : 0.0;
    }
    node[v] = n;
  }
}

// path heads, in BFS order: the sources and every vertex that is not its
// parent's smallest-index child
__global__ void k_head_flags(const int32_t* __restrict__ order, const int32_t* __restrict__ parent,
                             const int32_t* __restrict__ dchild, int64_t b, int64_t e, uint8_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = order[i];
    flag[i] = i < b || dchild[parent[v]] != v;
  }
}

__device__ __forceinline__ void st_pub(double* p, double x) {
  asm volatile("st.volatile.global.f64 [%0], %1;" ::"l"(p), "d"(x) : "memory");
}

// d along every path (run_levels, integrate.hpp:19-36). Each thread takes its
// paths in increasing BFS order of their first vertex, and all threads are
// co-resident: the unfinished path with the smallest first vertex can always
// proceed (its first vertex's parent lies on a path that starts earlier, so
// that path is finished or being walked), hence no deadlock.
__global__ void __launch_bounds__(B) k_chain_paths(const int32_t* __restrict__ heads, const int32_t* __restrict__ nheads,
                                                   const int32_t* __restrict__ parent, const int32_t* __restrict__ level,
                                                   const double* __restrict__ inc, const PathNode* __restrict__ node,
                                                   double* __restrict__ d) {
  const int64_t n = *nheads;
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < n; h += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = heads[h];
    double dv = 0.0;  // sources: d = 0 (integrate.hpp:20)
    if (level[v] > 0) {
      const int32_t p = parent[v];
      const double step = inc[v];
      unsigned long long x;
      unsigned ns = 0;
      for (;;) {
        asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(x) : "l"(d + p) : "memory");
        if (x != kPending) break;
        __nanosleep(ns);
        ns = ns < 256 ? ns + 32 : 256;
      }
      dv = __longlong_as_double((long long)x) + step;
      st_pub(d + v, dv);
    }
    int32_t cur = v;
    for (;;) {
      const PathNode nd = node[cur];
      int32_t last = -1;
#pragma unroll
      for (int k = 0; k < kSkip; ++k) {
        if (nd.next[k] < 0) break;
        dv = dv + nd.inc[k];
        st_pub(d + nd.next[k], dv);
        last = nd.next[k];
      }
      if (last < 0 || nd.next[kSkip - 1] < 0) break;
      cur = last;
    }
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
  gh::Scratch<int32_t> dchild(m->nv, s), heads(e, s), nheads(1, s);
  gh::Scratch<PathNode> node(m->nv, s);
  gh::Scratch<uint8_t> flag(e, s);
  GH_CUDA(cudaMemsetAsync(dchild.p, 0x7f, sizeof(int32_t) * m->nv, s));  // 0x7f7f7f7f > any vertex: "none"
  k_dchild<<<gh::grid_for(e - b), B, 0, s>>>(L->order.p, L->parent.p, b, e, dchild.p);
  k_path_nodes<<<gh::grid_for(m->nv), B, 0, s>>>(dchild.p, inc, m->nv, node.p);
  k_head_flags<<<gh::grid_for(e), B, 0, s>>>(L->order.p, L->parent.p, dchild.p, b, e, flag.p);
  GH_LAUNCH_CHECK();
  size_t tmp = 0;
  GH_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, L->order.p, flag.p, heads.p, nheads.p, (int)e, s));
  {
    gh::Scratch<unsigned char> t(tmp, s);
    GH_CUDA(cub::DeviceSelect::Flagged(t.p, tmp, L->order.p, flag.p, heads.p, nheads.p, (int)e, s));
  }
  int nsm = 0, per_sm = 0;
  GH_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device));
  GH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chain_paths, B, 0));
  const int64_t want = (e + B - 1) / B;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * std::max(1, per_sm), want));
  const int32_t* hp = heads.p;
  const int32_t* np = nheads.p;
  const int32_t* par = L->parent.p;
  const int32_t* lev = L->level.p;
  const PathNode* nodes = node.p;
  void* args[] = {&hp, &np, &par, &lev, &inc, &nodes, &d};
  GH_CUDA(cudaLaunchCooperativeKernel((void*)k_chain_paths, grid, B, args, 0, s));
  GH_LAUNCH_CHECK();
  m->launches += 6;
}

}  // namespace

namespace gh {

void integrate_face_dev(gh_levels* L, const double* d_g, double* d_d) {
  gh_mesh* m = L->mesh;
  Scratch<double> inc(m->nv + 1, m->stream);
  const int64_t b = L->h_offsets.size() > 1 ? L->h_offsets[1] : 0, e = L->nreach;
  if (e > b) {
    k_inc_face<<<grid_for(e - b), B, 0, m->stream>>>(L->order.p, L->parent.p, b, e, m->vv_offset.p, m->vv_index.p,
                                                     m->vv_edge.p, m->edge_he.p, m->pos.p, d_g, inc.p);
    GH_LAUNCH_CHECK();
    m->launches++;
  }
  run_chain(L, inc.p, d_d);
}

void integrate_edge_dev(gh_levels* L, const double* d_x, double* d_d) {
  gh_mesh* m = L->mesh;
  Scratch<double> inc(m->nv + 1, m->stream);
  const int64_t b = L->h_offsets.size() > 1 ? L->h_offsets[1] : 0, e = L->nreach;
  if (e > b) {
    k_inc_edge<<<grid_for(e - b), B, 0, m->stream>>>(L->order.p, L->parent.p, b, e, m->vv_offset.p, m->vv_index.p,
                                                     m->vv_edge.p, m->edge_v.p, d_x, inc.p);
    GH_LAUNCH_CHECK();
    m->launches++;
  }
  run_chain(L, inc.p, d_d);
}

}  // namespace gh
