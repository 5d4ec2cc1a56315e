// BFS level sets (reference bfs.hpp:26-72) and the BFS-renumbered diffusion
// layout derived from them.
//
// BFS: a cooperative persistent kernel expands one ring per grid barrier;
// atomicCAS claims a vertex for the ring, so the level of every vertex is the
// graph distance and does not depend on the claim order. Rings are then
// stable-sorted by (level, vertex) — exactly the reference's per-ring
// std::sort — and parent(v) = first neighbour one level up in v's
// ascending row (bfs.hpp:57-65).
//
// The diffusion layout derived from the levels is built in gh_band.cu.

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "gh_internal.cuh"

namespace {

constexpr int B = gh::kBlock;
constexpr int32_t kPartialLevels = 2048;  // levels of a partial main band (bfs_build)

__global__ void k_bfs_init(int32_t* __restrict__ level, int64_t nv) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x)
    level[v] = -1;
}

// D_0: level 0 and the first frontier (vertex, row begin, row end)
__global__ void k_bfs_seed(const int32_t* __restrict__ vv_off, int32_t* __restrict__ level,
                           const int32_t* __restrict__ src, int32_t ns, int4* __restrict__ frontier) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x) {
    const int32_t v = src[i];
    level[v] = 0;
    frontier[i] = make_int4(v, vv_off[v], vv_off[v + 1], 0);
  }
}

// One ring per iteration; level_size[d] counts ring d. Returns nlev in *out.
// Frontier entries carry their row bounds (read by the claiming thread while
// its append slot is reserved), so expanding a ring starts at vv_idx.
constexpr int kBfsBlock = 512;
constexpr int kBfsStage = 2048;       // claims a block stages per ring before one global append
constexpr int kBfsStageRing = 12288;  // rings wider than this stage their appends
__global__ void __launch_bounds__(kBfsBlock) k_bfs(const int32_t* __restrict__ vv_off, const int32_t* __restrict__ vv_idx,
                                                   int32_t* __restrict__ level, int4* __restrict__ fa,
                                                   int4* __restrict__ fb, int32_t* __restrict__ level_size,
                                                   int32_t* __restrict__ out, unsigned* __restrict__ bar) {
  // 8 lanes per frontier vertex, one neighbour each, so a ring costs a few
  // dependent memory round trips instead of one per neighbour. A block's new
  // frontier entries are staged in shared memory and appended with one global
  // atomic per block and ring (a per-warp atomic on the one ring counter
  // serialised thousands of atomics per ring on wide rings).
  __shared__ int4 stage[kBfsStage];
  __shared__ int32_t s_cnt, s_base;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t groups = ((int64_t)gridDim.x * blockDim.x) >> 3;
  const int sub = threadIdx.x & 7, lane = threadIdx.x & 31;
  int4* cur = fa;
  int4* nxt = fb;
  int32_t ncur = __ldcg(level_size);
  int32_t depth = 1;
  for (;;) {
    // wide rings stage (the ring counter's contention dominates there); narrow
    // ones append per warp (two block barriers per ring cost more than they save)
    const bool staged = ncur > kBfsStageRing;
    if (staged) {
      if (threadIdx.x == 0) s_cnt = 0;
      __syncthreads();
    }
    const int64_t rounds = (ncur + groups - 1) / groups;
    for (int64_t k = 0; k < rounds; ++k) {
      const int64_t i = (tid >> 3) + k * groups;
      int32_t a = 0, a1 = 0;
      if (i < ncur) {
        const int4 e = __ldcg(cur + i);
        a = e.y + sub;
        a1 = e.z;
      }
      for (; __any_sync(0xffffffffu, a < a1); a += 8) {
        bool claimed = false;
        int32_t w = 0, w0 = 0, w1 = 0;
        if (a < a1) {
          w = vv_idx[a];
          claimed = atomicCAS(level + w, -1, depth) == -1;
        }
        if (claimed) {
          w0 = vv_off[w];
          w1 = vv_off[w + 1];
        }
        const unsigned mask = __ballot_sync(0xffffffffu, claimed);
        if (!mask) continue;
        if (!staged) {
          int32_t base = 0;
          if (lane == 0) base = atomicAdd(level_size + depth, __popc(mask));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (claimed) nxt[base + __popc(mask & ((1u << lane) - 1u))] = make_int4(w, w0, w1, 0);
          continue;
        }
        int32_t off = 0;
        if (lane == 0) off = atomicAdd(&s_cnt, __popc(mask));
        off = __shfl_sync(0xffffffffu, off, 0);
        const int32_t p = off + __popc(mask & ((1u << lane) - 1u));
        // past the stage: straight to the global frontier
        const unsigned spill = __ballot_sync(0xffffffffu, claimed && p >= kBfsStage);
        int32_t gbase = 0;
        if (lane == 0 && spill) gbase = atomicAdd(level_size + depth, __popc(spill));
        gbase = __shfl_sync(0xffffffffu, gbase, 0);
        if (claimed) {
          const int4 ent = make_int4(w, w0, w1, 0);
          if (p < kBfsStage) stage[p] = ent;
          else nxt[gbase + __popc(spill & ((1u << lane) - 1u))] = ent;
        }
      }
    }
    if (staged) {
      __syncthreads();
      const int32_t n = s_cnt < kBfsStage ? s_cnt : kBfsStage;
      if (threadIdx.x == 0 && n) s_base = atomicAdd(level_size + depth, n);
      __syncthreads();
      for (int32_t j = threadIdx.x; j < n; j += blockDim.x) nxt[s_base + j] = stage[j];
    }
    ghd::grid_barrier(bar, (unsigned)(depth - 1));
    const int32_t nn = __ldcg(level_size + depth);
    if (nn == 0) break;
    int4* t = cur;
    cur = nxt;
    nxt = t;
    ncur = nn;
    ++depth;
  }
  if (tid == 0) *out = depth;
}

// parent(v) = smallest-index neighbour at depth - 1 (bfs.hpp:57-65)
// (and the edge (parent, v): the CSR entry that found the parent carries it,
// so integration needs no edge_between search)
__global__ void k_parent(const int32_t* __restrict__ vv_off, const int32_t* __restrict__ vv_idx,
                         const int32_t* __restrict__ vv_edge, const int32_t* __restrict__ level, int64_t nv,
                         int32_t* __restrict__ parent, int32_t* __restrict__ parent_edge,
                         uint32_t* __restrict__ key, int32_t* __restrict__ val, uint32_t unreach_key) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t L = level[v];
    int32_t p = -1, pe = -1;
    if (L > 0)
      for (int32_t a = vv_off[v]; a < vv_off[v + 1]; ++a) {
        const int32_t w = vv_idx[a];
        if (level[w] == L - 1) {
          p = w;
          pe = vv_edge[a];
          break;
        }
      }
    parent[v] = p;
    parent_edge[v] = pe;
    key[v] = L >= 0 ? (uint32_t)L : unreach_key;
    val[v] = (int32_t)v;
  }
}

// Spatial order inside each ring for the diffusion layout: key = (level,
// 30-bit Morton code of the position in the mesh's bounding box). Rows of a
// ring keep their arithmetic (each row sums its neighbours in the reference's
// order, whatever its position); only which rows share a chunk changes.
__device__ __forceinline__ uint64_t spread3(uint32_t x) {
  uint64_t r = 0;
  for (int b = 0; b < 10; ++b) r |= (uint64_t)((x >> b) & 1u) << (3 * b);
  return r;
}
__global__ void k_morton_keys(const double* __restrict__ pos, const int32_t* __restrict__ level,
                              const double* __restrict__ box, int64_t nv, uint64_t* __restrict__ key,
                              int32_t* __restrict__ val) {
  const double lo[3] = {box[0], box[1], box[2]};
  double ext = 0.0;
  for (int k = 0; k < 3; ++k) ext = fmax(ext, box[3 + k] - box[k]);
  const double sc = ext > 0.0 ? 1023.0 / ext : 0.0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t L = level[v];
    uint64_t k = ~0ull;
    if (L >= 0) {
      uint64_t m = 0;
      for (int a = 0; a < 3; ++a) {
        const double q = (pos[3 * v + a] - lo[a]) * sc;
        const uint32_t qi = q > 0.0 ? (q < 1023.0 ? (uint32_t)q : 1023u) : 0u;
        m |= spread3(qi) << a;
      }
      k = (uint64_t)L << 32 | m;
    }
    key[v] = k;
    val[v] = (int32_t)v;
  }
}

// mean |v - w| over the CSR's (v, w) pairs, scaled down by 2^10 per term to
// stay within int64 (a locality test of the vertex numbering)
__global__ void k_index_spread(const int32_t* __restrict__ vv_off, const int32_t* __restrict__ vv_idx, int64_t nv,
                               unsigned long long* __restrict__ acc) {
  unsigned long long sum = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x)
    for (int32_t i = vv_off[v]; i < vv_off[v + 1]; ++i) {
      const int64_t d = (int64_t)vv_idx[i] - v;
      sum += (unsigned long long)((d < 0 ? -d : d) >> 10);
    }
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0 && sum) atomicAdd(acc, sum);
}

template <class T>
T read_scalar(const T* d, cudaStream_t s) {
  T v;
  GH_CUDA(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
  return v;
}

}  // namespace

uint64_t gh_levels::device_bytes() const {
  return level.bytes() + parent.bytes() + parent_edge.bytes() + order.bytes() + offsets.bytes() + u_orig.bytes() +
         main.device_bytes();
}

namespace gh {

void bfs_build(gh_levels* L, const int32_t* h_sources, int32_t ns) {
  gh_mesh* m = L->mesh;
  cudaStream_t s = m->stream;
  const int64_t V = m->nv;
  // D_0 = sorted unique sources (bfs.hpp:27-30, 55-60)
  if (ns <= 0) fail(GH_ERR_INVALID, "bfs_levels: empty source set");
  std::vector<int32_t> src(h_sources, h_sources + ns);
  for (int32_t x : src)
    if (x < 0 || x >= m->nv) fail(GH_ERR_INVALID, "bfs_levels: source index out of range");
  std::sort(src.begin(), src.end());
  src.erase(std::unique(src.begin(), src.end()), src.end());
  const int32_t n0 = (int32_t)src.size();

  L->level.alloc(V, s);
  L->parent.alloc(V, s);
  Scratch<int4> fa(V + 1, s), fb(V + 1, s);
  Scratch<int32_t> level_size(V + 2, s), dsrc(n0, s), nlev_d(2, s);
  GH_CUDA(cudaMemsetAsync(level_size.p, 0, sizeof(int32_t) * (V + 2), s));
  GH_CUDA(cudaMemcpyAsync(level_size.p, &n0, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  GH_CUDA(cudaMemcpyAsync(dsrc.p, src.data(), sizeof(int32_t) * n0, cudaMemcpyHostToDevice, s));
  k_bfs_init<<<grid_for(V), B, 0, s>>>(L->level.p, V);
  k_bfs_seed<<<grid_for(n0), B, 0, s>>>(m->vv_offset.p, L->level.p, dsrc.p, n0, fa.p);
  GH_LAUNCH_CHECK();

  // cooperative ring expansion
  {
    int dev = m->device, nsm = 0, per_sm = 0;
    GH_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    GH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bfs, kBfsBlock, 0));
    if (per_sm < 1) fail(GH_ERR_CUDA, "BFS kernel cannot be resident");
    int grid = nsm;  // one block per SM: the barrier cost grows with the block count
    const int32_t* vo = m->vv_offset.p;
    const int32_t* vi = m->vv_index.p;
    int32_t* lv = L->level.p;
    int4* pa = fa.p;
    int4* pb = fb.p;
    int32_t* ls = level_size.p;
    int32_t* out = nlev_d.p;
    unsigned* bar = reinterpret_cast<unsigned*>(nlev_d.p + 1);
    GH_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned), s));
    void* args[] = {&vo, &vi, &lv, &pa, &pb, &ls, &out, &bar};
    GH_CUDA(cudaLaunchCooperativeKernel((void*)k_bfs, grid, kBfsBlock, args, 0, s));
    GH_LAUNCH_CHECK();
  }
  const int32_t nlev = read_scalar(nlev_d.p, s);
  L->nlev = nlev;
  std::vector<int32_t> sizes(nlev);
  GH_CUDA(cudaMemcpyAsync(sizes.data(), level_size.p, sizeof(int32_t) * nlev, cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
  L->h_offsets.assign(nlev + 1, 0);
  L->max_width = 0;
  for (int32_t i = 0; i < nlev; ++i) {
    L->h_offsets[i + 1] = L->h_offsets[i] + sizes[i];
    L->max_width = std::max(L->max_width, sizes[i]);
  }
  L->nreach = L->h_offsets[nlev];
  L->unreachable = (int32_t)(V - L->nreach);

  // parents + ring order: stable radix sort by level over ascending vertex ids
  L->order.alloc(V, s);
  {
    Scratch<uint32_t> k0(V, s), k1(V, s);
    Scratch<int32_t> v1(V, s);
    L->parent_edge.alloc(V, s);
    k_parent<<<grid_for(V), B, 0, s>>>(m->vv_offset.p, m->vv_index.p, m->vv_edge.p, L->level.p, V, L->parent.p,
                                       L->parent_edge.p, k0.p, L->order.p,
                                       (uint32_t)nlev);
    GH_LAUNCH_CHECK();
    int end_bit = 1;
    while (end_bit < 32 && ((uint32_t)nlev >> end_bit) != 0) ++end_bit;
    cub::DoubleBuffer<uint32_t> kb(k0.p, k1.p);
    cub::DoubleBuffer<int32_t> vb(L->order.p, v1.p);
    size_t tmp = 0;
    GH_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, (int)V, 0, end_bit, s));
    Scratch<char> t(tmp, s);
    GH_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, kb, vb, (int)V, 0, end_bit, s));
    if (vb.Current() != L->order.p)
      GH_CUDA(cudaMemcpyAsync(L->order.p, vb.Current(), sizeof(int32_t) * V, cudaMemcpyDeviceToDevice, s));
  }
  L->offsets.alloc(nlev + 1, s);
  GH_CUDA(cudaMemcpyAsync(L->offsets.p, L->h_offsets.data(), sizeof(int32_t) * (nlev + 1), cudaMemcpyHostToDevice, s));

  L->u_orig.alloc(V, s);
  L->u_valid = 0;
  m->launches += 4;
  // Rings in vertex-id order are spatially coherent on grid-like numberings;
  // when they are not (ring neighbours scattered over the ring, as with the
  // icosphere's subdivision numbering) no 16-bit column format fits, and the
  // layout is built with each ring in Morton order (GH_LAYOUT=id|morton
  // forces one, for tests). A numbering whose neighbours lie on average more
  // than V/64 apart goes to Morton order directly (config 4: saves building
  // the id-order layout first); otherwise the id-order layout is tried and
  // rebuilt in Morton order when no 16-bit format fits.
  const char* lay = getenv("GH_LAYOUT");
  const bool force_morton = lay && std::strcmp(lay, "morton") == 0;
  const bool force_id = lay && std::strcmp(lay, "id") == 0;
  bool scattered = false;
  if (!force_id && !force_morton && L->nreach > 0 && m->vv_index.n > 0) {
    Scratch<unsigned long long> acc(1, s);
    GH_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(unsigned long long), s));
    k_index_spread<<<grid_for(V), B, 0, s>>>(m->vv_offset.p, m->vv_index.p, V, acc.p);
    GH_LAUNCH_CHECK();
    m->launches++;
    const double mean = 1024.0 * (double)read_scalar(acc.p, s) / (double)m->vv_index.n;
    scattered = mean > (double)V / 64.0;
  }
  L->layout_order.release();
  // diffusion layout: one band, no ghosts. A mesh whose first 2048 rings hold
  // less than half the vertices gets those rings only (the heat underflows to
  // +0 long before the rest: config 5 builds 13 of 201 M rows);
  // main_layout_ensure extends the band when a solve needs more levels.
  int32_t main_le = nlev, part = kPartialLevels;
  if (const char* e = getenv("GH_PARTIAL_LEVELS")) part = std::max(2, atoi(e));  // tests: small partial bands
  if (zero_level_truncation() && nlev > part && 2 * (int64_t)L->h_offsets[part] <= (int64_t)L->nreach) main_le = part;
  if (!(scattered || force_morton)) band_build(L, &L->main, 0, main_le);
  if (L->nreach > 0 && (force_morton || scattered || (!force_id && L->main.col16_windows == 0))) {
    L->layout_order.alloc(V, s);
    {
      Scratch<uint64_t> k0(V, s), k1(V, s);
      Scratch<int32_t> v1(V, s);
      k_morton_keys<<<grid_for(V), B, 0, s>>>(m->pos.p, L->level.p, m->scalars.p + 5, V, k0.p, L->layout_order.p);
      GH_LAUNCH_CHECK();
      int end_bit = 33;
      while (end_bit < 64 && ((uint64_t)nlev >> (end_bit - 32)) != 0) ++end_bit;
      cub::DoubleBuffer<uint64_t> kb(k0.p, k1.p);
      cub::DoubleBuffer<int32_t> vb(L->layout_order.p, v1.p);
      size_t tmp = 0;
      GH_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, (int)V, 0, end_bit, s));
      Scratch<char> t(tmp, s);
      GH_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, kb, vb, (int)V, 0, end_bit, s));
      if (vb.Current() != L->layout_order.p)
        GH_CUDA(cudaMemcpyAsync(L->layout_order.p, vb.Current(), sizeof(int32_t) * V, cudaMemcpyDeviceToDevice, s));
    }
    m->launches += 2;
    band_build(L, &L->main, 0, main_le);
  }
}

void main_layout_ensure(gh_levels* L, int32_t le) {
  le = std::min(le, L->nlev);
  if (L->main.le >= le || L->nreach <= 0) return;
  L->main.release_state();
  band_build(L, &L->main, 0, le);  // in the ring order bfs_build chose (order or layout_order)
  L->u_valid = 0;
}

}  // namespace gh
