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
// Diffusion layout: rows are renumbered by (level parity,
// level, original index). Every step of the sweep-pipelined schedule then
// touches one contiguous row range. The CSR is re-laid out as SELL-32 (32
// rows per chunk, entry k of lane j at chunk_ptr + 32k + j) so a warp's k-th
// neighbour loads are one coalesced 128 B (col) + 256 B (weight) access.
// Each row keeps the reference's neighbour order (ascending original index),
// and each column carries a flag bit saying "this neighbour sits one level
// closer to the sources", which selects the sweep buffer to read.

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "gh_internal.cuh"

namespace {

constexpr int B = gh::kBlock;

__global__ void k_bfs_init(int32_t* __restrict__ level, int64_t nv) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x)
    level[v] = -1;
}

__global__ void k_bfs_seed(int32_t* __restrict__ level, const int32_t* __restrict__ src, int32_t ns) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x) level[src[i]] = 0;
}

// One ring per iteration; level_size[d] counts ring d. Returns nlev in *out.
constexpr int kBfsBlock = 512;
__global__ void __launch_bounds__(kBfsBlock) k_bfs(const int32_t* __restrict__ vv_off, const int32_t* __restrict__ vv_idx,
                                                   int32_t* __restrict__ level, int32_t* __restrict__ fa,
                                                   int32_t* __restrict__ fb, int32_t* __restrict__ level_size,
                                                   int32_t* __restrict__ out, unsigned* __restrict__ bar) {
  // 8 lanes per frontier vertex, one neighbour each, so a ring costs a few
  // dependent memory round trips instead of one per neighbour
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t groups = ((int64_t)gridDim.x * blockDim.x) >> 3;
  const int sub = threadIdx.x & 7, lane = threadIdx.x & 31;
  int32_t* cur = fa;
  int32_t* nxt = fb;
  int32_t ncur = __ldcg(level_size);
  int32_t depth = 1;
  for (;;) {
    const int64_t rounds = (ncur + groups - 1) / groups;
    for (int64_t k = 0; k < rounds; ++k) {
      const int64_t i = (tid >> 3) + k * groups;
      int32_t a = 0, a1 = 0;
      if (i < ncur) {
        const int32_t v = __ldcg(cur + i);
        a = vv_off[v] + sub;
        a1 = vv_off[v + 1];
      }
      for (; __any_sync(0xffffffffu, a < a1); a += 8) {
        bool claimed = false;
        int32_t w = 0;
        if (a < a1) {
          w = vv_idx[a];
          claimed = atomicCAS(level + w, -1, depth) == -1;
        }
        const unsigned mask = __ballot_sync(0xffffffffu, claimed);
        int32_t base = 0;
        if (lane == 0 && mask) base = atomicAdd(level_size + depth, __popc(mask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (claimed) nxt[base + __popc(mask & ((1u << lane) - 1u))] = w;
      }
    }
    ghd::grid_barrier(bar, (unsigned)(depth - 1));
    const int32_t nn = __ldcg(level_size + depth);
    if (nn == 0) break;
    int32_t* t = cur;
    cur = nxt;
    nxt = t;
    ncur = nn;
    ++depth;
  }
  if (tid == 0) *out = depth;
}

// parent(v) = smallest-index neighbour at depth - 1 (bfs.hpp:57-65)
__global__ void k_parent(const int32_t* __restrict__ vv_off, const int32_t* __restrict__ vv_idx,
                         const int32_t* __restrict__ level, int64_t nv, int32_t* __restrict__ parent,
                         uint32_t* __restrict__ key, int32_t* __restrict__ val, uint32_t unreach_key) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t L = level[v];
    int32_t p = -1;
    if (L > 0)
      for (int32_t a = vv_off[v]; a < vv_off[v + 1]; ++a) {
        const int32_t w = vv_idx[a];
        if (level[w] == L - 1) {
          p = w;
          break;
        }
      }
    parent[v] = p;
    key[v] = L >= 0 ? (uint32_t)L : unreach_key;
    val[v] = (int32_t)v;
  }
}

// new row index of every reachable vertex
__global__ void k_renumber(const int32_t* __restrict__ order, const int32_t* __restrict__ level, int64_t nreach,
                           const int32_t* __restrict__ boff, const int32_t* __restrict__ pstart,
                           int32_t* __restrict__ perm, int32_t* __restrict__ newidx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nreach; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = order[i];
    const int32_t L = level[v];
    const int32_t r = pstart[L] + (int32_t)(i - boff[L]);
    perm[r] = v;
    newidx[v] = r;
  }
}

// per chunk: level of the first row, width = max row length
__global__ void k_chunk_meta(const int32_t* __restrict__ perm, const int32_t* __restrict__ level,
                             const int32_t* __restrict__ vv_off, int64_t nchunks, int32_t* __restrict__ chunk_level,
                             int64_t* __restrict__ width, uint16_t* __restrict__ deg, int32_t* __restrict__ maxdeg) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = warp; c < nchunks; c += nwarps) {
    const int64_t r = c * 32 + lane;
    const int32_t v = perm[r];
    int32_t d = v >= 0 ? vv_off[v + 1] - vv_off[v] : 0;
    int32_t m = d;
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    deg[r] = (uint16_t)(d > 65535 ? 65535 : d);
    if (lane == 0) {
      width[c] = 32 * (int64_t)m;
      chunk_level[c] = level[perm[c * 32]];
      if (m > 65535) atomicMax(maxdeg, m);
    }
  }
}

__global__ void k_sell_fill(const int32_t* __restrict__ perm, const int32_t* __restrict__ level,
                            const int32_t* __restrict__ newidx, const int32_t* __restrict__ vv_off,
                            const int32_t* __restrict__ vv_idx, const double* __restrict__ vv_w,
                            const double* __restrict__ va, const double* __restrict__ wsum,
                            const int64_t* __restrict__ chunk_ptr, int64_t nrows, int32_t* __restrict__ col,
                            double* __restrict__ wt, double* __restrict__ area_r, double* __restrict__ wsum_r) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = perm[r];
    if (v < 0) {
      area_r[r] = 0.0;
      wsum_r[r] = 0.0;
      continue;
    }
    const int32_t L = level[v];
    const int64_t base = chunk_ptr[r >> 5] + (r & 31);
    const int32_t a0 = vv_off[v], a1 = vv_off[v + 1];
    for (int32_t a = a0; a < a1; ++a) {
      const int32_t nb = vv_idx[a];
      const uint32_t flag = level[nb] == L - 1 ? 0x80000000u : 0u;
      col[base + 32 * (int64_t)(a - a0)] = (int32_t)((uint32_t)newidx[nb] | flag);
      wt[base + 32 * (int64_t)(a - a0)] = vv_w[a];
    }
    area_r[r] = va[v];
    wsum_r[r] = wsum[v];
  }
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
  return level.bytes() + parent.bytes() + order.bytes() + offsets.bytes() + pstart.bytes() + pend.bytes() +
         perm.bytes() + chunk_level.bytes() + chunk_ptr.bytes() + deg.bytes() + col.bytes() + wt.bytes() +
         area_r.bytes() + wsum_r.bytes() + den.bytes() + ubuf.bytes() + u_orig.bytes();
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
  Scratch<int32_t> fa(V + 1, s), fb(V + 1, s), level_size(V + 2, s), dsrc(n0, s), nlev_d(2, s);
  GH_CUDA(cudaMemsetAsync(level_size.p, 0, sizeof(int32_t) * (V + 2), s));
  GH_CUDA(cudaMemcpyAsync(level_size.p, &n0, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  GH_CUDA(cudaMemcpyAsync(dsrc.p, src.data(), sizeof(int32_t) * n0, cudaMemcpyHostToDevice, s));
  GH_CUDA(cudaMemcpyAsync(fa.p, src.data(), sizeof(int32_t) * n0, cudaMemcpyHostToDevice, s));
  k_bfs_init<<<grid_for(V), B, 0, s>>>(L->level.p, V);
  k_bfs_seed<<<grid_for(n0), B, 0, s>>>(L->level.p, dsrc.p, n0);
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
    int32_t* pa = fa.p;
    int32_t* pb = fb.p;
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
    k_parent<<<grid_for(V), B, 0, s>>>(m->vv_offset.p, m->vv_index.p, L->level.p, V, L->parent.p, k0.p, L->order.p,
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

  // ---- diffusion layout: (parity, level, index) row order, SELL-32
  L->h_pstart.assign(nlev, 0);
  L->h_pend.assign(nlev, 0);
  // every level starts on a 32-row chunk boundary, even levels first
  int64_t cursor = 0;
  for (int p = 0; p < 2; ++p) {
    for (int32_t l = p; l < nlev; l += 2) {
      cursor = (cursor + 31) & ~int64_t(31);
      L->h_pstart[l] = (int32_t)cursor;
      cursor += sizes[l];
      L->h_pend[l] = (int32_t)cursor;
    }
  }
  cursor = (cursor + 31) & ~int64_t(31);
  if (cursor > 0x7fffffffLL) fail(GH_ERR_INVALID, "mesh too large for the diffusion layout");
  L->nrows = (int32_t)cursor;
  L->nchunks = L->nrows / 32;
  L->pstart.alloc(nlev, s);
  L->pend.alloc(nlev, s);
  GH_CUDA(cudaMemcpyAsync(L->pstart.p, L->h_pstart.data(), sizeof(int32_t) * nlev, cudaMemcpyHostToDevice, s));
  GH_CUDA(cudaMemcpyAsync(L->pend.p, L->h_pend.data(), sizeof(int32_t) * nlev, cudaMemcpyHostToDevice, s));
  L->perm.alloc(L->nrows, s);
  GH_CUDA(cudaMemsetAsync(L->perm.p, 0xff, sizeof(int32_t) * L->nrows, s));
  Scratch<int32_t> newidx(V, s);
  GH_CUDA(cudaMemsetAsync(newidx.p, 0xff, sizeof(int32_t) * V, s));
  if (L->nreach) {
    k_renumber<<<grid_for(L->nreach), B, 0, s>>>(L->order.p, L->level.p, L->nreach, L->offsets.p, L->pstart.p,
                                                 L->perm.p, newidx.p);
    GH_LAUNCH_CHECK();
  }
  L->chunk_level.alloc(L->nchunks, s);
  L->deg.alloc(L->nrows, s);
  L->chunk_ptr.alloc(L->nchunks + 1, s);
  {
    Scratch<int64_t> width(L->nchunks + 1, s);
    Scratch<int32_t> maxdeg(1, s);
    GH_CUDA(cudaMemsetAsync(maxdeg.p, 0, sizeof(int32_t), s));
    GH_CUDA(cudaMemsetAsync(width.p + L->nchunks, 0, sizeof(int64_t), s));
    k_chunk_meta<<<grid_for((int64_t)L->nchunks * 32), B, 0, s>>>(L->perm.p, L->level.p, m->vv_offset.p, L->nchunks,
                                                                  L->chunk_level.p, width.p, L->deg.p, maxdeg.p);
    GH_LAUNCH_CHECK();
    if (read_scalar(maxdeg.p, s) > 65535) fail(GH_ERR_INVALID, "vertex valence above 65535 is not supported");
    size_t tmp = 0;
    GH_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, width.p, L->chunk_ptr.p, L->nchunks + 1, s));
    Scratch<char> t(tmp, s);
    GH_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, width.p, L->chunk_ptr.p, L->nchunks + 1, s));
  }
  const int64_t nnz_padded = read_scalar(L->chunk_ptr.p + L->nchunks, s);
  {
    std::vector<int64_t> cp(L->nchunks + 1);
    GH_CUDA(cudaMemcpyAsync(cp.data(), L->chunk_ptr.p, sizeof(int64_t) * cp.size(), cudaMemcpyDeviceToHost, s));
    GH_CUDA(cudaStreamSynchronize(s));
    int64_t wmax = 0;
    for (int32_t c = 0; c < L->nchunks; ++c) wmax = std::max(wmax, (cp[c + 1] - cp[c]) / 32);
    L->max_chunk_width = (int32_t)wmax;
  }
  L->col.alloc(nnz_padded, s);
  L->wt.alloc(nnz_padded, s);
  if (nnz_padded) {
    GH_CUDA(cudaMemsetAsync(L->col.p, 0, sizeof(int32_t) * nnz_padded, s));
    GH_CUDA(cudaMemsetAsync(L->wt.p, 0, sizeof(double) * nnz_padded, s));
  }
  L->area_r.alloc(L->nrows, s);
  L->wsum_r.alloc(L->nrows, s);
  k_sell_fill<<<grid_for(L->nrows), B, 0, s>>>(L->perm.p, L->level.p, newidx.p, m->vv_offset.p, m->vv_index.p,
                                               m->vv_weight.p, m->vertex_area.p, m->vertex_weight_sum.p,
                                               L->chunk_ptr.p, L->nrows, L->col.p, L->wt.p, L->area_r.p, L->wsum_r.p);
  GH_LAUNCH_CHECK();
  L->den.alloc(L->nrows, s);
  L->rows_done.alloc(nlev, s);
  L->ubuf.alloc(2 * (size_t)L->nrows, s);
  L->u_orig.alloc(V, s);
  L->den_t = 0.0;
  L->u_valid = 0;
  m->launches += 8;
  GH_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gh
