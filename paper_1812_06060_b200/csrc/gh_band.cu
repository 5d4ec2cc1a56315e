// Diffusion layout of a BFS band.
//
// Rows of the band's own levels [lb, le) are renumbered by (level parity,
// level, original index), every level starting on a 32-row chunk boundary, so
// the rows a pipeline step touches are one contiguous range and a chunk holds
// one level. The ghost levels lb-1 and le (copies of the neighbours' boundary
// levels) follow. The CSR of the own rows is laid out SELL-32 (entry k of lane
// j at chunk_ptr + 32k + j); each row keeps the reference's neighbour order
// (ascending original index, mesh.hpp:255-266) and each column carries a flag
// bit "one level closer to the sources", which selects the sweep buffer.
//
// Band plan: levels are cut into contiguous bands of about equal row counts.
// By the BFS property (|level difference| <= 1 across an edge) a band only
// touches its two neighbours, through one ring each.

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <cstdlib>

#include "gh_internal.cuh"

namespace {

constexpr int B = gh::kBlock;

// local row of every vertex of levels [glo, ghi] (own and ghost)
__global__ void k_band_renumber(const int32_t* __restrict__ order, const int32_t* __restrict__ level, int64_t b,
                                int64_t e, const int32_t* __restrict__ boff, const int32_t* __restrict__ pstart,
                                int32_t* __restrict__ perm, int32_t* __restrict__ local) {
  for (int64_t i = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = order[i];
    const int32_t L = level[v];
    const int32_t r = pstart[L] + (int32_t)(i - boff[L]);
    perm[r] = v;
    local[v] = r;
  }
}

__global__ void k_deg_big(const int32_t* __restrict__ perm, const int32_t* __restrict__ vv_off, int64_t nrows,
                          int32_t* __restrict__ deg) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = perm[r];
    deg[r] = v >= 0 ? vv_off[v + 1] - vv_off[v] : 0;
  }
}

// per own chunk: its level, width = longest row, and the row lengths; *maxdeg
// = the longest row of the band (one atomic per block)
__global__ void k_chunk_meta(const int32_t* __restrict__ perm, const int32_t* __restrict__ level,
                             const int32_t* __restrict__ vv_off, int64_t nchunks, int32_t* __restrict__ chunk_level,
                             int64_t* __restrict__ width, uint16_t* __restrict__ deg, int32_t* __restrict__ maxdeg) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int32_t wm = 0;
  for (int64_t c = warp; c < nchunks; c += nwarps) {
    const int64_t r = c * 32 + lane;
    const int32_t v = perm[r];
    const int32_t d = v >= 0 ? vv_off[v + 1] - vv_off[v] : 0;
    int32_t m = d;
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    deg[r] = (uint16_t)(d > 65535 ? 65535 : d);
    wm = max(wm, m);
    if (lane == 0) {
      width[c] = 32 * (int64_t)m;
      chunk_level[c] = level[perm[c * 32]];  // levels are chunk aligned: row 0 of a chunk is real
    }
  }
  __shared__ int32_t sm;
  if (threadIdx.x == 0) sm = 0;
  __syncthreads();
  if (lane == 0 && wm) atomicMax(&sm, wm);
  __syncthreads();
  if (threadIdx.x == 0 && sm) atomicMax(maxdeg, sm);
}

__global__ void k_sell_fill(const int32_t* __restrict__ perm, const int32_t* __restrict__ level,
                            const int32_t* __restrict__ local, const int32_t* __restrict__ vv_off,
                            const int32_t* __restrict__ vv_idx, const double* __restrict__ vv_w,
                            const double* __restrict__ va, const double* __restrict__ wsum,
                            const int64_t* __restrict__ chunk_ptr, int64_t own_rows, uint32_t* __restrict__ col,
                            double* __restrict__ wt, double* __restrict__ area_r, double* __restrict__ wsum_r) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < own_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = perm[r];
    if (v < 0) continue;
    const int32_t L = level[v];
    const int64_t base = chunk_ptr[r >> 5] + (r & 31);
    const int32_t a0 = vv_off[v], a1 = vv_off[v + 1];
    for (int32_t a = a0; a < a1; ++a) {
      const int32_t nb = vv_idx[a];
      // the neighbour's slot in the sweep buffers: parity bit 0 = the sweep being
      // written (one level closer to the sources), 1 = the previous sweep
      col[base + 32 * (int64_t)(a - a0)] = gh::uidx((uint32_t)local[nb], level[nb] == L - 1 ? 0u : 1u);
      wt[base + 32 * (int64_t)(a - a0)] = vv_w[a];
    }
    area_r[r] = va[v];
    wsum_r[r] = wsum[v];
  }
}

// 16-bit columns of one chunk per warp (format: gh::Band::col16). With 2
// windows the entries point into the chunk's own level (same parity half) or
// levels L-1, L+1 (adjacent in the other half); with 3 windows into L, L-1 and
// L+1 separately (for rings so wide that L-1 and L+1 are far apart in the
// other half). Each window gets a 64-aligned uidx base; an entry keeps its
// offset (parity bit included) below the window bits. A chunk whose window
// spans reach the limit keeps only its 32-bit columns.
__global__ void k_col16(const int32_t* __restrict__ chunk_level, const int32_t* __restrict__ pstart,
                        const int32_t* __restrict__ pend, const int64_t* __restrict__ chunk_ptr,
                        const uint16_t* __restrict__ deg, const int32_t* __restrict__ deg_big,
                        const uint32_t* __restrict__ col, int64_t nchunks, int windows, uint32_t span_limit,
                        uint32_t ghost_lo, uint16_t* __restrict__ col16, int4* __restrict__ cbase,
                        uint8_t* __restrict__ deg4, unsigned long long* __restrict__ nwide) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t limit = min(span_limit, windows == 2 ? 32768u : 16384u);
  for (int64_t c = warp; c < nchunks; c += nwarps) {
    const int32_t L = chunk_level[c];
    const uint32_t lo = (uint32_t)pstart[L], hi = (uint32_t)pend[L];
    const uint32_t lo1 = L > 0 ? (uint32_t)pstart[L - 1] : 0u, hi1 = L > 0 ? (uint32_t)pend[L - 1] : 0u;
    const int64_t p0 = chunk_ptr[c], w = (chunk_ptr[c + 1] - p0) / 32;
    int64_t d = deg[c * 32 + lane];
    if (d == 65535 && deg_big) d = deg_big[c * 32 + lane];
    // row lengths as nibbles, lane pairs to one byte (15: the kernel reads deg)
    const uint32_t nib = (uint32_t)(d < 15 ? d : 15);
    const uint32_t hi_nib = __shfl_down_sync(0xffffffffu, nib, 1);
    if ((lane & 1) == 0) deg4[c * 16 + (lane >> 1)] = (uint8_t)(nib | hi_nib << 4);
    // window of a neighbour: 0 = level L; else 1 (2 windows: the other half;
    // 3 windows: level L-1), 2 (level L+1) or 3 (a ghost row, from ghost_lo on)
    auto window = [&](uint32_t u) -> int {
      const uint32_t row = (u >> 6) << 5 | (u & 31u);
      if (row >= lo && row < hi) return 0;
      if (windows == 2) return 1;
      if (ghost_lo && row >= ghost_lo) return 3;
      return row >= lo1 && row < hi1 ? 1 : 2;
    };
    uint32_t mn[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu}, mx[4] = {0u, 0u, 0u, 0u};
    for (int64_t k = 0; k < d; ++k) {
      const uint32_t u = col[p0 + 32 * k + lane];
      const int o = window(u);
      mn[o] = min(mn[o], u);
      mx[o] = max(mx[o], u);
    }
    bool fits = true;
    uint32_t base[4];
    for (int o = 0; o < 4; ++o) {
      for (int x = 16; x > 0; x >>= 1) {
        mn[o] = min(mn[o], __shfl_xor_sync(0xffffffffu, mn[o], x));
        mx[o] = max(mx[o], __shfl_xor_sync(0xffffffffu, mx[o], x));
      }
      base[o] = mn[o] == 0xffffffffu ? 0u : mn[o] & ~63u;
      fits = fits && (mn[o] == 0xffffffffu || mx[o] - base[o] < limit);
    }
    const int shift = windows == 2 ? 15 : 14;
    for (int64_t k = 0; k < w; ++k) {
      uint16_t e = 0;
      if (fits && k < d) {
        const uint32_t u = col[p0 + 32 * k + lane];
        const int o = window(u);
        e = (uint16_t)((uint32_t)o << shift | (u - base[o]));
      }
      col16[p0 + 32 * k + lane] = e;
    }
    if (lane == 0) {
      if (!fits) {
        cbase[c] = make_int4(-1, 0, 0, 0);
        atomicAdd(nwide, 1ull);
      } else if (windows == 2) {
        cbase[c] = make_int4((int32_t)base[0], (int32_t)base[1], 0, 0);
      } else {
        cbase[c] = make_int4((int32_t)base[0], (int32_t)base[1] - (1 << 14), (int32_t)base[2] - (2 << 14),
                             (int32_t)base[3] - (3 << 14));
      }
    }
  }
}


// ---- sector slices

// slice of every reachable vertex: its position in its ring, cut into
// nslices contiguous parts ([ceil(q n / N), ceil((q + 1) n / N)) is slice q)
__global__ void k_slice_owner(const int32_t* __restrict__ ord, const int32_t* __restrict__ level,
                              const int32_t* __restrict__ off, int64_t nreach, int32_t nslices,
                              int32_t* __restrict__ owner) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nreach; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = ord[i];
    const int32_t L = level[v];
    const int64_t p = i - off[L], n = off[L + 1] - off[L];
    owner[v] = (int32_t)((p * nslices) / n);
  }
}

// flag[k] bit q: slice q reads vertex k, owned by another slice
__global__ void k_slice_flags(const int32_t* __restrict__ ord, int64_t nreach, const int32_t* __restrict__ owner,
                              const int32_t* __restrict__ vv_off, const int32_t* __restrict__ vv_idx,
                              uint32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nreach; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = ord[i];
    const int32_t q = owner[v];
    for (int32_t a = vv_off[v]; a < vv_off[v + 1]; ++a) {
      const int32_t k = vv_idx[a];
      if (owner[k] != q) atomicOr(flag + k, 1u << q);
    }
  }
}

// 1 where slice q ghosts the ring-order vertex ord[i]
__global__ void k_slice_pick(const int32_t* __restrict__ ord, int64_t nreach, const uint32_t* __restrict__ flag,
                             int32_t q, uint8_t* __restrict__ pick) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nreach; i += (int64_t)gridDim.x * blockDim.x)
    pick[i] = (uint8_t)((flag[ord[i]] >> q) & 1u);
}

// own rows of slice r: ring position p of level L in [sstart[L], sstart[L] + cnt) -> row pstart[L] + p - sstart[L]
__global__ void k_slice_rows(const int32_t* __restrict__ ord, const int32_t* __restrict__ level,
                             const int32_t* __restrict__ off, int64_t nreach, const int32_t* __restrict__ owner,
                             int32_t r, int32_t nslices, const int32_t* __restrict__ pstart, int32_t* __restrict__ perm,
                             int32_t* __restrict__ local) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nreach; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = ord[i];
    if (owner[v] != r) continue;
    const int32_t L = level[v];
    const int64_t p = i - off[L], n = off[L + 1] - off[L];
    const int64_t lo = ((int64_t)r * n + nslices - 1) / nslices;
    const int32_t row = pstart[L] + (int32_t)(p - lo);
    perm[row] = v;
    local[v] = row;
  }
}

// ghost j (ring order) -> row gbase + j; its level's source slice in src_mask
__global__ void k_ghost_rows(const int32_t* __restrict__ glist, int64_t ng, int32_t gbase,
                             const int32_t* __restrict__ level, const int32_t* __restrict__ owner,
                             int32_t* __restrict__ perm, int32_t* __restrict__ local, uint32_t* __restrict__ src_mask) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < ng; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = glist[j];
    perm[gbase + j] = v;
    local[v] = gbase + (int32_t)j;
    atomicOr(src_mask + level[v], 1u << owner[v]);
  }
}

// slots of one destination's ghosts: gslot[v] = gbase_d + j
__global__ void k_ghost_slots(const int32_t* __restrict__ glist, int64_t ng, int32_t gbase,
                              int32_t* __restrict__ gslot) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < ng; j += (int64_t)gridDim.x * blockDim.x)
    gslot[glist[j]] = gbase + (int32_t)j;
}

// exports of this slice's own rows to destination d (rows whose flag has bit d):
// key = row << 32 | d << 28 | the destination's ghost row; dst_mask per level
__global__ void k_slice_exports(const int32_t* __restrict__ perm, int64_t own_rows, const uint32_t* __restrict__ flag,
                                const int32_t* __restrict__ level, int32_t d, const int32_t* __restrict__ gslot,
                                unsigned long long* __restrict__ keys, unsigned long long* __restrict__ nkeys,
                                uint32_t* __restrict__ dst_mask) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < own_rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = perm[r];
    if (v < 0 || !((flag[v] >> d) & 1u)) continue;
    const unsigned long long at = atomicAdd(nkeys, 1ull);
    if (keys) keys[at] = (unsigned long long)r << 32 | (unsigned long long)((uint32_t)d << 28 | (uint32_t)gslot[v]);
    atomicOr(dst_mask + level[v], 1u << d);
  }
}

__global__ void k_own_mask(const int32_t* __restrict__ perm, int64_t own_rows, uint8_t* __restrict__ mask) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < own_rows; r += (int64_t)gridDim.x * blockDim.x)
    if (perm[r] >= 0) mask[perm[r]] = 1;
}

// sorted export keys -> entries and per-chunk counts
__global__ void k_export_entries(const unsigned long long* __restrict__ keys, int64_t n, int2* __restrict__ xent,
                                 int32_t* __restrict__ xcount) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    const int32_t row = (int32_t)(k >> 32);
    xent[i] = make_int2(row, (int32_t)(uint32_t)k);
    atomicAdd(xcount + (row >> 5), 1);
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

namespace gh {

Band::~Band() { release_state(); }

void Band::release_state() {
  if (!ubuf && !rows_done && !stalled && !gdone) return;
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  if (prev != device) cudaSetDevice(device);
  for (void* p : {(void*)ubuf, (void*)rows_done, (void*)stalled, (void*)gdone}) {
    if (!p) continue;
    if (ipc) cudaFree(p);
    else cudaFreeAsync(p, astream);
  }
  ubuf = nullptr;
  rows_done = nullptr;
  stalled = nullptr;
  gdone = nullptr;
  if (prev >= 0 && prev != device) cudaSetDevice(prev);  // the caller's current device stays
}

uint64_t Band::device_bytes() const {
  return pstart.bytes() + pend.bytes() + perm.bytes() + chunk_level.bytes() + chunk_ptr.bytes() + deg.bytes() +
         deg_big.bytes() + col.bytes() + col16.bytes() + cbase.bytes() + deg4.bytes() + wt.bytes() + area_r.bytes() +
         wsum_r.bytes() + den.bytes() + 2 * sizeof(double) * nrows + sizeof(unsigned long long) * nlev +
         src_mask.bytes() + dst_mask.bytes() + slice_cnt.bytes() + xoff.bytes() + xent.bytes() +
         sizeof(unsigned long long) * (size_t)nslices * nlev;
}

// Cut levels into nbands contiguous bands of about equal row counts; band r
// owns levels [cut[r], cut[r+1]). Mirrored in paper_1812_06060_b200/bands.py.
std::vector<int32_t> plan_bands(const std::vector<int32_t>& offsets, int32_t nbands) {
  const int32_t nlev = (int32_t)offsets.size() - 1;
  if (nbands < 1) fail(GH_ERR_INVALID, "plan_bands: need at least one band");
  if (nbands > nlev) fail(GH_ERR_INVALID, "plan_bands: more bands than BFS levels");
  const int64_t total = offsets[nlev];
  std::vector<int32_t> cut(nbands + 1, 0);
  cut[nbands] = nlev;
  int32_t L = 0;
  for (int32_t r = 1; r < nbands; ++r) {
    const int64_t target = total * r / nbands;
    while (L < nlev && offsets[L] < target) ++L;  // first level starting at or after the target row
    if (L > 0 && target - offsets[L - 1] < offsets[L] - target) --L;  // or the closer boundary before it
    L = std::max(L, cut[r - 1] + 1);              // every band owns at least one level
    L = std::min(L, nlev - (nbands - r));         // and leaves one for each later band
    cut[r] = L;
  }
  return cut;
}

// The band's CSR stream from its row layout (perm, pstart/pend, own_rows,
// nrows set; local[v] = row of v in this band, own or ghost): chunk metadata,
// SELL-32 columns and weights, 16-bit columns, den, and the state buffers.
static void build_rows(gh_levels* L, Band* b, const int32_t* local_p) {
  gh_mesh* m = L->mesh;
  cudaStream_t s = m->stream;
  const int32_t nlev = L->nlev;
  b->chunk_level.alloc(b->own_chunks, s);
  b->deg.alloc(b->nrows, s);
  GH_CUDA(cudaMemsetAsync(b->deg.p, 0, sizeof(uint16_t) * b->nrows, s));
  b->chunk_ptr.alloc(b->own_chunks + 1, s);
  {
    Scratch<int64_t> width(b->own_chunks + 1, s);
    Scratch<int32_t> maxdeg(1, s);
    GH_CUDA(cudaMemsetAsync(maxdeg.p, 0, sizeof(int32_t), s));
    GH_CUDA(cudaMemsetAsync(width.p + b->own_chunks, 0, sizeof(int64_t), s));
    if (b->own_chunks)
      k_chunk_meta<<<grid_for((int64_t)b->own_chunks * 32), B, 0, s>>>(b->perm.p, L->level.p, m->vv_offset.p,
                                                                       b->own_chunks, b->chunk_level.p, width.p,
                                                                       b->deg.p, maxdeg.p);
    GH_LAUNCH_CHECK();
    b->max_chunk_width = read_scalar(maxdeg.p, s);  // the widest chunk = the longest row
    if (b->max_chunk_width >= 65535) {
      // valences past the 16-bit row length: the kernel reads these rows' true
      // length here (deg holds the 65535 marker)
      b->deg_big.alloc(b->nrows, s);
      k_deg_big<<<grid_for(b->nrows), B, 0, s>>>(b->perm.p, m->vv_offset.p, b->nrows, b->deg_big.p);
      GH_LAUNCH_CHECK();
    }
    size_t tmp = 0;
    GH_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, width.p, b->chunk_ptr.p, b->own_chunks + 1, s));
    Scratch<char> t(tmp, s);
    GH_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, width.p, b->chunk_ptr.p, b->own_chunks + 1, s));
  }
  const int64_t nnz = read_scalar(b->chunk_ptr.p + b->own_chunks, s);
  b->col.alloc(nnz, s);
  b->wt.alloc(nnz, s);
  if (nnz) {
    GH_CUDA(cudaMemsetAsync(b->col.p, 0, sizeof(uint32_t) * nnz, s));
    GH_CUDA(cudaMemsetAsync(b->wt.p, 0, sizeof(double) * nnz, s));
  }
  b->area_r.alloc(b->nrows, s);
  b->wsum_r.alloc(b->nrows, s);
  GH_CUDA(cudaMemsetAsync(b->area_r.p, 0, sizeof(double) * b->nrows, s));
  GH_CUDA(cudaMemsetAsync(b->wsum_r.p, 0, sizeof(double) * b->nrows, s));
  if (b->own_rows)
    k_sell_fill<<<grid_for(b->own_rows), B, 0, s>>>(b->perm.p, L->level.p, local_p, m->vv_offset.p, m->vv_index.p,
                                                    m->vv_weight.p, m->vertex_area.p, m->vertex_weight_sum.p,
                                                    b->chunk_ptr.p, b->own_rows, b->col.p, b->wt.p, b->area_r.p,
                                                    b->wsum_r.p);
  GH_LAUNCH_CHECK();
  b->col16.alloc(nnz, s);
  b->cbase.alloc(b->own_chunks, s);
  b->deg4.alloc((size_t)b->own_chunks * 16, s);
  b->wide_chunks = 0;
  b->col16_windows = 0;
  if (b->own_chunks) {
    // 2 windows if at most 1/64 of the chunks fall back to 32 bits, else 3,
    // else none. Tests: GH_COL16_WINDOWS=2|3 forces a format, GH_COL16_SPAN
    // lowers the window limit (forcing fallback chunks).
    const char* env = getenv("GH_COL16_SPAN");
    const uint32_t span = env ? (uint32_t)std::max(1, std::min(32768, atoi(env))) : 32768u;
    const char* force = getenv("GH_COL16_WINDOWS");
    // slices read ghost rows in every level: only the 3-window format (its 4th
    // window is the ghost area) expresses them
    const int forced = b->nslices ? 3 : force ? atoi(force) : 0;
    Scratch<unsigned long long> nwide(1, s);
    // A band with ghost rows (a neighbour's boundary level, or a slice's
    // foreign neighbours) tries 3 windows first: only their 4th window reaches
    // the ghost rows, and chunks that fit no window take the global-memory
    // path — a few of them per step are stragglers the whole pipeline waits
    // for (2 BFS bands at config 3: 1.78x one band in 2-window format, 1.20x
    // with 3 windows; profiles/r2_partitions_emulated_*.json)
    const bool ghosts = b->nrows > b->own_rows;
    for (int windows : {ghosts ? 3 : 2, ghosts ? 2 : 3}) {
      if (forced && windows != forced) continue;
      GH_CUDA(cudaMemsetAsync(nwide.p, 0, sizeof(unsigned long long), s));
      k_col16<<<grid_for((int64_t)b->own_chunks * 32), B, 0, s>>>(
          b->chunk_level.p, b->pstart.p, b->pend.p, b->chunk_ptr.p, b->deg.p, b->deg_big.p, b->col.p, b->own_chunks,
          windows, span, b->nrows > b->own_rows ? (uint32_t)b->own_rows : 0u, b->col16.p, b->cbase.p, b->deg4.p,
          nwide.p);
      GH_LAUNCH_CHECK();
      m->launches++;
      b->wide_chunks = (int64_t)read_scalar(nwide.p, s);
      if (forced || b->wide_chunks * 64 <= b->own_chunks) {
        b->col16_windows = windows;
        break;
      }
    }
  }
  b->den.alloc(b->nrows, s);
  b->den_t = 0.0;
  if (!b->ubuf) {
    b->astream = s;
    const size_t sizes[4] = {sizeof(double) * 2 * (size_t)b->nrows, sizeof(unsigned long long) * nlev, sizeof(int32_t),
                             sizeof(unsigned long long) * (size_t)b->nslices * nlev};
    void** ptrs[4] = {reinterpret_cast<void**>(&b->ubuf), reinterpret_cast<void**>(&b->rows_done),
                      reinterpret_cast<void**>(&b->stalled), reinterpret_cast<void**>(&b->gdone)};
    for (int i = 0; i < 4; ++i) {
      if (!sizes[i]) continue;
      if (b->ipc) GH_CUDA(cudaMalloc(ptrs[i], sizes[i]));  // IPC handles need driver allocations
      else GH_CUDA(cudaMallocAsync(ptrs[i], sizes[i], s));
    }
  }
  m->launches += 4;
  GH_CUDA(cudaStreamSynchronize(s));
}


void band_build(gh_levels* L, Band* b, int32_t lb, int32_t le) {
  gh_mesh* m = L->mesh;
  cudaStream_t s = m->stream;
  const int32_t nlev = L->nlev;
  const int64_t V = m->nv;
  const std::vector<int32_t>& off = L->h_offsets;
  b->lb = lb;
  b->le = le;
  b->nlev = nlev;
  b->device = m->device;
  b->h_pstart.assign(nlev, 0);
  b->h_pend.assign(nlev, 0);
  int64_t cursor = 0;
  for (int p = 0; p < 2; ++p) {
    for (int32_t l = lb + ((lb & 1) != p); l < le; l += 2) {
      cursor = (cursor + 31) & ~int64_t(31);
      b->h_pstart[l] = (int32_t)cursor;
      cursor += off[l + 1] - off[l];
      b->h_pend[l] = (int32_t)cursor;
    }
  }
  cursor = (cursor + 31) & ~int64_t(31);
  b->own_rows = (int32_t)cursor;
  for (int32_t g : {lb - 1, le}) {
    if (g < 0 || g >= nlev) continue;
    b->h_pstart[g] = (int32_t)cursor;
    cursor += off[g + 1] - off[g];
    b->h_pend[g] = (int32_t)cursor;
    cursor = (cursor + 31) & ~int64_t(31);
  }
  if (cursor > 0x3fffffffLL) fail(GH_ERR_INVALID, "mesh too large for the diffusion layout");  // uidx < 2^31
  b->nrows = (int32_t)cursor;
  b->own_chunks = b->own_rows / 32;
  b->pstart.alloc(nlev, s);
  b->pend.alloc(nlev, s);
  GH_CUDA(cudaMemcpyAsync(b->pstart.p, b->h_pstart.data(), sizeof(int32_t) * nlev, cudaMemcpyHostToDevice, s));
  GH_CUDA(cudaMemcpyAsync(b->pend.p, b->h_pend.data(), sizeof(int32_t) * nlev, cudaMemcpyHostToDevice, s));
  b->perm.alloc(b->nrows, s);
  GH_CUDA(cudaMemsetAsync(b->perm.p, 0xff, sizeof(int32_t) * b->nrows, s));
  Scratch<int32_t> local(V, s);
  GH_CUDA(cudaMemsetAsync(local.p, 0xff, sizeof(int32_t) * V, s));
  const int32_t glo = std::max(lb - 1, 0), ghi = std::min(le, nlev - 1);
  const int64_t pb = off[glo], pe = off[ghi + 1];
  if (pe > pb) {
    const int32_t* ord = L->layout_order.p ? L->layout_order.p : L->order.p;
    k_band_renumber<<<grid_for(pe - pb), B, 0, s>>>(ord, L->level.p, pb, pe, L->offsets.p, b->pstart.p,
                                                    b->perm.p, local.p);
    GH_LAUNCH_CHECK();
  }
  build_rows(L, b, local.p);
}

void band_link(Band* lower, Band* upper) {
  // upper.lb == lower.le: the lower band's last level is upper's lower ghost,
  // the upper band's first level is lower's upper ghost
  lower->hi_ubuf = upper->ubuf;
  lower->hi_done = upper->rows_done;
  lower->hi_nrows = upper->nrows;
  lower->hi_ghost = upper->ghost_row(lower->le - 1);
  upper->lo_ubuf = lower->ubuf;
  upper->lo_done = lower->rows_done;
  upper->lo_nrows = lower->nrows;
  upper->lo_ghost = lower->ghost_row(upper->lb);
}


namespace {

// own rows of slice q in a ring of n: positions [slice_lo(n, q), slice_lo(n, q + 1))
int32_t slice_lo(int64_t n, int32_t q, int32_t nslices) { return (int32_t)(((int64_t)q * n + nslices - 1) / nslices); }

// the parity layout of slice q's own rows (band_build's order, lb = 0, le = nlev);
// returns the 32-aligned own row count
int64_t slice_layout(const std::vector<int32_t>& off, int32_t q, int32_t nslices, std::vector<int32_t>* ps,
                     std::vector<int32_t>* pe) {
  const int32_t nlev = (int32_t)off.size() - 1;
  int64_t cursor = 0;
  for (int p = 0; p < 2; ++p) {
    for (int32_t l = p; l < nlev; l += 2) {
      const int64_t n = off[l + 1] - off[l];
      cursor = (cursor + 31) & ~int64_t(31);
      if (ps) (*ps)[l] = (int32_t)cursor;
      cursor += slice_lo(n, q + 1, nslices) - slice_lo(n, q, nslices);
      if (pe) (*pe)[l] = (int32_t)cursor;
    }
  }
  return (cursor + 31) & ~int64_t(31);
}

// vertices slice q ghosts, in ring order; returns their count
int64_t ghost_list(const int32_t* ord, int64_t nreach, const uint32_t* flag, int32_t q, int32_t* glist,
                   uint8_t* pick, cudaStream_t s) {
  k_slice_pick<<<grid_for(nreach), B, 0, s>>>(ord, nreach, flag, q, pick);
  GH_LAUNCH_CHECK();
  Scratch<int64_t> ng(1, s);
  size_t tmp = 0;
  GH_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, ord, pick, glist, ng.p, nreach, s));
  Scratch<char> t(tmp, s);
  GH_CUDA(cub::DeviceSelect::Flagged(t.p, tmp, ord, pick, glist, ng.p, nreach, s));
  return read_scalar(ng.p, s);
}

}  // namespace

void slice_build(gh_levels* L, Band* b, int32_t rank, int32_t nslices) {
  gh_mesh* m = L->mesh;
  cudaStream_t s = m->stream;
  const int32_t nlev = L->nlev;
  const int64_t V = m->nv, nreach = L->nreach;
  const std::vector<int32_t>& off = L->h_offsets;
  if (nslices < 1 || nslices > Band::kMaxSlices) fail(GH_ERR_INVALID, "slices: 1 to 8 slices");
  if (rank < 0 || rank >= nslices) fail(GH_ERR_INVALID, "slices: bad rank");
  b->lb = 0;
  b->le = nlev;
  b->nlev = nlev;
  b->device = m->device;
  b->nslices = nslices;
  b->rank = rank;
  // every slice's own rows per level, and every slice's own row count (the
  // base of its ghost rows, where this slice's exports land)
  std::vector<int32_t> cnt((size_t)nslices * nlev);
  std::vector<int64_t> own(nslices);
  for (int32_t q = 0; q < nslices; ++q) {
    for (int32_t l = 0; l < nlev; ++l) {
      const int64_t n = off[l + 1] - off[l];
      cnt[(size_t)q * nlev + l] = slice_lo(n, q + 1, nslices) - slice_lo(n, q, nslices);
    }
    own[q] = slice_layout(off, q, nslices, nullptr, nullptr);
  }
  b->h_pstart.assign(nlev, 0);
  b->h_pend.assign(nlev, 0);
  slice_layout(off, rank, nslices, &b->h_pstart, &b->h_pend);
  b->own_rows = (int32_t)own[rank];
  b->own_chunks = b->own_rows / 32;
  const int32_t* ord = L->layout_order.p ? L->layout_order.p : L->order.p;
  Scratch<int32_t> owner(V, s);
  Scratch<uint32_t> flag(V, s);
  GH_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(uint32_t) * V, s));
  Scratch<uint8_t> pick(nreach, s);
  Scratch<int32_t> glist(nreach, s);
  if (nreach) {
    k_slice_owner<<<grid_for(nreach), B, 0, s>>>(ord, L->level.p, L->offsets.p, nreach, nslices, owner.p);
    k_slice_flags<<<grid_for(nreach), B, 0, s>>>(ord, nreach, owner.p, m->vv_offset.p, m->vv_index.p, flag.p);
    GH_LAUNCH_CHECK();
  }
  const int64_t ng = nreach ? ghost_list(ord, nreach, flag.p, rank, glist.p, pick.p, s) : 0;
  b->ghost_rows = ng;
  const int64_t nrows = (b->own_rows + ng + 31) & ~int64_t(31);
  if (nrows > 0x3fffffffLL) fail(GH_ERR_INVALID, "mesh too large for the diffusion layout");  // uidx < 2^31
  b->nrows = (int32_t)nrows;
  b->pstart.alloc(nlev, s);
  b->pend.alloc(nlev, s);
  GH_CUDA(cudaMemcpyAsync(b->pstart.p, b->h_pstart.data(), sizeof(int32_t) * nlev, cudaMemcpyHostToDevice, s));
  GH_CUDA(cudaMemcpyAsync(b->pend.p, b->h_pend.data(), sizeof(int32_t) * nlev, cudaMemcpyHostToDevice, s));
  b->perm.alloc(b->nrows, s);
  GH_CUDA(cudaMemsetAsync(b->perm.p, 0xff, sizeof(int32_t) * b->nrows, s));
  b->src_mask.alloc(nlev, s);
  b->dst_mask.alloc(nlev, s);
  GH_CUDA(cudaMemsetAsync(b->src_mask.p, 0, sizeof(uint32_t) * nlev, s));
  GH_CUDA(cudaMemsetAsync(b->dst_mask.p, 0, sizeof(uint32_t) * nlev, s));
  {
    Scratch<int32_t> local(V, s);
    GH_CUDA(cudaMemsetAsync(local.p, 0xff, sizeof(int32_t) * V, s));
    if (nreach)
      k_slice_rows<<<grid_for(nreach), B, 0, s>>>(ord, L->level.p, L->offsets.p, nreach, owner.p, rank, nslices,
                                                  b->pstart.p, b->perm.p, local.p);
    if (ng)
      k_ghost_rows<<<grid_for(ng), B, 0, s>>>(glist.p, ng, b->own_rows, L->level.p, owner.p, b->perm.p, local.p,
                                              b->src_mask.p);
    GH_LAUNCH_CHECK();
    build_rows(L, b, local.p);
  }
  // exports: for every other slice d, the rows of this slice that d ghosts,
  // with their rows in d's layout (d's ghost j sits at row own[d] + j)
  Scratch<int32_t> gslot(V, s);
  Scratch<unsigned long long> nkeys(1, s);
  GH_CUDA(cudaMemsetAsync(nkeys.p, 0, sizeof(unsigned long long), s));
  for (int pass = 0; pass < 2; ++pass) {
    const int64_t nk = pass ? (int64_t)read_scalar(nkeys.p, s) : 0;
    Scratch<unsigned long long> keys(pass ? nk : 0, s);
    if (pass) GH_CUDA(cudaMemsetAsync(nkeys.p, 0, sizeof(unsigned long long), s));
    for (int32_t d = 0; d < nslices && (pass == 0 || nk > 0); ++d) {
      if (d == rank || !nreach) continue;
      const int64_t gd = ghost_list(ord, nreach, flag.p, d, glist.p, pick.p, s);
      if (!gd) continue;
      k_ghost_slots<<<grid_for(gd), B, 0, s>>>(glist.p, gd, (int32_t)own[d], gslot.p);
      k_slice_exports<<<grid_for(b->own_rows), B, 0, s>>>(b->perm.p, b->own_rows, flag.p, L->level.p, d, gslot.p,
                                                          pass ? keys.p : nullptr, nkeys.p, b->dst_mask.p);
      GH_LAUNCH_CHECK();
    }
    if (!pass) continue;
    b->exports = nk;
    b->xent.alloc(nk, s);
    b->xoff.alloc(b->own_chunks + 1, s);
    Scratch<int32_t> xcount(b->own_chunks + 1, s);
    GH_CUDA(cudaMemsetAsync(xcount.p, 0, sizeof(int32_t) * (b->own_chunks + 1), s));
    if (nk) {
      Scratch<unsigned long long> sorted(nk, s);
      size_t tmp = 0;
      GH_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.p, sorted.p, nk, 0, 64, s));
      Scratch<char> t(tmp, s);
      GH_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, keys.p, sorted.p, nk, 0, 64, s));
      k_export_entries<<<grid_for(nk), B, 0, s>>>(sorted.p, nk, b->xent.p, xcount.p);
      GH_LAUNCH_CHECK();
    }
    size_t tmp = 0;
    GH_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, xcount.p, b->xoff.p, b->own_chunks + 1, s));
    Scratch<char> t(tmp, s);
    GH_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, xcount.p, b->xoff.p, b->own_chunks + 1, s));
  }
  b->slice_cnt.alloc(cnt.size(), s);
  GH_CUDA(cudaMemcpyAsync(b->slice_cnt.p, cnt.data(), sizeof(int32_t) * cnt.size(), cudaMemcpyHostToDevice, s));
  m->launches += 8 + 3 * nslices;
  GH_CUDA(cudaStreamSynchronize(s));
}

void band_own_mask(const Band* b, uint8_t* d_mask, int64_t nv, cudaStream_t s) {
  GH_CUDA(cudaMemsetAsync(d_mask, 0, nv, s));
  if (b->own_rows) k_own_mask<<<grid_for(b->own_rows), B, 0, s>>>(b->perm.p, b->own_rows, d_mask);
  GH_LAUNCH_CHECK();
}

void slice_link(std::vector<Band*>& sl) {
  for (Band* a : sl)
    for (size_t d = 0; d < sl.size(); ++d) {
      a->peer_ubuf[d] = sl[d]->ubuf;
      a->peer_gdone[d] = sl[d]->gdone;
      a->peer_sys = false;  // one device
    }
}

}  // namespace gh
