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

#include <cub/device/device_scan.cuh>

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
                        uint16_t* __restrict__ col16, int4* __restrict__ cbase, uint8_t* __restrict__ deg4,
                        unsigned long long* __restrict__ nwide) {
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
    // 3 windows: level L-1) or 2 (level L+1)
    auto window = [&](uint32_t u) -> int {
      const uint32_t row = (u >> 6) << 5 | (u & 31u);
      if (row >= lo && row < hi) return 0;
      if (windows == 2) return 1;
      return row >= lo1 && row < hi1 ? 1 : 2;
    };
    uint32_t mn[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, mx[3] = {0u, 0u, 0u};
    for (int64_t k = 0; k < d; ++k) {
      const uint32_t u = col[p0 + 32 * k + lane];
      const int o = window(u);
      mn[o] = min(mn[o], u);
      mx[o] = max(mx[o], u);
    }
    bool fits = true;
    uint32_t base[3];
    for (int o = 0; o < 3; ++o) {
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
        cbase[c] = make_int4((int32_t)base[0], (int32_t)base[1] - (1 << 14), (int32_t)base[2] - (2 << 14), 0);
      }
    }
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

Band::~Band() {
  if (!ubuf && !rows_done && !stalled) return;
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  if (prev != device) cudaSetDevice(device);
  for (void* p : {(void*)ubuf, (void*)rows_done, (void*)stalled}) {
    if (!p) continue;
    if (ipc) cudaFree(p);
    else cudaFreeAsync(p, astream);
  }
  if (prev >= 0 && prev != device) cudaSetDevice(prev);  // the caller's current device stays
}

uint64_t Band::device_bytes() const {
  return pstart.bytes() + pend.bytes() + perm.bytes() + chunk_level.bytes() + chunk_ptr.bytes() + deg.bytes() +
         deg_big.bytes() + col.bytes() + col16.bytes() + cbase.bytes() + deg4.bytes() + wt.bytes() + area_r.bytes() +
         wsum_r.bytes() + den.bytes() + 2 * sizeof(double) * nrows + sizeof(unsigned long long) * nlev;
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
    k_sell_fill<<<grid_for(b->own_rows), B, 0, s>>>(b->perm.p, L->level.p, local.p, m->vv_offset.p, m->vv_index.p,
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
    const int forced = force ? atoi(force) : 0;
    Scratch<unsigned long long> nwide(1, s);
    for (int windows : {2, 3}) {
      if (forced && windows != forced) continue;
      GH_CUDA(cudaMemsetAsync(nwide.p, 0, sizeof(unsigned long long), s));
      k_col16<<<grid_for((int64_t)b->own_chunks * 32), B, 0, s>>>(
          b->chunk_level.p, b->pstart.p, b->pend.p, b->chunk_ptr.p, b->deg.p, b->deg_big.p, b->col.p, b->own_chunks,
          windows, span, b->col16.p, b->cbase.p, b->deg4.p, nwide.p);
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
    const size_t sizes[3] = {sizeof(double) * 2 * (size_t)b->nrows, sizeof(unsigned long long) * nlev, sizeof(int32_t)};
    void** ptrs[3] = {reinterpret_cast<void**>(&b->ubuf), reinterpret_cast<void**>(&b->rows_done),
                      reinterpret_cast<void**>(&b->stalled)};
    for (int i = 0; i < 3; ++i) {
      if (b->ipc) GH_CUDA(cudaMalloc(ptrs[i], sizes[i]));  // IPC handles need driver allocations
      else GH_CUDA(cudaMallocAsync(ptrs[i], sizes[i], s));
    }
  }
  m->launches += 4;
  GH_CUDA(cudaStreamSynchronize(s));
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

}  // namespace gh
