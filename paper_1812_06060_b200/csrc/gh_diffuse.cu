// Breadth-first Gauss-Seidel heat diffusion, gs_diffuse (reference
// diffusion.hpp:57-124), sweep-pipelined for sm_100a.
//
// Reference semantics: sweep s visits levels D_0, D_1, ... in order; the
// update of j in D_L reads u^s of level L-1 and u^(s-1) of levels L and L+1
// ("Jacobi within a level, Gauss-Seidel across levels", diffusion.hpp:74-83).
//
// Pipelining: task U(s, L) writes buffer (s & 1) and reads
// level L-1 from buffer (s & 1), levels L and L+1 from buffer ((s-1) & 1).
// Then every task with L + 2s = tau ("step tau") is independent of the others
// of its step, and U(s, L) only needs levels L-1, L, L+1 to have finished the
// sweeps it reads. Operand values, and their summation order within a row, are
// exactly the reference's, so u is bit-identical (no FMA: -fmad=false).
//
// Kernel (k_diffuse_tma): one persistent cooperative launch for all S sweeps.
//  * rows renumbered by (level parity, level, original index), every level
//    32-row aligned, so a step's active rows are one contiguous range and a
//    32-row chunk holds one level; CSR in SELL-32 (entry k of lane j at
//    chunk_ptr + 32k + j).
//  * per block, a producer warp streams the step's chunk share (den, row
//    lengths, columns, weights: 68.5 B per update with 16-bit columns, 82 B
//    with 32-bit ones, of the ~100 algorithmic B) HBM -> shared memory
//    with cp.async.bulk + mbarrier complete_tx into a ring of tiles, running
//    ahead across steps (the CSR is read-only);
//  * 8 consumer warps each take 2 chunks of a tile, gather the neighbour u
//    values (ld.global.ca: L1, then L2) with all 12-16 gathers in flight,
//    store u;
//  * no grid barrier: a chunk of level L at step tau waits (acquire) on
//    per-level row counters of L-1, L, L+1; blocks publish their rows per
//    level after each step (release). Each task depends only on earlier
//    steps and all blocks are co-resident, so the schedule cannot deadlock.

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "gh_internal.cuh"

namespace {

constexpr int B = gh::kBlock;
constexpr int kMaxSmemLevels = 12 * 1024;  // pend table in shared memory (48 KB; pstart is derived from it)

__global__ void k_den(const double* __restrict__ area, const double* __restrict__ wsum, double t, int64_t n,
                      double* __restrict__ den) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    den[r] = area[r] + t * wsum[r];  // diffusion.hpp:81
}

// both sweep-parity buffers <- start state (initial, or u0 = 1 on D_0)
__global__ void k_init_buffers(const int32_t* __restrict__ perm, const int32_t* __restrict__ level,
                               const double* __restrict__ initial, int64_t nrows, double* __restrict__ ubuf) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = perm[r];
    double x = 0.0;
    if (v >= 0) x = initial ? initial[v] : (level[v] == 0 ? 1.0 : 0.0);
    ubuf[gh::uidx((uint32_t)r, 0)] = x;
    ubuf[gh::uidx((uint32_t)r, 1)] = x;
  }
}

__global__ void k_init_orig(const int32_t* __restrict__ level, const double* __restrict__ initial, int64_t nv,
                            double* __restrict__ u) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x)
    u[v] = initial ? initial[v] : (level[v] == 0 ? 1.0 : 0.0);
}

// own rows of a band -> original vertex order
__global__ void k_scatter(const int32_t* __restrict__ perm, const double* __restrict__ ubuf, uint32_t parity,
                          int64_t nrows, double* __restrict__ u) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = perm[r];
    if (v >= 0) u[v] = ubuf[gh::uidx((uint32_t)r, parity)];
  }
}

// ---------------------------------------------------------------- the kernel
constexpr int kConsumerWarps = 8;
constexpr int kChunksPerWarp = 2;                            // chunks a consumer warp has in flight
constexpr int kTileChunks = kConsumerWarps * kChunksPerWarp;  // chunks per ring slot
constexpr int kTmaThreads = 32 * (kConsumerWarps + 1);

// one BFS band (gh::Band) as the kernel sees it
struct BandArgs {
  const int32_t* pstart;
  const int32_t* pend;
  const int32_t* chunk_level;
  const int64_t* chunk_ptr;
  const uint16_t* deg;
  const int32_t* deg_big;         // true row lengths where deg holds 65535 (else null)
  const uint8_t* deg4;            // row lengths as nibbles, 16 B per chunk (15: look in deg)
  const uint32_t* col;            // gh::uidx(neighbour row, 1 unless one level closer to the sources)
  const uint16_t* col16;          // the same columns in 16 bits against per-chunk bases (gh::Band::col16)
  const int4* cbase;              // per chunk: window bases (gh::Band::cbase)
  const double* wt;
  const double* den;
  double* ubuf;                   // both sweep parities, gh::uidx layout
  unsigned long long* rows_done;  // [nlev]
  double* lo_ubuf;                // lower neighbour (holds our level lb as a ghost), or null
  unsigned long long* lo_done;
  double* hi_ubuf;                // upper neighbour (holds our level le-1 as a ghost), or null
  unsigned long long* hi_done;
  int32_t* stalled;               // set when a dependency never arrives (a dead peer): the kernel bails out
  int32_t lo_ghost, hi_ghost;     // first row of the ghost copy inside the neighbour
  int32_t lb, le;                 // own levels
  int32_t half2;                  // first row of the odd-level half
  int32_t gs_lo, gs_hi;           // first rows of the ghost levels lb-1, le (this band)
  // sector slices (gh::Band, kSlice kernels only)
  const uint32_t* src_mask;       // [nlev] slices this one reads ghost rows from
  const uint32_t* dst_mask;       // [nlev] slices that read rows of this one
  const int32_t* slice_cnt;       // [nslices][nlev] own rows per slice
  const int32_t* xoff;            // [own chunks + 1] export entries per chunk
  const int2* xent;               // (own row, dest << 28 | dest row)
  int32_t xoff_src;               // this slice has ghost rows (from some source slice)
  unsigned long long* gdone;      // [nslices][nlev] this slice's ghost rows finished, per source
  double* peer_ubuf[gh::Band::kMaxSlices];
  unsigned long long* peer_gdone[gh::Band::kMaxSlices];
  int32_t nslices, rank, peer_sys;
};

constexpr int kMaxBands = 8;  // bands per launch (one per GPU in production; more when emulated)

struct TmaArgs {
  BandArgs bands[kMaxBands];
  int32_t block_start[kMaxBands + 1];  // blocks of band i are [block_start[i], block_start[i+1])
  int32_t nbands;
  int32_t nlev, sweeps;
  int32_t wcap;        // widest chunk (neighbours per row) a slot holds
  int32_t nslots;      // ring slots per block
  int32_t slot_bytes;
  int32_t table_in_smem;
  int32_t stream_policy;    // L2 policy of the CSR stream copies: 0 evict_first, 1 evict_last, 2 evict_normal
  // Sweep groups: sweeps [gK, gK + K) run as one pipeline
  // over the levels, group g starting at step g * P. K = sweeps, P = huge is
  // the plain pipeline (step tau = L + 2s).
  int32_t group_sweeps, group_period;
  // the E1 early stop (gh_gs_diffuse_tol): every update's value also lands in
  // snap[s * snap_rows + row] (row order of the single band), so u of every
  // sweep of the launch is available afterwards; null otherwise
  double* snap;
  int64_t snap_rows;
  // zero-level truncation (diffuse_truncated_dev): set to 1 when a row of the
  // band's top own level (le - 1) gets a value with any bit set; null otherwise
  int32_t* top_nonzero;
  double t;
};

// step tau -> group g, local step tl = tau - g * P
__device__ __forceinline__ void step_group(const TmaArgs& a, int32_t tau, int32_t& g, int32_t& tl) {
  if (tau < a.group_period) {  // the plain pipeline (one group): no division per step
    g = 0;
    tl = tau;
    return;
  }
  g = tau / a.group_period;
  tl = tau - g * a.group_period;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// The CSR stream is read once per sweep: copy it with an L2 evict-first
// policy so it does not push the reused u values out of L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// ... unless the whole stream fits in L2 next to u: then it stays there
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_normal_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// contiguous share of the step's chunk range [c0, c1) for block b
// (measured, round 2: n / nb by a reciprocal multiply + fix-up instead of the
// division costs two registers, which spill: config 3 +1.5 %, config 2 +6 %)
__device__ __forceinline__ void block_share(int32_t c0, int32_t c1, int32_t b, int32_t nb, int32_t& cb,
                                            int32_t& ce) {
  const int32_t n = c1 - c0, q = n / nb, rem = n % nb;
  cb = c0 + b * q + (b < rem ? b : rem);
  ce = cb + q + (b < rem ? 1 : 0);
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// own levels are counted by this GPU's blocks; the two ghost levels by the
// neighbour band's GPU (system scope)
__device__ __forceinline__ unsigned long long ld_done(const unsigned long long* p, bool ghost) {
  return ghost ? ld_acquire_sys_u64(p) : ld_acquire_gpu_u64(p);
}

// spin until *ctr >= need (acquire); a dependency that never arrives (a dead
// peer) sets *stalled after ~17 s and gives up, so the launch can report it
__device__ __forceinline__ void wait_counter(const unsigned long long* ctr, unsigned long long need, bool sys,
                                             int32_t* stalled) {
  if (ld_done(ctr, sys) >= need) return;
  const long long t0 = clock64();
  unsigned ns = 64;
  for (unsigned it = 1;; ++it) {
    __nanosleep(ns);
    if (ld_done(ctr, sys) >= need) break;
    if (ns < 512) ns <<= 1;
    if ((it & 255) == 0 && clock64() - t0 > (1ll << 35)) {
      atomicExch(stalled, 1);
      break;
    }
  }
}

// rows [rb, re) of the band's own levels active at step tau: in group g
// (sweeps gK .. gK + Kg - 1) at local step tl, level L runs sweep
// gK + (tl - L) / 2 for tl - L even, 0 <= tl - L < 2 Kg
template <class PStart>
__device__ __forceinline__ bool step_range(const TmaArgs& a, int32_t lb, int32_t le, PStart pstart,
                                           const int32_t* pend, int32_t tau, int32_t& rb, int32_t& re) {
  int32_t g, tl;
  step_group(a, tau, g, tl);
  const int32_t s0 = g * a.group_sweeps;
  if (s0 >= a.sweeps) return false;
  const int32_t kg = a.sweeps - s0 < a.group_sweeps ? a.sweeps - s0 : a.group_sweeps;
  int32_t lhi = tl < le - 1 ? tl : le - 1;
  if ((lhi ^ tl) & 1) --lhi;
  int32_t llo = tl - 2 * (kg - 1);
  if (llo < lb) llo = lb;
  if ((llo ^ tl) & 1) ++llo;
  if (llo > lhi) return false;
  rb = pstart(llo);
  re = pend[lhi];
  return true;
}

// Make n more rows of level X (this band) visible to every waiter: after a
// release fence, the band's own counter and, for a boundary level, the
// neighbour band's copy of it (system scope: the neighbour is another GPU).
__device__ __forceinline__ void publish_rows(const BandArgs* vba, int32_t band_lb, int32_t band_le, int32_t X,
                                             unsigned long long n, bool sys) {
  unsigned long long* lo_done = vba->lo_done;
  unsigned long long* hi_done = vba->hi_done;
  const bool to_lo = X == band_lb && lo_done, to_hi = X == band_le - 1 && hi_done;
  // release: acq_rel fences (not the sequentially consistent __threadfence);
  // system scope only when the neighbour is another GPU
  if ((to_lo || to_hi) && sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
  else asm volatile("fence.acq_rel.gpu;" ::: "memory");
  atomicAdd(vba->rows_done + X, n);
  if (to_lo) sys ? (void)atomicAdd_system(lo_done + X, n) : (void)atomicAdd(lo_done + X, n);
  if (to_hi) sys ? (void)atomicAdd_system(hi_done + X, n) : (void)atomicAdd(hi_done + X, n);
}

// slot layout: header 512 B (int32: chunk offsets [0..kTileChunks], fits [31], chunk levels [32..],
//              16-bit column window bases [64 + 4q .. 67 + 4q])
//              | den kTileChunks x 256 B | row lengths kTileChunks x 64 B (u16; nibbles use 16 B)
//              | columns (u32, or u16 with kWin) | weights
constexpr int kHdr = 512;
constexpr int kBaseHdr = 64;
constexpr int kDenOff = kHdr;
constexpr int kDegOff = kDenOff + kTileChunks * 256;
constexpr int kColOff32 = kDegOff + kTileChunks * 64;  // u16 row lengths
constexpr int kColOff16 = kDegOff + kTileChunks * 16;  // nibbles (16-bit-column kernels)

// kUnroll: rows up to this valence are gathered fully unrolled (6 covers
// icosphere and torus meshes and saves the registers of two more gathers).
// kTable: the pend table is copied into shared memory (separate instances so
// every shared-memory access compiles to LDS, not a generic load); pstart is
// derived from it (levels of a parity half are consecutive, 32-row aligned),
// which halves the table and leaves room for a third ring slot.
// kWin: 0 = 32-bit columns; 2 or 3 = columns streamed as 16-bit offsets into
// 2 or 3 per-chunk windows (gh::Band::col16), 12 B less per
// row; chunks without 16-bit columns take the global-memory path.
// kSlice: the band is a sector slice (gh::Band::nslices): ghost rows of every
// level, counted per source slice; own rows exported to the readers' ghosts.
// kMode: what a row's store is followed by. 0 = everything decided at run time
// (snapshots for the E1 stop, copies into the neighbour bands' ghost rows);
// 1 = the single band on its own: nothing (the consumers are issue-bound: the
// three uniform tests cost the plain launch a few per cent — the top-level
// test alone 121.4 vs 118.4 ms at config 3, same box, alternating runs);
// 2 = a launch of the zero-level truncation (diffuse_truncated_dev): a row of
// the band's top level written with any bit set raises a.top_nonzero.
template <int kUnroll, bool kTable, int kWin, bool kSlice, int kMode>
__global__ void __launch_bounds__(kTmaThreads, 2) k_diffuse_tma(const __grid_constant__ TmaArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  // this block's band and its rank inside the band
  int bi = 0;
  while (bi + 1 < a.nbands && (int32_t)blockIdx.x >= a.block_start[bi + 1]) ++bi;
  // the band descriptor stays in the kernel's parameter (constant) bank: fields
  // are cheap to re-load there, which keeps them out of the register budget
  const BandArgs* vba = &a.bands[bi];
  const BandArgs& sba = a.bands[bi];
  const int32_t band_lb = sba.lb, band_le = sba.le;
  const int32_t b = (int32_t)blockIdx.x - a.block_start[bi];
  const int32_t nb = a.block_start[bi + 1] - a.block_start[bi];

  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + a.nslots;
  int32_t* sh_pend = reinterpret_cast<int32_t*>(empty + a.nslots);
  const uint32_t table_bytes = kTable ? ((4u * (uint32_t)a.nlev + 127u) & ~127u) : 0u;
  // slots start 128-byte aligned in the shared window (offsets from smem keep
  // the accesses in the shared address space)
  const uint32_t slots_at = 16u * (uint32_t)a.nslots + table_bytes;
  unsigned char* slots = smem + slots_at + ((128u - ((smem_u32(smem) + slots_at) & 127u)) & 127u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.nslots; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (kTable) {
    for (int i = threadIdx.x; i < a.nlev; i += blockDim.x) {
      sh_pend[i] = sba.pend[i];
    }
  }
  const int32_t* pend = kTable ? sh_pend : sba.pend;
  // first row of level X: the even and the odd half start at 0 and half2, a
  // later level right after the previous one of its half (rounded up to 32),
  // ghosts where the layout put them
  const int32_t half2 = sba.half2, gs_lo = sba.gs_lo, gs_hi = sba.gs_hi;
  auto pstart = [&](int32_t X) -> int32_t {
    if (!kTable) return sba.pstart[X];
    if (X < band_lb) return gs_lo;
    if (X >= band_le) return gs_hi;
    if (X <= band_lb + 1) return (X & 1) ? half2 : 0;
    return (pend[X - 2] + 31) & ~31;
  };
  __syncthreads();

  // the last group's last task: (band_le - 1) + 2 (kg - 1) steps after its start
  const int32_t last_g = (a.sweeps - 1) / a.group_sweeps;
  const int32_t nsteps = last_g * a.group_period + (band_le - 1) + 2 * (a.sweeps - 1 - last_g * a.group_sweeps) + 1;
  const uint32_t col_cap = (uint32_t)kTileChunks * 32u * a.wcap;  // entries
  constexpr bool kCol16 = kWin != 0;
  constexpr int kColOff = kCol16 ? kColOff16 : kColOff32;
  constexpr uint32_t kColBytes = kCol16 ? 2u : 4u;
  // ring position: slot index and its use parity advance tile by tile
  int slot = 0;
  uint32_t use = 0;
  int32_t issued = 0;

  if (warp == kConsumerWarps) {
    // ---- producer warp: streams the band's share of every step into the ring,
    // running ahead across steps (the CSR is read-only). Work is a stream of
    // batches of 32 chunks; the chunk pointers and levels of the next batch are
    // loaded while the current batch is issued.
    constexpr int kTilesPerBatch = 32 / kTileChunks;
    int32_t tau = -1, cb = 0, ce = 0, ntile = 0, t0 = -kTilesPerBatch;
    auto advance = [&](int32_t& xtau, int32_t& xcb, int32_t& xce, int32_t& xnt, int32_t& xt0) -> bool {
      xt0 += kTilesPerBatch;
      while (xt0 >= xnt) {
        if (++xtau >= nsteps) return false;
        int32_t rb, re;
        xt0 = 0;
        xnt = 0;
        if (!step_range(a, band_lb, band_le, pstart, pend, xtau, rb, re)) continue;
        block_share(rb >> 5, (re + 31) >> 5, b, nb, xcb, xce);
        xnt = (xce - xcb + kTileChunks - 1) / kTileChunks;
      }
      return true;
    };
    auto load = [&](int32_t xcb, int32_t xce, int32_t xt0, int64_t& p0, int32_t& lv0, int64_t& plast, int4& cb0) {
      const int32_t cbase = xcb + xt0 * kTileChunks;
      const int32_t cl = cbase + lane < xce ? cbase + lane : xce;
      p0 = __ldg(vba->chunk_ptr + cl);
      lv0 = cbase + lane < xce ? __ldg(vba->chunk_level + cl) : 0;
      if (kCol16) cb0 = cbase + lane < xce ? __ldg(vba->cbase + cl) : make_int4(-1, 0, 0, 0);
      plast = __ldg(vba->chunk_ptr + (cbase + 32 < xce ? cbase + 32 : xce));
    };
    int64_t p0 = 0, p_last = 0;
    int32_t lv0 = 0;
    int4 cb0 = make_int4(-1, 0, 0, 0);
    bool have = advance(tau, cb, ce, ntile, t0);
    if (have) load(cb, ce, t0, p0, lv0, p_last, cb0);
    while (have) {
      int32_t ntau = tau, ncb = cb, nce = ce, nnt = ntile, nt0 = t0;
      int64_t np0 = 0, np_last = 0;
      int32_t nlv0 = 0;
      int4 ncb0 = make_int4(-1, 0, 0, 0);
      const bool have_next = advance(ntau, ncb, nce, nnt, nt0);
      if (have_next) load(ncb, nce, nt0, np0, nlv0, np_last, ncb0);
      const int32_t cbase = cb + t0 * kTileChunks;
      for (int j = 0; j < kTilesPerBatch && t0 + j < ntile; ++j) {
        if (issued >= a.nslots) mbar_wait(empty + slot, use ^ 1u);
        const int off = j * kTileChunks;  // the tile's lanes in the batch
        const int32_t c0 = cbase + off;
        const int nch = (int)(ce - c0 < kTileChunks ? ce - c0 : kTileChunks);
        const int64_t base = __shfl_sync(0xffffffffu, p0, off);
        const int src = off + (lane <= kTileChunks ? lane : 0);
        int64_t pi = __shfl_sync(0xffffffffu, p0, src < 32 ? src : 31);
        const int32_t li = __shfl_sync(0xffffffffu, lv0, (off + (lane & (kTileChunks - 1))) & 31);
        if (off + lane == 32) pi = p_last;
        int32_t* hdr = reinterpret_cast<int32_t*>(slots + (size_t)slot * a.slot_bytes);
        if (lane <= nch) hdr[lane] = (int32_t)(pi - base);
        if (lane < kTileChunks) hdr[32 + lane] = li;
        if (kCol16) {
          const int qs = (off + (lane & (kTileChunks - 1))) & 31;
          const int32_t bx = __shfl_sync(0xffffffffu, cb0.x, qs), by = __shfl_sync(0xffffffffu, cb0.y, qs);
          const int32_t bz = __shfl_sync(0xffffffffu, cb0.z, qs), bw = __shfl_sync(0xffffffffu, cb0.w, qs);
          if (lane < kTileChunks) {
            hdr[kBaseHdr + 4 * lane] = bx;
            hdr[kBaseHdr + 4 * lane + 1] = by;
            hdr[kBaseHdr + 4 * lane + 2] = bz;
            hdr[kBaseHdr + 4 * lane + 3] = bw;  // 3 windows: the ghost rows (window 3)
          }
        }
        const int64_t pend_tile = __shfl_sync(0xffffffffu, pi, nch);
        const uint32_t ncol = (uint32_t)(pend_tile - base);
        const bool fits = ncol <= col_cap;
        if (lane == 0) hdr[31] = fits ? 1 : 0;
        __syncwarp();
        if (lane == 0) {
          unsigned char* sb = reinterpret_cast<unsigned char*>(hdr);
          const uint32_t bytes = (uint32_t)nch * (256u + (kCol16 ? 16u : 64u)) + (fits ? ncol * (kColBytes + 8u) : 0u);
          mbar_expect_tx(full + slot, bytes);
          const uint64_t pol = a.stream_policy == 1   ? l2_evict_last_policy()
                               : a.stream_policy == 2 ? l2_evict_normal_policy()
                                                      : l2_evict_first_policy();
          bulk_g2s(sb + kDenOff, vba->den + (int64_t)c0 * 32, (uint32_t)nch * 256u, full + slot, pol);
          if (kCol16) bulk_g2s(sb + kDegOff, vba->deg4 + (int64_t)c0 * 16, (uint32_t)nch * 16u, full + slot, pol);
          else bulk_g2s(sb + kDegOff, vba->deg + (int64_t)c0 * 32, (uint32_t)nch * 64u, full + slot, pol);
          if (fits && ncol) {
            if (kCol16) bulk_g2s(sb + kColOff, vba->col16 + base, ncol * 2u, full + slot, pol);
            else bulk_g2s(sb + kColOff, vba->col + base, ncol * 4u, full + slot, pol);
            bulk_g2s(sb + kColOff + col_cap * kColBytes, vba->wt + base, ncol * 8u, full + slot, pol);
          }
        }
        __syncwarp();
        if (issued < a.nslots) ++issued;
        if (++slot == a.nslots) {
          slot = 0;
          use ^= 1u;
        }
      }
      tau = ntau, cb = ncb, ce = nce, ntile = nnt, t0 = nt0;
      p0 = np0, p_last = np_last, lv0 = nlv0, cb0 = ncb0;
      have = have_next;
    }
    return;
  }

  // ---- consumer warps: warp w takes chunks w and w + 8 of every tile. No grid
  // barrier: before a chunk of level L at step tau the warp waits (acquire)
  // until levels L-1, L, L+1 have finished the sweeps its operands come from
  // (rows_done[X] >= ((tau - X + 1) / 2) * |D_X|; ghost levels are counted by
  // the neighbour band); after the step the block publishes its rows per
  // level (release), to the neighbour as well for a boundary level.
  int32_t seen_L = -1, seen_L2 = -1;
  int32_t seen_tau = -1;
  for (int32_t tau = 0; tau < nsteps; ++tau) {
    int32_t rb, re;
    if (!step_range(a, band_lb, band_le, pstart, pend, tau, rb, re)) continue;
    // sweep of level L at this step: s_base - L / 2 (tl - L is even)
    int32_t grp, tl;
    step_group(a, tau, grp, tl);
    const int32_t s_base = grp * a.group_sweeps + (tl >> 1);
    int32_t cb, ce;
    block_share(rb >> 5, (re + 31) >> 5, b, nb, cb, ce);
    const int32_t ntile = (ce - cb + kTileChunks - 1) / kTileChunks;
    if (ntile == 0) continue;
    int32_t lv_first = 0, lv_last = 0;
    if (warp == 0 && lane == 0) {
      lv_first = __ldg(vba->chunk_level + cb);
      lv_last = __ldg(vba->chunk_level + ce - 1);
    }
    if (kSlice) {
      // A slice's share of a step spans many levels (each slice holds 1/N of
      // every ring), so its dependencies are checked once per step, for all of
      // them, by warp 0 (own rows, and ghost rows per source slice): one round
      // of acquires and one L1 invalidation instead of one per level change;
      // the other warps start after the barrier, so their L1-cached gathers
      // see only data published before warp 0's acquires (see below).
      if (warp == 0) {
        const int32_t l0 = __shfl_sync(0xffffffffu, lv_first, 0), l1 = __shfl_sync(0xffffffffu, lv_last, 0);
        const int32_t npairs = ((l1 - l0) / 2 + 1) * 3;
        for (int32_t p = lane; p < npairs; p += 32) {
          const int32_t Lp = l0 + 2 * (p / 3), X = Lp - 1 + p % 3;
          if (X < 0 || X >= a.nlev) continue;
          // level L-1 through sweep s, levels L and L+1 through sweep s-1
          const unsigned long long sw = (unsigned long long)(s_base - (Lp >> 1) + (X < Lp ? 1 : 0));
          wait_counter(vba->rows_done + X, sw * (unsigned long long)(pend[X] - pstart(X)), false, vba->stalled);
          if (vba->xoff_src)
            for (uint32_t msk = __ldg(vba->src_mask + X); msk; msk &= msk - 1) {
              const int q = __ffs(msk) - 1;
              wait_counter(vba->gdone + (size_t)q * a.nlev + X,
                           sw * (unsigned long long)__ldg(vba->slice_cnt + (size_t)q * a.nlev + X), sba.peer_sys != 0,
                           vba->stalled);
            }
        }
        __syncwarp();
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * kConsumerWarps) : "memory");
    }
    for (int32_t j = 0; j < ntile; ++j) {
      mbar_wait(full + slot, use);
      const unsigned char* sb = slots + (size_t)slot * a.slot_bytes;
      const int32_t* hdr = reinterpret_cast<const int32_t*>(sb);
      const bool fits = hdr[31] != 0;
      int32_t Lq[kChunksPerWarp];
      bool live[kChunksPerWarp];
#pragma unroll
      for (int i = 0; i < kChunksPerWarp; ++i) {
        const int q = warp + kConsumerWarps * i;
        live[i] = cb + j * kTileChunks + q < ce;
        Lq[i] = live[i] ? hdr[32 + q] : -1;
      }
      // The u gathers below are L1-cached loads (ld.global.ca). That is safe
      // because every warp passes this check at the start of every step (tau
      // changes) and the acquire loads here are followed by CCTL.IVALL, which
      // drops the SM's whole L1: every value the step reads was published
      // before that acquire, so an L1 line is either refilled from L2 after it
      // or was filled after it — never older than the data the step needs.
      if (!kSlice && (Lq[0] != seen_L || Lq[kChunksPerWarp - 1] != seen_L2 || tau != seen_tau)) {
        // operands: wait for levels L-1, L, L+1 of each chunk (lanes 3i..3i+2)
        const int i = lane / 3;
        const int32_t Li = i == 0 ? Lq[0] : Lq[kChunksPerWarp - 1];  // no dynamic register-array index
        if (i < kChunksPerWarp && Li >= 0) {
          const int32_t X = Li - 1 + lane % 3;
          if (X >= 0 && X < a.nlev) {
            // level L-1 through sweep s, levels L and L+1 through sweep s-1
            const int32_t s = s_base - (Li >> 1);
            const unsigned long long need =
                (unsigned long long)(s + (X < Li ? 1 : 0)) * (unsigned long long)(pend[X] - pstart(X));
            wait_counter(vba->rows_done + X, need, (X < band_lb || X >= band_le) && sba.peer_sys, vba->stalled);
          }
        }
        __syncwarp();
        seen_L = Lq[0];
        seen_L2 = Lq[kChunksPerWarp - 1];
        seen_tau = tau;
      }
      double num[kChunksPerWarp], den[kChunksPerWarp], v[kChunksPerWarp][kUnroll];
      int32_t d[kChunksPerWarp];
      bool on[kChunksPerWarp], fast[kChunksPerWarp];
      uint32_t px[kChunksPerWarp];  // sweep parity of the step, as the uidx xor mask
      double* const ub = vba->ubuf;
      const double* ubs[kChunksPerWarp];  // 2 windows: u at the chunk's same-level base
      int32_t dlt[kChunksPerWarp];        // 2 windows: other-half base - same-level base - 0x8000
      const int32_t* wtab[kChunksPerWarp];  // 3 windows: the chunk's base table (base_c - c * 2^14)
#pragma unroll
      for (int i = 0; i < kChunksPerWarp; ++i) {
        const int q = warp + kConsumerWarps * i;
        const int32_t c = cb + j * kTileChunks + q;
        const int32_t r = c * 32 + lane;
        on[i] = live[i] && r < pend[Lq[i]];
        px[i] = (uint32_t)((s_base - (Lq[i] >> 1)) & 1) << 5;
        den[i] = reinterpret_cast<const double*>(sb + kDenOff)[q * 32 + lane];
        if (kCol16) {  // nibbles; 15 (a valence of 15 or more) takes the slow path, which reads deg
          const uint32_t nb = reinterpret_cast<const uint8_t*>(sb + kDegOff)[q * 16 + (lane >> 1)];
          d[i] = on[i] ? (int32_t)((nb >> ((lane & 1) << 2)) & 15u) : 0;
        } else {
          d[i] = on[i] ? reinterpret_cast<const uint16_t*>(sb + kDegOff)[q * 32 + lane] : 0;
        }
        fast[i] = fits && d[i] <= kUnroll;  // 65535 (valence past 16 bits) always takes the slow path
        if (kCol16) {
          const int32_t bs = hdr[kBaseHdr + 4 * q], bo = hdr[kBaseHdr + 4 * q + 1];
          fast[i] = fast[i] && bs >= 0;
          ubs[i] = ub + bs;
          dlt[i] = bo - bs - 0x8000;
          wtab[i] = hdr + kBaseHdr + 4 * q;
        }
        num[i] = 0.0;
      }
      // all gathers of both chunks in flight together; u gathers are L1-cached
      // (see the dependency check above)
#pragma unroll
      for (int i = 0; i < kChunksPerWarp; ++i) {
        if (kWin == 2) {
          // e ^ px keeps bit 15; the same-level base is 64-aligned, so the parity
          // xor commutes with adding it: u index = base(e >> 15) + (e & 0x7fff) ^ px
          const uint16_t* scol = reinterpret_cast<const uint16_t*>(sb + kColOff) + hdr[warp + kConsumerWarps * i] + lane;
#pragma unroll
          for (int k = 0; k < kUnroll; ++k)
            if (fast[i] && k < d[i]) {
              const int32_t e = (int32_t)((uint32_t)scol[32 * k] ^ px[i]);
              v[i][k] = __ldca(ubs[i] + ((e >> 15) * dlt[i] + e));
            }
        } else if (kWin == 3) {
          // window c = e >> 14 (same level, L-1, L+1); table entry c holds
          // base_c - c * 2^14, so u index = table[e >> 14] + e ^ px
          const uint16_t* scol = reinterpret_cast<const uint16_t*>(sb + kColOff) + hdr[warp + kConsumerWarps * i] + lane;
#pragma unroll
          for (int k = 0; k < kUnroll; ++k)
            if (fast[i] && k < d[i]) {
              const int32_t e = (int32_t)((uint32_t)scol[32 * k] ^ px[i]);
              v[i][k] = __ldca(ub + (wtab[i][e >> 14] + e));
            }
        } else {
          const uint32_t* scol = reinterpret_cast<const uint32_t*>(sb + kColOff) + hdr[warp + kConsumerWarps * i] + lane;
#pragma unroll
          for (int k = 0; k < kUnroll; ++k)
            if (fast[i] && k < d[i]) v[i][k] = __ldca(ub + (scol[32 * k] ^ px[i]));
        }
      }
      // row sums, each left to right (diffusion.hpp:79). The branch keeps the
      // scheduler from pulling products above the later gathers; the common
      // case interleaves the two rows' dependent chains.
      const double* swt[kChunksPerWarp];
#pragma unroll
      for (int i = 0; i < kChunksPerWarp; ++i)
        swt[i] = reinterpret_cast<const double*>(sb + kColOff + (size_t)col_cap * kColBytes) +
                 hdr[warp + kConsumerWarps * i] + lane;
      if (fast[0] && fast[kChunksPerWarp - 1]) {
#pragma unroll
        for (int k = 0; k < kUnroll; ++k)
#pragma unroll
          for (int i = 0; i < kChunksPerWarp; ++i)
            if (k < d[i]) num[i] += swt[i][32 * k] * v[i][k];
      } else {
#pragma unroll
        for (int i = 0; i < kChunksPerWarp; ++i)
          if (fast[i]) {
#pragma unroll
            for (int k = 0; k < kUnroll; ++k)
              if (k < d[i]) num[i] += swt[i][32 * k] * v[i][k];
          }
      }
#pragma unroll
      for (int i = 0; i < kChunksPerWarp; ++i) {
        const int q = warp + kConsumerWarps * i;
        const int32_t c = cb + j * kTileChunks + q;
        if (!fast[i] && on[i]) {  // wide rows or a tile past the slot: straight from global memory
          const int64_t q0 = __ldg(vba->chunk_ptr + c) + lane;
          // (a global load here, not above: a load in the fast path would share a
          // scoreboard with the gathers and serialise the two chunks)
          int32_t dd = d[i];
          if (kCol16) dd = vba->deg[c * 32 + lane];
          if (dd == 65535 && vba->deg_big) dd = vba->deg_big[c * 32 + lane];
          for (int32_t k = 0; k < dd; ++k) {
            const uint32_t cc = __ldg(vba->col + q0 + 32 * (int64_t)k);
            const double w = __ldg(vba->wt + q0 + 32 * (int64_t)k);
            num[i] += w * __ldca(ub + (cc ^ px[i]));
          }
        }
        double un = 0.0;
        if (on[i]) {
          const int32_t r = c * 32 + lane;
          const double u0 = Lq[i] == 0 ? 1.0 : 0.0;
          // (u0 + t num) / den (diffusion.hpp:82). Far from the sources the
          // numerator is exactly 0 for many sweeps (underflow), and a zero
          // quotient sends the IEEE division down its slow path; 0 / den with
          // den > 0 is that same zero, so skip the division there.
          const double nz = u0 + a.t * num[i];
          un = nz;
          if (!(nz == 0.0 && den[i] > 0.0))  // asm volatile: keeps the division under the branch
            asm volatile("div.rn.f64 %0, %1, %2;" : "=d"(un) : "d"(nz), "d"(den[i]));
          const uint32_t par = px[i] >> 5;
          __stcg(ub + gh::uidx((uint32_t)r, par), un);
          if (kMode == 0) {
            if (a.snap) __stcs(a.snap + (int64_t)(s_base - (Lq[i] >> 1)) * a.snap_rows + r, un);
            // boundary levels also land in the neighbour band's ghost copy
            if (Lq[i] == band_lb && vba->lo_ubuf)
              __stcg(vba->lo_ubuf + gh::uidx((uint32_t)(vba->lo_ghost + (r - pstart(Lq[i]))), par), un);
            if (Lq[i] == band_le - 1 && vba->hi_ubuf)
              __stcg(vba->hi_ubuf + gh::uidx((uint32_t)(vba->hi_ghost + (r - pstart(Lq[i]))), par), un);
          }
          // zero-level truncation: any bit set in the cap's top level flags the launch
          if (kMode == 2 && Lq[i] == band_le - 1 && __double_as_longlong(un) != 0) *a.top_nonzero = 1;
        }
        if (kSlice && live[i] && vba->xoff) {
          // rows other slices read: into their ghost rows (same sweep parity)
          const int32_t x0 = __ldg(vba->xoff + c), x1 = __ldg(vba->xoff + c + 1);
          for (int32_t e0 = x0; e0 < x1; e0 += 32) {
            const bool ok = e0 + lane < x1;
            const int2 en = ok ? __ldg(vba->xent + e0 + lane) : make_int2(0, 0);
            const double val = __shfl_sync(0xffffffffu, un, en.x & 31);
            if (ok) {
              const uint32_t d = (uint32_t)en.y >> 28, row = (uint32_t)en.y & 0x0fffffffu;
              __stcg(sba.peer_ubuf[d] + gh::uidx(row, px[i] >> 5), val);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + slot);
      if (++slot == a.nslots) {
        slot = 0;
        use ^= 1u;
      }
    }
    // publish this block's rows of the step, level by level
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kConsumerWarps) : "memory");
    if (warp == 0) {
      lv_first = __shfl_sync(0xffffffffu, lv_first, 0);
      lv_last = __shfl_sync(0xffffffffu, lv_last, 0);
      for (int32_t X = lv_first + 2 * lane; X <= lv_last; X += 64) {
        const int32_t px0 = pstart(X);
        const int32_t lo = cb * 32 > px0 ? cb * 32 : px0;
        const int32_t hi = ce * 32 < pend[X] ? ce * 32 : pend[X];
        if (hi > lo) {
          if (kSlice) {  // own counter, then every reader slice's count of this source
            const uint32_t dm = __ldg(vba->dst_mask + X);
            if (sba.peer_sys && dm) asm volatile("fence.acq_rel.sys;" ::: "memory");
            else asm volatile("fence.acq_rel.gpu;" ::: "memory");
            atomicAdd(vba->rows_done + X, (unsigned long long)(hi - lo));
            for (uint32_t msk = dm; msk; msk &= msk - 1) {
              unsigned long long* ctr = sba.peer_gdone[__ffs(msk) - 1] + (size_t)sba.rank * a.nlev + X;
              if (sba.peer_sys) atomicAdd_system(ctr, (unsigned long long)(hi - lo));
              else atomicAdd(ctr, (unsigned long long)(hi - lo));
            }
          } else {
            publish_rows(vba, band_lb, band_le, X, (unsigned long long)(hi - lo), sba.peer_sys != 0);
          }
        }
      }
    }
    // the block's own rows are published before any warp starts the next step:
    // otherwise the first tile of the next step polls for them
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kConsumerWarps) : "memory");
  }
}

template <class T>
T read_scalar(const T* d, cudaStream_t s) {
  T v;
  GH_CUDA(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
  return v;
}

// one sweep's snapshot (the single band's row order) -> original vertex order
__global__ void k_scatter_rows(const int32_t* __restrict__ perm, const double* __restrict__ snap, int64_t nrows,
                               double* __restrict__ u) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = perm[r];
    if (v >= 0) u[v] = snap[r];
  }
}

// r_j = A_j u_j - t * sum theta (u_k - u_j) - u0_j (diffusion.hpp:41-47); sq_j = r_j^2
__global__ void k_residual(const int32_t* __restrict__ vv_off, const int32_t* __restrict__ vv_idx,
                           const double* __restrict__ vv_w, const double* __restrict__ va,
                           const int32_t* __restrict__ level, const double* __restrict__ u, double t, int64_t nv,
                           double* __restrict__ sq) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nv; j += (int64_t)gridDim.x * blockDim.x) {
    double lap = 0.0;
    const double uj = u[j];
    for (int32_t i = vv_off[j]; i < vv_off[j + 1]; ++i) lap += vv_w[i] * (u[vv_idx[i]] - uj);
    const double r = va[j] * uj - t * lap - (level[j] == 0 ? 1.0 : 0.0);
    sq[j] = r * r;
  }
}

// vertex -> row of the single band (-1: unreachable), and the CSR's columns as rows
__global__ void k_rowof(const int32_t* __restrict__ perm, int64_t own_rows, int32_t* __restrict__ rowof) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < own_rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = perm[r];
    if (v >= 0) rowof[v] = (int32_t)r;
  }
}
__global__ void k_vv_row(const int32_t* __restrict__ vv_idx, const int32_t* __restrict__ rowof, int64_t nnz,
                         int32_t* __restrict__ vv_row) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nnz; c += (int64_t)gridDim.x * blockDim.x)
    vv_row[c] = rowof[vv_idx[c]];
}

// k_residual for the k sweeps of a group at once, in the band's row order
// straight from the sweeps' snapshots (snap_rows apart): thread = row, its
// vertex's CSR row (columns as rows) kept in registers (valence <= 8; larger
// rows loop over it) while it loops over the sweeps, so the CSR is read once
// per group, and per sweep only the gathers of neighbouring rows (levels L-1,
// L, L+1 near the same ring position: the diffusion kernel's own locality)
// and one coalesced store remain. The arithmetic and its order are
// k_residual's (diffusion.hpp:41-47), hence the same bits. r^2 goes to sqr
// (k x own_rows, row order); k_scatter_sq puts it in vertex order.
constexpr int kResRow = 8;
__global__ void __launch_bounds__(256) k_residual_rows(const int32_t* __restrict__ perm, int64_t own_rows,
                                                       const int32_t* __restrict__ vv_off,
                                                       const int32_t* __restrict__ vv_row,
                                                       const double* __restrict__ vv_w, const double* __restrict__ va,
                                                       const int32_t* __restrict__ level,
                                                       const double* __restrict__ snap, int64_t snap_rows, double t,
                                                       int32_t k, double* __restrict__ sqr) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < own_rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = perm[r];
    if (v < 0) continue;  // padding row
    const int32_t b = vv_off[v], e = vv_off[v + 1], n = e - b;
    const double a = va[v];
    const double u0 = level[v] == 0 ? 1.0 : 0.0;
    if (n <= kResRow) {
      int32_t rr[kResRow];
      double w[kResRow];
#pragma unroll
      for (int c = 0; c < kResRow; ++c) {
        rr[c] = c < n ? vv_row[b + c] : (int32_t)r;
        w[c] = c < n ? vv_w[b + c] : 0.0;
      }
      for (int32_t i = 0; i < k; ++i) {
        const double* __restrict__ sp = snap + (int64_t)i * snap_rows;
        const double uj = sp[r];
        double x[kResRow];
#pragma unroll
        for (int c = 0; c < kResRow; ++c) x[c] = c < n ? sp[rr[c]] : 0.0;
        double lap = 0.0;
#pragma unroll
        for (int c = 0; c < kResRow; ++c)
          if (c < n) lap += w[c] * (x[c] - uj);
        const double res = a * uj - t * lap - u0;
        __stcs(sqr + (int64_t)i * own_rows + r, res * res);
      }
    } else {
      for (int32_t i = 0; i < k; ++i) {
        const double* __restrict__ sp = snap + (int64_t)i * snap_rows;
        const double uj = sp[r];
        double lap = 0.0;
        for (int32_t c = b; c < e; ++c) lap += vv_w[c] * (sp[vv_row[c]] - uj);
        const double res = a * uj - t * lap - u0;
        __stcs(sqr + (int64_t)i * own_rows + r, res * res);
      }
    }
  }
}

// warp sum of r^2 (32 consecutive vertices, inside one 1024-vertex segment)
// into that segment's bound T (fp64 atomics: the order does not matter, T only
// chooses which binades the exact sum prepares)
__device__ __forceinline__ void seg_add(double val, int64_t jw, int64_t i, int64_t nseg, double* __restrict__ T) {
  for (int o = 16; o > 0; o >>= 1) val += __shfl_down_sync(0xffffffffu, val, o);
  if ((threadIdx.x & 31) == 0 && val != 0.0) atomicAdd(T + i * nseg + jw / gh::kSeqsumSegment, val);
}

// r^2 of the k sweeps, row order -> vertex order, as a gather: coalesced
// stores, and reads through vertex -> row (rows of one ring sit together, so
// the other rows of a sector are read a few thousand vertices later: L2
// hits). A scatter (8-byte stores to scattered vertices) made HBM fill and
// write back a 32-byte sector per store: 3x the bytes.
__global__ void k_gather_sq(const int32_t* __restrict__ rowof, const double* __restrict__ sqr, int64_t own_rows,
                            int32_t k, int64_t nv, int64_t nseg, double* __restrict__ sq, double* __restrict__ T) {
  const int lane = threadIdx.x & 31;
  constexpr int U = 4;  // grid-stride iterations in flight per thread
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int32_t i = 0; i < k; ++i) {
    const double* __restrict__ src = sqr + (int64_t)i * own_rows;
    double* __restrict__ dst = sq + (int64_t)i * nv;
    for (int64_t jw0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane; jw0 < nv; jw0 += U * stride) {
      double val[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = jw0 + u * stride + lane;
        val[u] = 0.0;
        if (v < nv) {
          const int32_t r = rowof[v];
          val[u] = r >= 0 ? src[r] : dst[v];  // unreachable: the fixed value
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t jw = jw0 + u * stride;
        if (jw + lane < nv) __stcs(dst + jw + lane, val[u]);
        if (jw < nv) seg_add(val[u], jw, i, nseg, T);
      }
    }
  }
}

// r^2 of the unreachable vertices: they and all their neighbours keep the
// start state, so the value is the same every sweep (k_residual's arithmetic)
__global__ void k_residual_fixed(const int32_t* __restrict__ vv_off, const int32_t* __restrict__ vv_idx,
                                 const double* __restrict__ vv_w, const double* __restrict__ va,
                                 const int32_t* __restrict__ level, const double* __restrict__ base, double t,
                                 int64_t nv, int32_t k, double* __restrict__ sq) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nv; j += (int64_t)gridDim.x * blockDim.x) {
    if (level[j] >= 0) continue;
    const double uj = base[j];
    double lap = 0.0;
    for (int32_t c = vv_off[j]; c < vv_off[j + 1]; ++c) lap += vv_w[c] * (base[vv_idx[c]] - uj);
    const double res = va[j] * uj - t * lap - 0.0;
    for (int32_t i = 0; i < k; ++i) sq[(int64_t)i * nv + j] = res * res;
  }
}

}  // namespace

namespace gh {

namespace {

BandArgs band_args(const Band& b) {
  BandArgs x{};
  x.pstart = b.pstart.p;
  x.half2 = 0;
  for (int32_t l = b.lb; l < b.le && l <= b.lb + 1; ++l)
    if (l & 1) x.half2 = b.h_pstart[l];
  x.gs_lo = b.lb > 0 ? b.h_pstart[b.lb - 1] : 0;
  x.gs_hi = b.le < b.nlev ? b.h_pstart[b.le] : 0;
  x.pend = b.pend.p;
  x.chunk_level = b.chunk_level.p;
  x.chunk_ptr = b.chunk_ptr.p;
  x.deg = b.deg.p;
  x.deg_big = b.deg_big.p;
  x.deg4 = b.deg4.p;
  x.col = b.col.p;
  x.col16 = b.col16.p;
  x.cbase = b.cbase.p;
  x.wt = b.wt.p;
  x.den = b.den.p;
  x.ubuf = b.ubuf;
  x.rows_done = b.rows_done;
  x.stalled = b.stalled;
  x.lo_ubuf = b.lo_ubuf;
  x.lo_done = b.lo_done;
  x.hi_ubuf = b.hi_ubuf;
  x.hi_done = b.hi_done;
  x.lo_ghost = b.lo_ghost;
  x.hi_ghost = b.hi_ghost;
  x.lb = b.lb;
  x.le = b.le;
  x.src_mask = b.src_mask.p;
  x.dst_mask = b.dst_mask.p;
  x.slice_cnt = b.slice_cnt.p;
  x.xoff = b.exports ? b.xoff.p : nullptr;  // no exports: no per-chunk lookups
  x.xent = b.xent.p;
  x.xoff_src = b.ghost_rows > 0 ? 1 : 0;
  x.gdone = b.gdone;
  for (int d = 0; d < Band::kMaxSlices; ++d) {
    x.peer_ubuf[d] = b.peer_ubuf[d];
    x.peer_gdone[d] = b.peer_gdone[d];
  }
  x.nslices = b.nslices;
  x.rank = b.rank;
  // GH_PEER_SYS=1: system-scope release and polls between same-device parts
  // too (the emulation then pays what links between GPUs cost)
  const bool force_sys = getenv("GH_PEER_SYS") && atoi(getenv("GH_PEER_SYS")) != 0;
  x.peer_sys = (b.peer_sys || force_sys) ? 1 : 0;
  return x;
}

}  // namespace

// Prepare bands for a solve: den for this t, both sweep buffers = the start
// state (own and ghost rows), progress counters zeroed. Across processes,
// every band must be prepared before any band is launched.
void bands_prepare(gh_levels* L, std::vector<Band*>& bands, double t, const double* d_initial) {
  gh_mesh* m = L->mesh;
  cudaStream_t s = m->stream;
  for (Band* b : bands) {
    if (b->den_t != t) {
      k_den<<<grid_for(b->nrows), B, 0, s>>>(b->area_r.p, b->wsum_r.p, t, b->nrows, b->den.p);
      GH_LAUNCH_CHECK();
      m->launches++;
      b->den_t = t;
    }
    k_init_buffers<<<grid_for(b->nrows), B, 0, s>>>(b->perm.p, L->level.p, d_initial, b->nrows, b->ubuf);
    GH_LAUNCH_CHECK();
    m->launches++;
    GH_CUDA(cudaMemsetAsync(b->rows_done, 0, sizeof(unsigned long long) * b->nlev, s));
    if (b->gdone) GH_CUDA(cudaMemsetAsync(b->gdone, 0, sizeof(unsigned long long) * b->nslices * b->nlev, s));
    GH_CUDA(cudaMemsetAsync(b->stalled, 0, sizeof(int32_t), s));
  }
}

// Run the bands in one cooperative launch on the current device, blocks split
// in proportion to their rows, then scatter their own rows to u_orig.
double bands_launch(gh_levels* L, std::vector<Band*>& bands, double t, int32_t sweeps, double* d_snap,
                    int32_t level_cap, int32_t* d_top_nonzero, bool scatter) {
  gh_mesh* m = L->mesh;
  cudaStream_t s = m->stream;
  int32_t wmax = 1;
  int64_t rows = 0;
  int32_t win = -1;  // the bands' common 16-bit column format (0: some band has none)
  const bool slices = bands[0]->nslices > 0;
  for (Band* b : bands) {
    if ((b->nslices > 0) != slices) fail(GH_ERR_INVALID, "diffusion: slices and level bands in one launch");
    wmax = std::max(wmax, b->max_chunk_width);
    rows += b->own_rows;
    if (!b->own_chunks) continue;
    win = win < 0 || win == b->col16_windows ? b->col16_windows : 0;
  }
  // 16-bit columns when every band has them in one format (gh::band_build
  // picks one only if at most 1/64 of its chunks fall back to 32 bits);
  // GH_DIFFUSE_COL32 forces 32-bit columns (tests)
  if (win < 0 || getenv("GH_DIFFUSE_COL32")) win = 0;
  if (slices && win == 2) win = 0;  // slices are laid out for 3 windows (ghost rows in window 3)
  const bool col16 = win != 0;
  // slot = 512 B header + per chunk (den 256 B + deg 64 B + wcap x 32 x (2 or 4 + 8) B of columns/weights)
  const int32_t wcap = std::min<int32_t>(wmax, 16);
  const int32_t col_off = col16 ? kColOff16 : kColOff32;
  const int32_t slot_bytes = ((col_off + kTileChunks * 32 * wcap * (col16 ? 10 : 12)) + 127) & ~127;
  const bool table = L->nlev <= kMaxSmemLevels;
  const size_t table_bytes = table ? ((sizeof(int32_t) * L->nlev + 127) & ~size_t(127)) : 0;
  // two blocks per SM with a ring of >= 2 slots each (228 KB per SM, 1 KB reserved per block)
  int32_t nslots = 0;
  for (int per = 2; per >= 1 && nslots < 2; --per) {
    const int64_t budget = 228 * 1024 / per - 1024;
    nslots = (int32_t)std::min<int64_t>(8, (budget - (int64_t)table_bytes - 256) / (slot_bytes + 16));
  }
  if (nslots < 2) nslots = 2;
  const size_t shmem = 16 * (size_t)nslots + table_bytes + 128 + (size_t)nslots * slot_bytes;
#define GH_DIFFUSE_FN(W, S, T)                                                                                 \
  (wmax <= 6 ? (table ? (void*)k_diffuse_tma<6, true, W, S, T> : (void*)k_diffuse_tma<6, false, W, S, T>)     \
             : (table ? (void*)k_diffuse_tma<8, true, W, S, T> : (void*)k_diffuse_tma<8, false, W, S, T>))
  // the single band on its own (no neighbour copies, no snapshots) takes the
  // lean instances, with the top-level test when it runs under a level cap
  // (GH_DIFFUSE_GENERAL=1: the run-time instances also there, for tests and A/B runs)
  const bool alone = !slices && bands.size() == 1 && !d_snap && !bands[0]->lo_ubuf && !bands[0]->hi_ubuf &&
                     (d_top_nonzero || !getenv("GH_DIFFUSE_GENERAL"));
  if (d_top_nonzero && !alone) fail(GH_ERR_INTERNAL, "diffusion: the level cap needs the single band on its own");
#define GH_DIFFUSE_MODE(M) \
  (win == 2 ? GH_DIFFUSE_FN(2, false, M) : win == 3 ? GH_DIFFUSE_FN(3, false, M) : GH_DIFFUSE_FN(0, false, M))
  void* fn = slices          ? (win == 3 ? GH_DIFFUSE_FN(3, true, 0) : GH_DIFFUSE_FN(0, true, 0))
             : d_top_nonzero ? GH_DIFFUSE_MODE(2)
             : alone         ? GH_DIFFUSE_MODE(1)
                             : GH_DIFFUSE_MODE(0);
#undef GH_DIFFUSE_MODE
#undef GH_DIFFUSE_FN
  L->last_col16 = win;
  GH_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem));
  int nsm = 0, per_sm = 0;
  GH_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device));
  GH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kTmaThreads, shmem));
  if (per_sm < 1) fail(GH_ERR_CUDA, "diffusion kernel cannot be resident");
  const int32_t nbands = (int32_t)bands.size();
  const int32_t grid = std::max<int32_t>(nsm * per_sm, nbands);
  // blocks per band in proportion to own rows, at least one each
  std::vector<int32_t> start(nbands + 1, 0);
  for (int32_t i = 0; i < nbands; ++i) {
    const int64_t share = rows ? (int64_t)(grid - nbands) * bands[i]->own_rows / rows : 0;
    start[i + 1] = start[i] + 1 + (int32_t)share;
  }
  start[nbands] = std::min(start[nbands], grid);
  if (nbands > kMaxBands) fail(GH_ERR_INVALID, "too many bands for one launch");
  TmaArgs a{};
  for (int32_t i = 0; i < nbands; ++i) a.bands[i] = band_args(*bands[i]);
  for (int32_t i = 0; i <= nbands; ++i) a.block_start[i] = start[i];

  a.nbands = nbands;
  a.nlev = L->nlev;
  a.sweeps = sweeps;
  a.wcap = wcap;
  a.nslots = nslots;
  a.slot_bytes = slot_bytes;
  a.table_in_smem = table ? 1 : 0;
  a.t = t;
  if (d_snap && nbands != 1) fail(GH_ERR_INTERNAL, "diffusion snapshots need the single band");
  a.snap = d_snap;
  a.snap_rows = bands[0]->nrows;
  a.top_nonzero = d_top_nonzero;
  if (level_cap > 0 && level_cap < L->nlev) {
    // the single band stops below level_cap: that level keeps its (zero) rows
    // and counts as finished for every sweep (its counter was set to ~0)
    if (nbands != 1 || slices || bands[0] != &L->main) fail(GH_ERR_INTERNAL, "diffusion: level cap needs the single band");
    a.bands[0].le = level_cap;
    a.bands[0].gs_hi = bands[0]->h_pstart[level_cap];
  }
  // sweep groups: one pipeline of all sweeps unless GH_SWEEP_GROUP=K (then
  // groups of K sweeps, each starting GH_SWEEP_PERIOD steps after the last,
  // at least nlev + 2K - 1 so that the groups never share a step)
  a.group_sweeps = sweeps;
  a.group_period = 0x3fffffff;
  if (const char* gk = getenv("GH_SWEEP_GROUP")) {
    const int32_t k = std::max(1, std::min(sweeps, atoi(gk)));
    if (k < sweeps) {
      const int64_t pmin = (int64_t)L->nlev + 2 * (int64_t)k - 1;
      const char* gp = getenv("GH_SWEEP_PERIOD");
      const int64_t p = std::max<int64_t>(pmin, gp ? atoll(gp) : 0);
      if ((int64_t)((sweeps - 1) / k + 1) * p >= 0x7fffffffLL) fail(GH_ERR_INVALID, "GH_SWEEP_GROUP: too many steps");
      a.group_sweeps = k;
      a.group_period = (int32_t)p;
    }
  }
  {
    // stream + both u buffers against L2 (GH_STREAM_L2=0|1|2 forces, for experiments): config 2 -2 %
    int l2 = 0;
    GH_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, m->device));
    uint64_t bytes = 0;
    for (Band* b : bands)
      bytes += b->den.bytes() + b->deg4.bytes() + b->col16.bytes() + b->wt.bytes() + 16ull * b->nrows;
    if (!col16)
      for (Band* b : bands) bytes += b->col.bytes() - b->col16.bytes() + b->deg.bytes();
    const char* env = getenv("GH_STREAM_L2");
    a.stream_policy = env ? atoi(env) : (bytes <= (uint64_t)l2 ? 1 : 0);
  }
  void* kargs[] = {&a};
  EventTimer timer(s);
  timer.start();
  GH_CUDA(cudaLaunchCooperativeKernel(fn, start[nbands], kTmaThreads, kargs, shmem, s));
  GH_LAUNCH_CHECK();
  timer.stop();
  m->launches++;
  const double ms = timer.ms();
  for (Band* b : bands) {
    int32_t stalled = 0;
    GH_CUDA(cudaMemcpyAsync(&stalled, b->stalled, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    GH_CUDA(cudaStreamSynchronize(s));
    if (stalled) fail(GH_ERR_INTERNAL, "diffusion: a band dependency never arrived (neighbour band not running?)");
    if (!scatter) continue;
    k_scatter<<<grid_for(b->own_rows), B, 0, s>>>(b->perm.p, b->ubuf, (uint32_t)((sweeps - 1) & 1), b->own_rows,
                                                  L->u_orig.p);
    GH_LAUNCH_CHECK();
    m->launches++;
  }
  return ms;
}


namespace {
}  // namespace

// ---------------------------------------------------------------- zero-level truncation
// Far from the sources the heat underflows to exactly +0 and stays there: the
// update of a row whose neighbours are all +0 is (0 + t * 0) / den = +0 for
// den > 0, whatever the weights. So if level C - 1 holds only +0 after every
// sweep, every level >= C stays +0 for all sweeps (induction over levels and
// sweeps, diffusion.hpp:73-82), and running the pipeline on levels [0, C)
// alone — level C read as the zeros it holds — gives the reference's u bit for
// bit. The solve runs in a few launches of an even number of sweeps (so the
// state is back in the parity buffer a launch starts from): each launch covers
// the levels below a cap beyond the nonzero front seen so far, the kernel
// flags any nonzero bit written to the cap's top level, and a flagged launch
// is undone (saved rows restored) and redone with a larger cap. Only meshes
// whose first 1024 rings hold less than half the vertices try it (a single
// source on a large mesh: configs 4 and 5); the others take the plain launch.
namespace {

std::atomic<int> g_zero_levels{-1};  // -1: from GH_ZERO_LEVELS on first use (default off)

// den of every reachable vertex (k_den's expression on the mesh's arrays: the
// rows a truncated launch skips are the ones that must give +0)
__global__ void k_den_nonpositive(const double* __restrict__ area, const double* __restrict__ wsum,
                                  const int32_t* __restrict__ level, double t, int64_t nv, int32_t* __restrict__ flag) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const double den = area[v] + t * wsum[v];
    // finite and positive: then every weight of the row is finite too (den = A + t * their sum)
    if (level[v] >= 0 && !(den > 0.0 && den < INFINITY)) *flag = 1;
  }
}

// largest level below `cap` with a nonzero value in sweep buffer `parity` (warp per chunk)
__global__ void k_nonzero_front(const double* __restrict__ ubuf, const int32_t* __restrict__ chunk_level,
                                int64_t nchunks, int32_t cap, uint32_t parity, int32_t* __restrict__ front) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int32_t best = -1;
  for (int64_t c = w0; c < nchunks; c += nw) {
    const int32_t lv = chunk_level[c];
    if (lv >= cap || lv <= best) continue;
    const bool nz = __double_as_longlong(ubuf[gh::uidx((uint32_t)(c * 32 + lane), parity)]) != 0;
    if (__any_sync(0xffffffffu, nz)) best = lv;
  }
  if (lane == 0 && best >= 0) atomicMax(front, best);
}

// uidx ranges (in doubles) holding both parities of the rows of levels [0, cap): the even and the odd half
void capped_ranges(const Band& b, int32_t cap, int64_t off[2], int64_t len[2]) {
  for (int h = 0; h < 2; ++h) {
    off[h] = len[h] = 0;
    int32_t top = cap - 1;
    if ((top & 1) != h) --top;
    if (top < h) continue;
    const int64_t r0 = b.h_pstart[h], r1 = ((int64_t)b.h_pend[top] + 31) & ~int64_t(31);
    off[h] = 2 * r0;
    len[h] = 2 * (r1 - r0);
  }
}

}  // namespace

void set_zero_level_truncation(bool on) { g_zero_levels.store(on ? 1 : 0); }
bool zero_level_truncation() {
  int v = g_zero_levels.load();
  if (v < 0) {
    const char* e = getenv("GH_ZERO_LEVELS");  // off unless asked for: by default every update the reference runs is run
    v = (e && atoi(e) != 0) ? 1 : 0;
    g_zero_levels.store(v);
  }
  return v != 0;
}

namespace {

// first cap tried (one sweep carries the heat ~500-900 rings before it
// underflows) and the least margin between the front and the next cap;
// GH_ZERO_LEVELS_FIRST / GH_ZERO_LEVELS_MARGIN shrink them so tests reach the redo paths
int32_t cap_first() {
  const char* e = getenv("GH_ZERO_LEVELS_FIRST");
  return e && atoi(e) > 1 ? atoi(e) : 1024;
}
int32_t margin_min() {
  const char* e = getenv("GH_ZERO_LEVELS_MARGIN");
  return e && atoi(e) > 0 ? atoi(e) : 160;
}

// sweeps in the next launch: short launches first (the front moves fastest
// early: it advances like sqrt(sweeps)), then half of what is done so far, at
// least 256; always even unless it is the last one
int32_t next_group(int32_t done, int32_t sweeps) {
  static const int32_t plan[] = {2, 14, 48, 192};
  int32_t acc = 0, k = std::max(256, done / 2);
  for (int32_t p : plan) {
    if (done == acc) {
      k = p;
      break;
    }
    acc += p;
  }
  k = std::min(k, sweeps - done);
  if (k < sweeps - done && (k & 1)) ++k;
  // a short tail joins this launch
  if (sweeps - done - k < k / 2) k = sweeps - done;
  return k;
}

double diffuse_truncated_dev(gh_levels* L, double t, int32_t sweeps) {
  gh_mesh* m = L->mesh;
  cudaStream_t s = m->stream;
  Band& b = L->main;
  std::vector<Band*> one{&b};
  bands_prepare(L, one, t, nullptr);
  Scratch<int32_t> flags(2, s);  // [0] top level nonzero, [1] front
  const auto rows_below = [&](int32_t cap) { return (int64_t)L->h_offsets[std::min(cap, L->nlev)]; };
  const auto dense_enough = [&](int32_t cap) { return cap >= L->nlev || 2 * rows_below(cap) > (int64_t)L->nreach; };
  EventTimer span(s);
  span.start();
  const int32_t mmin = margin_min();
  const bool trace = getenv("GH_ZERO_LEVELS_TRACE") != nullptr;  // per-launch lines on stderr (tuning)
  int32_t done = 0, cap = cap_first(), front = -1, margin = mmin, last_k = 0;
  L->last_launches = L->last_retries = 0;
  L->last_row_updates = 0;
  // the band covers levels [0, b.le) (bfs_build lays out the first rings only
  // on meshes like this one); a cap past it rebuilds the band with more levels
  // and carries the state over through u_orig
  const auto extend = [&](int32_t le) {
    if (b.le >= std::min(le, L->nlev)) return;
    const bool carry = done > 0;
    if (carry) {
      k_scatter<<<grid_for(b.own_rows), B, 0, s>>>(b.perm.p, b.ubuf, 1u, b.own_rows, L->u_orig.p);
      GH_LAUNCH_CHECK();
      m->launches++;
    }
    main_layout_ensure(L, le);
    bands_prepare(L, one, t, carry ? L->u_orig.p : nullptr);
  };
  while (done < sweeps) {
    if (dense_enough(cap)) {
      extend(L->nlev);
      // the rest in one plain launch over every level (it continues from the
      // state in parity buffer 1; the levels never run so far hold zeros)
      const int32_t k = sweeps - done;
      // (counters: earlier launches, also undone ones, left theirs)
      GH_CUDA(cudaMemsetAsync(b.rows_done, 0, sizeof(unsigned long long) * b.nlev, s));
      GH_CUDA(cudaMemsetAsync(b.stalled, 0, sizeof(int32_t), s));
      bands_launch(L, one, t, k, nullptr, 0, nullptr, false);
      L->last_launches++;
      L->last_row_updates += (uint64_t)L->nreach * (uint64_t)k;
      L->last_active_levels = L->nlev;
      last_k = k;
      done = sweeps;
      break;
    }
    const int32_t k = next_group(done, sweeps);
    if (cap > b.le) extend((int32_t)std::min<int64_t>(L->nlev, std::max<int64_t>(2 * (int64_t)b.le, (int64_t)cap + cap / 2)));
    // the rows this launch may write, saved for a redo
    int64_t off[2], len[2];
    capped_ranges(b, cap, off, len);
    Scratch<double> saved((size_t)(len[0] + len[1]), s);
    GH_CUDA(cudaMemcpyAsync(saved.p, b.ubuf + off[0], sizeof(double) * len[0], cudaMemcpyDeviceToDevice, s));
    GH_CUDA(cudaMemcpyAsync(saved.p + len[0], b.ubuf + off[1], sizeof(double) * len[1], cudaMemcpyDeviceToDevice, s));
    GH_CUDA(cudaMemsetAsync(b.rows_done, 0, sizeof(unsigned long long) * b.nlev, s));
    GH_CUDA(cudaMemsetAsync(b.rows_done + cap, 0xff, sizeof(unsigned long long), s));  // level `cap`: done for every sweep
    GH_CUDA(cudaMemsetAsync(b.stalled, 0, sizeof(int32_t), s));
    GH_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int32_t), s));
    GH_CUDA(cudaMemsetAsync(flags.p + 1, 0xff, sizeof(int32_t), s));
    const double launch_ms = bands_launch(L, one, t, k, nullptr, cap, flags.p, false);
    L->last_launches++;
    L->last_row_updates += (uint64_t)rows_below(cap) * (uint64_t)k;
    k_nonzero_front<<<grid_for(std::min<int64_t>((int64_t)b.own_chunks * 32, 1 << 22)), B, 0, s>>>(
        b.ubuf, b.chunk_level.p, b.own_chunks, cap, (uint32_t)((k - 1) & 1), flags.p + 1);
    GH_LAUNCH_CHECK();
    m->launches++;
    int32_t h[2];
    GH_CUDA(cudaMemcpyAsync(h, flags.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    GH_CUDA(cudaStreamSynchronize(s));
    if (trace)
      fprintf(stderr, "zero_levels: sweeps [%d, %d) cap %d rows %lld front %d flagged %d %.3f ms\n", done, done + k, cap,
              (long long)rows_below(cap), h[1], h[0], launch_ms);
    if (h[0]) {
      // the top level saw a nonzero value: level `cap` would have too. Undo, widen, redo.
      GH_CUDA(cudaMemcpyAsync(b.ubuf + off[0], saved.p, sizeof(double) * len[0], cudaMemcpyDeviceToDevice, s));
      GH_CUDA(cudaMemcpyAsync(b.ubuf + off[1], saved.p + len[0], sizeof(double) * len[1], cudaMemcpyDeviceToDevice, s));
      L->last_retries++;
      margin *= 2;
      cap = done == 0 ? (cap > L->nlev / 2 ? L->nlev : 2 * cap) : std::min<int64_t>(L->nlev, (int64_t)cap + margin);
      continue;
    }
    L->last_active_levels = cap;
    const int32_t grown = front >= 0 ? std::max(0, h[1] - front) : 0;
    front = h[1];
    done += k;
    if (done < sweeps) {
      // margin for the next launch: the front advances like sqrt(sweeps)
      // (diffusively), so this launch's growth scaled by the ratio of the
      // launches' sqrt-spans predicts the next one's; 1.5 x that + 32, at
      // least margin_min() levels
      const int32_t kn = next_group(done, sweeps);
      const double span = std::sqrt((double)done) - std::sqrt((double)(done - k));
      const double next_span = std::sqrt((double)(done + kn)) - std::sqrt((double)done);
      const double scaled = 1.5 * (double)grown * next_span / span + 32.0;
      margin = std::max<int32_t>(mmin, (int32_t)std::min<double>(scaled, 1e9));
      cap = (int32_t)std::min<int64_t>(L->nlev, std::max<int64_t>(cap, (int64_t)front + 1 + margin));
    }
    last_k = k;
  }
  span.stop();
  const double ms = span.ms();
  k_scatter<<<grid_for(b.own_rows), B, 0, s>>>(b.perm.p, b.ubuf, (uint32_t)((last_k - 1) & 1), b.own_rows, L->u_orig.p);
  GH_LAUNCH_CHECK();
  m->launches++;
  return ms;
}

}  // namespace

double diffuse_dev(gh_levels* L, double t, int32_t sweeps, const double* d_initial, double* d_snap) {
  std::vector<Band*> one{&L->main};
  gh_mesh* m = L->mesh;
  // zero-level truncation: from u0 only (a warm start may be nonzero anywhere),
  // no snapshots, a mesh whose first rings hold a minority of the vertices,
  // and every den finite and > 0 (w * 0 must be a zero and 0 / den must be +0)
  bool truncate = zero_level_truncation() && !d_initial && !d_snap && sweeps >= 2 && t > 0.0 && L->nreach > 0 &&
                  L->nlev > cap_first() && 2 * (int64_t)L->h_offsets[cap_first()] <= (int64_t)L->nreach &&
                  !getenv("GH_SWEEP_GROUP") && (int64_t)L->nlev + 2 * (int64_t)sweeps < 0x7fffffffLL;
  if (truncate) {
    if (L->den_positive < 0 || L->den_positive_t != t) {
      Scratch<int32_t> flag(1, m->stream);
      GH_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int32_t), m->stream));
      k_den_nonpositive<<<grid_for(m->nv), B, 0, m->stream>>>(m->vertex_area.p, m->vertex_weight_sum.p, L->level.p, t,
                                                              m->nv, flag.p);
      GH_LAUNCH_CHECK();
      m->launches++;
      L->den_positive = read_scalar(flag.p, m->stream) ? 0 : 1;
      L->den_positive_t = t;
    }
    truncate = L->den_positive == 1;
  }
  if (!truncate) {
    main_layout_ensure(L, L->nlev);  // the plain launch runs every level
    const double ms = diffuse_bands_dev(L, one, t, sweeps, d_initial, d_snap);
    L->last_active_levels = L->nlev;
    L->last_launches = sweeps > 0 && L->nreach > 0 ? 1 : 0;
    L->last_retries = 0;
    L->last_row_updates = (uint64_t)L->nreach * (uint64_t)std::max(sweeps, 0);
    return ms;
  }
  k_init_orig<<<grid_for(m->nv), B, 0, m->stream>>>(L->level.p, nullptr, m->nv, L->u_orig.p);
  GH_LAUNCH_CHECK();
  m->launches++;
  const double ms = diffuse_truncated_dev(L, t, sweeps);
  L->u_valid = 1;
  L->u_sweeps = sweeps;
  return ms;
}

double diffuse_bands_dev(gh_levels* L, std::vector<Band*>& bands, double t, int32_t sweeps, const double* d_initial,
                         double* d_snap) {
  gh_mesh* m = L->mesh;
  cudaStream_t s = m->stream;
  if (sweeps < 0) fail(GH_ERR_INVALID, "DiffusionConfig: sweeps must be >= 0");
  // the pipeline's step index tau < nlev + 2 * sweeps is an int32
  if ((int64_t)L->nlev + 2 * (int64_t)sweeps >= 0x7fffffffLL)
    fail(GH_ERR_INVALID, "gs_diffuse: sweeps must be below (2^31 - levels) / 2 for the sweep pipeline");
  if (!(t > 0.0)) fail(GH_ERR_INVALID, "gs_diffuse: t must be positive");
  k_init_orig<<<grid_for(m->nv), B, 0, s>>>(L->level.p, d_initial, m->nv, L->u_orig.p);
  GH_LAUNCH_CHECK();
  m->launches++;
  double ms = 0.0;
  if (sweeps > 0 && L->nreach > 0) {
    bands_prepare(L, bands, t, d_initial);
    ms = bands_launch(L, bands, t, sweeps, d_snap);
  }
  L->u_valid = 1;
  L->u_sweeps = sweeps;
  return ms;
}

void band_own_u(const Band* b, int32_t sweeps, double* d_u, cudaStream_t s) {
  if (!b->own_rows) return;
  k_scatter<<<grid_for(b->own_rows), B, 0, s>>>(b->perm.p, b->ubuf, (uint32_t)((sweeps - 1) & 1), b->own_rows, d_u);
  GH_LAUNCH_CHECK();
}

void snapshot_to_orig(gh_levels* L, const double* d_snap_sweep, double* d_u) {
  gh_mesh* m = L->mesh;
  const Band& b = L->main;
  if (b.own_rows)
    k_scatter_rows<<<grid_for(b.own_rows), B, 0, m->stream>>>(b.perm.p, d_snap_sweep, b.own_rows, d_u);
  GH_LAUNCH_CHECK();
  m->launches++;
}

void e1_setup_dev(gh_levels* L, int32_t* d_rowof, int32_t* d_vv_row, const double* d_base, double t, int32_t kmax,
                  double* d_sq) {
  gh_mesh* m = L->mesh;
  const Band& b = L->main;
  GH_CUDA(cudaMemsetAsync(d_rowof, 0xff, sizeof(int32_t) * m->nv, m->stream));
  if (b.own_rows) k_rowof<<<grid_for(b.own_rows), B, 0, m->stream>>>(b.perm.p, b.own_rows, d_rowof);
  const int64_t nnz = (int64_t)m->vv_index.n;
  if (nnz) k_vv_row<<<grid_for(nnz), B, 0, m->stream>>>(m->vv_index.p, d_rowof, nnz, d_vv_row);
  GH_LAUNCH_CHECK();
  m->launches += 2;
  if (L->nreach < m->nv) {
    k_residual_fixed<<<grid_for(m->nv), B, 0, m->stream>>>(m->vv_offset.p, m->vv_index.p, m->vv_weight.p,
                                                           m->vertex_area.p, L->level.p, d_base, t, m->nv, kmax, d_sq);
    GH_LAUNCH_CHECK();
    m->launches++;
  }
}

int resident_grid(const void* kernel, int block, int device) {
  int nsm = 0, per_sm = 0;
  GH_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  GH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0));
  return std::max(1, nsm * std::max(1, per_sm));
}

void e1_group_dev(gh_levels* L, const double* d_snap, int32_t k, double t, const int32_t* d_rowof,
                  const int32_t* d_vv_row, double* d_sqr, double* d_sq, double* d_sums) {
  gh_mesh* m = L->mesh;
  const Band& b = L->main;
  if (k <= 0) return;
  const int64_t nseg = seqsum_segments(m->nv);
  Scratch<double> T((size_t)nseg * k, m->stream);
  GH_CUDA(cudaMemsetAsync(T.p, 0, sizeof(double) * nseg * k, m->stream));
  // r^2 in row order: one resident wave grid-striding over the rows, so the
  // rows of neighbouring levels are worked on together, sweep by sweep, and
  // their snapshot values are L2 hits; then gathered into vertex order
  if (b.own_rows) {
    static const int rg_max = resident_grid((const void*)k_residual_rows, 256, m->device);
    const unsigned rg = (unsigned)std::min<int64_t>(rg_max, (b.own_rows + 255) / 256);
    k_residual_rows<<<rg, 256, 0, m->stream>>>(b.perm.p, b.own_rows, m->vv_offset.p, d_vv_row, m->vv_weight.p,
                                               m->vertex_area.p, L->level.p, d_snap, b.nrows, t, k, d_sqr);
    m->launches++;
  }
  k_gather_sq<<<grid_for(m->nv), B, 0, m->stream>>>(d_rowof, d_sqr, b.own_rows, k, m->nv, nseg, d_sq, T.p);
  GH_LAUNCH_CHECK();
  m->launches++;
  sequential_sums_from_T(d_sq, m->nv, m->nv, k, T.p, d_sums, m->stream);
  m->launches += 3;
}

double diffusion_residual_dev(gh_levels* L, const double* d_u, double t) {
  gh_mesh* m = L->mesh;
  // u0 from the level-0 flags: sources are exactly D_0 (diffusion.hpp:38-39)
  Scratch<double> sq(m->nv, m->stream);
  k_residual<<<grid_for(m->nv), B, 0, m->stream>>>(m->vv_offset.p, m->vv_index.p, m->vv_weight.p,
                                                   m->vertex_area.p, L->level.p, d_u, t, m->nv, sq.p);
  GH_LAUNCH_CHECK();
  m->launches++;
  // sqrt(deterministic_sum(sq)) (diffusion.hpp:48): the left-to-right sum, bit for bit
  static const bool prof = getenv("GH_E1_PROFILE") != nullptr;  // stage times on stderr (experiments)
  if (!prof) return std::sqrt(sequential_sum_nonneg(sq.p, m->nv, m->stream, &m->launches));
  EventTimer ts(m->stream);
  ts.start();
  const double sum = sequential_sum_nonneg(sq.p, m->nv, m->stream, &m->launches);
  ts.stop();
  fprintf(stderr, "e1_sum_ms %.4f\n", ts.ms());
  return std::sqrt(sum);
}

}  // namespace gh
