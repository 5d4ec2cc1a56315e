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
//  * per block, a producer warp streams the step's chunk share (den, deg,
//    columns, weights: ~86 of the ~100 B per update) HBM -> shared memory
//    with cp.async.bulk + mbarrier complete_tx into a ring of tiles, running
//    ahead across steps (the CSR is read-only);
//  * 8 consumer warps each take 2 chunks of a tile, gather the neighbour u
//    values from L2 (ld.global.cg) with all 12-16 gathers in flight, store u;
//  * no grid barrier: a chunk of level L at step tau waits (acquire) on
//    per-level row counters of L-1, L, L+1; blocks publish their rows per
//    level after each step (release). Each task depends only on earlier
//    steps and all blocks are co-resident, so the schedule cannot deadlock.

#include <algorithm>

#include "gh_internal.cuh"

namespace {

constexpr int B = gh::kBlock;
constexpr int kMaxSmemLevels = 6 * 1024;  // pstart/pend tables in shared memory (48 KB)
constexpr int kUnroll = 8;                  // rows up to this valence take the unrolled path

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
    ubuf[r] = x;
    ubuf[nrows + r] = x;
  }
}

__global__ void k_init_orig(const int32_t* __restrict__ level, const double* __restrict__ initial, int64_t nv,
                            double* __restrict__ u) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x)
    u[v] = initial ? initial[v] : (level[v] == 0 ? 1.0 : 0.0);
}

__global__ void k_scatter(const int32_t* __restrict__ perm, const double* __restrict__ src, int64_t nrows,
                          double* __restrict__ u) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = perm[r];
    if (v >= 0) u[v] = src[r];
  }
}

// ---------------------------------------------------------------- bulk-staged schedule
// Same step/barrier schedule, but the streamed operands of each 32-row chunk
// (SELL columns + weights, den, deg: ~86 B of the ~100 B per update) are moved
// HBM -> shared memory by the bulk-copy engine (cp.async.bulk + mbarrier
// complete_tx), issued by one producer warp into a ring of chunk slots, while
// kConsumerWarps warps consume chunks: read the row from shared memory, gather
// the 6-ish neighbour u values (L2), and store u. The DRAM stream no longer
// waits behind the gather latency of the warps, so many more bytes are in
// flight per SM. Rows are still summed in the reference's order (bitwise).
constexpr int kConsumerWarps = 8;
constexpr int kChunksPerWarp = 2;                            // chunks a consumer warp has in flight
constexpr int kTileChunks = kConsumerWarps * kChunksPerWarp;  // chunks per ring slot
constexpr int kTmaThreads = 32 * (kConsumerWarps + 1);

struct TmaArgs {
  const int32_t* pstart;
  const int32_t* pend;
  const int32_t* chunk_level;
  const int64_t* chunk_ptr;
  const uint16_t* deg;
  const int32_t* col;
  const double* wt;
  const double* den;
  double* ubuf;
  int64_t nrows;
  int32_t nlev, sweeps;
  int32_t wcap;      // widest chunk (neighbours per row) a slot holds
  int32_t nslots;    // ring slots per block
  int32_t slot_bytes;
  int32_t table_in_smem;
  unsigned long long* rows_done;  // per level: rows finished over all sweeps (zeroed per launch)
  double t;
};

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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// contiguous share of the step's chunk range [c0, c1) for block b
__device__ __forceinline__ void block_share(int64_t c0, int64_t c1, int64_t b, int64_t nb, int64_t& cb,
                                            int64_t& ce) {
  const int64_t n = c1 - c0, q = n / nb, rem = n % nb;
  cb = c0 + b * q + (b < rem ? b : rem);
  ce = cb + q + (b < rem ? 1 : 0);
}

__device__ __forceinline__ bool step_range(const TmaArgs& a, const int32_t* pstart, const int32_t* pend, int64_t tau,
                                           int64_t& rb, int64_t& re) {
  int64_t lhi = tau < a.nlev - 1 ? tau : a.nlev - 1;
  if ((lhi ^ tau) & 1) --lhi;
  int64_t llo = tau - 2 * (int64_t)(a.sweeps - 1);
  if (llo < 0) llo = tau & 1;
  if (llo > lhi) return false;
  rb = pstart[llo];
  re = pend[lhi];
  return true;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int32_t ld_acquire_gpu(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// slot layout: header 256 B (int32: chunk offsets [0..kTileChunks], fits [31], chunk levels [32..])
//              | den kTileChunks x 256 B | deg kTileChunks x 64 B | columns | weights
constexpr int kHdr = 256;
constexpr int kDenOff = kHdr;
constexpr int kDegOff = kDenOff + kTileChunks * 256;
constexpr int kColOff = kDegOff + kTileChunks * 64;

__global__ void __launch_bounds__(kTmaThreads, 2) k_diffuse_tma(TmaArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + a.nslots;
  int32_t* sh_pend = reinterpret_cast<int32_t*>(empty + a.nslots);
  int32_t* sh_pstart = sh_pend + a.nlev;
  const size_t table_bytes = a.table_in_smem ? ((2 * sizeof(int32_t) * a.nlev + 127) & ~size_t(127)) : 0;
  unsigned char* slots = reinterpret_cast<unsigned char*>(empty + a.nslots) + table_bytes;
  slots = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(slots) + 127) & ~uintptr_t(127));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.nslots; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int32_t* pend = a.pend;
  const int32_t* pstart = a.pstart;
  if (a.table_in_smem) {
    for (int i = threadIdx.x; i < a.nlev; i += blockDim.x) {
      sh_pend[i] = a.pend[i];
      sh_pstart[i] = a.pstart[i];
    }
    pend = sh_pend;
    pstart = sh_pstart;
  }
  __syncthreads();

  const int64_t nb = gridDim.x, b = blockIdx.x;
  const int64_t nsteps = (int64_t)(a.nlev - 1) + 2 * (int64_t)(a.sweeps - 1) + 1;
  const uint32_t col_cap = (uint32_t)kTileChunks * 32u * a.wcap;  // entries
  // ring position: slot index and its use parity advance tile by tile (no 64-bit modulo)
  int slot = 0;
  uint32_t use = 0;
  int64_t issued = 0;

  if (warp == kConsumerWarps) {
    // ---- producer warp: runs ahead across steps, bounded by the ring. Work is a
    // stream of batches of 32 chunks (4 tiles); the chunk pointers and levels
    // of the next batch are loaded while the current batch is issued.
    constexpr int kTilesPerBatch = 32 / kTileChunks;
    int64_t tau = -1, cb = 0, ce = 0, ntile = 0, t0 = -kTilesPerBatch;
    auto advance = [&](int64_t& xtau, int64_t& xcb, int64_t& xce, int64_t& xnt, int64_t& xt0) -> bool {
      xt0 += kTilesPerBatch;
      while (xt0 >= xnt) {
        if (++xtau >= nsteps) return false;
        int64_t rb, re;
        xt0 = 0;
        xnt = 0;
        if (!step_range(a, pstart, pend, xtau, rb, re)) continue;
        block_share(rb >> 5, (re + 31) >> 5, b, nb, xcb, xce);
        xnt = (xce - xcb + kTileChunks - 1) / kTileChunks;
      }
      return true;
    };
    auto load = [&](int64_t xcb, int64_t xce, int64_t xt0, int64_t& p0, int32_t& lv0, int64_t& plast) {
      const int64_t cbase = xcb + xt0 * kTileChunks;
      const int64_t cl = cbase + lane < xce ? cbase + lane : xce;
      p0 = __ldg(a.chunk_ptr + cl);
      lv0 = cbase + lane < xce ? __ldg(a.chunk_level + cl) : 0;
      plast = __ldg(a.chunk_ptr + (cbase + 32 < xce ? cbase + 32 : xce));
    };
    int64_t p0 = 0, p_last = 0;
    int32_t lv0 = 0;
    bool have = advance(tau, cb, ce, ntile, t0);
    if (have) load(cb, ce, t0, p0, lv0, p_last);
    while (have) {
      int64_t ntau = tau, ncb = cb, nce = ce, nnt = ntile, nt0 = t0;
      int64_t np0 = 0, np_last = 0;
      int32_t nlv0 = 0;
      const bool have_next = advance(ntau, ncb, nce, nnt, nt0);
      if (have_next) load(ncb, nce, nt0, np0, nlv0, np_last);
      const int64_t cbase = cb + t0 * kTileChunks;
      for (int j = 0; j < kTilesPerBatch && t0 + j < ntile; ++j) {
        if (issued >= a.nslots) mbar_wait(empty + slot, use ^ 1u);
        const int64_t c0 = cbase + j * kTileChunks;
        const int nch = (int)(ce - c0 < kTileChunks ? ce - c0 : kTileChunks);
        const int64_t base = __shfl_sync(0xffffffffu, p0, j * kTileChunks);
        const int src = j * kTileChunks + (lane <= kTileChunks ? lane : 0);
        int64_t pi = __shfl_sync(0xffffffffu, p0, src < 32 ? src : 31);
        const int32_t li = __shfl_sync(0xffffffffu, lv0, (j * kTileChunks + (lane & (kTileChunks - 1))) & 31);
        if (j * kTileChunks + lane == 32) pi = p_last;
        int32_t* hdr = reinterpret_cast<int32_t*>(slots + (size_t)slot * a.slot_bytes);
        if (lane <= nch) hdr[lane] = (int32_t)(pi - base);
        if (lane < kTileChunks) hdr[32 + lane] = li;
        const int64_t pend_tile = __shfl_sync(0xffffffffu, pi, nch);
        const uint32_t ncol = (uint32_t)(pend_tile - base);
        const bool fits = ncol <= col_cap;
        if (lane == 0) hdr[31] = fits ? 1 : 0;
        __syncwarp();
        if (lane == 0) {
          unsigned char* sb = reinterpret_cast<unsigned char*>(hdr);
          const uint32_t bytes = (uint32_t)nch * (256u + 64u) + (fits ? ncol * 12u : 0u);
          mbar_expect_tx(full + slot, bytes);
          bulk_g2s(sb + kDenOff, a.den + c0 * 32, (uint32_t)nch * 256u, full + slot);
          bulk_g2s(sb + kDegOff, a.deg + c0 * 32, (uint32_t)nch * 64u, full + slot);
          if (fits && ncol) {
            bulk_g2s(sb + kColOff, a.col + base, ncol * 4u, full + slot);
            bulk_g2s(sb + kColOff + col_cap * 4u, a.wt + base, ncol * 8u, full + slot);
          }
        }
        __syncwarp();
        ++issued;
        if (++slot == a.nslots) {
          slot = 0;
          use ^= 1u;
        }
      }
      tau = ntau, cb = ncb, ce = nce, ntile = nnt, t0 = nt0;
      p0 = np0, p_last = np_last, lv0 = nlv0;
      have = have_next;
    }
    return;
  }

  // ---- consumer warps: warp w takes chunk w of every tile. No grid barrier:
  // before a chunk of level L at step tau, the warp waits (acquire) until
  // levels L-1, L, L+1 have completed the sweeps its operands come from
  // (rows_done[X] >= ((tau - X + 1) / 2) * |D_X|); after the step the block
  // publishes its rows per level (release). Every level starts on a chunk
  // boundary, so a chunk holds rows of exactly one level.
  int32_t seen_L = -1, seen_L2 = -1;
  int64_t seen_tau = -1;
  for (int64_t tau = 0; tau < nsteps; ++tau) {
    int64_t rb, re;
    if (!step_range(a, pstart, pend, tau, rb, re)) continue;
    int64_t cb, ce;
    block_share(rb >> 5, (re + 31) >> 5, b, nb, cb, ce);
    const int64_t ntile = (ce - cb + kTileChunks - 1) / kTileChunks;
    if (ntile == 0) continue;
    int32_t lv_first = 0, lv_last = 0;
    if (warp == 0 && lane == 0) {
      lv_first = __ldg(a.chunk_level + cb);
      lv_last = __ldg(a.chunk_level + ce - 1);
    }
    for (int64_t j = 0; j < ntile; ++j) {
      mbar_wait(full + slot, use);
      const unsigned char* sb = slots + (size_t)slot * a.slot_bytes;
      const int32_t* hdr = reinterpret_cast<const int32_t*>(sb);
      const bool fits = hdr[31] != 0;
      // this warp's chunks in the tile: q = warp + kConsumerWarps * i
      int32_t Lq[kChunksPerWarp];
      bool live[kChunksPerWarp];
#pragma unroll
      for (int i = 0; i < kChunksPerWarp; ++i) {
        const int q = warp + kConsumerWarps * i;
        live[i] = cb + j * kTileChunks + q < ce;
        Lq[i] = live[i] ? hdr[32 + q] : -1;
      }
      if (Lq[0] != seen_L || Lq[kChunksPerWarp - 1] != seen_L2 || tau != seen_tau) {
        // operands: wait for levels L-1, L, L+1 of each chunk (lanes 3i..3i+2)
        const int i = lane / 3;
        if (i < kChunksPerWarp && Lq[i] >= 0) {
          const int32_t X = Lq[i] - 1 + lane % 3;
          if (X >= 0 && X < a.nlev) {
            const unsigned long long need =
                (unsigned long long)((tau - X + 1) >> 1) * (unsigned long long)(pend[X] - pstart[X]);
            unsigned ns = 32;
            while (ld_acquire_u64(a.rows_done + X) < need) {
              __nanosleep(ns);
              if (ns < 256) ns <<= 1;
            }
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
      double* cur[kChunksPerWarp];
      const double* prev[kChunksPerWarp];
#pragma unroll
      for (int i = 0; i < kChunksPerWarp; ++i) {
        const int q = warp + kConsumerWarps * i;
        const int64_t c = cb + j * kTileChunks + q;
        const int64_t r = c * 32 + lane;
        on[i] = live[i] && r < pend[Lq[i]];
        const int32_t sweep = (int32_t)((tau - Lq[i]) >> 1);
        cur[i] = a.ubuf + (sweep & 1) * a.nrows;
        prev[i] = a.ubuf + ((sweep & 1) ^ 1) * a.nrows;
        den[i] = reinterpret_cast<const double*>(sb + kDenOff)[q * 32 + lane];
        d[i] = on[i] ? reinterpret_cast<const uint16_t*>(sb + kDegOff)[q * 32 + lane] : 0;
        fast[i] = fits && d[i] <= kUnroll;
        num[i] = 0.0;
      }
      // all gathers of both chunks in flight together
#pragma unroll
      for (int i = 0; i < kChunksPerWarp; ++i) {
        const int32_t* scol = reinterpret_cast<const int32_t*>(sb + kColOff) + hdr[warp + kConsumerWarps * i] + lane;
#pragma unroll
        for (int k = 0; k < kUnroll; ++k)
          if (fast[i] && k < d[i]) {
            const int32_t cc = scol[32 * k];
            v[i][k] = __ldcg((cc < 0 ? cur[i] : prev[i]) + (cc & 0x7fffffff));
          }
      }
#pragma unroll
      for (int i = 0; i < kChunksPerWarp; ++i) {
        const int q = warp + kConsumerWarps * i;
        const int64_t c = cb + j * kTileChunks + q;
        if (fast[i]) {
          const double* swt =
              reinterpret_cast<const double*>(sb + kColOff + (size_t)col_cap * 4u) + hdr[q] + lane;
#pragma unroll
          for (int k = 0; k < kUnroll; ++k)
            if (k < d[i]) num[i] += swt[32 * k] * v[i][k];  // diffusion.hpp:79
        } else if (on[i]) {
          const int64_t q0 = __ldg(a.chunk_ptr + c) + lane;
          for (int32_t k = 0; k < d[i]; ++k) {
            const int32_t cc = __ldg(a.col + q0 + 32 * (int64_t)k);
            const double w = __ldg(a.wt + q0 + 32 * (int64_t)k);
            num[i] += w * __ldcg((cc < 0 ? cur[i] : prev[i]) + (cc & 0x7fffffff));
          }
        }
        if (on[i]) {
          const double u0 = Lq[i] == 0 ? 1.0 : 0.0;
          __stcg(cur[i] + c * 32 + lane, (u0 + a.t * num[i]) / den[i]);  // diffusion.hpp:82
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
        const int64_t lo = cb * 32 > pstart[X] ? cb * 32 : pstart[X];
        const int64_t hi = ce * 32 < pend[X] ? ce * 32 : pend[X];
        if (hi > lo) {
          __threadfence();
          atomicAdd(a.rows_done + X, (unsigned long long)(hi - lo));
        }
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

// r_j = A_j u_j - t * sum theta (u_k - u_j) - u0_j (diffusion.hpp:41-47)
__global__ void k_residual(const int32_t* __restrict__ vv_off, const int32_t* __restrict__ vv_idx,
                           const double* __restrict__ vv_w, const double* __restrict__ va,
                           const int32_t* __restrict__ level, const double* __restrict__ u, double t, int64_t nv,
                           double* __restrict__ part) {
  double s = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nv; j += (int64_t)gridDim.x * blockDim.x) {
    double lap = 0.0;
    const double uj = u[j];
    for (int32_t i = vv_off[j]; i < vv_off[j + 1]; ++i) lap += vv_w[i] * (u[vv_idx[i]] - uj);
    const double r = va[j] * uj - t * lap - (level[j] == 0 ? 1.0 : 0.0);
    s += r * r;
  }
  s = ghd::block_sum<B>(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

}  // namespace

namespace gh {

double diffuse_dev(gh_levels* L, double t, int32_t sweeps, const double* d_initial) {
  gh_mesh* m = L->mesh;
  cudaStream_t s = m->stream;
  const int64_t V = m->nv;
  if (sweeps < 0) fail(GH_ERR_INVALID, "DiffusionConfig: sweeps must be >= 0");
  if (!(t > 0.0)) fail(GH_ERR_INVALID, "gs_diffuse: t must be positive");
  if (L->den_t != t) {
    k_den<<<grid_for(L->nrows), B, 0, s>>>(L->area_r.p, L->wsum_r.p, t, L->nrows, L->den.p);
    GH_LAUNCH_CHECK();
    m->launches++;
    L->den_t = t;
  }
  k_init_orig<<<grid_for(V), B, 0, s>>>(L->level.p, d_initial, V, L->u_orig.p);
  GH_LAUNCH_CHECK();
  m->launches++;
  double ms = 0.0;
  if (sweeps > 0 && L->nreach > 0) {
    k_init_buffers<<<grid_for(L->nrows), B, 0, s>>>(L->perm.p, L->level.p, d_initial, L->nrows, L->ubuf.p);
    GH_LAUNCH_CHECK();
    m->launches++;
    int nsm = 0, per_sm = 0;
    GH_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device));
    EventTimer timer(s);
    {
      // slot = 64 B header + per chunk (den 256 B + deg 64 B + wcap x 32 x 12 B of columns/weights)
      const int32_t wcap = std::min<int32_t>(std::max<int32_t>(L->max_chunk_width, 1), 16);
      const int32_t slot_bytes = ((kColOff + kTileChunks * 32 * wcap * 12) + 127) & ~127;
      const bool table = L->nlev <= kMaxSmemLevels;
      const size_t table_bytes = table ? ((2 * sizeof(int32_t) * L->nlev + 127) & ~size_t(127)) : 0;
      // two blocks per SM with a ring of >= 2 slots each (228 KB per SM, 1 KB reserved per block)
      int32_t nslots = 0;
      for (int per = 2; per >= 1 && nslots < 2; --per) {
        const int64_t budget = 228 * 1024 / per - 1024;
        nslots = (int32_t)std::min<int64_t>(8, (budget - (int64_t)table_bytes - 256) / (slot_bytes + 16));
      }
      if (nslots < 2) nslots = 2;
      const size_t shmem = 16 * (size_t)nslots + table_bytes + 128 + (size_t)nslots * slot_bytes;
      GH_CUDA(cudaFuncSetAttribute((void*)k_diffuse_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem));
      TmaArgs a{L->pstart.p, L->pend.p, L->chunk_level.p, L->chunk_ptr.p, L->deg.p, L->col.p, L->wt.p, L->den.p,
                L->ubuf.p, L->nrows, L->nlev, sweeps, wcap, nslots, slot_bytes, table ? 1 : 0, L->rows_done.p, t};
      GH_CUDA(cudaMemsetAsync(L->rows_done.p, 0, sizeof(unsigned long long) * L->nlev, s));
      GH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_diffuse_tma, kTmaThreads, shmem));
      if (per_sm < 1) fail(GH_ERR_CUDA, "diffusion kernel cannot be resident");
      void* args[] = {&a};
      timer.start();
      GH_CUDA(cudaLaunchCooperativeKernel((void*)k_diffuse_tma, nsm * per_sm, kTmaThreads, args, shmem, s));
      GH_LAUNCH_CHECK();
      timer.stop();
    }
    m->launches++;
    ms = timer.ms();
    const double* result = L->ubuf.p + ((sweeps - 1) & 1) * (int64_t)L->nrows;
    k_scatter<<<grid_for(L->nrows), B, 0, s>>>(L->perm.p, result, L->nrows, L->u_orig.p);
    GH_LAUNCH_CHECK();
    m->launches++;
  }
  L->u_valid = 1;
  L->u_sweeps = sweeps;
  return ms;
}

double diffusion_residual_dev(gh_levels* L, const double* d_u, double t) {
  gh_mesh* m = L->mesh;
  // u0 from the level-0 flags: sources are exactly D_0 (diffusion.hpp:38-39)
  k_residual<<<kReduceGrid, B, 0, m->stream>>>(m->vv_offset.p, m->vv_index.p, m->vv_weight.p, m->vertex_area.p,
                                               L->level.p, d_u, t, m->nv, m->partials.p);
  GH_LAUNCH_CHECK();
  m->launches++;
  reduce_partials(m, m->scalars.p + 3);
  return std::sqrt(read_scalar(m->scalars.p + 3, m->stream));
}

}  // namespace gh
