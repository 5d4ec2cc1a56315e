// Bit-exact left-to-right sums of non-negative doubles on the device.
//
// The reference accumulates global sums sequentially (`double s = 0.0;
// for (x : terms) s += x;`, e.g. average_edge_length, mesh.hpp:289-293, and
// deterministic_sum, parallel.hpp:50-54). A tree sum is reproducible but
// rounds differently. For non-negative terms the sequential result can be
// reproduced exactly in parallel: while the running sum s stays inside one
// binade [2^e, 2^(e+1)) every partial sum is a multiple of u = 2^(e-52), and
// fl(s + x) = s + rint(x / u) * u unless x / u has fractional part exactly
// 1/2 (a tie, whose rounding depends on the parity of s / u) or the addition
// leaves the binade. So, with 1024-term segments:
//   1. the first K terms are summed sequentially (one block);
//   2. a tree prefix over the segment sums bounds the running sum at the
//      start of every segment (relative error <= (n + 2^11) 2^-52), giving at
//      most two candidate binades per segment; for each, the segment's
//      sum(rint(x / u)) and a flag (a tie, or a term >= 2^e) are recorded;
//   3. one block walks the segments 1024 at a time: every thread takes a
//      segment's integer sum for the current binade, a block scan finds the
//      first segment that is flagged, has no candidate for that binade, or
//      would carry s out of it; the segments before it are added exactly as
//      integers, that segment is added term by term in double (exactly the
//      reference's operations), and the walk goes on from the next one.
// Ties do not stop the walk: their rounding depends only on the parity of
// the running count, so every term, segment and run of segments is a 2-state
// transducer (quanta added and outgoing parity per incoming parity), and the
// sums are scans of those (see Tx below). The walk stops once per binade
// change; everything else is a parallel pass over the terms plus one scan per
// 1024 segments.

#include <cmath>

#include <cub/device/device_scan.cuh>

#include "gh_internal.cuh"

namespace {

constexpr int kSeg = 1024;         // terms per segment
constexpr int kSeqPrefix = 4096;   // leading terms summed sequentially
constexpr int kWalkThreads = 1024;
constexpr int kSegThreads = 256;
constexpr int kPerThread = kSeg / kSegThreads;
constexpr int kNoBinade = -100000;

// s += x[b..e) in order: the block stages 1024 terms at a time in shared
// memory (coalesced) and thread 0 adds them one by one.
__device__ double block_ordered_add(double s, const double* __restrict__ x, int64_t b, int64_t e, double* sh) {
  for (int64_t c = b; c < e; c += kWalkThreads) {
    const int64_t m = e - c < kWalkThreads ? e - c : kWalkThreads;
    __syncthreads();
    if (threadIdx.x < m) sh[threadIdx.x] = x[c + threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < m; ++k) s += sh[k];
  }
  return s;  // valid in thread 0
}

__global__ void k_seq_block(const double* __restrict__ x, int64_t b, int64_t e, double* __restrict__ acc) {
  __shared__ double sh[kWalkThreads];
  const double s = block_ordered_add(acc[0], x, b, e, sh);
  if (threadIdx.x == 0) acc[0] = s;
}

// The grid of the running sum: u = 2^(e-52) inside binade e; every double
// below 2^-1021 is a multiple of 2^-1074, so 0, the subnormals and binade
// -1022 form one "binade" with u = 2^-1074 (sums there are exact integers).
__device__ __forceinline__ int binade_of(double s) {
  if (s == 0.0) return -1022;
  const int e = ilogb(s);
  return e < -1022 ? -1022 : e;
}
// x * 2^k, exact for k up to 1074 (two finite factors)
__device__ __forceinline__ double scale2(double x, int k) {
  const int k1 = k > 1000 ? 1000 : k;
  return x * ldexp(1.0, k1) * ldexp(1.0, k - k1);
}

// step 2a: per-segment tree sums (any order: they only bound the running sum)
__global__ void __launch_bounds__(kSegThreads) k_seg_sums(const double* __restrict__ x, int64_t b, int64_t n,
                                                          int64_t nseg, double* __restrict__ T) {
  for (int64_t g = blockIdx.x; g < nseg; g += gridDim.x) {
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      const int64_t k = b + g * kSeg + i * kSegThreads + threadIdx.x;
      if (k < n) v += x[k];
    }
    v = ghd::block_sum<kSegThreads>(v);
    if (threadIdx.x == 0) T[g] = v;
    __syncthreads();
  }
}

// Ties: fl(s + x) with x / u = m + 1/2 rounds to the even multiple of u, so
// it adds m + ((A + m) & 1) quanta (A = s / u) and leaves an even count. A
// term's effect on the integer running count is therefore a function of the
// incoming parity only: (q(p), out(p)) for p in {0, 1}, with q the quanta
// added and out the parity after (a tie: q(p) = m + ((p + m) & 1), out = 0;
// else q = rint(x / u), out = p ^ (q & 1)). These 2-state transducers compose
// associatively, so a segment (and a run of segments) reduces to one, and the
// walk scans them in parallel: ties never stop it, only a change of binade.
// saturating non-negative int64 sums (cap 2^62: a saturated count is past any binade)
constexpr unsigned long long kCap = 1ull << 62;
__device__ __forceinline__ unsigned long long sat_add(unsigned long long a, unsigned long long b) {
  const unsigned long long c = a + b;  // both <= 2^62: no wrap
  return c < kCap ? c : kCap;
}

struct Tx {
  unsigned long long q0, q1;  // quanta added for incoming parity 0 / 1 (saturating at 2^62)
  uint32_t o;                 // bit p: outgoing parity for incoming parity p
};
__device__ __forceinline__ Tx tx_identity() { return Tx{0ull, 0ull, 2u}; }
// a then b
__device__ __forceinline__ Tx tx_then(const Tx& a, const Tx& b) {
  const uint32_t a0 = a.o & 1u, a1 = (a.o >> 1) & 1u;
  Tx r;
  r.q0 = sat_add(a.q0, a0 ? b.q1 : b.q0);
  r.q1 = sat_add(a.q1, a1 ? b.q1 : b.q0);
  r.o = ((b.o >> a0) & 1u) | (((b.o >> a1) & 1u) << 1);
  return r;
}
__device__ __forceinline__ Tx tx_shfl_down(const Tx& t, int d) {
  return Tx{__shfl_down_sync(0xffffffffu, t.q0, d), __shfl_down_sync(0xffffffffu, t.q1, d),
            __shfl_down_sync(0xffffffffu, t.o, d)};
}
__device__ __forceinline__ Tx tx_shfl_up(const Tx& t, int d) {
  return Tx{__shfl_up_sync(0xffffffffu, t.q0, d), __shfl_up_sync(0xffffffffu, t.q1, d),
            __shfl_up_sync(0xffffffffu, t.o, d)};
}
// the transducer of term x in binade e; *flag when x >= 2^e (leaves the binade)
__device__ __forceinline__ Tx tx_term(double x, int e, double lim, bool& flag) {
  if (x >= lim) {
    flag = true;
    return tx_identity();
  }
  const double y = scale2(x, 52 - e);  // exact
  const double m = floor(y);
  const unsigned long long mi = (unsigned long long)m;
  if (y - m == 0.5) {
    const unsigned long long odd = mi & 1ull;
    return Tx{mi + odd, mi + (odd ^ 1ull), 0u};
  }
  const unsigned long long q = (unsigned long long)rint(y);
  const uint32_t b = (uint32_t)(q & 1ull);
  return Tx{q, q, b | ((1u ^ b) << 1)};
}

// step 2b: candidate binades from the bounded prefix, then per candidate the
// segment's transducer and a flag (a term that leaves the binade). Thread t
// takes the 4 consecutive terms 4t .. 4t+3 of the segment.
__global__ void __launch_bounds__(kSegThreads) k_seg_q(const double* __restrict__ x, int64_t b, int64_t n, int64_t nseg,
                                                       const double* __restrict__ P, const double* __restrict__ acc,
                                                       double rel, int32_t* __restrict__ elo,
                                                       Tx* __restrict__ Q, int32_t* __restrict__ F) {
  __shared__ Tx sq[kSegThreads / 32][2];
  __shared__ int32_t sf[kSegThreads / 32][2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t g = blockIdx.x; g < nseg; g += gridDim.x) {
    const double pre = acc[0] + P[g];  // ~ running sum before segment g
    const double lo = pre * (1.0 - rel);  // at most the running sum (terms >= 0)
    const int e0 = isfinite(pre) ? binade_of(lo > 0.0 ? lo : 0.0) : kNoBinade;
    const bool ok = e0 != kNoBinade && e0 + 2 < 1023;
    double xv[kPerThread];
    bool in[kPerThread];
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      const int64_t k = b + g * kSeg + kPerThread * threadIdx.x + i;
      in[i] = k < n;
      xv[i] = in[i] ? x[k] : 0.0;
    }
    for (int c = 0; c < 2; ++c) {
      const int e = e0 + c;
      const double lim = ok ? ldexp(1.0, e + (e == -1022 ? 1 : 0)) : 0.0;  // the lowest "binade" ends at 2^-1021
      Tx t = tx_identity();
      bool flag = !ok;
      if (ok) {
#pragma unroll
        for (int i = 0; i < kPerThread; ++i)
          if (in[i]) t = tx_then(t, tx_term(xv[i], e, lim, flag));
      }
      // ordered warp reduction: lane l composes with lanes above it
      for (int o = 1; o < 32; o <<= 1) {
        const Tx up = tx_shfl_down(t, o);
        if ((lane & (2 * o - 1)) == 0) t = tx_then(t, up);
      }
      const unsigned any = __ballot_sync(0xffffffffu, flag);
      if (lane == 0) {
        sq[w][c] = t;
        sf[w][c] = any ? 1 : 0;
      }
    }
    __syncthreads();
    if (threadIdx.x < 2) {
      Tx tq = tx_identity();
      int32_t tf = 0;
      for (int v = 0; v < kSegThreads / 32; ++v) {
        tq = tx_then(tq, sq[v][threadIdx.x]);
        tf |= sf[v][threadIdx.x];
      }
      Q[2 * g + threadIdx.x] = tq;
      F[2 * g + threadIdx.x] = tf;
      if (threadIdx.x == 0) elo[g] = ok ? e0 : kNoBinade;
    }
    __syncthreads();
  }
}

// block-wide inclusive scan of transducers in thread order
__device__ Tx block_scan_tx(Tx v, Tx* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const Tx t = tx_shfl_up(v, o);
    if (lane >= o) v = tx_then(t, v);
  }
  __syncthreads();
  if (lane == 31) wsum[w] = v;
  __syncthreads();
  if (w == 0) {
    Tx a = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const Tx t = tx_shfl_up(a, o);
      if (lane >= o) a = tx_then(t, a);
    }
    wsum[lane] = a;
  }
  __syncthreads();
  return w ? tx_then(wsum[w - 1], v) : v;
}

// step 3: one block of 1024 threads
__global__ void __launch_bounds__(kWalkThreads) k_walk(const double* __restrict__ x, int64_t b, int64_t n,
                                                       int64_t nseg, const int32_t* __restrict__ elo,
                                                       const Tx* __restrict__ Q, const int32_t* __restrict__ F,
                                                       double* __restrict__ acc) {
  __shared__ double sh[kWalkThreads];
  __shared__ Tx wsum[32];
  __shared__ double s_sh;
  __shared__ int64_t stop_at;
  __shared__ unsigned long long cum_before;
  double s = acc[0];
  int64_t g = 0;
  const unsigned long long top = 1ull << 53;
  while (g < nseg) {
    if (threadIdx.x == 0) s_sh = s;
    __syncthreads();
    const double sc = s_sh;
    if (sc == INFINITY) break;  // inf + (x >= 0) stays inf
    // the current binade (none if s is not finite: term by term)
    const bool has = isfinite(sc);
    const int e = has ? binade_of(sc) : kNoBinade;
    const double u = has ? ldexp(1.0, e - 52) : 0.0;
    const unsigned long long A = has ? (unsigned long long)scale2(sc, 52 - e) : 0;  // s / u, exact
    const uint32_t p0 = (uint32_t)(A & 1ull);
    const int64_t gi = g + threadIdx.x;
    bool simple = false;
    Tx q = tx_identity();
    if (gi < nseg && has) {
      const int c = e - elo[gi];
      if (elo[gi] != kNoBinade && (c == 0 || c == 1) && !F[2 * gi + c]) {
        simple = true;
        q = Q[2 * gi + c];
      }
    }
    const Tx pre = block_scan_tx(q, wsum);  // inclusive
    const unsigned long long cum = p0 ? pre.q1 : pre.q0;
    const bool stop = gi < nseg && (!simple || A + cum >= top);
    if (threadIdx.x == 0) stop_at = INT64_MAX;
    __syncthreads();
    if (stop) atomicMin(reinterpret_cast<unsigned long long*>(&stop_at), (unsigned long long)gi);
    __syncthreads();
    const int64_t sa = stop_at;
    // exact integer sum of the simple segments before the stop (or the whole batch)
    const int64_t last = sa == INT64_MAX ? (nseg < g + kWalkThreads ? nseg : g + kWalkThreads) - 1 : sa - 1;
    if (threadIdx.x == 0) cum_before = 0;
    __syncthreads();
    if (last >= g && gi == last) cum_before = cum;
    __syncthreads();
    if (threadIdx.x == 0 && has) s = (double)(A + cum_before) * u;  // a multiple of u below 2^(e+1): exact
    if (sa == INT64_MAX) {
      g = last + 1;
      continue;
    }
    const int64_t kb = b + sa * kSeg;
    s = block_ordered_add(s, x, kb, kb + kSeg < n ? kb + kSeg : n, sh);  // the reference's own additions
    g = sa + 1;
  }
  if (threadIdx.x == 0) acc[0] = s;
}

__global__ void k_any_negative(const double* __restrict__ x, int64_t n, int32_t* __restrict__ flag) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    if (!(x[k] >= 0.0)) *flag = 1;  // negative, -0.0 is fine; NaN also takes the ordered path
}

}  // namespace

namespace gh {

double sequential_sum_nonneg(const double* d_x, int64_t n, cudaStream_t s, int* launches) {
  if (n == 0) return 0.0;
  Scratch<double> acc(1, s);
  GH_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(double), s));
  const int64_t K = n < kSeqPrefix ? n : kSeqPrefix;
  k_seq_block<<<1, kWalkThreads, 0, s>>>(d_x, 0, K, acc.p);
  int nl = 1;
  if (n > K) {
    const int64_t nseg = (n - K + kSeg - 1) / kSeg;
    Scratch<double> T(nseg, s), P(nseg, s);
    Scratch<int32_t> elo(nseg, s), F(2 * nseg, s);
    Scratch<Tx> Q(2 * nseg, s);
    const unsigned grid = (unsigned)std::min<int64_t>(nseg, 148 * 32);
    k_seg_sums<<<grid, kSegThreads, 0, s>>>(d_x, K, n, nseg, T.p);
    size_t tmp_bytes = 0;
    GH_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, T.p, P.p, (int)nseg, s));
    {
      Scratch<unsigned char> tmp(tmp_bytes, s);
      GH_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, T.p, P.p, (int)nseg, s));
    }
    // |sequential - exact| and |scan - exact| are both <= (n + 2^11) 2^-53 of the sum
    const double rel = (double)(n + 4096) * 2.3e-16;
    k_seg_q<<<grid, kSegThreads, 0, s>>>(d_x, K, n, nseg, P.p, acc.p, rel, elo.p, Q.p, F.p);
    k_walk<<<1, kWalkThreads, 0, s>>>(d_x, K, n, nseg, elo.p, Q.p, F.p, acc.p);
    GH_LAUNCH_CHECK();
    nl += 4;
  }
  double h = 0.0;
  GH_CUDA(cudaMemcpyAsync(&h, acc.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
  if (launches) *launches += nl;
  return h;
}

double deterministic_sum_dev(const double* d_x, int64_t n, cudaStream_t s) {
  if (n == 0) return 0.0;
  Scratch<int32_t> neg(1, s);
  GH_CUDA(cudaMemsetAsync(neg.p, 0, sizeof(int32_t), s));
  k_any_negative<<<grid_for(n), kBlock, 0, s>>>(d_x, n, neg.p);
  GH_LAUNCH_CHECK();
  int32_t h = 0;
  GH_CUDA(cudaMemcpyAsync(&h, neg.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
  if (!h) return sequential_sum_nonneg(d_x, n, s, nullptr);
  Scratch<double> acc(1, s);
  GH_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(double), s));
  k_seq_block<<<1, kWalkThreads, 0, s>>>(d_x, 0, n, acc.p);
  GH_LAUNCH_CHECK();
  double out = 0.0;
  GH_CUDA(cudaMemcpyAsync(&out, acc.p, sizeof(out), cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
  return out;
}

}  // namespace gh
