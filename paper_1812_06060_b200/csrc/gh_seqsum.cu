// Bit-exact left-to-right sums on the device, one or many at a time.
//
// The reference accumulates global sums sequentially (`double s = 0.0;
// for (x : terms) s += x;`, e.g. average_edge_length, mesh.hpp:289-293,
// deterministic_sum, parallel.hpp:50-54, and E1 after every sweep,
// diffusion.hpp:48, 110-117). A tree sum is reproducible but rounds
// differently. For non-negative terms the sequential result can be reproduced
// exactly in parallel: while the running sum s stays inside one binade
// [2^e, 2^(e+1)) every partial sum is a multiple of u = 2^(e-52), and
// fl(s + x) = s + rint(x / u) * u unless x / u has fractional part exactly
// 1/2 (a tie, whose rounding depends on the parity of s / u) or the addition
// leaves the binade. Ties do not break this: a term's effect on the integer
// count s / u is a function of the incoming parity only, so every term,
// segment and run of segments is a 2-state transducer (quanta added and
// outgoing parity per incoming parity; Tx below) and sums of them are scans.
//
// Several sums (count, stride apart) run at once, one block per sum in the
// walk, everything else as fully parallel passes; with 1024-term segments:
//   1. T = each segment's tree sum (any order: only a bound). The E1 path
//      gets T from its residual kernel, for free;
//   2. P = exclusive prefix of T per sum: about the running sum at the start of
//      every segment, so almost always in the binade there (P only chooses the
//      binade to prepare; results never depend on it);
//   3. per segment, its transducer in that binade and a flag (a term >= 2^e,
//      negative or NaN);
//   4. the walk: one block per sum takes 1024 segments per step, each thread
//      one segment's transducer, and a block scan finds the first segment
//      that was prepared for another binade, is flagged,
//      or would carry s out of it; the segments before it are added exactly as
//      integers, that one term by term in double (its nonzero terms, in
//      order: zeros are exact no-ops), and the walk goes on after it. A
//      negative or non-finite running sum (terms of any sign are accepted)
//      stops the walk at every segment, which is then added the same way.

#include <climits>
#include <cmath>

#include "gh_internal.cuh"

namespace {

constexpr int kSeg = 1024;          // terms per segment
constexpr int kWalkThreads = 1024;  // = kSeg: one term per thread when a segment is walked term by term
constexpr int kSegThreads = 256;
constexpr int kPerThread = kSeg / kSegThreads;
constexpr int kNoBinade = -100000;

// s += x[b..e) in order: the block stages terms in shared memory (coalesced)
// and thread 0 adds them one by one.
__device__ double block_ordered_add(double s, const double* __restrict__ x, int64_t b, int64_t e, double* sh) {
  for (int64_t c = b; c < e; c += blockDim.x) {
    const int64_t m = e - c < (int64_t)blockDim.x ? e - c : (int64_t)blockDim.x;
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
// the two factors of 2^(52-e) that scale2 uses
__device__ __forceinline__ void quantum_factors(int e, double& f1, double& f2) {
  const int k = 52 - e, k1 = k > 1000 ? 1000 : k;
  f1 = ldexp(1.0, k1);
  f2 = ldexp(1.0, k - k1);
}

// Ties: fl(s + x) with x / u = m + 1/2 rounds to the even multiple of u, so
// it adds m + ((A + m) & 1) quanta (A = s / u) and leaves an even count: a
// tie's transducer is q(p) = m + ((p + m) & 1), out = 0; any other term's is
// q = rint(x / u), out = p ^ (q & 1). Counts saturate at 2^62 (a saturated
// count is past any binade).
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
// the transducer of term x in binade e; *flag when x >= lim = 2^e (it leaves
// the binade) or x is negative or NaN
// (f1 * f2 = 2^(52-e), split so that both factors are finite: see scale2)
__device__ __forceinline__ Tx tx_term(double x, double f1, double f2, double lim, bool& flag) {
  if (!(x >= 0.0) || x >= lim) {
    flag = true;
    return tx_identity();
  }
  const double y = x * f1 * f2;  // x / u, exact
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

// exclusive block scan of transducers in thread order (NT threads); *total = all of them
template <int NT>
__device__ Tx block_exscan_tx(Tx v, Tx* wsum, Tx* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Tx inc = v;
  for (int o = 1; o < 32; o <<= 1) {
    const Tx t = tx_shfl_up(inc, o);
    if (lane >= o) inc = tx_then(t, inc);
  }
  Tx ex = tx_shfl_up(inc, 1);
  if (lane == 0) ex = tx_identity();
  __syncthreads();
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    constexpr int nw = NT / 32;
    Tx a = lane < nw ? wsum[lane] : tx_identity();
    for (int o = 1; o < 32; o <<= 1) {
      const Tx t = tx_shfl_up(a, o);
      if (lane >= o) a = tx_then(t, a);
    }
    if (lane < nw) wsum[lane] = a;  // inclusive over warps
  }
  __syncthreads();
  *total = wsum[NT / 32 - 1];
  return w ? tx_then(wsum[w - 1], ex) : ex;
}

struct WalkShared {
  Tx wsum[32];
  double sh[kWalkThreads];
  int cnt[kWalkThreads / 32];
  int total;
  unsigned long long cum;
  double x;
  long long stop;
};

// s += one segment's terms in order, exactly as the reference's additions
// (one term per thread, v; zeros past the end). Zero terms are exact no-ops
// (s + 0 = s for every s, signed zeros and NaN included), so the block keeps
// the nonzero terms in order (warp ballots, a prefix over the warps) and
// thread 0 adds just those, one by one: a walked segment is where the running
// sum leaves its binade, often several times in a few terms (E1: ~1000 binade
// changes in ~300 of 8192 segments at config 3), where a block scan per change
// costs more than the additions. s is the same in every thread on return.
__device__ double walk_segment(double s, double v, WalkShared& W) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool nz = !(v == 0.0);
  const unsigned m = __ballot_sync(0xffffffffu, nz);
  if (lane == 0) W.cnt[w] = __popc(m);
  __syncthreads();
  if (w == 0) {  // exclusive prefix over the warps
    const int c = lane < kWalkThreads / 32 ? W.cnt[lane] : 0;
    int inc = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane < kWalkThreads / 32) W.cnt[lane] = inc - c;
    if (lane == 31) W.total = inc;
  }
  __syncthreads();
  if (nz) W.sh[W.cnt[w] + __popc(m & ((1u << lane) - 1u))] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    const int n = W.total;
    for (int k = 0; k < n; ++k) s += W.sh[k];
    W.x = s;
  }
  __syncthreads();
  s = W.x;
  __syncthreads();  // W is reused by the next segment
  return s;
}

// 1. per-segment tree sums T[y * nseg + g] of sum y = blockIdx.y
__global__ void __launch_bounds__(kSegThreads) k_seg_sums(const double* __restrict__ X, int64_t n, int64_t stride,
                                                          int64_t nseg, double* __restrict__ T) {
  const double* __restrict__ x = X + (int64_t)blockIdx.y * stride;
  for (int64_t g = blockIdx.x; g < nseg; g += gridDim.x) {
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      const int64_t k = g * kSeg + i * kSegThreads + threadIdx.x;
      if (k < n) v += x[k];
    }
    v = ghd::block_sum<kSegThreads>(v);
    if (threadIdx.x == 0) T[(int64_t)blockIdx.y * nseg + g] = v;
    __syncthreads();
  }
}

// 2. P = exclusive prefix of T, per sum (one block each)
__global__ void __launch_bounds__(1024) k_seg_scan(const double* __restrict__ T, int64_t nseg, double* __restrict__ P) {
  __shared__ double ws[32];
  __shared__ double carry_sh;
  const double* __restrict__ t = T + (int64_t)blockIdx.x * nseg;
  double* __restrict__ p = P + (int64_t)blockIdx.x * nseg;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double carry = 0.0;
  for (int64_t b = 0; b < nseg; b += 1024) {
    const int64_t g = b + threadIdx.x;
    const double v = g < nseg ? t[g] : 0.0;
    double inc = v;
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    if (w == 0) {
      double a = ws[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, a, o);
        if (lane >= o) a += y;
      }
      ws[lane] = a;
      if (lane == 31) carry_sh = a;
    }
    __syncthreads();
    if (g < nseg) p[g] = carry + (w ? ws[w - 1] : 0.0) + (inc - v);
    carry += carry_sh;
    __syncthreads();
  }
}

// 3. the binade of P (the running sum at the segment's start is within ~n 2^-53
// of P: another binade only for P within that of a power of two, and then the
// walk just takes the segment term by term), the segment's transducer in it
// and a flag. Thread t takes the 4 consecutive terms 4t .. 4t+3; terms below
// half a quantum (E1's far field: zeros and terms far below the running sum)
// are the identity and skipped.
__global__ void __launch_bounds__(kSegThreads) k_seg_q(const double* __restrict__ X, int64_t n, int64_t stride,
                                                       int64_t nseg, const double* __restrict__ P,
                                                       int32_t* __restrict__ elo, Tx* __restrict__ Q,
                                                       int32_t* __restrict__ F) {
  __shared__ Tx sq[kSegThreads / 32];
  __shared__ int32_t sf[kSegThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t y = blockIdx.y;
  const double* __restrict__ x = X + y * stride;
  for (int64_t g = blockIdx.x; g < nseg; g += gridDim.x) {
    const int64_t gy = y * nseg + g;
    const double pre = P[gy];  // ~ the running sum before segment g
    const int e = isfinite(pre) ? binade_of(pre > 0.0 ? pre : 0.0) : kNoBinade;
    const bool ok = e != kNoBinade && e + 1 < 1023;
    double xv[kPerThread];
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      const int64_t k = g * kSeg + kPerThread * threadIdx.x + i;
      xv[i] = k < n ? x[k] : 0.0;
    }
    Tx t = tx_identity();
    bool flag = !ok;
    if (ok) {
      const double lim = ldexp(1.0, e + (e == -1022 ? 1 : 0));  // the lowest "binade" ends at 2^-1021
      const double halfu = e > -1022 ? ldexp(1.0, e - 53) : 0.0;
      double f1, f2;
      quantum_factors(e, f1, f2);
#pragma unroll
      for (int i = 0; i < kPerThread; ++i) {
        if (xv[i] >= 0.0 && (e > -1022 ? xv[i] < halfu : xv[i] == 0.0)) continue;  // a no-op term
        t = tx_then(t, tx_term(xv[i], f1, f2, lim, flag));
      }
    }
    // ordered warp reduction: lane l composes with lanes above it
    if (__any_sync(0xffffffffu, t.o != 2u || t.q0 || t.q1)) {
      for (int o = 1; o < 32; o <<= 1) {
        const Tx up = tx_shfl_down(t, o);
        if ((lane & (2 * o - 1)) == 0) t = tx_then(t, up);
      }
    }
    const unsigned any = __ballot_sync(0xffffffffu, flag);
    if (lane == 0) {
      sq[w] = t;
      sf[w] = any ? 1 : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      Tx tq = tx_identity();
      int32_t tf = 0;
      for (int v = 0; v < kSegThreads / 32; ++v) {
        tq = tx_then(tq, sq[v]);
        tf |= sf[v];
      }
      Q[gy] = tq;
      F[gy] = tf;
      elo[gy] = ok ? e : kNoBinade;
    }
    __syncthreads();
  }
}

// 4. the walk: one block of kWalkThreads per sum (sum y = blockIdx.x)
__global__ void __launch_bounds__(kWalkThreads) k_walk(const double* __restrict__ X, int64_t n, int64_t stride,
                                                       int64_t nseg, const int32_t* __restrict__ elo_all,
                                                       const Tx* __restrict__ Q_all, const int32_t* __restrict__ F_all,
                                                       double* __restrict__ out) {
  __shared__ WalkShared W;
  const int64_t y = blockIdx.x;
  const double* __restrict__ x = X + y * stride;
  const int32_t* __restrict__ elo = elo_all + y * nseg;
  const Tx* __restrict__ Q = Q_all + y * nseg;
  const int32_t* __restrict__ F = F_all + y * nseg;
  const unsigned long long top = 1ull << 53;
  double s = 0.0;  // the running sum, the same in every thread
  int64_t g = 0;
  while (g < nseg) {
    if (s != s) break;  // NaN + anything = NaN
    const bool has = s >= 0.0 && s < INFINITY;
    const int e = has ? binade_of(s) : kNoBinade;
    const unsigned long long A = has ? (unsigned long long)scale2(s, 52 - e) : 0;  // s / u, exact
    const uint32_t p0 = (uint32_t)(A & 1ull);
    const int64_t gi = g + threadIdx.x;
    bool simple = false;
    Tx q = tx_identity();
    if (gi < nseg && has && elo[gi] == e && !F[gi]) {
      simple = true;
      q = Q[gi];
    }
    Tx total;
    const Tx ex = block_exscan_tx<kWalkThreads>(q, W.wsum, &total);
    const Tx pre = tx_then(ex, q);  // inclusive
    const unsigned long long cum = p0 ? pre.q1 : pre.q0;
    const bool stop = gi < nseg && (!simple || A + cum >= top);
    if (threadIdx.x == 0) W.stop = LLONG_MAX;
    __syncthreads();
    if (stop) atomicMin(&W.stop, (long long)gi);
    __syncthreads();
    const int64_t sa = W.stop;
    // exact integer sum of the simple segments before the stop (or the whole batch)
    const int64_t last = sa == LLONG_MAX ? (nseg < g + kWalkThreads ? nseg : g + kWalkThreads) - 1 : sa - 1;
    if (last >= g && gi == last) W.cum = cum;
    __syncthreads();
    if (has && last >= g) s = (double)(A + W.cum) * ldexp(1.0, e - 52);  // a multiple of u below 2^(e+1): exact
    __syncthreads();
    if (sa == LLONG_MAX) {
      g = last + 1;
      continue;
    }
    // segment sa term by term
    const int64_t kb = sa * kSeg;
    const int len = (int)(n - kb < kSeg ? n - kb : kSeg);
    s = walk_segment(s, (int)threadIdx.x < len ? x[kb + threadIdx.x] : 0.0, W);
    g = sa + 1;
  }
  if (threadIdx.x == 0) out[y] = s;
}

__global__ void k_any_negative(const double* __restrict__ x, int64_t n, int32_t* __restrict__ flag) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    if (!(x[k] >= 0.0)) *flag = 1;  // negative, -0.0 is fine; NaN also takes the ordered path
}

}  // namespace

namespace gh {

int64_t seqsum_segments(int64_t n) { return (n + kSeg - 1) / kSeg; }

void sequential_sums_from_T(const double* d_x, int64_t n, int64_t stride, int32_t count, const double* d_T,
                            double* d_out, cudaStream_t s) {
  if (count <= 0) return;
  if (n == 0) {
    GH_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double) * count, s));
    return;
  }
  const int64_t nseg = seqsum_segments(n);
  Scratch<double> P((size_t)nseg * count, s);
  Scratch<int32_t> elo((size_t)nseg * count, s), F((size_t)nseg * count, s);
  Scratch<Tx> Q((size_t)nseg * count, s);
  k_seg_scan<<<count, 1024, 0, s>>>(d_T, nseg, P.p);
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nseg, (148LL * 16 + count - 1) / count));
  k_seg_q<<<dim3(gx, (unsigned)count), kSegThreads, 0, s>>>(d_x, n, stride, nseg, P.p, elo.p, Q.p, F.p);
  k_walk<<<count, kWalkThreads, 0, s>>>(d_x, n, stride, nseg, elo.p, Q.p, F.p, d_out);
  GH_LAUNCH_CHECK();
}

void sequential_sums_group(const double* d_x, int64_t n, int64_t stride, int32_t count, double* d_out,
                           cudaStream_t s) {
  if (count <= 0) return;
  const int64_t nseg = seqsum_segments(n);
  Scratch<double> T((size_t)std::max<int64_t>(1, nseg) * count, s);
  if (nseg) {
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nseg, (148LL * 16 + count - 1) / count));
    k_seg_sums<<<dim3(gx, (unsigned)count), kSegThreads, 0, s>>>(d_x, n, stride, nseg, T.p);
    GH_LAUNCH_CHECK();
  }
  sequential_sums_from_T(d_x, n, stride, count, T.p, d_out, s);
}

double sequential_sum_nonneg(const double* d_x, int64_t n, cudaStream_t s, int* launches) {
  if (n == 0) return 0.0;
  Scratch<double> out(1, s);
  sequential_sums_group(d_x, n, n, 1, out.p, s);
  double h = 0.0;
  GH_CUDA(cudaMemcpyAsync(&h, out.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
  if (launches) *launches += 4;
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
