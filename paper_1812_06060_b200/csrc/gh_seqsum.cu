// Bit-exact left-to-right sums of non-negative doubles on the device.
//
// The reference accumulates global sums sequentially (`double s = 0.0;
// for (x : terms) s += x;`, e.g. average_edge_length, mesh.hpp:289-293).
// A tree sum is reproducible but rounds differently. For non-negative terms
// the sequential result can be reproduced exactly in parallel: while the
// running sum s stays inside one binade [2^e, 2^(e+1)) every partial sum is a
// multiple of u = 2^(e-52), and fl(s + x) = s + rint(x / u) * u unless x / u
// has fractional part exactly 1/2 (a tie, whose rounding depends on the
// parity of s / u) or the addition leaves the binade. So:
//   1. the first K terms are summed sequentially (one thread);
//   2. for every binade e the running sum can visit (bounded from a tree sum
//      of the rest), each 1024-term segment records sum(rint(x / u_e)) and
//      whether it holds a tie or a term >= 2^e (one parallel pass);
//   3. per binade, prefix sums over the segments;
//   4. one thread walks the segments: it jumps (binary search) to the first
//      segment that holds a flagged term or would carry s out of its binade,
//      adds the exact integer sum of the skipped segments, and adds that
//      segment term by term in double, exactly as the reference does.
// Step 4 runs once per binade change or flagged segment (tens of times for
// millions of terms), so the sum costs a few passes over the terms.

#include <cmath>

#include "gh_internal.cuh"

namespace {

constexpr int kSeg = 1024;        // terms per segment
constexpr int kSeqPrefix = 4096;  // leading terms summed sequentially
constexpr int kMaxBinades = 48;
constexpr int kWalkThreads = 1024;

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

__global__ void k_tree_partial(const double* __restrict__ x, int64_t b, int64_t n, double* __restrict__ part) {
  double s = 0.0;
  for (int64_t k = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    s += x[k];
  s = ghd::block_sum<gh::kBlock>(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// the binades [e0, e0 + nb) the running sum can visit, from the sequential
// prefix acc[0] and an upper bound of the rest (nb = 0: no fast path)
__global__ void k_binades(const double* __restrict__ part, int nparts, const double* __restrict__ acc,
                          int32_t* __restrict__ prm) {
  double r = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) r += part[i];
  const double rest = ghd::block_sum<1024>(r);  // any order: only a bound
  if (threadIdx.x != 0) return;
  const double s0 = acc[0];
  int nb = 0, e0 = 0;
  if (s0 > 0.0 && isfinite(rest)) {
    e0 = ilogb(s0);
    const int e1 = ilogb((s0 + rest) * (1.0 + 1.0 / (1 << 20)));
    nb = e1 - e0 + 1;
    if (nb < 1 || nb > kMaxBinades || e0 - 52 < -1000 || e0 + nb > 1000) nb = 0;  // keep 2^(52-e) finite
  }
  prm[0] = e0;
  prm[1] = nb;
}

// per segment g and binade j: Q[j][g] = sum rint(x * 2^(52 - e0 - j)), F[j][g] = tie or big term present
constexpr int kSegThreads = 256;
constexpr int kPerThread = kSeg / kSegThreads;
__global__ void __launch_bounds__(kSegThreads) k_segments(const double* __restrict__ x, int64_t b, int64_t n,
                                                          int64_t nseg, const int32_t* __restrict__ prm,
                                                          long long* __restrict__ Q, int32_t* __restrict__ F) {
  const int e0 = prm[0], nb = prm[1];
  __shared__ long long sq[kSegThreads / 32][kMaxBinades];
  __shared__ int32_t sf[kSegThreads / 32][kMaxBinades];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t g = blockIdx.x; g < nseg && nb > 0; g += gridDim.x) {
    double xv[kPerThread];
    bool in[kPerThread];
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      const int64_t k = b + g * kSeg + i * kSegThreads + threadIdx.x;
      in[i] = k < n;
      xv[i] = in[i] ? x[k] : 0.0;
    }
    double scale = ldexp(1.0, 52 - e0), lim = ldexp(1.0, e0);  // exact powers of two
    for (int j = 0; j < nb; ++j) {
      long long q = 0;
      bool flag = false;
#pragma unroll
      for (int i = 0; i < kPerThread; ++i) {
        const double y = xv[i] * scale;  // exact scaling
        const bool f = in[i] && (xv[i] >= lim || y - floor(y) == 0.5);
        flag |= f;
        q += f ? 0 : (long long)rint(y);
      }
      for (int o = 16; o > 0; o >>= 1) q += __shfl_down_sync(0xffffffffu, q, o);
      const unsigned any = __ballot_sync(0xffffffffu, flag);
      if (lane == 0) {
        sq[w][j] = q;
        sf[w][j] = any ? 1 : 0;
      }
      scale *= 0.5;
      lim *= 2.0;
    }
    __syncthreads();
    if (threadIdx.x < nb) {
      long long tq = 0;
      int32_t tf = 0;
      for (int v = 0; v < kSegThreads / 32; ++v) {
        tq += sq[v][threadIdx.x];
        tf |= sf[v][threadIdx.x];
      }
      Q[(int64_t)threadIdx.x * nseg + g] = tq;
      F[(int64_t)threadIdx.x * nseg + g] = tf;
    }
    __syncthreads();
  }
}

// per binade: exclusive prefix with a leading 0, P[j][0..nseg]. The sums
// saturate at 2^62: only comparisons against < 2^53 matter, and the prefix of
// the binade the walk is in stays below 2^53 up to its position (those terms
// summed to less than 2^(e+1)), while lower binades' prefixes may grow past
// the int64 range.
constexpr unsigned long long kCap = 1ull << 62;
__device__ __forceinline__ unsigned long long sat_add(unsigned long long a, unsigned long long b) {
  const unsigned long long c = a + b;  // both <= 2^62: no wrap
  return c < kCap ? c : kCap;
}
__global__ void k_prefix(const long long* __restrict__ Q, const int32_t* __restrict__ F, int64_t nseg,
                         const int32_t* __restrict__ prm, long long* __restrict__ PQ, int32_t* __restrict__ PF) {
  const int j = blockIdx.x;
  if (j >= prm[1]) return;
  __shared__ unsigned long long carry_q;
  __shared__ int32_t carry_f;
  __shared__ unsigned long long wq[32];
  __shared__ int32_t wf[32];
  if (threadIdx.x == 0) {
    carry_q = 0;
    carry_f = 0;
    PQ[(int64_t)j * (nseg + 1)] = 0;
    PF[(int64_t)j * (nseg + 1)] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = 0; base < nseg; base += blockDim.x) {
    const int64_t g = base + threadIdx.x;
    unsigned long long q = g < nseg ? (unsigned long long)Q[(int64_t)j * nseg + g] : 0;
    int32_t f = g < nseg ? F[(int64_t)j * nseg + g] : 0;
    for (int o = 1; o < 32; o <<= 1) {  // warp inclusive scan
      const unsigned long long tq = __shfl_up_sync(0xffffffffu, q, o);
      const int32_t tf = __shfl_up_sync(0xffffffffu, f, o);
      if (lane >= o) {
        q = sat_add(q, tq);
        f += tf;
      }
    }
    if (lane == 31) {
      wq[w] = q;
      wf[w] = f;
    }
    __syncthreads();
    if (w == 0) {
      unsigned long long a = lane < (int)(blockDim.x >> 5) ? wq[lane] : 0;
      int32_t c = lane < (int)(blockDim.x >> 5) ? wf[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long ta = __shfl_up_sync(0xffffffffu, a, o);
        const int32_t tc = __shfl_up_sync(0xffffffffu, c, o);
        if (lane >= o) {
          a = sat_add(a, ta);
          c += tc;
        }
      }
      wq[lane] = a;
      wf[lane] = c;
    }
    __syncthreads();
    const unsigned long long off_q = sat_add(carry_q, w ? wq[w - 1] : 0);
    const int32_t off_f = carry_f + (w ? wf[w - 1] : 0);
    if (g < nseg) {
      PQ[(int64_t)j * (nseg + 1) + g + 1] = (long long)sat_add(off_q, q);
      PF[(int64_t)j * (nseg + 1) + g + 1] = off_f + f;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) {
      carry_q = sat_add(off_q, q);
      carry_f = off_f + f;
    }
    __syncthreads();
  }
}

// Step 4, one block: thread 0 keeps the running sum and searches; the block
// stages each segment that has to be added term by term. acc[0]: the
// sequential prefix on entry, the sum on exit.
__global__ void k_walk(const double* __restrict__ x, int64_t b, int64_t n, int64_t nseg,
                       const int32_t* __restrict__ prm, const long long* __restrict__ PQ,
                       const int32_t* __restrict__ PF, double* __restrict__ acc) {
  __shared__ double sh[kWalkThreads];
  __shared__ int64_t seg;   // next segment to add term by term, -1: done, -2: rest term by term
  __shared__ int64_t from;  // segment the walk continues at
  __shared__ int64_t first; // search: first stopping candidate
  __shared__ int walk_j;
  __shared__ long long walk_A;
  __shared__ double walk_u;
  const int e0 = prm[0], nb = prm[1];
  double s = acc[0];
  int64_t g = 0;
  const long long top = 1ll << 53;
  while (true) {
    if (threadIdx.x == 0) {
      if (g >= nseg) {
        seg = -1;
      } else {
        const int e = ilogb(s);
        const int j = e - e0;
        if (nb == 0 || !(s > 0.0) || j < 0 || j >= nb) {
          seg = -2;  // outside the precomputed binades
          from = g;
        } else {
          const double u = ldexp(1.0, e - 52);
          const long long A = (long long)(s / u);
          walk_j = j;
          walk_A = A;
          walk_u = u;
          seg = -3;  // search below
        }
      }
    }
    __syncthreads();
    if (seg == -3) {
      // first segment >= g that is flagged or would leave the binade: the block
      // tests 1024 evenly spaced candidates, then the 1024 segments of the hit
      const long long* pq = PQ + (int64_t)walk_j * (nseg + 1);
      const int32_t* pf = PF + (int64_t)walk_j * (nseg + 1);
      const long long A = walk_A, q0 = pq[g];
      const int32_t f0 = pf[g];
      auto stop = [&](int64_t m) { return pf[m + 1] > f0 || A + (pq[m + 1] - q0) >= top; };
      int64_t lo = g, hi = nseg;  // the answer lies in [lo, hi]; hi = nseg: none
      while (hi - lo > 1) {
        const int64_t step = (hi - lo + kWalkThreads - 1) / kWalkThreads;
        const int64_t m = lo + threadIdx.x * step;
        if (threadIdx.x == 0) first = hi;
        __syncthreads();
        if (m < hi && stop(m)) atomicMin(reinterpret_cast<unsigned long long*>(&first), (unsigned long long)m);
        __syncthreads();
        const int64_t f = first;
        __syncthreads();
        // the first stop lies in (f - step, f]; when f = hi none of the candidates stopped
        const int64_t nlo = f - step + 1 > lo ? f - step + 1 : lo;
        if (f == hi) {
          lo = hi - step + 1 > lo ? hi - step + 1 : lo;
        } else {
          hi = f;
          lo = nlo;
        }
        if (step == 1) break;
      }
      if (threadIdx.x == 0) {
        int64_t r = lo;
        while (r < hi && !stop(r)) ++r;  // at most one candidate left
        s = (double)(A + (pq[r] - q0)) * walk_u;  // exact: a multiple of u below 2^(e+1)
        seg = r < nseg ? r : -1;
      }
      __syncthreads();
    }
    const int64_t sg = seg;
    if (sg == -1) break;
    if (sg == -2) {
      s = block_ordered_add(s, x, b + from * kSeg, n, sh);
      break;
    }
    const int64_t kb = b + sg * kSeg;
    s = block_ordered_add(s, x, kb, kb + kSeg < n ? kb + kSeg : n, sh);  // the reference's own additions
    g = sg + 1;
    __syncthreads();
  }
  if (threadIdx.x == 0) acc[0] = s;
}

__global__ void k_any_negative(const double* __restrict__ x, int64_t n, int32_t* __restrict__ flag) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    if (!(x[k] >= 0.0)) *flag = 1;  // negative, -0.0 is fine; NaN also takes the ordered path
}

}  // namespace

namespace gh {

// Device-resident: one host synchronisation (the result) per sum.
double sequential_sum_nonneg(const double* d_x, int64_t n, cudaStream_t s, int* launches) {
  if (n == 0) return 0.0;
  Scratch<double> acc(1, s);
  GH_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(double), s));
  const int64_t K = n < kSeqPrefix ? n : kSeqPrefix;
  k_seq_block<<<1, kWalkThreads, 0, s>>>(d_x, 0, K, acc.p);
  int nl = 1;
  if (n > K) {
    const int64_t nseg = (n - K + kSeg - 1) / kSeg;
    Scratch<double> part(kReduceGrid, s);
    Scratch<int32_t> prm(2, s);
    Scratch<long long> Q((size_t)kMaxBinades * nseg, s), PQ((size_t)kMaxBinades * (nseg + 1), s);
    Scratch<int32_t> F((size_t)kMaxBinades * nseg, s), PF((size_t)kMaxBinades * (nseg + 1), s);
    k_tree_partial<<<kReduceGrid, kBlock, 0, s>>>(d_x, K, n, part.p);
    k_binades<<<1, 1024, 0, s>>>(part.p, kReduceGrid, acc.p, prm.p);
    k_segments<<<(unsigned)std::min<int64_t>(nseg, 148 * 32), kSegThreads, 0, s>>>(d_x, K, n, nseg, prm.p, Q.p, F.p);
    k_prefix<<<kMaxBinades, 1024, 0, s>>>(Q.p, F.p, nseg, prm.p, PQ.p, PF.p);
    k_walk<<<1, kWalkThreads, 0, s>>>(d_x, K, n, nseg, prm.p, PQ.p, PF.p, acc.p);
    nl += 5;
  }
  GH_LAUNCH_CHECK();
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
