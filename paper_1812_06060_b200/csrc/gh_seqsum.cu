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

constexpr int kSeg = 1024;       // terms per segment
constexpr int kSeqPrefix = 4096; // leading terms summed sequentially
constexpr int kMaxBinades = 48;

__global__ void k_seq(const double* __restrict__ x, int64_t b, int64_t e, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = out[0];
  for (int64_t k = b; k < e; ++k) s += x[k];
  out[0] = s;
}

__global__ void k_tree_partial(const double* __restrict__ x, int64_t b, int64_t n, double* __restrict__ part) {
  double s = 0.0;
  for (int64_t k = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    s += x[k];
  s = ghd::block_sum<gh::kBlock>(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// per segment g and binade j: Q[j][g] = sum rint(x * 2^(52 - e0 - j)), F[j][g] = tie or big term present
__global__ void k_segments(const double* __restrict__ x, int64_t b, int64_t n, int64_t nseg, int e0, int nb,
                           long long* __restrict__ Q, int32_t* __restrict__ F) {
  __shared__ long long sq[kMaxBinades];
  __shared__ int32_t sf[kMaxBinades];
  for (int64_t g = blockIdx.x; g < nseg; g += gridDim.x) {
    if (threadIdx.x < nb) {
      sq[threadIdx.x] = 0;
      sf[threadIdx.x] = 0;
    }
    __syncthreads();
    const int64_t k = b + g * kSeg + threadIdx.x;
    const bool in = k < n;
    const double xv = in ? x[k] : 0.0;
    for (int j = 0; j < nb; ++j) {
      const int e = e0 + j;
      const double y = ldexp(xv, 52 - e);  // exact scaling
      const double r = rint(y);
      const bool flag = in && (xv >= ldexp(1.0, e) || y - floor(y) == 0.5);
      long long q = flag ? 0 : (long long)r;
      for (int o = 16; o > 0; o >>= 1) q += __shfl_down_sync(0xffffffffu, q, o);
      const unsigned any = __ballot_sync(0xffffffffu, flag);
      if ((threadIdx.x & 31) == 0) {
        if (q) atomicAdd(reinterpret_cast<unsigned long long*>(&sq[j]), (unsigned long long)q);
        if (any) sf[j] = 1;
      }
    }
    __syncthreads();
    if (threadIdx.x < nb) {
      Q[(int64_t)threadIdx.x * nseg + g] = sq[threadIdx.x];
      F[(int64_t)threadIdx.x * nseg + g] = sf[threadIdx.x];
    }
    __syncthreads();
  }
}

// inclusive -> stored as exclusive prefix with a leading 0: P[j][0..nseg]
__global__ void k_prefix(const long long* __restrict__ Q, const int32_t* __restrict__ F, int64_t nseg,
                         long long* __restrict__ PQ, int32_t* __restrict__ PF) {
  const int j = blockIdx.x;
  __shared__ long long carry_q;
  __shared__ int32_t carry_f;
  __shared__ long long wq[32];
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
    long long q = g < nseg ? Q[(int64_t)j * nseg + g] : 0;
    int32_t f = g < nseg ? F[(int64_t)j * nseg + g] : 0;
    for (int o = 1; o < 32; o <<= 1) {  // warp inclusive scan
      const long long tq = __shfl_up_sync(0xffffffffu, q, o);
      const int32_t tf = __shfl_up_sync(0xffffffffu, f, o);
      if (lane >= o) {
        q += tq;
        f += tf;
      }
    }
    if (lane == 31) {
      wq[w] = q;
      wf[w] = f;
    }
    __syncthreads();
    if (w == 0) {
      long long a = lane < (int)(blockDim.x >> 5) ? wq[lane] : 0;
      int32_t c = lane < (int)(blockDim.x >> 5) ? wf[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const long long ta = __shfl_up_sync(0xffffffffu, a, o);
        const int32_t tc = __shfl_up_sync(0xffffffffu, c, o);
        if (lane >= o) {
          a += ta;
          c += tc;
        }
      }
      wq[lane] = a;
      wf[lane] = c;
    }
    __syncthreads();
    const long long off_q = carry_q + (w ? wq[w - 1] : 0);
    const int32_t off_f = carry_f + (w ? wf[w - 1] : 0);
    if (g < nseg) {
      PQ[(int64_t)j * (nseg + 1) + g + 1] = off_q + q;
      PF[(int64_t)j * (nseg + 1) + g + 1] = off_f + f;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) {
      carry_q = off_q + q;
      carry_f = off_f + f;
    }
    __syncthreads();
  }
}

// the walk of step 4; out[0] holds s on entry (the sequential prefix) and on exit
__global__ void k_walk(const double* __restrict__ x, int64_t b, int64_t n, int64_t nseg, int e0, int nb,
                       const long long* __restrict__ PQ, const int32_t* __restrict__ PF, double* __restrict__ out,
                       int32_t* __restrict__ fail) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = out[0];
  int64_t g = 0;
  const long long top = 1ll << 53;
  while (g < nseg) {
    const int e = ilogb(s);
    const int j = e - e0;
    if (s <= 0.0 || j < 0 || j >= nb) {  // outside the precomputed binades: finish term by term
      for (int64_t k = b + g * kSeg; k < n; ++k) s += x[k];
      *fail = 1;
      break;
    }
    const double u = ldexp(1.0, e - 52);
    const long long A = (long long)(s / u);
    const long long* pq = PQ + (int64_t)j * (nseg + 1);
    const int32_t* pf = PF + (int64_t)j * (nseg + 1);
    // first segment g' >= g that is flagged or would leave the binade
    int64_t lo = g, hi = nseg;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      const bool stop = pf[mid + 1] > pf[g] || A + (pq[mid + 1] - pq[g]) >= top;
      if (stop) hi = mid;
      else lo = mid + 1;
    }
    s = (double)(A + (pq[lo] - pq[g])) * u;  // exact: a multiple of u below 2^(e+1)
    if (lo == nseg) break;
    const int64_t kb = b + lo * kSeg, ke = kb + kSeg < n ? kb + kSeg : n;
    for (int64_t k = kb; k < ke; ++k) s += x[k];  // the reference's own additions
    g = lo + 1;
  }
  out[0] = s;
}

__global__ void k_any_negative(const double* __restrict__ x, int64_t n, int32_t* __restrict__ flag) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    if (!(x[k] >= 0.0)) *flag = 1;  // negative, -0.0 is fine; NaN also takes the ordered path
}

}  // namespace

namespace gh {

double sequential_sum_nonneg(const double* d_x, int64_t n, cudaStream_t s, int* launches) {
  Scratch<double> acc(2, s);
  GH_CUDA(cudaMemsetAsync(acc.p, 0, 2 * sizeof(double), s));
  const int64_t K = n < kSeqPrefix ? n : kSeqPrefix;
  k_seq<<<1, 32, 0, s>>>(d_x, 0, K, acc.p);
  GH_LAUNCH_CHECK();
  int nl = 1;
  double h[2] = {0.0, 0.0};
  if (n > K) {
    Scratch<double> part(kReduceGrid, s);
    k_tree_partial<<<kReduceGrid, kBlock, 0, s>>>(d_x, K, n, part.p);
    Scratch<double> tot(1, s);
    std::vector<double> hp(kReduceGrid);
    GH_CUDA(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * kReduceGrid, cudaMemcpyDeviceToHost, s));
    GH_CUDA(cudaMemcpyAsync(h, acc.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    GH_CUDA(cudaStreamSynchronize(s));
    nl += 1;
    double rest = 0.0;  // an upper bound only (bounds the binades the walk can visit)
    for (double v : hp) rest += v;
    const double s0 = h[0];
    const int e0 = s0 > 0.0 ? std::ilogb(s0) : 0;
    const int e1 = std::ilogb((s0 + rest) * (1.0 + 1.0 / (1 << 20)) + 1e-300);
    const int nb = e1 - e0 + 1;
    Scratch<int32_t> fail(1, s);
    GH_CUDA(cudaMemsetAsync(fail.p, 0, sizeof(int32_t), s));
    if (!(s0 > 0.0) || nb < 1 || nb > kMaxBinades) {
      k_seq<<<1, 32, 0, s>>>(d_x, K, n, acc.p);  // pathological ranges: plain sequential
      nl += 1;
    } else {
      const int64_t nseg = (n - K + kSeg - 1) / kSeg;
      Scratch<long long> Q((size_t)nb * nseg, s), PQ((size_t)nb * (nseg + 1), s);
      Scratch<int32_t> F((size_t)nb * nseg, s), PF((size_t)nb * (nseg + 1), s);
      k_segments<<<(unsigned)std::min<int64_t>(nseg, 148 * 16), kSeg, 0, s>>>(d_x, K, n, nseg, e0, nb, Q.p, F.p);
      k_prefix<<<nb, 1024, 0, s>>>(Q.p, F.p, nseg, PQ.p, PF.p);
      k_walk<<<1, 32, 0, s>>>(d_x, K, n, nseg, e0, nb, PQ.p, PF.p, acc.p, fail.p);
      GH_LAUNCH_CHECK();
      nl += 3;
    }
  }
  GH_CUDA(cudaMemcpyAsync(h, acc.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
  if (launches) *launches += nl;
  return h[0];
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
  k_seq<<<1, 32, 0, s>>>(d_x, 0, n, acc.p);
  GH_LAUNCH_CHECK();
  double out = 0.0;
  GH_CUDA(cudaMemcpyAsync(&out, acc.p, sizeof(out), cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
  return out;
}

}  // namespace gh
