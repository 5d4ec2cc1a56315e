// Gradient normalisation and the two integrability-constrained ADMM
// optimisers as fused gather kernels:
//   normalized_target_gradients (reference diffusion.hpp:132-145)
//   FaceAdmmSolver / admm_face_optimize (grad_face.hpp:51-206, 228-237)
//   EdgeAdmmSolver / admm_edge_optimize (grad_edge.hpp:57-198, 207-216)
//
// Per iteration the face method runs two kernels instead of the reference's
// five loops: G-update (+ dual partials) per face, and lambda-update (+ primal
// partials) fused with the NEXT iteration's Y-update per interior edge (Y only
// needs the new g and the new lambda, both final once the edge thread has
// written lambda). The edge method likewise runs X-update (+ dual) per edge
// and lambda-update (+ primal) fused with the next W-update per face.
// Element values are bit-identical to the reference. The residual norms use a
// fixed-shape tree (kReduceGrid blocks x 256 threads, then one block), which
// is reproducible run to run but not the reference's left-to-right sum; the
// stop rule compares them against thresholds with the same formulas.

#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "gh_internal.cuh"

using namespace ghd;

namespace {

constexpr int B = gh::kBlock;
constexpr unsigned G = gh::kReduceGrid;

#define GRID_STRIDE(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------- normalisation
__global__ void k_normalize(const double* __restrict__ pos, const int32_t* __restrict__ faces,
                            const double* __restrict__ normal, const double* __restrict__ area,
                            const double* __restrict__ u, int64_t nf, double* __restrict__ h,
                            double* __restrict__ part) {
  double zeros = 0.0;
  GRID_STRIDE(f, nf) {
    const int32_t t[3] = {faces[3 * f], faces[3 * f + 1], faces[3 * f + 2]};
    const v3 n = ld3(normal, f);
    v3 g = mk(0.0, 0.0, 0.0);
    for (int k = 0; k < 3; ++k) {  // face_gradient (mesh.hpp:316-325)
      v3 opp = sub(ld3(pos, t[(k + 2) % 3]), ld3(pos, t[(k + 1) % 3]));
      g = add(g, scale(u[t[k]], cross(n, opp)));
    }
    g = divs(g, 2.0 * area[f]);
    const double nrm = ghd::norm(g);
    if (nrm >= 1e-20) {
      st3(h, f, divs(mk(-g.x, -g.y, -g.z), nrm));
    } else {
      st3(h, f, mk(0.0, 0.0, 0.0));
      zeros += 1.0;
    }
  }
  zeros = block_sum<B>(zeros);
  if (threadIdx.x == 0) part[blockIdx.x] = zeros;
}

// ---------------------------------------------------------------- face ADMM
// Slot of face f's k-th edge in the interior-edge state: 2i + side, or -1.
__global__ void k_face_slots(const int32_t* __restrict__ he_edge, const int32_t* __restrict__ iei,
                             const int32_t* __restrict__ edge_he, int64_t nf, int32_t* __restrict__ slot) {
  GRID_STRIDE(f, nf) {
    for (int k = 0; k < 3; ++k) {
      const int32_t e = he_edge[3 * f + k];
      const int32_t i = iei[e];
      slot[3 * f + k] = i < 0 ? -1 : 2 * i + (edge_he[2 * e] / 3 == f ? 0 : 1);
    }
  }
}


// Y-update for interior edge i (grad_face.hpp:126-137 + y_update_edge 31-36)
// from the two side faces' g and lambda; d = lambda / (mu sqrt(A)) per side is
// returned too (the G-update adds the same quotient, grad_face.hpp:150).
// msa = mu * sqrt(A) of each side face and w = (A2 / (A1 + A2), A1 / (A1 + A2))
// of the edge are computed once per solve (k_face_consts, k_face_init_edges):
// the same operations on the same operands as the reference's per-iteration
// expressions, so the same bits, without 2 sqrt + 2 divisions per call.
__device__ __forceinline__ void face_y_update(int64_t i, v3 g1, v3 g2, double msa1, double msa2, double w1,
                                              double w2, const double* __restrict__ edir, v3 l1, v3 l2, v3& y1,
                                              v3& y2, v3& d1, v3& d2) {
  d1 = divs(l1, msa1);
  d2 = divs(l2, msa2);
  const v3 q1 = sub(g1, d1);
  const v3 q2 = sub(g2, d2);
  const v3 ed = ld3(edir, i);
  const double mismatch = dot(ed, sub(q2, q1));
  const v3 shift = mk(ed.x * mismatch, ed.y * mismatch, ed.z * mismatch);
  y1 = add(q1, scale(w1, shift));
  y2 = sub(q2, scale(w2, shift));
}

// per face: sqrt(A) (the primal rows' weight, grad_face.hpp:163-164); the dual
// offset's divisor mu sqrt(A) (grad_face.hpp:130-131, 150) is mu * sa[f], the
// same operation on the same operands, formed where it is used
__global__ void k_face_consts(const double* __restrict__ area, int64_t nf, double* __restrict__ sa) {
  GRID_STRIDE(f, nf) sa[f] = sqrt(area[f]);
}

// ctor (grad_face.hpp:76-85): edge_dir, incident faces, lambda = 0, scale
// partials; with C set, also the first iteration's c per slot: y1, y2 start
// at h of the side faces (grad_face.hpp:82-83), which is the Y-update from
// g = h, lambda = 0 (computed exactly like later ones, see k_face_lambda_pair)
__global__ void k_face_init_edges(const double* __restrict__ pos, const int32_t* __restrict__ interior_edges,
                                  const int32_t* __restrict__ edge_v, const int32_t* __restrict__ edge_he,
                                  const double* __restrict__ area, const double* __restrict__ h, int64_t ni,
                                  double mu, const double* __restrict__ sa, double* __restrict__ edir,
                                  int32_t* __restrict__ ef, double* __restrict__ wq, double* __restrict__ lam,
                                  double* __restrict__ C, double* __restrict__ part, double* __restrict__ term,
                                  const uint8_t* __restrict__ act) {
  double s = 0.0;
  GRID_STRIDE(i, ni) {
    const int32_t e = interior_edges[i];
    const int32_t f1 = edge_he[2 * e] / 3, f2 = edge_he[2 * e + 1] / 3;
    const double a1 = area[f1], a2 = area[f2];
    const double tt = a1 + a2;  // scale2 += A1 + A2 (grad_face.hpp:83)
    term[i] = tt;
    s += tt;
    if (act && !act[i]) continue;  // an edge that stays zero: only its scale term (lambda, c were zeroed)
    st3(edir, i, normalized(sub(ld3(pos, edge_v[2 * e + 1]), ld3(pos, edge_v[2 * e]))));
    ef[2 * i] = f1;
    ef[2 * i + 1] = f2;
    const v3 zero = mk(0.0, 0.0, 0.0);
    st3(lam, 2 * i, zero);
    st3(lam, 2 * i + 1, zero);
    const double w1 = ddiv(a2, a1 + a2), w2 = ddiv(a1, a1 + a2);  // y_update_edge (grad_face.hpp:35)
    wq[2 * i] = w1;
    wq[2 * i + 1] = w2;
    if (C) {
      v3 y1, y2, d1, d2;
      face_y_update(i, ld3(h, f1), ld3(h, f2), mu * sa[f1], mu * sa[f2], w1, w2, edir, zero, zero, y1, y2, d1, d2);
      st3(C, 2 * i, add(y1, d1));
      st3(C, 2 * i + 1, add(y2, d2));
    }
  }
  s = block_sum<B>(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// The face kernel needs, per slot (interior edge i, side), only
// c = y + lambda / (mu sqrt(A_side)) (grad_face.hpp:150): the edge kernel writes
// c instead of Y, and recomputes Y from the previous g (kept in a second
// buffer) and lambda when it needs it. 48 B per face less to read, no Y
// round trip; every value is the reference's expression, so bits are unchanged.

// G-update per face (grad_face.hpp:139-155) + dual partials (170-171, 104-111):
// g_out = (2h + mu sum_k c_k) / (2 + mu count), dual term from g_out - g_in
__global__ void k_face_g(const int32_t* __restrict__ slot, const double* __restrict__ area,
                         const double* __restrict__ h, const double* __restrict__ C, int64_t nf, double mu,
                         const double* __restrict__ gin, double* __restrict__ gout, double* __restrict__ part,
                         double* __restrict__ term, const int32_t* __restrict__ halt,
                         const uint8_t* __restrict__ act) {
  if (*halt) return;  // the device stop rule ended the loop (see admm_loop)
  double s = 0.0;
  GRID_STRIDE(f, nf) {
    if (act && !act[f]) continue;  // g stays +0 here (both buffers hold it), its dual term 0
    const double A = area[f];
    v3 sum = mk(0.0, 0.0, 0.0);
    int count = 0;
    for (int k = 0; k < 3; ++k) {
      const int32_t sl = slot[3 * f + k];
      if (sl < 0) continue;
      sum = add(sum, ld3(C, sl));
      ++count;
    }
    const v3 gold = ld3(gin, f);
    const v3 gnew = divs(add(scale(2.0, ld3(h, f)), scale(mu, sum)), 2.0 + mu * (double)count);
    st3(gout, f, gnew);
    const v3 dg = sub(gnew, gold);
    const double tt = (double)count * A * sqnorm(dg);
    term[f] = tt;
    s += tt;
  }
  s = block_sum<B>(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// lambda-update + primal rows per interior edge (grad_face.hpp:158-168) with
// this iteration's Y recomputed from g_in (the previous g) and the old lambda,
// then the next iteration's Y and c from the same registers; two lanes per
// edge (lane 2k + side handles side
// `side` of edge i = k >> 1: face ef[2i + side], its lambda / c slots), so each
// thread holds one side's state (half the registers, twice the resident warps)
// and the per-side streams (ef, wq, lambda, c) are contiguous across lanes.
// The two sides meet only in the mismatch dot(e, q2 - q1) and in the primal
// term |r1|^2 + |r2|^2: their q and |r|^2 cross the pair with one shuffle, and
// both lanes evaluate the reference's expressions on the same operands in the
// same order (grad_face.hpp:31-36, 126-168), so every value keeps its bits.
// Only side-0 lanes add the primal term into the block's tree sum.
__device__ __forceinline__ v3 shfl_pair(const v3& a) {
  return mk(__shfl_xor_sync(0xffffffffu, a.x, 1), __shfl_xor_sync(0xffffffffu, a.y, 1),
            __shfl_xor_sync(0xffffffffu, a.z, 1));
}
// y for this side from both sides' q (y_update_edge, grad_face.hpp:31-36)
__device__ __forceinline__ v3 pair_y(int side, const v3& q, const v3& ed, double w) {
  const v3 qo = shfl_pair(q);
  const v3 q1 = side ? qo : q, q2 = side ? q : qo;
  const double mismatch = dot(ed, sub(q2, q1));
  const v3 shift = mk(ed.x * mismatch, ed.y * mismatch, ed.z * mismatch);
  return side ? sub(q, scale(w, shift)) : add(q, scale(w, shift));
}
// 4 blocks per SM (64 registers; g_out is loaded after the first y so that
// fits): config 3 18.3 vs 19.0 ms, config 4 103 vs 107.5 ms per 10 iterations
// against one thread per edge at 3 blocks per SM (same box, interleaved runs).
// kAct: activity flags per interior edge (admm_active_flags, padded to a
// multiple of 16 bytes): a warp iteration covers 16 consecutive edges, and lane
// j of a warp looks at the 16 flags of the warp's j-th next iteration in one
// 16-byte load, so 32 iterations are screened per round trip and only the
// active ones run (in the same ascending order: the partial sums keep their
// bits).
template <bool kAct>
__global__ void __launch_bounds__(B, 4) k_face_lambda_pair(const int32_t* __restrict__ ef, const double* __restrict__ sa,
                                                        const double* __restrict__ wq, const double* __restrict__ gin,
                                                        const double* __restrict__ gout,
                                                        const double* __restrict__ edir, int64_t ni, double mu,
                                                        double* __restrict__ C, double* __restrict__ lam,
                                                        double* __restrict__ part, double* __restrict__ term,
                                                        const int32_t* __restrict__ halt,
                                                        const uint8_t* __restrict__ act) {
  if (*halt) return;
  double s = 0.0;
  const int side = threadIdx.x & 1;
  const int64_t n = 2 * ni, stride = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  // the whole warp steps together (the pair shuffles need every lane)
  const auto body = [&](int64_t k0) {
    const int64_t k = k0 + lane;
    const int64_t i = k >> 1;
    // n even: both lanes of a pair agree; an edge that stays zero is skipped (lambda, c, term keep their 0)
    const bool valid = k < n && (!kAct || act[i]);
    const int32_t f = valid ? ef[k] : 0;
    const double sf = valid ? sa[f] : 1.0;
    const double m = mu * sf, w = valid ? wq[k] : 0.0;
    const v3 ed = valid ? ld3(edir, i) : mk(0.0, 0.0, 0.0);
    const v3 lold = valid ? ld3(lam, k) : mk(0.0, 0.0, 0.0);
    const v3 gi = valid ? ld3(gin, f) : mk(0.0, 0.0, 0.0);
    // this iteration's y from g_in and the old lambda (grad_face.hpp:126-137)
    const v3 d = divs(lold, m);
    const v3 y = pair_y(side, sub(gi, d), ed, w);
    asm volatile("" ::: "memory");  // g_out's load after y: fewer live registers
    const v3 go = valid ? ld3(gout, f) : mk(0.0, 0.0, 0.0);
    // lambda += mu r, r = sqrt(A) (y - g) (grad_face.hpp:158-168)
    const v3 r = scale(sf, sub(y, go));
    const v3 l = add(lold, scale(mu, r));
    const double sq = sqnorm(r), sqo = __shfl_xor_sync(0xffffffffu, sq, 1);
    if (valid) {
      st3(lam, k, l);
      if (!side) {
        const double tt = sq + sqo;
        term[i] = tt;
        s += tt;
      }
    }
    // the next iteration's y and c = y + lambda / (mu sqrt(A)) from the same registers
    const v3 d2 = divs(l, m);
    const v3 y2 = pair_y(side, sub(go, d2), ed, w);
    if (valid) st3(C, k, add(y2, d2));
  };
  const int64_t first = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31);
  if (!kAct) {
    for (int64_t k0 = first; k0 < n; k0 += stride) body(k0);
  } else {
    for (int64_t base = first; base < n; base += 32 * stride) {
      const int64_t kk = base + lane * stride;  // the warp's k0 `lane` iterations from now
      bool any = false;
      if (kk < n) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(act + (kk >> 1)));
        any = (a.x | a.y | a.z | a.w) != 0;
      }
      for (unsigned msk = __ballot_sync(0xffffffffu, any); msk; msk &= msk - 1)
        body(base + (int64_t)(__ffs(msk) - 1) * stride);
    }
  }
  s = block_sum<B>(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// ---------------------------------------------------------------- edge ADMM
// ctor (grad_edge.hpp:84-89): z = H_f . e per corner, signs (mesh.hpp:81-83)
__global__ void k_edge_init_faces(const double* __restrict__ pos, const int32_t* __restrict__ faces,
                                  const int32_t* __restrict__ he_edge, const int32_t* __restrict__ edge_v,
                                  const double* __restrict__ h, int64_t nf, double* __restrict__ w,
                                  double* __restrict__ lam, int8_t* __restrict__ sgn,
                                  const uint8_t* __restrict__ act) {
  GRID_STRIDE(f, nf) {
    if (act && !act[f]) continue;  // w, lambda were zeroed
    const v3 hf = ld3(h, f);
    for (int k = 0; k < 3; ++k) {
      const int64_t hh = 3 * f + k;
      const int32_t e = he_edge[hh];
      const int32_t a = edge_v[2 * e], b = edge_v[2 * e + 1];
      w[hh] = dot(hf, sub(ld3(pos, b), ld3(pos, a)));
      lam[hh] = 0.0;
      sgn[hh] = faces[hh] == a ? (int8_t)1 : (int8_t)-1;
    }
  }
}

// target_sum in ascending halfedge order from 0.0; x = target_sum / deg (85-93)
__global__ void k_edge_init_edges(const int32_t* __restrict__ edge_he, const double* __restrict__ z, int64_t ne,
                                  double* __restrict__ tsum, double* __restrict__ x,
                                  const uint8_t* __restrict__ act) {
  GRID_STRIDE(e, ne) {
    if (act && !act[e]) continue;  // x was zeroed
    int32_t h0 = edge_he[2 * e], h1 = edge_he[2 * e + 1];
    if (h0 >= 0 && h1 >= 0 && h1 < h0) {
      const int32_t t = h0;
      h0 = h1;
      h1 = t;
    }
    double s = 0.0;
    int deg = 0;
    if (h0 >= 0) {
      s += z[h0];
      ++deg;
    }
    if (h1 >= 0) {
      s += z[h1];
      ++deg;
    }
    tsum[e] = s;
    x[e] = ddiv(s, (double)deg);
  }
}

// W-update for face f (grad_edge.hpp:131-141)
__device__ __forceinline__ void edge_w_update(int64_t f, const int32_t* __restrict__ he_edge,
                                              const double* __restrict__ x, const double l[3],
                                              const int8_t* __restrict__ sgn, double mu, double* __restrict__ w) {
  double v[3], dotv = 0.0;
  for (int k = 0; k < 3; ++k) {
    v[k] = x[he_edge[3 * f + k]] - ddiv(l[k], mu);
    dotv += (double)sgn[3 * f + k] * v[k];
  }
  const double shift = ddiv(dotv, 3.0);
  for (int k = 0; k < 3; ++k) w[3 * f + k] = v[k] - shift * (double)sgn[3 * f + k];
}

__global__ void k_edge_first_w(const int32_t* __restrict__ he_edge, const double* __restrict__ x,
                               const double* __restrict__ lam, const int8_t* __restrict__ sgn, int64_t nf, double mu,
                               double* __restrict__ w, const uint8_t* __restrict__ act) {
  GRID_STRIDE(f, nf) {
    if (act && !act[f]) continue;
    const double l[3] = {lam[3 * f], lam[3 * f + 1], lam[3 * f + 2]};
    edge_w_update(f, he_edge, x, l, sgn, mu, w);
  }
}

// X-update per edge (143-149) + dual partials (163-164, 117-123)
__global__ void k_edge_x(const int32_t* __restrict__ edge_he, const double* __restrict__ tsum,
                         const double* __restrict__ lam, const double* __restrict__ w, int64_t ne, double mu,
                         double* __restrict__ x, double* __restrict__ part, double* __restrict__ term,
                         const int32_t* __restrict__ halt, const uint8_t* __restrict__ act) {
  if (*halt) return;
  double s = 0.0;
  GRID_STRIDE(e, ne) {
    if (act && !act[e]) continue;
    const double xold = x[e];
    double sum = tsum[e];
    const int32_t h0 = edge_he[2 * e], h1 = edge_he[2 * e + 1];
    if (h0 >= 0) sum += lam[h0] + mu * w[h0];
    if (h1 >= 0) sum += lam[h1] + mu * w[h1];
    const double deg = (h0 >= 0 && h1 >= 0) ? 2.0 : 1.0;
    const double xn = ddiv(sum, deg * (1.0 + mu));
    x[e] = xn;
    const double d = xn - xold;
    const double tt = deg * d * d;
    term[e] = tt;
    s += tt;
  }
  s = block_sum<B>(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// lambda-update + primal (151-158), then the next W-update per face
__global__ void k_edge_lambda_w(const int32_t* __restrict__ he_edge, const double* __restrict__ x,
                                const int8_t* __restrict__ sgn, int64_t nf, double mu, double* __restrict__ w,
                                double* __restrict__ lam, double* __restrict__ part, double* __restrict__ term,
                                const int32_t* __restrict__ halt, const uint8_t* __restrict__ act) {
  if (*halt) return;
  double s = 0.0;
  GRID_STRIDE(f, nf) {
    if (act && !act[f]) continue;
    double l[3], rs = 0.0;
    for (int k = 0; k < 3; ++k) {
      const int64_t hh = 3 * f + k;
      const double r = w[hh] - x[he_edge[hh]];
      l[k] = lam[hh] + mu * r;
      lam[hh] = l[k];
      rs += r * r;
    }
    term[f] = rs;
    s += rs;
    edge_w_update(f, he_edge, x, l, sgn, mu, w);
  }
  s = block_sum<B>(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// Fixed-order sum of kReduceGrid partials by one 1024-thread block (the same
// order as k_reduce_block below).
__device__ double block_reduce_1024(const double* __restrict__ part, double* sh) {
  double s = 0.0;
  for (int i = threadIdx.x; i < (int)G; i += 1024) s += part[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int k = 512; k > 0; k >>= 1) {
    if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

// Stop rule of iteration `it` on the device: residual norms from the partials
// (primal = sqrt(sum), dual = mu sqrt(sum), grad_face.hpp:170-177 /
// grad_edge.hpp:163-170), recorded in hist[2 it], hist[2 it + 1]. halt = 1 when
// both thresholds are met, 2 when either norm is inside the guard band where
// the tree sum might decide differently from the reference's left-to-right sum
// (the host then decides from the exact sums), and stays 0 otherwise. Once set,
// the later iterations' kernels return at once, so the state is that of `it`.
__global__ void k_admm_stop(const double* __restrict__ part_primal, const double* __restrict__ part_dual, double mu,
                            double thr1, double thr2, double gp, double gd, int32_t it, double* __restrict__ hist,
                            double* __restrict__ halted_at, int32_t* __restrict__ halt) {
  __shared__ double sh[1024];
  if (*halt) return;
  const double sp = block_reduce_1024(part_primal, sh);
  const double sd = block_reduce_1024(part_dual, sh);
  if (threadIdx.x == 0) {
    const double primal = sqrt(sp), dual = mu * sqrt(sd);
    hist[2 * it] = primal;
    hist[2 * it + 1] = dual;
    const bool near1 = fabs(primal - thr1) <= gp * fmax(fabs(primal), thr1);
    const bool near2 = fabs(dual - thr2) <= gd * fmax(fabs(dual), thr2);
    const int32_t state = (near1 || near2) ? 2 : (primal <= thr1 && dual <= thr2) ? 1 : 0;
    if (state) {
      *halt = state;
      *halted_at = (double)it;  // read back with the history
    }
  }
}

void validate(const gh_admm_config& c) {
  if (c.max_iterations < 0) gh::fail(GH_ERR_INVALID, "AdmmConfig: max_iterations must be >= 0");
  if (!(c.eps1 > 0.0) || !(c.eps2 > 0.0)) gh::fail(GH_ERR_INVALID, "AdmmConfig: eps must be positive");
  if (!(c.mu > 0.0)) gh::fail(GH_ERR_INVALID, "AdmmConfig: mu must be positive");
}

}  // namespace

namespace {
__global__ void k_reduce_block(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) s += part[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int k = 512; k > 0; k >>= 1) {
    if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}
}  // namespace

void reduce_into(gh_mesh* m, const double* partials, double* slot) {
  k_reduce_block<<<1, 1024, 0, m->stream>>>(partials, (int)G, slot);
  GH_LAUNCH_CHECK();
  m->launches++;
}

namespace gh {

int32_t normalize_dev(gh_mesh* m, const double* d_u, double* d_h) {
  if (!m->nf) return 0;
  k_normalize<<<G, B, 0, m->stream>>>(m->pos.p, m->faces.p, m->face_normal.p, m->face_area.p, d_u, m->nf, d_h,
                                      m->partials.p);
  GH_LAUNCH_CHECK();
  m->launches++;
  reduce_into(m, m->partials.p, m->scalars.p + 4);
  double z = 0.0;
  GH_CUDA(cudaMemcpyAsync(&z, m->scalars.p + 4, sizeof(double), cudaMemcpyDeviceToHost, m->stream));
  GH_CUDA(cudaStreamSynchronize(m->stream));
  return (int32_t)z;
}

namespace {

// The stop rule primal <= scale*eps1 && dual <= scale*eps2 on the residual
// norms of the reference's left-to-right sums. The tree sums (already on the
// host) decide whenever both comparisons clear a guard band wider than the
// worst-case gap between the two summation orders ((n + 64) * 2^-52
// relative); inside the band the per-element terms are summed exactly in the
// reference's order (gh_seqsum.cu) and those values decide. So iteration
// counts and converged flags equal the reference's by construction; the
// reported residuals are the tree values (within ~1e-14 of the reference's)
// except where the band forced the exact sums.
double guard(int64_t n) { return (double)(n + 64) * 2.220446049250313e-16; }

bool stop_rule(gh_mesh* m, AdmmResult& res, int it, const gh_admm_config& cfg, double scale, double mu,
               double primal, double dual, const double* term_p, int64_t np, const double* term_d, int64_t nd) {
  const double thr1 = scale * cfg.eps1, thr2 = scale * cfg.eps2;
  const double gp = guard(np), gd = guard(nd);
  auto near = [](double v, double thr, double g) { return std::fabs(v - thr) <= g * std::fmax(std::fabs(v), thr); };
  if (near(primal, thr1, gp) || near(dual, thr2, gd)) {
    primal = std::sqrt(sequential_sum_nonneg(term_p, np, m->stream, &m->launches));
    dual = mu * std::sqrt(sequential_sum_nonneg(term_d, nd, m->stream, &m->launches));
  }
  const bool met = primal <= thr1 && dual <= thr2;
  res.primal.push_back(primal);
  res.dual.push_back(dual);
  res.final_primal = primal;
  res.final_dual = dual;
  res.iterations = it + 1;
  res.converged = met;
  (void)it;
  return met;
}

// The iteration loop without a host round trip per iteration: all remaining
// iterations are enqueued at once, each followed by k_admm_stop; the first
// iteration whose stop rule fires (or lands in the guard band) halts the rest
// on the device. One read-back then gives the history; a guard-band iteration
// is decided on the host from the exact sums (stop_rule) and the loop resumes
// after it if the thresholds are not met.
template <class Iterate>
void admm_loop(gh_mesh* m, AdmmResult& res, const gh_admm_config& cfg, double scale, double mu,
               const double* term_p, int64_t np, const double* term_d, int64_t nd, Iterate iterate) {
  constexpr int32_t kBatch = 16;  // iterations enqueued per host check (no-ops after a halt)
  const int32_t imax = cfg.max_iterations;
  if (imax <= 0) return;
  cudaStream_t s = m->stream;
  Scratch<double> hist(2 * (size_t)imax + 1, s);  // [primal, dual] per iteration, then the halting iteration
  Scratch<int32_t> halt(1, s);
  std::vector<double> h(2 * (size_t)imax + 1);
  const double thr1 = scale * cfg.eps1, thr2 = scale * cfg.eps2;
  int32_t it0 = 0;
  bool armed = false;
  while (it0 < imax) {
    if (!armed) GH_CUDA(cudaMemsetAsync(halt.p, 0, sizeof(int32_t), s));
    armed = true;
    const int32_t end = std::min(imax, it0 + kBatch);
    for (int32_t it = it0; it < end; ++it) {
      iterate(it, halt.p);
      k_admm_stop<<<1, 1024, 0, s>>>(m->partials.p + G, m->partials.p, mu, thr1, thr2, guard(np), guard(nd), it,
                                     hist.p, hist.p + 2 * (size_t)imax, halt.p);
      GH_LAUNCH_CHECK();
      m->launches += 3;
    }
    int32_t state = 0;
    GH_CUDA(cudaMemcpyAsync(h.data() + 2 * (size_t)it0, hist.p + 2 * (size_t)it0, sizeof(double) * 2 * (end - it0),
                            cudaMemcpyDeviceToHost, s));
    GH_CUDA(cudaMemcpyAsync(h.data() + 2 * (size_t)imax, hist.p + 2 * (size_t)imax, sizeof(double),
                            cudaMemcpyDeviceToHost, s));
    GH_CUDA(cudaMemcpyAsync(&state, halt.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    GH_CUDA(cudaStreamSynchronize(s));
    if (!state && end < imax) {  // the whole batch cleared both guard bands without meeting the rule
      for (int32_t it = it0; it < end; ++it) {
        res.primal.push_back(h[2 * it]);
        res.dual.push_back(h[2 * it + 1]);
      }
      it0 = end;
      continue;
    }
    const int32_t last = state ? (int32_t)h[2 * (size_t)imax] : imax - 1;  // iteration that halted (or the final one)
    for (int32_t it = it0; it < last; ++it) {
      res.primal.push_back(h[2 * it]);
      res.dual.push_back(h[2 * it + 1]);
    }
    if (stop_rule(m, res, last, cfg, scale, mu, h[2 * last], h[2 * last + 1], term_p, np, term_d, nd)) return;
    it0 = last + 1;
    armed = false;  // the guard-band halt is cleared before resuming
  }
}

}  // namespace

// ---------------------------------------------------------------- zero skipping
// The targets H are exactly +0 on every face whose heat gradient is below
// 1e-20 (diffusion.hpp:138-143) — all but the faces within ~100-150 rings of
// the sources at t = h^2. Both optimisers keep +0 where everything around is
// +0 (every update is a sum/difference/product/quotient of +0 operands with
// positive divisors: grad_face.hpp:31-36, 126-168; grad_edge.hpp:131-158), and a
// nonzero value moves by one face per iteration. With D(f) = the least BFS
// level of f's vertices (neighbouring faces differ by at most 1 in D), a face
// can differ from +0 after k iterations only if D(f) <= D_H + k, D_H = the
// largest D of a face with a nonzero target; an edge only if the lower level
// of its end points is <= D_H + k + 1. Elements past those bounds (+1 to
// spare) are skipped: their state is zero-filled once and their residual terms
// are 0, which a sum does not see.
namespace {

__global__ void k_target_front(const double* __restrict__ h, const int32_t* __restrict__ faces,
                               const int32_t* __restrict__ level, int64_t nf, int32_t* __restrict__ front) {
  int32_t best = -1;
  GRID_STRIDE(f, nf) {
    const v3 hf = ld3(h, f);
    if ((__double_as_longlong(hf.x) | __double_as_longlong(hf.y) | __double_as_longlong(hf.z)) == 0) continue;
    int32_t d = 0x7fffffff;
    for (int k = 0; k < 3; ++k) {
      const int32_t l = level[faces[3 * f + k]];
      d = l >= 0 && l < d ? l : d;
    }
    // a nonzero target on an unreachable face cannot happen (u = 0 there); if it did, every level is active
    best = d == 0x7fffffff ? 0x7ffffff0 : (d > best ? d : best);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const int32_t other = __shfl_down_sync(0xffffffffu, best, o);
    best = other > best ? other : best;
  }
  if ((threadIdx.x & 31) == 0 && best >= 0) atomicMax(front, best);
}

__global__ void k_active_faces(const int32_t* __restrict__ faces, const int32_t* __restrict__ level, int64_t nf,
                               int32_t bound, uint8_t* __restrict__ act) {
  GRID_STRIDE(f, nf) {
    bool on = false;
    for (int k = 0; k < 3; ++k) {
      const int32_t l = level[faces[3 * f + k]];
      on = on || (l >= 0 && l <= bound);
    }
    act[f] = on ? 1 : 0;
  }
}

// list == null: act[e] for every edge e; else act[i] for interior edge i = list[i]
__global__ void k_active_edges(const int32_t* __restrict__ list, const int32_t* __restrict__ edge_v,
                               const int32_t* __restrict__ level, int64_t n, int32_t bound, uint8_t* __restrict__ act) {
  GRID_STRIDE(i, n) {
    const int64_t e = list ? list[i] : i;
    const int32_t la = level[edge_v[2 * e]], lb = level[edge_v[2 * e + 1]];
    act[i] = ((la >= 0 && la <= bound) || (lb >= 0 && lb <= bound)) ? 1 : 0;
  }
}

}  // namespace

int32_t admm_active_level(gh_levels* L, const double* d_h, int32_t iterations) {
  gh_mesh* m = L->mesh;
  if (!zero_level_truncation() || iterations <= 0 || !m->nf || L->nreach <= 0) return -1;
  cudaStream_t s = m->stream;
  Scratch<int32_t> front(1, s);
  GH_CUDA(cudaMemsetAsync(front.p, 0xff, sizeof(int32_t), s));
  k_target_front<<<G, B, 0, s>>>(d_h, m->faces.p, L->level.p, m->nf, front.p);
  GH_LAUNCH_CHECK();
  m->launches++;
  int32_t dh = -1;
  GH_CUDA(cudaMemcpyAsync(&dh, front.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
  const int64_t bound = (int64_t)dh + iterations + 1;
  // worth it when the levels past the edges' bound hold at least 30 % of the vertices
  const int64_t lim = bound + 2;
  if (lim >= L->nlev || 10 * (int64_t)L->h_offsets[lim] > 7 * (int64_t)L->nreach) return -1;
  return (int32_t)bound;
}

void admm_active_flags(gh_levels* L, int32_t level_bound, bool interior_edges, uint8_t* act_f, uint8_t* act_e) {
  gh_mesh* m = L->mesh;
  cudaStream_t s = m->stream;
  k_active_faces<<<G, B, 0, s>>>(m->faces.p, L->level.p, m->nf, level_bound, act_f);
  const int64_t n = interior_edges ? m->ni : m->ne;
  if (n)
    k_active_edges<<<G, B, 0, s>>>(interior_edges ? m->interior_edges.p : nullptr, m->edge_v.p, L->level.p, n,
                                   level_bound + 1, act_e);
  GH_LAUNCH_CHECK();
  m->launches += 2;
}

AdmmResult admm_face_dev(gh_mesh* m, const double* d_h, const gh_admm_config& cfg, double* d_g, const uint8_t* act_f,
                         const uint8_t* act_e) {
  validate(cfg);
  cudaStream_t s = m->stream;
  const int64_t F = m->nf, NI = m->ni;
  const double mu = cfg.mu;
  AdmmResult res;
  Scratch<double> Cs(6 * NI + 6, s), lam(6 * NI + 6, s), edir(3 * NI + 3, s), gtmp(3 * F + 3, s);
  Scratch<int32_t> ef(2 * NI + 2, s), slot(3 * F + 3, s);
  res.state_bytes = sizeof(double) * (3 * F /*g*/ + 3 * F /*targets*/ + 15 * NI + F /*sqrt A*/ + 2 * NI /*w*/) +
                    sizeof(int32_t) * (2 * NI + 3 * F);
  double* part_dual = m->partials.p;  // admm_loop's k_admm_stop reads both halves
  double* part_primal = m->partials.p + G;
  EventTimer timer(s);
  timer.start();
  // g ping-pongs between d_g and gtmp: iteration it reads gbuf[(it + 1) & 1] and
  // writes gbuf[it & 1]; g = h starts in gbuf[1] (and in d_g for 0 iterations)
  double* gbuf[2] = {d_g, gtmp.p};
  GH_CUDA(cudaMemcpyAsync(d_g, d_h, sizeof(double) * 3 * F, cudaMemcpyDeviceToDevice, s));  // g = h
  GH_CUDA(cudaMemcpyAsync(gtmp.p, d_h, sizeof(double) * 3 * F, cudaMemcpyDeviceToDevice, s));
  if (F) k_face_slots<<<G, B, 0, s>>>(m->he_edge.p, m->interior_edge_index.p, m->edge_he.p, F, slot.p);
  Scratch<double> term_p(NI + 1, s), term_d(F + 1, s);  // per-element residual terms
  Scratch<double> sa(F + 1, s), wq(2 * NI + 2, s);  // per-solve constants (face_y_update)
  if (F) k_face_consts<<<G, B, 0, s>>>(m->face_area.p, F, sa.p);
  if (act_e) {
    // edges outside the active set (admm_active_level) keep lambda = c = +0 for
    // the whole solve, as in the reference; their terms stay 0 in both sums
    GH_CUDA(cudaMemsetAsync(lam.p, 0, sizeof(double) * 6 * NI, s));
    GH_CUDA(cudaMemsetAsync(Cs.p, 0, sizeof(double) * 6 * NI, s));
    GH_CUDA(cudaMemsetAsync(term_d.p, 0, sizeof(double) * F, s));
  }
  k_face_init_edges<<<G, B, 0, s>>>(m->pos.p, m->interior_edges.p, m->edge_v.p, m->edge_he.p, m->face_area.p, d_h,
                                    NI, mu, sa.p, edir.p, ef.p, wq.p, lam.p,
                                    cfg.max_iterations > 0 ? Cs.p : nullptr, part_primal, term_p.p, act_e);
  GH_LAUNCH_CHECK();
  m->launches += 3;
  // ||M||_F (grad_face.hpp:85): the reference's left-to-right sum, exactly
  const double scale = std::sqrt(sequential_sum_nonneg(term_p.p, NI, s, &m->launches));
  if (act_e) GH_CUDA(cudaMemsetAsync(term_p.p, 0, sizeof(double) * NI, s));  // from here on: primal terms
  // grad_face.hpp:175-177
  admm_loop(m, res, cfg, scale, mu, term_p.p, NI, term_d.p, F, [&](int32_t it, const int32_t* halt) {
    const double* gin = gbuf[(it + 1) & 1];
    double* gout = gbuf[it & 1];
    k_face_g<<<G, B, 0, s>>>(slot.p, m->face_area.p, d_h, Cs.p, F, mu, gin, gout, part_dual, term_d.p, halt, act_f);
    if (act_e)
      k_face_lambda_pair<true><<<G, B, 0, s>>>(ef.p, sa.p, wq.p, gin, gout, edir.p, NI, mu, Cs.p, lam.p, part_primal,
                                               term_p.p, halt, act_e);
    else
      k_face_lambda_pair<false><<<G, B, 0, s>>>(ef.p, sa.p, wq.p, gin, gout, edir.p, NI, mu, Cs.p, lam.p, part_primal,
                                                term_p.p, halt, nullptr);
  });
  // the last iteration's g: odd iterations wrote gtmp
  if (res.iterations > 0 && ((res.iterations - 1) & 1))
    GH_CUDA(cudaMemcpyAsync(d_g, gtmp.p, sizeof(double) * 3 * F, cudaMemcpyDeviceToDevice, s));
  timer.stop();
  res.device_ms = timer.ms();
  return res;
}

AdmmResult admm_edge_dev(gh_mesh* m, const double* d_h, const gh_admm_config& cfg, double* d_x, const uint8_t* act_f,
                         const uint8_t* act_e) {
  validate(cfg);
  cudaStream_t s = m->stream;
  const int64_t F = m->nf, E = m->ne;
  const double mu = cfg.mu;
  AdmmResult res;
  Scratch<double> w(3 * F + 3, s), lam(3 * F + 3, s), tsum(E + 1, s);
  Scratch<int8_t> sgn(3 * F + 3, s);
  res.state_bytes = sizeof(double) * (2 * E + 6 * F) + 3 * F;  // x, target_sum, w, lambda, sign
  double* part_dual = m->partials.p;  // admm_loop's k_admm_stop reads both halves
  double* part_primal = m->partials.p + G;
  const double scale = std::sqrt(3.0 * (double)F);  // ||R||_F (grad_edge.hpp:79)
  EventTimer timer(s);
  timer.start();
  Scratch<double> term_p(F + 1, s), term_d(E + 1, s);  // per-element residual terms
  if (act_f) {
    // faces and edges outside the active set (admm_active_level) keep w = lambda
    // = x = +0 for the whole solve, as in the reference (an active edge next to
    // such a face reads those zeros), and their terms stay 0 in both sums
    GH_CUDA(cudaMemsetAsync(w.p, 0, sizeof(double) * 3 * F, s));
    GH_CUDA(cudaMemsetAsync(lam.p, 0, sizeof(double) * 3 * F, s));
    GH_CUDA(cudaMemsetAsync(d_x, 0, sizeof(double) * E, s));
    GH_CUDA(cudaMemsetAsync(term_p.p, 0, sizeof(double) * F, s));
    GH_CUDA(cudaMemsetAsync(term_d.p, 0, sizeof(double) * E, s));
  }
  if (F)
    k_edge_init_faces<<<G, B, 0, s>>>(m->pos.p, m->faces.p, m->he_edge.p, m->edge_v.p, d_h, F, w.p, lam.p, sgn.p, act_f);
  if (E) k_edge_init_edges<<<G, B, 0, s>>>(m->edge_he.p, w.p, E, tsum.p, d_x, act_e);
  GH_LAUNCH_CHECK();
  m->launches += 2;
  if (cfg.max_iterations > 0 && F) {
    k_edge_first_w<<<G, B, 0, s>>>(m->he_edge.p, d_x, lam.p, sgn.p, F, mu, w.p, act_f);
    GH_LAUNCH_CHECK();
    m->launches++;
  }
  // grad_edge.hpp:168-170
  admm_loop(m, res, cfg, scale, mu, term_p.p, F, term_d.p, E, [&](int32_t, const int32_t* halt) {
    k_edge_x<<<G, B, 0, s>>>(m->edge_he.p, tsum.p, lam.p, w.p, E, mu, d_x, part_dual, term_d.p, halt, act_e);
    k_edge_lambda_w<<<G, B, 0, s>>>(m->he_edge.p, d_x, sgn.p, F, mu, w.p, lam.p, part_primal, term_p.p, halt, act_f);
  });
  timer.stop();
  res.device_ms = timer.ms();
  return res;
}

}  // namespace gh
