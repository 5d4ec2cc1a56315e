// The classic heat method on a CG backend:
// poisson_heat_method (reference.hpp:175-216) = Jacobi-preconditioned CG on
// the heat operator A - t*Lc (HeatOperator, reference.hpp:86-104), gradient
// normalisation, integrated divergence (reference.hpp:142-160), and CG on the
// reduced Poisson operator -Lc over the reachable non-source vertices
// (ReducedPoissonOperator, reference.hpp:107-139).
//
// The CG iteration (cg_solve, reference.hpp:35-84) runs device-driven: the
// scalars (alpha, beta, r.z, |r|) live in device memory, small single-block
// kernels compute them, every kernel of an iteration returns at once when the
// solve has finished, and a chunk of iterations is captured once as a CUDA
// graph and replayed until the host sees the done flag. Element values follow
// the reference's formulas exactly (-fmad=false); the dot products use the
// library's fixed-shape tree instead of the reference's left-to-right
// deterministic_sum (parallel.hpp:50-54), so iterates agree to rounding and
// iteration counts agree except when |r| lands within rounding of tol*|b|.

#include <chrono>
#include <cmath>

#include "gh_internal.cuh"

using namespace ghd;

namespace {

constexpr int B = gh::kBlock;
constexpr unsigned G = gh::kReduceGrid;
constexpr int kChunk = 16;  // CG iterations per captured graph

#define GRID_STRIDE(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

struct CgState {
  double rz, rhs_norm, alpha, beta, rnorm, curvature;
  int32_t done;  // 0 running, 1 converged, 2 breakdown
  int32_t iterations;
  int32_t max_iters;
  int32_t pad;
  double tol;
};

// Matrix-free operators over the mesh's vertex-vertex CSR (reference order).
struct HeatOp {  // y_j = A_j x_j - t * sum_i w_i (x_k - x_j)
  const int32_t *off, *idx;
  const double *w, *area, *wsum;
  double t;
  int64_t n;
  __device__ double apply(const double* x, int64_t j) const {
    double lap = 0.0;
    const double xj = x[j];
    for (int32_t i = off[j]; i < off[j + 1]; ++i) lap += w[i] * (x[idx[i]] - xj);
    return area[j] * xj - t * lap;
  }
  __device__ double diag(int64_t j) const { return area[j] + t * wsum[j]; }
};

struct ReducedOp {  // y_r = sum_i w_i (x_r - (x_rk or 0)) over the kept rows
  const int32_t *off, *idx, *subset, *reduced_of;
  const double *w, *wsum;
  int64_t n;
  __device__ double apply(const double* x, int64_t row) const {
    const int32_t j = subset[row];
    double sum = 0.0;
    const double xr = x[row];
    for (int32_t i = off[j]; i < off[j + 1]; ++i) {
      const int32_t rk = reduced_of[idx[i]];
      sum += w[i] * (xr - (rk >= 0 ? x[rk] : 0.0));
    }
    return sum;
  }
  __device__ double diag(int64_t row) const { return wsum[subset[row]]; }
};

template <class Op>
__global__ void k_cg_init(Op op, const double* __restrict__ rhs, double* __restrict__ x, double* __restrict__ r,
                          double* __restrict__ diag, double* __restrict__ z, double* __restrict__ p,
                          double* __restrict__ part_rz, double* __restrict__ part_rr) {
  double rz = 0.0, rr = 0.0;
  GRID_STRIDE(i, op.n) {
    const double ri = rhs[i], di = op.diag(i);
    const double zi = ddiv(ri, di);
    x[i] = 0.0;
    r[i] = ri;
    diag[i] = di;
    z[i] = zi;
    p[i] = zi;
    rz += ri * zi;
    rr += ri * ri;
  }
  rz = block_sum<B>(rz);
  rr = block_sum<B>(rr);
  if (threadIdx.x == 0) {
    part_rz[blockIdx.x] = rz;
    part_rr[blockIdx.x] = rr;
  }
}

// one block of 1024: the fixed tree of gh::reduce_partials
__device__ double reduce_fixed(const double* __restrict__ part, int n) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) s += part[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int k = 512; k > 0; k >>= 1) {
    if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
    __syncthreads();
  }
  const double out = sh[0];
  __syncthreads();
  return out;
}

__global__ void k_cg_start(const double* __restrict__ part_rz, const double* __restrict__ part_rr, CgState* st) {
  const double rz = reduce_fixed(part_rz, G);
  const double rr = reduce_fixed(part_rr, G);
  if (threadIdx.x == 0) {
    st->rz = rz;
    st->rhs_norm = sqrt(rr);
    st->rnorm = st->rhs_norm;
    st->iterations = 0;
    st->done = (st->rhs_norm == 0.0) ? 1 : (st->max_iters <= 0 ? 3 : 0);
  }
}

// q = Op p, partial p.q
template <class Op>
__global__ void k_cg_apply(Op op, const double* __restrict__ p, double* __restrict__ q, double* __restrict__ part,
                           const CgState* st) {
  if (st->done) return;
  double pq = 0.0;
  GRID_STRIDE(i, op.n) {
    const double qi = op.apply(p, i);
    q[i] = qi;
    pq += p[i] * qi;
  }
  pq = block_sum<B>(pq);
  if (threadIdx.x == 0) part[blockIdx.x] = pq;
}

__global__ void k_cg_alpha(const double* __restrict__ part, CgState* st) {
  if (st->done) return;
  const double curvature = reduce_fixed(part, G);
  if (threadIdx.x == 0) {
    st->curvature = curvature;
    if (!(curvature > 0.0) || !isfinite(curvature)) st->done = 2;
    else st->alpha = st->rz / curvature;
  }
}

// x += alpha p; r -= alpha q; z = r / diag; partials r.r and r.z
__global__ void k_cg_update(int64_t n, const double* __restrict__ p, const double* __restrict__ q,
                            const double* __restrict__ diag, double* __restrict__ x, double* __restrict__ r,
                            double* __restrict__ z, double* __restrict__ part_rr, double* __restrict__ part_rz,
                            const CgState* st) {
  if (st->done) return;
  const double alpha = st->alpha;
  double rr = 0.0, rz = 0.0;
  GRID_STRIDE(i, n) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    const double zi = ddiv(ri, diag[i]);
    z[i] = zi;
    rr += ri * ri;
    rz += ri * zi;
  }
  rr = block_sum<B>(rr);
  rz = block_sum<B>(rz);
  if (threadIdx.x == 0) {
    part_rr[blockIdx.x] = rr;
    part_rz[blockIdx.x] = rz;
  }
}

__global__ void k_cg_check(const double* __restrict__ part_rr, const double* __restrict__ part_rz, CgState* st) {
  if (st->done) return;
  const double rr = reduce_fixed(part_rr, G);
  const double rz_next = reduce_fixed(part_rz, G);
  if (threadIdx.x == 0) {
    const double rnorm = sqrt(rr);
    st->rnorm = rnorm;
    st->iterations += 1;
    if (!isfinite(rnorm)) {
      st->done = 2;
    } else if (rnorm <= st->tol * st->rhs_norm) {
      st->done = 1;
    } else if (st->iterations >= st->max_iters) {
      st->done = 3;  // iteration cap: not converged, not a breakdown
    } else {
      st->beta = rz_next / st->rz;
      st->rz = rz_next;
    }
  }
}

__global__ void k_cg_direction(int64_t n, const double* __restrict__ z, double* __restrict__ p, const CgState* st) {
  if (st->done) return;
  const double beta = st->beta;
  GRID_STRIDE(i, n) p[i] = z[i] + beta * p[i];
}

struct CgOut {
  int iterations = 0;
  double relative_residual = 0.0;
  bool converged = false, breakdown = false;
};

// cg_solve (reference.hpp:35-84) on the device; x receives the solution.
template <class Op>
CgOut cg_solve_dev(gh_mesh* m, const Op& op, const double* d_rhs, double tol, int64_t max_iters, double* d_x) {
  cudaStream_t s = m->stream;
  const int64_t n = op.n;
  CgOut out;
  if (n == 0) {
    out.converged = true;
    return out;
  }
  gh::Scratch<double> r(n, s), diag(n, s), z(n, s), p(n, s), q(n, s), part(4 * G, s);
  gh::Scratch<CgState> st(1, s);
  CgState init{};
  init.tol = tol;
  init.max_iters = (int32_t)std::min<int64_t>(max_iters, 0x7fffffff);
  GH_CUDA(cudaMemcpyAsync(st.p, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  double *p_a = part.p, *p_b = part.p + G;
  k_cg_init<Op><<<G, B, 0, s>>>(op, d_rhs, d_x, r.p, diag.p, z.p, p.p, p_a, p_b);
  k_cg_start<<<1, 1024, 0, s>>>(p_a, p_b, st.p);
  GH_LAUNCH_CHECK();
  m->launches += 2;

  auto enqueue = [&](int iters) {
    for (int k = 0; k < iters; ++k) {
      k_cg_apply<Op><<<G, B, 0, s>>>(op, p.p, q.p, p_a, st.p);
      k_cg_alpha<<<1, 1024, 0, s>>>(p_a, st.p);
      k_cg_update<<<G, B, 0, s>>>(n, p.p, q.p, diag.p, d_x, r.p, z.p, p_a, p_b, st.p);
      k_cg_check<<<1, 1024, 0, s>>>(p_a, p_b, st.p);
      k_cg_direction<<<G, B, 0, s>>>(n, z.p, p.p, st.p);
    }
  };
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  GH_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  enqueue(kChunk);
  GH_CUDA(cudaStreamEndCapture(s, &graph));
  GH_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  CgState h{};
  int64_t issued = 0;
  try {
    while (true) {
      GH_CUDA(cudaGraphLaunch(exec, s));
      m->launches += 5 * kChunk;
      issued += kChunk;
      GH_CUDA(cudaMemcpyAsync(&h, st.p, sizeof(h), cudaMemcpyDeviceToHost, s));
      GH_CUDA(cudaStreamSynchronize(s));
      if (h.done) break;
      if (issued > max_iters + kChunk) gh::fail(GH_ERR_INTERNAL, "cg: iteration cap not honoured");
    }
  } catch (...) {
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    throw;
  }
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  out.iterations = h.iterations;
  out.converged = h.done == 1;
  out.breakdown = h.done == 2;
  out.relative_residual = h.rnorm / h.rhs_norm;
  if (h.rhs_norm == 0.0) out.relative_residual = 0.0;
  return out;
}

// integrated_divergence (reference.hpp:142-160)
__global__ void k_divergence(const double* __restrict__ pos, const int32_t* __restrict__ faces,
                             const double* __restrict__ cot, const int32_t* __restrict__ vc_off,
                             const int32_t* __restrict__ vc_corner, const double* __restrict__ X, int64_t nv,
                             double* __restrict__ b) {
  GRID_STRIDE(v, nv) {
    double sum = 0.0;
    for (int32_t ci = vc_off[v]; ci < vc_off[v + 1]; ++ci) {
      const int32_t h = vc_corner[ci];
      const int32_t f = h / 3, k = h % 3;
      const int32_t t[3] = {faces[3 * f], faces[3 * f + 1], faces[3 * f + 2]};
      const v3 p = ld3(pos, t[k]);
      const v3 e1 = sub(ld3(pos, t[(k + 1) % 3]), p);
      const v3 e2 = sub(ld3(pos, t[(k + 2) % 3]), p);
      const v3 xf = ld3(X, f);
      sum += cot[3 * f + k] * dot(e1, xf) + cot[3 * f + (k + 2) % 3] * dot(e2, xf);
    }
    b[v] = 0.5 * sum;
  }
}

__global__ void k_heat_rhs(const int32_t* __restrict__ order, int32_t n0, double* __restrict__ u0) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n0; i += gridDim.x * blockDim.x) u0[order[i]] = 1.0;
}

// keep = level > 0 (reachable non-source): flags for the stable compaction
__global__ void k_keep(const int32_t* __restrict__ level, int64_t nv, int32_t* __restrict__ flag) {
  GRID_STRIDE(v, nv) flag[v] = level[v] > 0 ? 1 : 0;
}

__global__ void k_reduced_map(const int32_t* __restrict__ flag, const int32_t* __restrict__ scan, int64_t nv,
                              int32_t* __restrict__ subset, int32_t* __restrict__ reduced_of,
                              const double* __restrict__ b, double* __restrict__ rhs) {
  GRID_STRIDE(v, nv) {
    if (flag[v]) {
      const int32_t row = scan[v];
      subset[row] = (int32_t)v;
      reduced_of[v] = row;
      rhs[row] = -b[v];
    } else {
      reduced_of[v] = -1;
    }
  }
}

__global__ void k_poisson_out(const int32_t* __restrict__ level, const int32_t* __restrict__ reduced_of,
                              const double* __restrict__ x, int64_t nv, double* __restrict__ d) {
  GRID_STRIDE(v, nv) {
    const int32_t lv = level[v];
    d[v] = lv == 0 ? 0.0 : (reduced_of[v] >= 0 ? x[reduced_of[v]] : INFINITY);
  }
}

}  // namespace

// exclusive scan used by the compaction (CUB, gh_bfs.cu / gh_band.cu style)
#include <cub/device/device_scan.cuh>

namespace gh {

PoissonOut poisson_heat_dev(gh_levels* L, double t, double tol, double* d_d) {
  gh_mesh* m = L->mesh;
  cudaStream_t s = m->stream;
  const int64_t nv = m->nv;
  PoissonOut out;
  auto t0 = std::chrono::steady_clock::now();
  Scratch<double> u0(nv, s), u(nv, s);
  GH_CUDA(cudaMemsetAsync(u0.p, 0, sizeof(double) * nv, s));
  const int32_t n0 = L->h_offsets.size() > 1 ? L->h_offsets[1] : 0;
  if (n0) k_heat_rhs<<<grid_for(n0), B, 0, s>>>(L->order.p, n0, u0.p);
  m->launches++;
  HeatOp heat{m->vv_offset.p, m->vv_index.p, m->vv_weight.p, m->vertex_area.p, m->vertex_weight_sum.p, t, nv};
  CgOut hs = cg_solve_dev(m, heat, u0.p, tol, 20 * nv + 100, u.p);
  if (hs.breakdown) fail(GH_ERR_SOLVER, "poisson_heat_method: CG breakdown in the heat solve");
  out.heat_iterations = hs.iterations;
  out.heat_residual = hs.relative_residual;
  auto t1 = std::chrono::steady_clock::now();
  out.heat_seconds = std::chrono::duration<double>(t1 - t0).count();

  Scratch<double> H(3 * (size_t)m->nf + 3, s), bdiv(nv, s);
  normalize_dev(m, u.p, H.p);
  k_divergence<<<grid_for(nv), B, 0, s>>>(m->pos.p, m->faces.p, m->he_cot.p, m->vc_offset.p, m->vc_corner.p, H.p, nv,
                                          bdiv.p);
  m->launches++;
  Scratch<int32_t> flag(nv + 1, s), scan(nv + 1, s), subset(nv + 1, s), reduced_of(nv + 1, s);
  Scratch<double> rhs(nv + 1, s), x(nv + 1, s);
  k_keep<<<grid_for(nv), B, 0, s>>>(L->level.p, nv, flag.p);
  m->launches++;
  GH_CUDA(cudaMemsetAsync(flag.p + nv, 0, sizeof(int32_t), s));
  size_t tmp_bytes = 0;
  GH_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flag.p, scan.p, (int)(nv + 1), s));
  {
    Scratch<unsigned char> tmp(tmp_bytes, s);
    GH_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, flag.p, scan.p, (int)(nv + 1), s));
  }
  int32_t nred = 0;
  GH_CUDA(cudaMemcpyAsync(&nred, scan.p + nv, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  k_reduced_map<<<grid_for(nv), B, 0, s>>>(flag.p, scan.p, nv, subset.p, reduced_of.p, bdiv.p, rhs.p);
  m->launches++;
  GH_CUDA(cudaStreamSynchronize(s));
  ReducedOp pois{m->vv_offset.p, m->vv_index.p, subset.p, reduced_of.p, m->vv_weight.p, m->vertex_weight_sum.p, nred};
  CgOut ps = cg_solve_dev(m, pois, rhs.p, tol, 40 * nv + 100, x.p);
  if (ps.breakdown) fail(GH_ERR_SOLVER, "poisson_heat_method: CG breakdown in the Poisson solve");
  out.poisson_iterations = ps.iterations;
  out.poisson_residual = ps.relative_residual;
  k_poisson_out<<<grid_for(nv), B, 0, s>>>(L->level.p, reduced_of.p, x.p, nv, d_d);
  GH_LAUNCH_CHECK();
  m->launches++;
  GH_CUDA(cudaStreamSynchronize(s));
  out.poisson_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
  return out;
}

}  // namespace gh
