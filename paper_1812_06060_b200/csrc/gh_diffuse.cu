// Breadth-first Gauss-Seidel heat diffusion, gs_diffuse (reference
// diffusion.hpp:57-124), sweep-pipelined for sm_100a.
//
// Reference semantics: sweep s visits levels D_0, D_1, ... in order; the
// update of j in D_L reads u^s of level L-1 and u^(s-1) of levels L and L+1
// ("Jacobi within a level, Gauss-Seidel across levels", diffusion.hpp:74-83).
//
// Pipelining: write task U(s, L) into buffer (s & 1), read
// level L-1 from buffer (s & 1) and levels L, L+1 from buffer ((s-1) & 1).
// Then all tasks with L + 2s = tau are independent and every read-after-write
// crosses a step boundary, so one grid barrier per step tau replaces the
// reference's two barriers per (sweep, level): nlev + 2(S-1) barriers in all
// instead of 2 * nlev * S. Operand values, and their summation order within a
// row, are exactly the reference's, so u is bit-identical.
//
// Row order inside the kernel is (level parity, level, original index), so
// the active rows of a step are one contiguous range; the CSR is SELL-32.

#include <cooperative_groups.h>

#include <algorithm>

#include "gh_internal.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int B = gh::kBlock;
constexpr int kMaxSmemLevels = 12 * 1024;  // pend table in shared memory (48 KB)

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

struct DiffuseArgs {
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
  int32_t nlev;
  int32_t sweeps;
  double t;
};

template <bool kSmemTable>
__global__ void __launch_bounds__(B) k_diffuse_pipelined(DiffuseArgs a) {
  extern __shared__ int32_t sh_pend[];
  cg::grid_group grid = cg::this_grid();
  const int32_t* pend = a.pend;
  if (kSmemTable) {
    for (int i = threadIdx.x; i < a.nlev; i += blockDim.x) sh_pend[i] = a.pend[i];
    __syncthreads();
    pend = sh_pend;
  }
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nsteps = (int64_t)(a.nlev - 1) + 2 * (int64_t)(a.sweeps - 1) + 1;
  const double t = a.t;

  for (int64_t tau = 0; tau < nsteps; ++tau) {
    // active levels: L = tau - 2s, 0 <= s < S, 0 <= L < nlev, all of parity tau & 1
    int64_t lhi = tau < a.nlev - 1 ? tau : a.nlev - 1;
    if ((lhi ^ tau) & 1) --lhi;
    int64_t llo = tau - 2 * (int64_t)(a.sweeps - 1);
    if (llo < 0) llo = tau & 1;
    if (llo <= lhi) {
      const int64_t rb = a.pstart[llo], re = pend[lhi];
      const int64_t c0 = rb >> 5, c1 = (re + 31) >> 5;
      for (int64_t c = c0 + warp; c < c1; c += nwarps) {
        const int64_t r = c * 32 + lane;
        if (r < rb || r >= re) continue;
        int32_t L = __ldg(a.chunk_level + c);
        while (r >= pend[L]) L += 2;
        const int32_t sweep = (int32_t)((tau - L) >> 1);
        double* cur = a.ubuf + (sweep & 1) * a.nrows;
        const double* prev = a.ubuf + ((sweep & 1) ^ 1) * a.nrows;
        const int32_t d = __ldg(a.deg + r);
        const int64_t base = __ldg(a.chunk_ptr + c) + lane;
        double num = 0.0;
        for (int32_t k = 0; k < d; ++k) {
          const int32_t cc = __ldg(a.col + base + 32 * (int64_t)k);
          const double w = __ldg(a.wt + base + 32 * (int64_t)k);
          const double* src = cc < 0 ? cur : prev;
          num += w * __ldcg(src + (cc & 0x7fffffff));  // diffusion.hpp:79
        }
        const double u0 = L == 0 ? 1.0 : 0.0;
        __stcg(cur + r, (u0 + t * num) / __ldg(a.den + r));  // diffusion.hpp:82
      }
    }
    grid.sync();
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
    DiffuseArgs a{L->pstart.p, L->pend.p, L->chunk_level.p, L->chunk_ptr.p, L->deg.p, L->col.p, L->wt.p, L->den.p,
                  L->ubuf.p, L->nrows, L->nlev, sweeps, t};
    const bool smem = L->nlev <= kMaxSmemLevels;
    void* fn = smem ? (void*)k_diffuse_pipelined<true> : (void*)k_diffuse_pipelined<false>;
    const size_t shmem = smem ? sizeof(int32_t) * (size_t)L->nlev : 0;
    int nsm = 0, per_sm = 0;
    GH_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device));
    GH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, B, shmem));
    if (per_sm < 1) fail(GH_ERR_CUDA, "diffusion kernel cannot be resident");
    const int grid = nsm * per_sm;
    void* args[] = {&a};
    EventTimer timer(s);
    timer.start();
    GH_CUDA(cudaLaunchCooperativeKernel(fn, grid, B, args, shmem, s));
    GH_LAUNCH_CHECK();
    timer.stop();
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
