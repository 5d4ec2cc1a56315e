// The reference's evaluation layer on the device, for the CLI drop-in
// (tools/geoheat.cpp:71-100, 164-181, 265-275):
//   triangulation_quality   mesh.hpp:297-310
//   midpoint_subdivide      subdivide.hpp:14-44
//   analytic_oracle         reference.hpp:283-321
//   dijkstra_edge_distance  reference.hpp:220-245
//   mean_relative_error     reference.hpp:250-266
//   recovery_error          reference.hpp:269-276
// Per-element values follow the reference formulas (-fmad=false), and the
// sums of non-negative terms (tau, the sphere's radius, both error metrics)
// are the reference's left-to-right sums bit for bit (gh_seqsum.cu); only
// the sphere's centre (a signed sum of positions) is a fixed-shape tree, so
// the sphere oracle agrees to rounding. Plane and Dijkstra distances and
// subdivided meshes are bit-identical.

#include <cmath>

#include "gh_internal.cuh"

using namespace ghd;

namespace {

constexpr int B = gh::kBlock;
constexpr unsigned G = gh::kReduceGrid;

#define GRID_STRIDE(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

template <class T>
T read_scalar(const T* d, cudaStream_t s) {
  T v;
  GH_CUDA(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
  return v;
}

__global__ void k_quality_terms(const double* __restrict__ pos, const int32_t* __restrict__ faces,
                                const double* __restrict__ area, int64_t nf, double* __restrict__ term) {
  const double k = 2.0 * sqrt(3.0);
  GRID_STRIDE(f, nf) {
    const v3 p0 = ld3(pos, faces[3 * f]), p1 = ld3(pos, faces[3 * f + 1]), p2 = ld3(pos, faces[3 * f + 2]);
    const double a = ghd::norm(sub(p1, p2)), b = ghd::norm(sub(p2, p0)), c = ghd::norm(sub(p0, p1));
    const double s = 0.5 * ((a + b) + c);
    const double inradius = area[f] / s;
    const double longest = fmax(fmax(a, b), c);  // std::max({a, b, c}) on finite lengths
    term[f] = k * inradius / longest;
  }
}

// subdivide.hpp:14-36: originals, then one midpoint per edge in edge order;
// four faces per face.
__global__ void k_subdivide(const double* __restrict__ pos, const int32_t* __restrict__ faces,
                            const int32_t* __restrict__ he_edge, const int32_t* __restrict__ edge_v, int64_t nv,
                            int64_t nf, int64_t ne, double* __restrict__ pos2, int32_t* __restrict__ faces2) {
  GRID_STRIDE(v, nv) st3(pos2, v, ld3(pos, v));
  GRID_STRIDE(e, ne) {
    const v3 a = ld3(pos, edge_v[2 * e]), b = ld3(pos, edge_v[2 * e + 1]);
    st3(pos2, nv + e, scale(0.5, add(a, b)));
  }
  GRID_STRIDE(f, nf) {
    const int32_t t0 = faces[3 * f], t1 = faces[3 * f + 1], t2 = faces[3 * f + 2];
    const int32_t m01 = (int32_t)nv + he_edge[3 * f], m12 = (int32_t)nv + he_edge[3 * f + 1];
    const int32_t m20 = (int32_t)nv + he_edge[3 * f + 2];
    const int32_t out[12] = {t0, m01, m20, m01, t1, m12, m20, m12, t2, m01, m12, m20};
    for (int k = 0; k < 12; ++k) faces2[12 * f + k] = out[k];
  }
}

__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }  // std::min(a, b)

// plane: d[v] = min over sources of |p_v - p_s|; flags off-plane vertices
__global__ void k_plane(const double* __restrict__ pos, int64_t nv, const int32_t* __restrict__ src, int32_t ns,
                        double z0, double tol, double* __restrict__ d, int32_t* __restrict__ bad) {
  GRID_STRIDE(v, nv) {
    const v3 p = ld3(pos, v);
    if (fabs(p.z - z0) > tol) atomicExch(bad, 1);
    double best = INFINITY;
    for (int32_t i = 0; i < ns; ++i) best = dmin(best, ghd::norm(sub(p, ld3(pos, src[i]))));
    d[v] = best;
  }
}

__global__ void k_bbox(const double* __restrict__ pos, int64_t nv, double* __restrict__ part) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  GRID_STRIDE(v, nv) {
    for (int k = 0; k < 3; ++k) {
      const double x = pos[3 * v + k];
      lo[k] = fmin(lo[k], x);  // cwiseMin / cwiseMax on finite input
      hi[k] = fmax(hi[k], x);
    }
  }
  __shared__ double sh[6][B];
  for (int k = 0; k < 3; ++k) {
    sh[k][threadIdx.x] = lo[k];
    sh[3 + k][threadIdx.x] = hi[k];
  }
  __syncthreads();
  for (int o = B / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int k = 0; k < 3; ++k) {
        sh[k][threadIdx.x] = fmin(sh[k][threadIdx.x], sh[k][threadIdx.x + o]);
        sh[3 + k][threadIdx.x] = fmax(sh[3 + k][threadIdx.x], sh[3 + k][threadIdx.x + o]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) part[6 * blockIdx.x + k] = sh[k][0];
}

__global__ void k_bbox_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double r[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int b = 0; b < n; ++b)
    for (int k = 0; k < 3; ++k) {
      r[k] = fmin(r[k], part[6 * b + k]);
      r[3 + k] = fmax(r[3 + k], part[6 * b + 3 + k]);
    }
  for (int k = 0; k < 6; ++k) out[k] = r[k];
}

// sphere: component sums of the positions (centre), then of |p - c| (radius)
__global__ void k_sum3(const double* __restrict__ pos, int64_t nv, double* __restrict__ part) {
  double s[3] = {0.0, 0.0, 0.0};
  GRID_STRIDE(v, nv) for (int k = 0; k < 3; ++k) s[k] += pos[3 * v + k];
  for (int k = 0; k < 3; ++k) {
    const double r = block_sum<B>(s[k]);
    if (threadIdx.x == 0) part[k * G + blockIdx.x] = r;
  }
}

__global__ void k_radius_terms(const double* __restrict__ pos, int64_t nv, v3 c, double* __restrict__ term) {
  GRID_STRIDE(v, nv) term[v] = ghd::norm(sub(ld3(pos, v), c));
}

__global__ void k_sphere(const double* __restrict__ pos, int64_t nv, const int32_t* __restrict__ src, int32_t ns,
                         v3 c, double radius, double* __restrict__ d, int32_t* __restrict__ bad) {
  GRID_STRIDE(v, nv) {
    const v3 pc = sub(ld3(pos, v), c);
    if (fabs(ghd::norm(pc) - radius) > 1e-6 * radius) atomicExch(bad, 1);
    const v3 pv = normalized(pc);
    double best = INFINITY;
    for (int32_t i = 0; i < ns; ++i) {
      const v3 ps = normalized(sub(ld3(pos, src[i]), c));
      const double cosine = fmin(fmax(dot(pv, ps), -1.0), 1.0);  // std::clamp
      best = dmin(best, radius * acos(cosine));
    }
    d[v] = best;
  }
}

// ---- Dijkstra by label-correcting relaxation: distances are non-negative,
// so their bit patterns order like the values and atomicMin on them finds
// the same fixed point d[w] = min_v fl(d[v] + |p_w - p_v|) Dijkstra settles.
__global__ void k_dij_init(int64_t nv, unsigned long long* __restrict__ d, int32_t* __restrict__ front) {
  GRID_STRIDE(v, nv) {
    d[v] = 0x7ff0000000000000ull;  // +inf
    front[v] = 0;
  }
}

__global__ void k_dij_sources(const int32_t* __restrict__ src, int32_t ns, unsigned long long* __restrict__ d,
                              int32_t* __restrict__ front) {
  for (int i = threadIdx.x; i < ns; i += blockDim.x) {
    d[src[i]] = 0ull;
    front[src[i]] = 1;
  }
}

__global__ void k_dij_relax(const double* __restrict__ pos, const int32_t* __restrict__ off,
                            const int32_t* __restrict__ idx, int64_t nv, unsigned long long* d,
                            const int32_t* __restrict__ front, int32_t* __restrict__ next, int32_t* __restrict__ any) {
  GRID_STRIDE(v, nv) {
    if (!front[v]) continue;
    const double dv = __longlong_as_double((long long)d[v]);
    const v3 pv = ld3(pos, v);
    for (int32_t i = off[v]; i < off[v + 1]; ++i) {
      const int32_t w = idx[i];
      const double cand = dv + ghd::norm(sub(ld3(pos, w), pv));
      const unsigned long long cb = (unsigned long long)__double_as_longlong(cand);
      if (cb < d[w] && atomicMin(&d[w], cb) > cb) {
        next[w] = 1;
        *any = 1;
      }
    }
  }
}

__global__ void k_clear(int64_t n, int32_t* __restrict__ a) {
  GRID_STRIDE(i, n) a[i] = 0;
}

// mean_relative_error / recovery_error terms (zeros where the reference skips
// a vertex: adding +0 to a non-negative running sum changes nothing)
__global__ void k_error_terms(const double* __restrict__ d, const double* __restrict__ r,
                              const uint8_t* __restrict__ is_src, int64_t n, double* __restrict__ mre_t,
                              double* __restrict__ e2_t, int32_t* __restrict__ skipped) {
  int32_t sk = 0;
  GRID_STRIDE(v, n) {
    const double diff = d[v] - r[v];
    e2_t[v] = diff * diff;
    double m = 0.0;
    if (!is_src[v]) {
      if (r[v] == 0.0 || !isfinite(r[v]) || !isfinite(d[v])) ++sk;
      else m = fabs(d[v] - r[v]) / fabs(r[v]);
    }
    mre_t[v] = m;
  }
  if (sk) atomicAdd(skipped, sk);
}

__global__ void k_mark_sources(const int32_t* __restrict__ src, int32_t ns, int64_t n, uint8_t* __restrict__ f) {
  for (int i = threadIdx.x; i < ns; i += blockDim.x)
    if (src[i] >= 0 && src[i] < n) f[src[i]] = 1;
}

}  // namespace

namespace gh {

double triangulation_quality_dev(gh_mesh* m) {
  Scratch<double> term(m->nf, m->stream);
  k_quality_terms<<<grid_for(m->nf), B, 0, m->stream>>>(m->pos.p, m->faces.p, m->face_area.p, m->nf, term.p);
  GH_LAUNCH_CHECK();
  m->launches++;
  return sequential_sum_nonneg(term.p, m->nf, m->stream, &m->launches) / (double)m->nf;
}

void subdivide_once(gh_mesh* src, gh_mesh* dst) {
  cudaStream_t s = dst->stream;
  const int64_t nv = src->nv, nf = src->nf, ne = src->ne;
  if (nv + ne > 0x7fffffffLL || 12 * nf > 0x7fffffffLL) fail(GH_ERR_INVALID, "midpoint_subdivide: mesh too large");
  GH_CUDA(cudaStreamSynchronize(src->stream));
  dst->nv = (int32_t)(nv + ne);
  dst->nf = (int32_t)(4 * nf);
  dst->pos.alloc(3 * (size_t)(nv + ne), s);
  dst->faces.alloc(12 * (size_t)nf, s);
  k_subdivide<<<grid_for(std::max(nv + ne, nf)), B, 0, s>>>(src->pos.p, src->faces.p, src->he_edge.p, src->edge_v.p,
                                                             nv, nf, ne, dst->pos.p, dst->faces.p);
  GH_LAUNCH_CHECK();
  dst->launches++;
  mesh_build(dst, nullptr, nullptr);
}

void copy_mesh_arrays(gh_mesh* src, gh_mesh* dst) {
  cudaStream_t s = dst->stream;
  GH_CUDA(cudaStreamSynchronize(src->stream));
  dst->nv = src->nv;
  dst->nf = src->nf;
  dst->pos.alloc(3 * (size_t)src->nv, s);
  dst->faces.alloc(3 * (size_t)src->nf, s);
  if (src->nv)
    GH_CUDA(cudaMemcpyAsync(dst->pos.p, src->pos.p, 24 * (size_t)src->nv, cudaMemcpyDeviceToDevice, s));
  if (src->nf)
    GH_CUDA(cudaMemcpyAsync(dst->faces.p, src->faces.p, 12 * (size_t)src->nf, cudaMemcpyDeviceToDevice, s));
  mesh_build(dst, nullptr, nullptr);
}

void analytic_dev(gh_mesh* m, int kind, const int32_t* d_src, int32_t ns, double* d_out) {
  cudaStream_t s = m->stream;
  const int64_t nv = m->nv;
  Scratch<int32_t> bad(1, s);
  GH_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int32_t), s));
  if (kind == 0) {
    Scratch<double> part(6 * (size_t)G, s), box(6, s);
    k_bbox<<<G, B, 0, s>>>(m->pos.p, nv, part.p);
    k_bbox_final<<<1, 32, 0, s>>>(part.p, (int)G, box.p);
    m->launches += 2;
    double bx[6];
    GH_CUDA(cudaMemcpyAsync(bx, box.p, sizeof(bx), cudaMemcpyDeviceToHost, s));
    double z0 = 0.0;
    if (nv) GH_CUDA(cudaMemcpyAsync(&z0, m->pos.p + 2, sizeof(double), cudaMemcpyDeviceToHost, s));
    GH_CUDA(cudaStreamSynchronize(s));
    const double dx = bx[3] - bx[0], dy = bx[4] - bx[1], dz = bx[5] - bx[2];
    const double scale = std::sqrt((dx * dx + dy * dy) + dz * dz);
    k_plane<<<grid_for(nv), B, 0, s>>>(m->pos.p, nv, d_src, ns, z0, 1e-6 * scale, d_out, bad.p);
    m->launches++;
    if (read_scalar(bad.p, s)) fail(GH_ERR_INVALID, "analytic_oracle: mesh is not planar (z = const)");
    return;
  }
  Scratch<double> part(3 * (size_t)G, s), sums(4, s);
  k_sum3<<<G, B, 0, s>>>(m->pos.p, nv, part.p);
  m->launches++;
  double* slot = m->scalars.p + 13;
  double c3[3];
  for (int k = 0; k < 3; ++k) {
    GH_CUDA(cudaMemcpyAsync(m->partials.p, part.p + k * G, sizeof(double) * G, cudaMemcpyDeviceToDevice, s));
    reduce_partials(m, slot);
    c3[k] = read_scalar(slot, s) / (double)nv;
  }
  const v3 c{c3[0], c3[1], c3[2]};
  Scratch<double> term(nv, s);
  k_radius_terms<<<grid_for(nv), B, 0, s>>>(m->pos.p, nv, c, term.p);
  m->launches++;
  const double radius = sequential_sum_nonneg(term.p, nv, s, &m->launches) / (double)nv;
  k_sphere<<<grid_for(nv), B, 0, s>>>(m->pos.p, nv, d_src, ns, c, radius, d_out, bad.p);
  m->launches++;
  if (read_scalar(bad.p, s)) fail(GH_ERR_INVALID, "analytic_oracle: mesh vertices are not on a common sphere");
}

void dijkstra_dev(gh_mesh* m, const int32_t* d_src, int32_t ns, double* d_out) {
  cudaStream_t s = m->stream;
  const int64_t nv = m->nv;
  if (!nv) return;
  unsigned long long* d = reinterpret_cast<unsigned long long*>(d_out);
  Scratch<int32_t> fa(nv, s), fb(nv, s), any(1, s);
  k_dij_init<<<grid_for(nv), B, 0, s>>>(nv, d, fa.p);
  k_dij_sources<<<1, 256, 0, s>>>(d_src, ns, d, fa.p);
  k_clear<<<grid_for(nv), B, 0, s>>>(nv, fb.p);
  m->launches += 3;
  int32_t* front = fa.p;
  int32_t* next = fb.p;
  for (int64_t round = 0;; ++round) {
    GH_CUDA(cudaMemsetAsync(any.p, 0, sizeof(int32_t), s));
    k_dij_relax<<<grid_for(nv), B, 0, s>>>(m->pos.p, m->vv_offset.p, m->vv_index.p, nv, d, front, next, any.p);
    k_clear<<<grid_for(nv), B, 0, s>>>(nv, front);
    m->launches += 2;
    if (read_scalar(any.p, s) == 0) break;
    std::swap(front, next);
    if (round > 4 * nv + 16) fail(GH_ERR_INTERNAL, "dijkstra_edge_distance: relaxation did not settle");
  }
}

void errors_dev(cudaStream_t s, const double* d, const double* r, int64_t n, const int32_t* src, int32_t ns,
                double* mre, int32_t* excluded, double* e2) {
  Scratch<double> dd(n, s), rr(n, s), mt(n, s), et(n, s);
  Scratch<uint8_t> is_src(n, s);
  Scratch<int32_t> ds(ns, s), sk(1, s);
  GH_CUDA(cudaMemcpyAsync(dd.p, d, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  GH_CUDA(cudaMemcpyAsync(rr.p, r, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  GH_CUDA(cudaMemsetAsync(is_src.p, 0, n, s));
  GH_CUDA(cudaMemsetAsync(sk.p, 0, sizeof(int32_t), s));
  if (ns) {
    GH_CUDA(cudaMemcpyAsync(ds.p, src, sizeof(int32_t) * ns, cudaMemcpyHostToDevice, s));
    k_mark_sources<<<1, 256, 0, s>>>(ds.p, ns, n, is_src.p);
  }
  k_error_terms<<<grid_for(n), B, 0, s>>>(dd.p, rr.p, is_src.p, n, mt.p, et.p, sk.p);
  GH_LAUNCH_CHECK();
  // left-to-right sums as the reference (reference.hpp:250-276); the e2 terms
  // may be inf/nan when a field is infinite, which takes the ordered path
  *mre = deterministic_sum_dev(mt.p, n, s) / (double)n;
  *e2 = std::sqrt(deterministic_sum_dev(et.p, n, s)) / (double)n;
  *excluded = read_scalar(sk.p, s);
}

}  // namespace gh
