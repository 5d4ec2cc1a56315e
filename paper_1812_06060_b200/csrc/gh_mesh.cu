// Device mesh preprocessing: the solver-relevant part of build_mesh
// (reference mesh.hpp:113-286), average_edge_length (289-293) and
// face_gradient (314-327), as sm_100a kernels.
//
// Every per-element value is produced with the reference's operation order
// (no FMA; sequential per-row sums in the reference's row order), so the
// device TriMesh arrays equal the reference's bit for bit. Orders that the
// reference gets from std::sort are produced by stable radix sorts:
//   edges      : halfedge keys (vmin, vmax) stable-sorted over h ascending
//   vc CSR     : corners stable-sorted by vertex (face order within a vertex)
//   vv CSR     : (row, neighbour) keys, unique per row

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cmath>
#include <cstring>

#include "gh_internal.cuh"

using namespace ghd;

namespace {

constexpr int B = gh::kBlock;

__global__ void k_bbox_partial(const double* __restrict__ pos, int64_t nv, double* __restrict__ part) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    for (int k = 0; k < 3; ++k) {
      double p = pos[3 * i + k];
      lo[k] = p < lo[k] ? p : lo[k];
      hi[k] = hi[k] < p ? p : hi[k];
    }
  }
  __shared__ double sh[6][B];
  for (int k = 0; k < 3; ++k) {
    sh[k][threadIdx.x] = lo[k];
    sh[3 + k][threadIdx.x] = hi[k];
  }
  __syncthreads();
  for (int s = B / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int k = 0; k < 3; ++k) {
        double a = sh[k][threadIdx.x + s];
        sh[k][threadIdx.x] = a < sh[k][threadIdx.x] ? a : sh[k][threadIdx.x];
        double b = sh[3 + k][threadIdx.x + s];
        sh[3 + k][threadIdx.x] = sh[3 + k][threadIdx.x] < b ? b : sh[3 + k][threadIdx.x];
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) part[6 * blockIdx.x + threadIdx.x] = sh[threadIdx.x][0];
}

// degenerate threshold 1e-14 * |hi - lo|^2 (mesh.hpp:120-126)
__global__ void k_bbox_final(const double* __restrict__ part, int nparts, int64_t nv, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int b = 0; b < nparts; ++b)
    for (int k = 0; k < 3; ++k) {
      double a = part[6 * b + k], c = part[6 * b + 3 + k];
      lo[k] = a < lo[k] ? a : lo[k];
      hi[k] = hi[k] < c ? c : hi[k];
    }
  v3 d = sub(mk(hi[0], hi[1], hi[2]), mk(lo[0], lo[1], lo[2]));
  const double diag2 = nv > 0 ? sqnorm(d) : 0.0;
  out[0] = 1e-14 * diag2;
  for (int k = 0; k < 3; ++k) {  // the box itself (the diffusion layout's spatial order, gh_bfs.cu)
    out[5 + k] = lo[k];
    out[8 + k] = hi[k];
  }
}

// face checks + area + unit normal (mesh.hpp:128-145); first failing face via atomicMin
__global__ void k_faces(const double* __restrict__ pos, const int32_t* __restrict__ faces, int64_t nf, int32_t nv,
                        const double* __restrict__ degen, double* __restrict__ area, double* __restrict__ normal,
                        int32_t* __restrict__ err_face) {
  const double thr = degen[0];
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = faces[3 * f], b = faces[3 * f + 1], c = faces[3 * f + 2];
    bool bad = a < 0 || a >= nv || b < 0 || b >= nv || c < 0 || c >= nv || a == b || b == c || a == c;
    if (!bad) {
      v3 p0 = ld3(pos, a), p1 = ld3(pos, b), p2 = ld3(pos, c);
      v3 n = cross(sub(p1, p0), sub(p2, p0));
      double A = 0.5 * norm(n);
      if (!(A > thr)) {
        bad = true;
      } else {
        area[f] = A;
        st3(normal, f, divs(n, 2.0 * A));
      }
    }
    if (bad) atomicMin(err_face, (int32_t)f);
  }
}

// the index part of the face checks (mesh.hpp:133-137): first face with a
// vertex out of range or repeated; needs no positions
__global__ void k_face_indices(const int32_t* __restrict__ faces, int64_t nf, int32_t nv,
                               int32_t* __restrict__ err_face) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = faces[3 * f], b = faces[3 * f + 1], c = faces[3 * f + 2];
    if (a < 0 || a >= nv || b < 0 || b >= nv || c < 0 || c >= nv || a == b || b == c || a == c)
      atomicMin(err_face, (int32_t)f);
  }
}

// halfedge keys: (vmin * nv + vmax, h) (mesh.hpp:147-158)
__global__ void k_he_keys(const int32_t* __restrict__ faces, int64_t nh, uint64_t nv, uint64_t* __restrict__ key,
                          int32_t* __restrict__ val) {
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nh; h += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = h / 3;
    const int32_t a = faces[h], b = faces[3 * f + (h % 3 + 1) % 3];
    const uint64_t lo = (uint64_t)(a < b ? a : b), hi = (uint64_t)(a < b ? b : a);
    key[h] = lo * nv + hi;
    val[h] = (int32_t)h;
  }
}

__global__ void k_heads(const uint64_t* __restrict__ key, int64_t n, int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// per sorted position: record the start of its edge group
__global__ void k_edge_starts(const int32_t* __restrict__ flag, const int32_t* __restrict__ eid, int64_t n,
                              int32_t* __restrict__ start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) start[eid[i]] = (int32_t)i;
}

// edges from sorted groups: endpoints, sides, twins, checks (mesh.hpp:159-192)
__global__ void k_edges(const uint64_t* __restrict__ key, const int32_t* __restrict__ val,
                        const int32_t* __restrict__ start, int64_t ne, int64_t nh, uint64_t nv,
                        const int32_t* __restrict__ faces, int32_t* __restrict__ edge_v, int32_t* __restrict__ edge_he,
                        int32_t* __restrict__ he_edge, int32_t* __restrict__ he_twin,
                        unsigned long long* __restrict__ err_edge) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = start[e], t = e + 1 < ne ? start[e + 1] : nh;
    const uint64_t k = key[s];
    const int32_t vmin = (int32_t)(k / nv), vmax = (int32_t)(k % nv);
    edge_v[2 * e] = vmin;
    edge_v[2 * e + 1] = vmax;
    const int64_t incident = t - s;
    if (incident > 2) {
      unsigned long long inc = incident > 0xFFFFFF ? 0xFFFFFFull : (unsigned long long)incident;
      atomicMin(err_edge, ((unsigned long long)e << 32) | (1ull << 24) | inc);
      continue;
    }
    int32_t halves[2] = {-1, -1};
    bool winding = false;
    for (int64_t i = s; i < t; ++i) {
      const int32_t h = val[i];
      he_edge[h] = (int32_t)e;
      const int side = faces[h] == vmin ? 0 : 1;
      if (halves[side] >= 0) winding = true;
      halves[side] = h;
    }
    if (winding) {
      atomicMin(err_edge, ((unsigned long long)e << 32) | (2ull << 24));
      continue;
    }
    if (incident == 2) {
      he_twin[halves[0]] = halves[1];
      he_twin[halves[1]] = halves[0];
    }
    edge_he[2 * e] = halves[0];
    edge_he[2 * e + 1] = halves[1];
  }
}

__global__ void k_interior_flag(const int32_t* __restrict__ edge_he, int64_t ne, int32_t* __restrict__ flag) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x)
    flag[e] = (edge_he[2 * e] >= 0 && edge_he[2 * e + 1] >= 0) ? 1 : 0;
}

__global__ void k_interior_fill(const int32_t* __restrict__ flag, const int32_t* __restrict__ idx, int64_t ne,
                                int32_t* __restrict__ interior_edges, int32_t* __restrict__ interior_edge_index) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    if (flag[e]) {
      interior_edge_index[e] = idx[e];
      interior_edges[idx[e]] = (int32_t)e;
    } else {
      interior_edge_index[e] = -1;
    }
  }
}

// cot_at (mesh.hpp:102-106), halfedge k opposite v_{k+2} (203-213)
__device__ __forceinline__ double cot_at(v3 apex, v3 p, v3 q) {
  v3 u = sub(p, apex), v = sub(q, apex);
  return dot(u, v) / norm(cross(u, v));
}

__global__ void k_cot(const double* __restrict__ pos, const int32_t* __restrict__ faces, int64_t nf,
                      double* __restrict__ cot) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
    v3 p0 = ld3(pos, faces[3 * f]), p1 = ld3(pos, faces[3 * f + 1]), p2 = ld3(pos, faces[3 * f + 2]);
    cot[3 * f + 0] = cot_at(p2, p0, p1);
    cot[3 * f + 1] = cot_at(p0, p1, p2);
    cot[3 * f + 2] = cot_at(p1, p2, p0);
  }
}

// theta_e = 0.5 * ((0 + cot side0) + cot side1) (mesh.hpp:214-220); boundary flags (226-232)
__global__ void k_edge_weight(const int32_t* __restrict__ edge_he, const int32_t* __restrict__ edge_v,
                              const double* __restrict__ cot, int64_t ne, double* __restrict__ w,
                              uint8_t* __restrict__ on_boundary) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t h0 = edge_he[2 * e], h1 = edge_he[2 * e + 1];
    double sum = 0.0;
    if (h0 >= 0) sum += cot[h0];
    if (h1 >= 0) sum += cot[h1];
    w[e] = 0.5 * sum;
    if (h0 < 0 || h1 < 0) {
      on_boundary[edge_v[2 * e]] = 1;
      on_boundary[edge_v[2 * e + 1]] = 1;
    }
  }
}

__global__ void k_count_i32(const int32_t* __restrict__ idx, int64_t n, int32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[idx[i]], 1);
}

// vertex -> corner keys: vertex * H + h (bucket = vertex, order = corner)
__global__ void k_corner_keys(const int32_t* __restrict__ faces, int64_t n, uint64_t* __restrict__ key,
                              int32_t* __restrict__ val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = (uint64_t)faces[i] * (uint64_t)n + (uint64_t)i;
    val[i] = (int32_t)i;
  }
}

__global__ void k_iota_u32(uint32_t* __restrict__ keys, const int32_t* __restrict__ src, int32_t* __restrict__ val,
                           int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = (uint32_t)src[i];
    val[i] = (int32_t)i;
  }
}

// A_v = sum over incident corners in face order of A_f / 3 (mesh.hpp:222-224)
__global__ void k_vertex_area(const int32_t* __restrict__ vc_off, const int32_t* __restrict__ vc_corner,
                              const double* __restrict__ face_area, int64_t nv, double* __restrict__ va) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int32_t i = vc_off[v]; i < vc_off[v + 1]; ++i) s += face_area[vc_corner[i] / 3] / 3.0;
    va[v] = s;
  }
}

// CSR entries: (row * nv + neighbour, edge) for both directions (mesh.hpp:234-249)
__global__ void k_vv_keys(const int32_t* __restrict__ edge_v, int64_t ne, uint64_t nv, uint64_t* __restrict__ key,
                          int32_t* __restrict__ val, int32_t* __restrict__ degree) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = (uint64_t)edge_v[2 * e], b = (uint64_t)edge_v[2 * e + 1];
    key[2 * e] = a * nv + b;
    val[2 * e] = (int32_t)e;
    key[2 * e + 1] = b * nv + a;
    val[2 * e + 1] = (int32_t)e;
    atomicAdd(&degree[a], 1);
    atomicAdd(&degree[b], 1);
  }
}

__global__ void k_vv_fill(const uint64_t* __restrict__ key, const int32_t* __restrict__ val, int64_t n, uint64_t nv,
                          const double* __restrict__ edge_w, int32_t* __restrict__ vv_index,
                          int32_t* __restrict__ vv_edge, double* __restrict__ vv_w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    vv_index[i] = (int32_t)(key[i] % nv);
    vv_edge[i] = val[i];
    vv_w[i] = edge_w[val[i]];
  }
}

// sequential row sums (mesh.hpp:267-270)
__global__ void k_row_sum(const int32_t* __restrict__ off, const double* __restrict__ w, int64_t nv,
                          double* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int32_t i = off[v]; i < off[v + 1]; ++i) s += w[i];
    out[v] = s;
  }
}

__global__ void k_boundary_count(const uint8_t* __restrict__ f, int64_t n, double* __restrict__ part) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += f[i];
  s = block_sum<B>(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// per-edge lengths for average_edge_length (mesh.hpp:289-293)
__global__ void k_edge_len(const double* __restrict__ pos, const int32_t* __restrict__ edge_v, int64_t ne,
                           double* __restrict__ len) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x)
    len[e] = norm(sub(ld3(pos, edge_v[2 * e + 1]), ld3(pos, edge_v[2 * e])));
}

__global__ void k_reduce_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  // one block of 1024 threads, fixed tree => reproducible
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

// face_gradient (mesh.hpp:314-327)
__global__ void k_face_gradient(const double* __restrict__ pos, const int32_t* __restrict__ faces,
                                const double* __restrict__ normal, const double* __restrict__ area,
                                const double* __restrict__ u, int64_t nf, double* __restrict__ grad) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t[3] = {faces[3 * f], faces[3 * f + 1], faces[3 * f + 2]};
    const v3 n = ld3(normal, f);
    v3 g = mk(0.0, 0.0, 0.0);
    for (int k = 0; k < 3; ++k) {
      v3 opp = sub(ld3(pos, t[(k + 2) % 3]), ld3(pos, t[(k + 1) % 3]));
      g = add(g, scale(u[t[k]], cross(n, opp)));
    }
    st3(grad, f, divs(g, 2.0 * area[f]));
  }
}

int bits_for(uint64_t maxval) {
  int b = 1;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

template <class K>
void radix_sort_pairs(K*& keys, K*& keys_alt, int32_t*& vals, int32_t*& vals_alt, int64_t n, int end_bit,
                      cudaStream_t s) {
  cub::DoubleBuffer<K> kb(keys, keys_alt);
  cub::DoubleBuffer<int32_t> vb(vals, vals_alt);
  size_t tmp = 0;
  GH_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, (int)n, 0, end_bit, s));
  gh::Scratch<char> t(tmp, s);
  GH_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, kb, vb, (int)n, 0, end_bit, s));
  if (kb.Current() != keys) std::swap(keys, keys_alt);
  if (vb.Current() != vals) std::swap(vals, vals_alt);
}

template <class T>
T read_scalar(const T* d, cudaStream_t s) {
  T v;
  GH_CUDA(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
  return v;
}

// ---- bucketed sort for mesh keys key = bucket * div + rest with small buckets
// (a vertex's incident halfedges / neighbours): count, scan, scatter, then each
// bucket is insertion-sorted by (key, value) by one thread. The result equals
// the stable radix sort's (equal keys keep ascending value = input order).
constexpr int kMaxBucket = 64;

__global__ void k_bucket_count(const uint64_t* __restrict__ key, int64_t n, uint64_t div, int32_t* __restrict__ cnt,
                               int32_t* __restrict__ maxb) {
  int32_t mx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = atomicAdd(&cnt[key[i] / div], 1) + 1;
    mx = c > mx ? c : mx;
  }
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_down_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(maxb, mx);
}

__global__ void k_bucket_scatter(const uint64_t* __restrict__ key, const int32_t* __restrict__ val, int64_t n,
                                 uint64_t div, const int32_t* __restrict__ off, int32_t* __restrict__ cur,
                                 uint64_t* __restrict__ key_out, int32_t* __restrict__ val_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    const uint64_t b = k / div;
    const int32_t pos = off[b] + atomicAdd(&cur[b], 1);
    key_out[pos] = k;
    val_out[pos] = val[i];
  }
}

// insertion sort of one bucket [s, e) by (key, value)
template <class K, class V>
__device__ __forceinline__ void insertion_sort(K* key, V* val, int32_t s, int32_t e) {
  for (int32_t i = s + 1; i < e; ++i) {
    const uint64_t k = key[i];
    const int32_t v = val[i];
    int32_t j = i - 1;
    while (j >= s && (key[j] > k || (key[j] == k && val[j] > v))) {
      key[j + 1] = key[j];
      val[j + 1] = val[j];
      --j;
    }
    key[j + 1] = k;
    val[j + 1] = v;
  }
}

// A block takes B consecutive buckets: their entries are one contiguous range,
// staged in shared memory with coalesced loads, each thread insertion-sorts
// its bucket there, and the range goes back coalesced (a range too large for
// the stage is sorted in place in global memory).
constexpr int kStageEntries = 3072;
__global__ void __launch_bounds__(B) k_bucket_sort(const int32_t* __restrict__ off, int64_t nb,
                                                   uint64_t* __restrict__ key, int32_t* __restrict__ val) {
  __shared__ uint64_t sk[kStageEntries];
  __shared__ int32_t sv[kStageEntries];
  for (int64_t b0 = (int64_t)blockIdx.x * B; b0 < nb; b0 += (int64_t)gridDim.x * B) {
    const int64_t b1 = b0 + B < nb ? b0 + B : nb;
    const int32_t lo = off[b0], hi = off[b1];
    const int64_t b = b0 + threadIdx.x;
    if (hi - lo <= kStageEntries) {
      for (int32_t i = lo + threadIdx.x; i < hi; i += B) {
        sk[i - lo] = key[i];
        sv[i - lo] = val[i];
      }
      __syncthreads();
      if (b < b1) insertion_sort(sk - lo, sv - lo, off[b], off[b + 1]);
      __syncthreads();
      for (int32_t i = lo + threadIdx.x; i < hi; i += B) {
        key[i] = sk[i - lo];
        val[i] = sv[i - lo];
      }
      __syncthreads();
    } else if (b < b1) {
      insertion_sort(key, val, off[b], off[b + 1]);
    }
  }
}

void exclusive_scan(const int32_t* in, int32_t* out, int64_t n, cudaStream_t s);

// Sorts (keys, vals) into (keys_out, vals_out) by (key, val); nb buckets of
// key / div. Returns false (outputs untouched) when a bucket exceeds
// kMaxBucket, for the caller's radix sort.
bool bucket_sort_pairs(const uint64_t* keys, const int32_t* vals, int64_t n, uint64_t div, int64_t nb,
                       uint64_t* keys_out, int32_t* vals_out, cudaStream_t s, int32_t* offsets_out = nullptr) {
  gh::Scratch<int32_t> cnt(nb + 1, s), off(nb + 1, s), cur(nb + 1, s), maxb(1, s);
  GH_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (nb + 1), s));
  GH_CUDA(cudaMemsetAsync(cur.p, 0, sizeof(int32_t) * (nb + 1), s));
  GH_CUDA(cudaMemsetAsync(maxb.p, 0, sizeof(int32_t), s));
  k_bucket_count<<<gh::grid_for(n), B, 0, s>>>(keys, n, div, cnt.p, maxb.p);
  GH_LAUNCH_CHECK();
  const int32_t mb = read_scalar(maxb.p, s);
  if (mb > kMaxBucket) return false;
  exclusive_scan(cnt.p, off.p, nb + 1, s);
  k_bucket_scatter<<<gh::grid_for(n), B, 0, s>>>(keys, vals, n, div, off.p, cur.p, keys_out, vals_out);
  k_bucket_sort<<<gh::grid_for(nb, B, 148 * 8), B, 0, s>>>(off.p, nb, keys_out, vals_out);
  GH_LAUNCH_CHECK();
  if (offsets_out) GH_CUDA(cudaMemcpyAsync(offsets_out, off.p, sizeof(int32_t) * (nb + 1), cudaMemcpyDeviceToDevice, s));
  return true;
}

void exclusive_scan(const int32_t* in, int32_t* out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  GH_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, s));
  gh::Scratch<char> t(tmp, s);
  GH_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, (int)n, s));
}

// Host restatement of one face's checks, only to word the error message of the
// first failing face exactly like mesh.hpp:133-142 (std::to_string = "%f").
// Inputs are the face's three indices and, once they are in range, the
// three corner positions (fetched from wherever the mesh arrays live).
std::string face_error(const int32_t t[3], int64_t f, int32_t nv, const double* (*corner)(const void*, int32_t),
                       const void* ctx) {
  for (int k = 0; k < 3; ++k)
    if (t[k] < 0 || t[k] >= nv) return "face " + std::to_string(f) + ": vertex index out of range";
  if (t[0] == t[1] || t[1] == t[2] || t[0] == t[2])
    return "face " + std::to_string(f) + ": repeated vertex (degenerate face)";
  double P[3][3];
  for (int k = 0; k < 3; ++k) {
    const double* c = corner(ctx, t[k]);
    P[k][0] = c[0];
    P[k][1] = c[1];
    P[k][2] = c[2];
  }
  double ux = P[1][0] - P[0][0], uy = P[1][1] - P[0][1], uz = P[1][2] - P[0][2];
  double vx = P[2][0] - P[0][0], vy = P[2][1] - P[0][1], vz = P[2][2] - P[0][2];
  double nx = uy * vz - uz * vy, ny = uz * vx - ux * vz, nz = ux * vy - uy * vx;
  double area = 0.5 * std::sqrt((nx * nx + ny * ny) + nz * nz);
  return "face " + std::to_string(f) + ": degenerate (area " + std::to_string(area) + ")";
}

struct DeviceCorners {
  const double* pos;
  cudaStream_t s;
  double buf[3];
};
const double* device_corner(const void* ctx, int32_t v) {
  DeviceCorners* c = (DeviceCorners*)const_cast<void*>(ctx);
  GH_CUDA(cudaMemcpyAsync(c->buf, c->pos + 3 * (int64_t)v, 3 * sizeof(double), cudaMemcpyDeviceToHost, c->s));
  GH_CUDA(cudaStreamSynchronize(c->s));
  return c->buf;
}

}  // namespace

uint64_t gh_mesh::device_bytes() const {
  return pos.bytes() + face_area.bytes() + face_normal.bytes() + vertex_area.bytes() + he_cot.bytes() +
         edge_weight.bytes() + vertex_weight_sum.bytes() + vv_weight.bytes() + faces.bytes() + he_twin.bytes() +
         he_edge.bytes() + edge_v.bytes() + edge_he.bytes() + interior_edges.bytes() + interior_edge_index.bytes() +
         vv_offset.bytes() + vv_index.bytes() + vv_edge.bytes() + vc_offset.bytes() + vc_corner.bytes() +
         on_boundary.bytes() + partials.bytes() + scalars.bytes();
}

namespace gh {

void reduce_partials(gh_mesh* m, double* d_result_slot) {
  k_reduce_final<<<1, 1024, 0, m->stream>>>(m->partials.p, kReduceGrid, d_result_slot);
  GH_LAUNCH_CHECK();
  m->launches++;
}

// The upload is split so the face-only topology work (halfedge sort, edges,
// interior edges, the corner and adjacency orderings) runs while the
// positions are still crossing PCIe: faces first on the mesh stream,
// positions behind them on the thread's copy stream. Errors keep the
// reference's precedence: every face check (mesh.hpp:128-145) before any
// edge check (170-183).
void mesh_build(gh_mesh* m, const double* h_pos, const int32_t* h_faces) {
  cudaStream_t s = m->stream;
  const int64_t V = m->nv, F = m->nf, H = 3 * F;
  const uint64_t nvu = (uint64_t)(V > 0 ? V : 1);
  m->partials.alloc(kReduceGrid * 6, s);
  m->scalars.alloc(16, s);
  Event pos_ready;  // positions on the device (recorded on the copy stream)
  bool pos_pending = false;
  // h_pos == h_faces == nullptr: the loader already decoded the arrays into
  // m->pos / m->faces on the device.
  if (h_pos || h_faces || m->pos.n != (size_t)(3 * V) || m->faces.n != (size_t)(3 * F)) {
    m->pos.alloc(3 * V, s);
    m->faces.alloc(3 * F, s);
    // large pageable arrays (std::vector / numpy, as the reference's callers
    // hold them): staged through pinned slots by host threads (~4x the
    // driver's own pageable copy); pinned or device arrays: async copies
    const uint64_t fbytes = sizeof(int32_t) * 3 * (uint64_t)F, pbytes = sizeof(double) * 3 * (uint64_t)V;
    constexpr uint64_t kStageMin = 32ull << 20;
    const bool stage_f = F && fbytes >= kStageMin && host_pageable(h_faces);
    const bool stage_p = V && pbytes >= kStageMin && host_pageable(h_pos);
    if (stage_f || stage_p) GH_CUDA(cudaStreamSynchronize(s));  // the pool allocations above, before other streams write
    if (stage_f) host_to_device_staged(h_faces, fbytes, m->faces.p, m->device);
    else if (F) GH_CUDA(cudaMemcpyAsync(m->faces.p, h_faces, fbytes, cudaMemcpyHostToDevice, s));
    if (stage_p) {
      host_to_device_staged(h_pos, pbytes, m->pos.p, m->device);
    } else if (V) {
      Event faces_done;
      faces_done.record(s);  // also orders the pos allocation before the copy stream uses it
      GH_CUDA(cudaStreamWaitEvent(m->copy_stream, faces_done.e, 0));
      GH_CUDA(cudaMemcpyAsync(m->pos.p, h_pos, sizeof(double) * 3 * V, cudaMemcpyHostToDevice, m->copy_stream));
      pos_ready.record(m->copy_stream);
      pos_pending = true;
    }
  }
  auto wait_pos = [&] {
    if (pos_pending) GH_CUDA(cudaStreamWaitEvent(s, pos_ready.e, 0));
    pos_pending = false;
  };
  // on an early exit, the buffers freed on the mesh stream must not be reused
  // before the upload into them has landed
  struct PosGuard {
    cudaStream_t s;
    cudaEvent_t e;
    bool& pending;
    ~PosGuard() {
      if (pending) cudaStreamWaitEvent(s, e, 0);
    }
  } pos_guard{s, pos_ready.e, pos_pending};
  m->face_area.alloc(F, s);
  m->face_normal.alloc(3 * F, s);
  const int32_t big = 0x7fffffff;
  Scratch<int32_t> err_face(1, s);
  // the face checks in full (range, repeat, degenerate; first failing face
  // wins), then fail with the reference's message
  auto face_checks = [&] {
    wait_pos();
    const unsigned gb = grid_for(V, B, 512);
    k_bbox_partial<<<gb, B, 0, s>>>(m->pos.p, V, m->partials.p);
    k_bbox_final<<<1, 32, 0, s>>>(m->partials.p, (int)gb, V, m->scalars.p);
    GH_LAUNCH_CHECK();
    GH_CUDA(cudaMemcpyAsync(err_face.p, &big, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    if (F) {
      k_faces<<<grid_for(F), B, 0, s>>>(m->pos.p, m->faces.p, F, m->nv, m->scalars.p, m->face_area.p,
                                        m->face_normal.p, err_face.p);
      GH_LAUNCH_CHECK();
    }
    m->launches += 3;
    const int32_t bad_face = read_scalar(err_face.p, s);
    if (bad_face != big) {
      int32_t t[3];
      GH_CUDA(cudaMemcpyAsync(t, m->faces.p + 3 * (int64_t)bad_face, sizeof(t), cudaMemcpyDeviceToHost, s));
      GH_CUDA(cudaStreamSynchronize(s));
      DeviceCorners ctx{m->pos.p, s, {0, 0, 0}};
      fail(GH_ERR_MESH, face_error(t, bad_face, m->nv, device_corner, &ctx));
    }
  };
  // indices first: the topology kernels need them in range
  if (F) {
    GH_CUDA(cudaMemcpyAsync(err_face.p, &big, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    k_face_indices<<<grid_for(F), B, 0, s>>>(m->faces.p, F, m->nv, err_face.p);
    GH_LAUNCH_CHECK();
    m->launches++;
    if (read_scalar(err_face.p, s) != big) face_checks();  // fails (an earlier degenerate face may win)
  }

  // edges: stable sort of halfedge keys
  const int end_bit = bits_for(nvu * nvu - 1 > 0 ? nvu * nvu - 1 : 1);
  int64_t E = 0;
  std::string edge_error;  // reported after the face checks (reference order)
  m->he_twin.alloc(H, s);
  m->he_edge.alloc(H, s);
  GH_CUDA(cudaMemsetAsync(m->he_twin.p, 0xff, sizeof(int32_t) * H, s));
  GH_CUDA(cudaMemsetAsync(m->he_edge.p, 0xff, sizeof(int32_t) * H, s));
  {
    Scratch<uint64_t> k0(H, s), k1(H, s);
    Scratch<int32_t> v0(H, s), v1(H, s);
    uint64_t *ka = k0.p, *kb = k1.p;
    int32_t *va = v0.p, *vb = v1.p;
    if (H) {
      k_he_keys<<<grid_for(H), B, 0, s>>>(m->faces.p, H, nvu, ka, va);
      GH_LAUNCH_CHECK();
      if (bucket_sort_pairs(ka, va, H, nvu, V, kb, vb, s)) {
        std::swap(ka, kb);
        std::swap(va, vb);
        m->launches += 4;
      } else {
        radix_sort_pairs(ka, kb, va, vb, H, end_bit, s);
      }
    }
    Scratch<int32_t> flag(H + 1, s), eid(H + 1, s);
    if (H) {
      k_heads<<<grid_for(H), B, 0, s>>>(ka, H, flag.p);
      GH_LAUNCH_CHECK();
      exclusive_scan(flag.p, eid.p, H, s);
      int32_t last_id = read_scalar(eid.p + H - 1, s), last_flag = read_scalar(flag.p + H - 1, s);
      E = (int64_t)last_id + last_flag;
    }
    m->ne = (int32_t)E;
    m->edge_v.alloc(2 * E, s);
    m->edge_he.alloc(2 * E, s);
    if (E) {
      Scratch<int32_t> start(E, s);
      k_edge_starts<<<grid_for(H), B, 0, s>>>(flag.p, eid.p, H, start.p);
      Scratch<unsigned long long> err_edge(1, s);
      const unsigned long long none = ~0ull;
      GH_CUDA(cudaMemcpyAsync(err_edge.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));
      k_edges<<<grid_for(E), B, 0, s>>>(ka, va, start.p, E, H, nvu, m->faces.p, m->edge_v.p, m->edge_he.p,
                                        m->he_edge.p, m->he_twin.p, err_edge.p);
      GH_LAUNCH_CHECK();
      const unsigned long long ee = read_scalar(err_edge.p, s);
      if (ee != none) {
        const int64_t e = (int64_t)(ee >> 32);
        const int code = (int)((ee >> 24) & 0xff);
        const long long inc = (long long)(ee & 0xffffff);
        int32_t ev[2];
        GH_CUDA(cudaMemcpyAsync(ev, m->edge_v.p + 2 * e, sizeof(ev), cudaMemcpyDeviceToHost, s));
        GH_CUDA(cudaStreamSynchronize(s));
        const std::string pair = "(" + std::to_string(ev[0]) + "," + std::to_string(ev[1]) + ")";
        edge_error = code == 1 ? "non-manifold edge " + pair + ": " + std::to_string(inc) + " incident faces"
                               : "inconsistent winding across edge " + pair;
      }
      m->launches += 4;
    }
  }
  if (!edge_error.empty()) {
    face_checks();  // a face error anywhere takes precedence
    fail(GH_ERR_MESH, edge_error);
  }

  // interior edges (mesh.hpp:194-201)
  {
    Scratch<int32_t> flag(E + 1, s), idx(E + 1, s);
    int32_t ni = 0;
    m->interior_edge_index.alloc(E, s);
    if (E) {
      k_interior_flag<<<grid_for(E), B, 0, s>>>(m->edge_he.p, E, flag.p);
      exclusive_scan(flag.p, idx.p, E, s);
      ni = read_scalar(idx.p + E - 1, s) + read_scalar(flag.p + E - 1, s);
    }
    m->ni = ni;
    m->interior_edges.alloc(ni, s);
    if (E) {
      k_interior_fill<<<grid_for(E), B, 0, s>>>(flag.p, idx.p, E, m->interior_edges.p, m->interior_edge_index.p);
      GH_LAUNCH_CHECK();
      m->launches += 3;
    }
  }

  // vertex -> corner CSR (mesh.hpp:272-283): faces only
  m->vc_offset.alloc(V + 1, s);
  m->vc_corner.alloc(H, s);
  {
    Scratch<int32_t> cnt(V + 1, s);
    GH_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (V + 1), s));
    if (H) k_count_i32<<<grid_for(H), B, 0, s>>>(m->faces.p, H, cnt.p);
    exclusive_scan(cnt.p, m->vc_offset.p, V + 1, s);
    Scratch<uint32_t> k0(H, s), k1(H, s);
    Scratch<int32_t> v1(H, s);
    uint32_t *ka = k0.p, *kb = k1.p;
    int32_t *va = m->vc_corner.p, *vb = v1.p;
    if (H) {
      bool done = false;
      {
        Scratch<uint64_t> wk(H, s), wk2(H, s);
        Scratch<int32_t> wv(H, s);
        k_corner_keys<<<grid_for(H), B, 0, s>>>(m->faces.p, H, wk.p, wv.p);
        GH_LAUNCH_CHECK();
        done = bucket_sort_pairs(wk.p, wv.p, H, (uint64_t)H, V, wk2.p, m->vc_corner.p, s);
      }
      if (!done) {
        k_iota_u32<<<grid_for(H), B, 0, s>>>(ka, m->faces.p, va, H);
        GH_LAUNCH_CHECK();
        radix_sort_pairs(ka, kb, va, vb, H, bits_for(nvu), s);
        if (va != m->vc_corner.p)
          GH_CUDA(cudaMemcpyAsync(m->vc_corner.p, va, sizeof(int32_t) * H, cudaMemcpyDeviceToDevice, s));
      }
    }
    m->launches += 2;
  }

  // vertex adjacency ordering (mesh.hpp:234-266): rows sorted by neighbour
  m->vv_offset.alloc(V + 1, s);
  m->vv_index.alloc(2 * E, s);
  m->vv_edge.alloc(2 * E, s);
  m->vv_weight.alloc(2 * E, s);
  m->vertex_weight_sum.alloc(V, s);
  Scratch<uint64_t> vk0(2 * E, s), vk1(2 * E, s);
  Scratch<int32_t> vv0(2 * E, s), vv1(2 * E, s);
  uint64_t* vka = vk0.p;
  int32_t* vva = vv0.p;
  {
    Scratch<int32_t> degree(V + 1, s);
    GH_CUDA(cudaMemsetAsync(degree.p, 0, sizeof(int32_t) * (V + 1), s));
    uint64_t* kb = vk1.p;
    int32_t* vb = vv1.p;
    if (E) {
      k_vv_keys<<<grid_for(E), B, 0, s>>>(m->edge_v.p, E, nvu, vka, vva, degree.p);
      GH_LAUNCH_CHECK();
      if (bucket_sort_pairs(vka, vva, 2 * E, nvu, V, kb, vb, s)) {
        std::swap(vka, kb);
        std::swap(vva, vb);
      } else {
        radix_sort_pairs(vka, kb, vva, vb, 2 * E, end_bit, s);
      }
    }
    exclusive_scan(degree.p, m->vv_offset.p, V + 1, s);
    m->launches += 2;
  }

  // ---- geometry: needs the positions
  face_checks();

  // cotangents, weights, boundary flags
  m->he_cot.alloc(H, s);
  m->edge_weight.alloc(E, s);
  m->on_boundary.alloc(V, s);
  if (V) GH_CUDA(cudaMemsetAsync(m->on_boundary.p, 0, V, s));
  if (F) k_cot<<<grid_for(F), B, 0, s>>>(m->pos.p, m->faces.p, F, m->he_cot.p);
  if (E) k_edge_weight<<<grid_for(E), B, 0, s>>>(m->edge_he.p, m->edge_v.p, m->he_cot.p, E, m->edge_weight.p,
                                                  m->on_boundary.p);
  GH_LAUNCH_CHECK();
  m->launches += 2;

  // vertex areas (mesh.hpp:222-224)
  m->vertex_area.alloc(V, s);
  if (V) k_vertex_area<<<grid_for(V), B, 0, s>>>(m->vc_offset.p, m->vc_corner.p, m->face_area.p, V, m->vertex_area.p);
  GH_LAUNCH_CHECK();
  m->launches++;

  // adjacency weights + row sums (mesh.hpp:259-270)
  if (E) {
    k_vv_fill<<<grid_for(2 * E), B, 0, s>>>(vka, vva, 2 * E, nvu, m->edge_weight.p, m->vv_index.p, m->vv_edge.p,
                                             m->vv_weight.p);
    GH_LAUNCH_CHECK();
  }
  if (V) k_row_sum<<<grid_for(V), B, 0, s>>>(m->vv_offset.p, m->vv_weight.p, V, m->vertex_weight_sum.p);
  GH_LAUNCH_CHECK();
  m->launches += 2;

  // boundary vertex count (for gh_mesh_info)
  if (V) {
    k_boundary_count<<<kReduceGrid, B, 0, s>>>(m->on_boundary.p, V, m->partials.p);
    reduce_partials(m, m->scalars.p + 1);
    m->boundary_vertices = (int32_t)read_scalar(m->scalars.p + 1, s);
  }
  GH_CUDA(cudaStreamSynchronize(s));
}

// the reference's edge-order sum, bit for bit, so t = m h^2 matches too
double mesh_average_edge_length(gh_mesh* m) {
  if (m->ne == 0) return NAN;
  Scratch<double> len(m->ne, m->stream);
  k_edge_len<<<grid_for(m->ne), B, 0, m->stream>>>(m->pos.p, m->edge_v.p, m->ne, len.p);
  GH_LAUNCH_CHECK();
  m->launches++;
  return sequential_sum_nonneg(len.p, m->ne, m->stream, &m->launches) / (double)m->ne;
}

void face_gradient_dev(gh_mesh* m, const double* d_u, double* d_grad) {
  if (!m->nf) return;
  k_face_gradient<<<grid_for(m->nf), B, 0, m->stream>>>(m->pos.p, m->faces.p, m->face_normal.p, m->face_area.p, d_u,
                                                        m->nf, d_grad);
  GH_LAUNCH_CHECK();
  m->launches++;
}

}  // namespace gh
