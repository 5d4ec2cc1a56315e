// Internal declarations of the geoheat_b200 CUDA library (sm_100a).
//
// All fp64 arithmetic in this library is compiled with -fmad=false: every
// product and sum is rounded exactly where the reference (compiled without
// FMA contraction) rounds it, so the per-element results are bit-identical to
// the reference. Only the residual norms of the ADMM stop rule use a
// different (deterministic, tree) summation order; see DESIGN.md §3.6.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/geoheat_b200.h"

namespace gh {

struct Error {
  int code;
  std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error{code, msg}; }

#define GH_CUDA(x)                                                                                     \
  do {                                                                                                 \
    cudaError_t gh_e_ = (x);                                                                           \
    if (gh_e_ != cudaSuccess)                                                                          \
      ::gh::fail(GH_ERR_CUDA, std::string(#x) + " failed: " + cudaGetErrorString(gh_e_) + " (" +      \
                                  __FILE__ + ":" + std::to_string(__LINE__) + ")");                   \
  } while (0)

#define GH_LAUNCH_CHECK() GH_CUDA(cudaGetLastError())

constexpr int kBlock = 256;
constexpr int kReduceGrid = 4096;  // fixed partial count => reproducible reductions

// Sweep buffers: rows in blocks of 32, each block holding parity 0 then parity 1,
// so a gather's parity is one xor with (sweep & 1) << 5 of the stored column.
__host__ __device__ __forceinline__ uint32_t uidx(uint32_t row, uint32_t parity) {
  return ((row >> 5) << 6) | (parity << 5) | (row & 31u);
}

inline unsigned grid_for(int64_t n, int block = kBlock, int64_t cap = 148 * 32) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

// Device buffer owned by a handle: stream-ordered allocation on the handle's
// stream from the device's default memory pool, whose release threshold is
// raised once per device (gh_mesh_create) so freed handle memory stays cached
// for the next solve instead of going back to the driver.
// Stream-ordered allocation with an exact-size cache for mid-size blocks
// (gh_alloc.cu). The default pool keeps freed memory (release threshold
// raised), but it fragments: an end-to-end solve that repeats the previous
// one's allocations still made the pool map new memory now and then (one
// 134 MB request taking 134 ms). Blocks from 1 MB to 2 GB are therefore kept
// by size on free (with an event recorded on the freeing stream) and handed
// back to the next request of exactly that size (the requesting stream waits
// on the event). The cache is bounded (an eighth of device memory, oldest
// blocks go back to the pool first) and flushed when an allocation fails.
void* dev_alloc(size_t bytes, cudaStream_t s);
void dev_free(void* p, size_t bytes, cudaStream_t s);
void dev_cache_flush();

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    n = count;
    s = stream;
    if (count) p = static_cast<T*>(dev_alloc(sizeof(T) * count, stream));
  }
  void release() {
    if (p) dev_free(p, sizeof(T) * n, s);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// Scratch allocation from the stream-ordered pool (freed in stream order).
template <class T>
struct Scratch {
  T* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  Scratch(size_t count, cudaStream_t stream) : bytes(sizeof(T) * count), s(stream) {
    if (count) p = static_cast<T*>(dev_alloc(bytes, stream));
  }
  ~Scratch() {
    if (p) dev_free(p, bytes, s);
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
};

struct Event {  // an ordering-only event
  cudaEvent_t e = nullptr;
  Event() { GH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
  ~Event() {
    if (e) cudaEventDestroy(e);
  }
  Event(const Event&) = delete;
  Event& operator=(const Event&) = delete;
  void record(cudaStream_t s) { GH_CUDA(cudaEventRecord(e, s)); }
};

struct EventTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  explicit EventTimer(cudaStream_t stream) : s(stream) {
    GH_CUDA(cudaEventCreate(&a));
    GH_CUDA(cudaEventCreate(&b));
  }
  ~EventTimer() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
  void start() { GH_CUDA(cudaEventRecord(a, s)); }
  void stop() { GH_CUDA(cudaEventRecord(b, s)); }
  double ms() {
    GH_CUDA(cudaEventSynchronize(b));
    float f = 0.f;
    GH_CUDA(cudaEventElapsedTime(&f, a, b));
    return (double)f;
  }
};

}  // namespace gh

// ---------------------------------------------------------------- handles

struct gh_mesh {
  int device = 0;
  cudaStream_t stream = nullptr;
  int32_t nv = 0, nf = 0, ne = 0, ni = 0, boundary_vertices = 0;
  gh::DevBuf<double> pos, face_area, face_normal, vertex_area, he_cot, edge_weight, vertex_weight_sum, vv_weight;
  gh::DevBuf<int32_t> faces, he_twin, he_edge, edge_v, edge_he, interior_edges, interior_edge_index;
  gh::DevBuf<int32_t> vv_offset, vv_index, vv_edge, vc_offset, vc_corner;
  gh::DevBuf<uint8_t> on_boundary;
  // reduction scratch: kReduceGrid partials + result slots
  gh::DevBuf<double> partials, scalars;
  cudaStream_t copy_stream = nullptr;  // the thread's second stream: uploads overlapping kernels
  int launches = 0;                  // kernels launched since the counter was last read
  int level_refs = 0;                // live gh_levels built on this mesh
  bool destroy_pending = false;      // gh_mesh_destroy called while levels were alive
  // Every C-ABI entry point holds this while it uses the handle (or a gh_levels /
  // gh_band built on it): the per-call state above (reduction scratch, launch
  // counter, the levels' u buffers) and the one work stream are shared, so two
  // host threads calling into the same mesh are serialised instead of
  // interleaving on the stream (the reference's functions are pure on const
  // objects, so concurrent calls must stay safe).
  mutable std::recursive_mutex mtx;
  uint64_t device_bytes() const;
};

namespace gh {
// Sets a device for the scope and restores the caller's current device after
// (a host application or torch on another GPU keeps its own current device).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      (void)cudaGetLastError();
      prev = -1;
    }
    if (device != prev) {
      const cudaError_t e = cudaSetDevice(device);
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        throw Error{GH_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)};
      }
    }
  }
  ~DeviceScope() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
};
}  // namespace gh

namespace gh {

// Diffusion layout of one BFS band: own levels [lb, le) plus ghost copies of
// the neighbouring levels lb-1 and le. The single-GPU
// path is one band [0, nlev) without ghosts; multi-GPU runs one band per GPU,
// and the single-GPU emulation runs several bands in one launch.
//   rows: own levels in (parity, level, original index) order, each level
//   32-row aligned; then the ghost levels, each 32-row aligned.
struct Band {
  int32_t lb = 0, le = 0, nlev = 0;
  int32_t nrows = 0;      // own + ghost rows (32-aligned)
  int32_t own_rows = 0;   // rows [0, own_rows) are own levels
  int32_t own_chunks = 0;
  int32_t max_chunk_width = 0;
  int32_t device = 0;
  std::vector<int32_t> h_pstart, h_pend;  // by level; valid on own and ghost levels
  DevBuf<int32_t> pstart, pend;
  DevBuf<int32_t> perm;         // row -> original vertex (-1 for padding)
  DevBuf<int32_t> chunk_level;  // level of each own chunk (a chunk holds one level)
  DevBuf<int64_t> chunk_ptr;    // SELL-32 chunk offsets (own chunks)
  DevBuf<uint16_t> deg;         // row lengths (65535: look in deg_big)
  DevBuf<int32_t> deg_big;      // full row lengths, only when some valence >= 65535
  DevBuf<uint32_t> col;         // uidx(local row of the neighbour, 0 if one level closer to the sources else 1)
  DevBuf<double> wt;            // cotan weights in the reference's row order
  // 16-bit copy of col, in one of two formats:
  //  2 windows: bit 15 = the neighbour is one level away (the other parity
  //    half), bits 0-14 = its uidx minus the chunk's base for that half;
  //    cbase = (same-level base, other-half base, -, -);
  //  3 windows: bits 14-15 = window (0 same level, 1 level L-1, 2 level L+1),
  //    bits 0-13 = uidx minus the window's base; cbase = (base_0, base_1 - 2^14,
  //    base_2 - 2^15, -).
  // cbase.x = -1 marks a chunk whose windows do not fit (kept 32-bit).
  DevBuf<uint16_t> col16;
  DevBuf<int4> cbase;
  DevBuf<uint8_t> deg4;       // row lengths as nibbles (min(deg, 15)), 16 B per own chunk
  int32_t col16_windows = 0;  // format of col16: 2, 3, or 0 when too many chunks do not fit
  int64_t wide_chunks = 0;    // own chunks with cbase.x == -1
  DevBuf<double> area_r, wsum_r, den;
  double den_t = 0.0;
  // state shared with neighbour bands: plain cudaMalloc when it is IPC-exported
  // (ipc), else from the stream-ordered pool like every other buffer
  bool ipc = false;
  cudaStream_t astream = nullptr;
  double* ubuf = nullptr;                   // both sweep parities of every row, uidx layout
  unsigned long long* rows_done = nullptr;  // [nlev] rows finished per level over all sweeps
  int32_t* stalled = nullptr;               // dependency-timeout flag of the last launch
  // links to the neighbours' copies of this band's boundary levels
  double* lo_ubuf = nullptr;
  unsigned long long* lo_done = nullptr;
  int64_t lo_nrows = 0;
  int32_t lo_ghost = 0;  // row of level lb inside the lower neighbour
  double* hi_ubuf = nullptr;
  unsigned long long* hi_done = nullptr;
  int64_t hi_nrows = 0;
  int32_t hi_ghost = 0;  // row of level le-1 inside the upper neighbour
  // Sector slices: nslices > 0 when this is slice `rank` of a
  // partition that gives every slice a contiguous 1/nslices of every ring (so
  // every slice has work at every pipeline step). Rows: own rows as above
  // (lb = 0, le = nlev), then the ghost rows — every foreign neighbour of an
  // own row, in ring order — from `own_rows` on. The owner of a ghosted row
  // stores its new value into the reader's ghost row (export list) and counts
  // its finished rows per level into the reader's gdone[source][level].
  int32_t nslices = 0, rank = 0;
  DevBuf<uint32_t> src_mask;    // [nlev] slices whose rows this slice ghosts, per level
  DevBuf<uint32_t> dst_mask;    // [nlev] slices that ghost rows of this slice, per level
  DevBuf<int32_t> slice_cnt;    // [nslices * nlev] own rows of every slice per level
  DevBuf<int32_t> xoff;         // [own_chunks + 1] export entries of each own chunk
  DevBuf<int2> xent;            // (own row, dest slice << 28 | dest ghost row), by own row
  unsigned long long* gdone = nullptr;  // [nslices * nlev] ghost rows finished per (source, level)
  static constexpr int kMaxSlices = 8;
  double* peer_ubuf[kMaxSlices] = {};
  unsigned long long* peer_gdone[kMaxSlices] = {};
  bool peer_sys = false;        // peers on other devices: system-scope release and polls
  int64_t ghost_rows = 0;       // rows [own_rows, own_rows + ghost_rows) are ghosts
  int64_t exports = 0;          // export entries
  Band() = default;
  Band(const Band&) = delete;
  Band& operator=(const Band&) = delete;
  ~Band();
  void release_state();  // frees ubuf / rows_done / stalled / gdone (a rebuild with another size)
  uint64_t device_bytes() const;
  int32_t ghost_row(int32_t level) const { return h_pstart[level]; }
};

}  // namespace gh

struct gh_levels {
  gh_mesh* mesh = nullptr;
  int32_t nlev = 0, unreachable = 0, nreach = 0, max_width = 0;
  std::vector<int32_t> h_offsets;  // BFS order ring boundaries (nlev + 1)
  gh::DevBuf<int32_t> level, parent, order, offsets;  // level/parent [V], order [nreach], offsets [nlev+1]
  gh::DevBuf<int32_t> parent_edge;  // [V] edge id of (parent(v), v), -1 for sources / unreachable
  gh::DevBuf<int32_t> layout_order;  // rings in the diffusion layout's order when not `order` (spatial, see gh_bfs.cu)
  gh::Band main;                                       // the whole level range
  int32_t u_valid = 0;
  int32_t u_sweeps = 0;
  int32_t last_col16 = 0;  // the last diffusion launch streamed 16-bit columns
  // the last gs_diffuse: levels its last launch updated (nlev when nothing was
  // truncated), pipelined launches, launches redone after a truncation proved
  // too tight, and row updates executed (reachable x sweeps without truncation)
  int32_t last_active_levels = 0, last_launches = 0, last_retries = 0;
  uint64_t last_row_updates = 0;
  int32_t den_positive = -1;  // every den of the main band is > 0 for den_positive_t (-1: not checked)
  double den_positive_t = 0.0;
  gh::DevBuf<double> u_orig;  // last diffusion result, original order [V]
  uint64_t device_bytes() const;
};

namespace gh {

// mesh build / queries (gh_mesh.cu)
// host -> device copies from pageable memory: up to 16 host threads copy
// through pinned 16 MiB slots, each overlapping its memcpy with the H2D of
// the previous slot (gh_load.cu); returns when the data is on the device
bool host_pageable(const void* p);
void host_to_device_staged(const void* src, uint64_t n, void* dst, int device);
void device_to_host_staged(const void* src, uint64_t n, void* dst, int device);
void mesh_build(gh_mesh* m, const double* h_pos, const int32_t* h_faces);
// gh_load.cu: load_mesh into an initialised handle (device, stream set).
void load_mesh_bytes(gh_mesh* m, const unsigned char* bytes, uint64_t n, int format, int threads, gh_load_report* rep);
void load_mesh_file(gh_mesh* m, const char* path, int threads, gh_load_report* rep);
std::string serialize_mesh(gh_mesh* m, int format, const double* quality);
double mesh_average_edge_length(gh_mesh* m);
void face_gradient_dev(gh_mesh* m, const double* d_u, double* d_grad);

// BFS (gh_bfs.cu)
void bfs_build(gh_levels* L, const int32_t* h_sources, int32_t ns);

// band layouts (gh_band.cu)
std::vector<int32_t> plan_bands(const std::vector<int32_t>& offsets, int32_t nbands);
void band_build(gh_levels* L, Band* b, int32_t lb, int32_t le);
void band_link(Band* lower, Band* upper);  // same-process neighbours (emulation)
// slice `rank` of `nslices` (sector sharding); slice_link connects the slices of
// one process (emulation) to each other
void slice_build(gh_levels* L, Band* b, int32_t rank, int32_t nslices);
void slice_link(std::vector<Band*>& slices);
void band_own_mask(const Band* b, uint8_t* d_mask, int64_t nv, cudaStream_t s);  // 1 on the band's own vertices

// diffusion (gh_diffuse.cu): result stays in L->u_orig (original order)
// d_snap (optional, [sweeps][main.nrows]): every sweep's u in the band's row order
double diffuse_dev(gh_levels* L, double t, int32_t sweeps, const double* d_initial, double* d_snap = nullptr);
// the same solve split into bands that each compute their own levels and
// exchange boundary levels; all bands on the current device in one launch
double diffuse_bands_dev(gh_levels* L, std::vector<Band*>& bands, double t, int32_t sweeps, const double* d_initial,
                         double* d_snap = nullptr);
// the two halves of diffuse_bands_dev, for bands that live in other processes
void bands_prepare(gh_levels* L, std::vector<Band*>& bands, double t, const double* d_initial);
// level_cap in (0, nlev): the single band runs levels [0, level_cap) only;
// d_top_nonzero is set when a row of its top level gets a nonzero value
double bands_launch(gh_levels* L, std::vector<Band*>& bands, double t, int32_t sweeps, double* d_snap = nullptr,
                    int32_t level_cap = 0, int32_t* d_top_nonzero = nullptr, bool scatter = true);
// exact-zero skipping: off by default, GH_ZERO_LEVELS=1 or this switch turn it on
// The single band L->main may cover only the first levels of a mesh whose
// heat cannot reach the rest (bfs_build); this rebuilds it to
// cover levels [0, le) when it does not yet (its u state is lost).
void main_layout_ensure(gh_levels* L, int32_t le);
void set_zero_level_truncation(bool on);
bool zero_level_truncation();
// the single band's reachable rows of one snapshot sweep into d_u (original order; unreachable untouched)
void snapshot_to_orig(gh_levels* L, const double* d_snap_sweep, double* d_u);
// a band's own rows of u after `sweeps` sweeps -> vertex order
void band_own_u(const Band* b, int32_t sweeps, double* d_u, cudaStream_t s);
double diffusion_residual_dev(gh_levels* L, const double* d_u, double t);
// E1 of a group of k sweeps from their snapshots (k x main.nrows, row order):
// e1_setup_dev once per solve (vertex -> row and the CSR's columns as rows,
// nv and nnz int32; the fixed r^2 of unreachable vertices into every one of
// the kmax vertex-order arrays of d_sq, from the start state d_base), then per
// group r^2 in row order into d_sqr (k x own_rows), in vertex order into d_sq
// (k x nv) and the k left-to-right sums into d_sums (device; E1 = sqrt).
void e1_setup_dev(gh_levels* L, int32_t* d_rowof, int32_t* d_vv_row, const double* d_base, double t, int32_t kmax,
                  double* d_sq);
void e1_group_dev(gh_levels* L, const double* d_snap, int32_t k, double t, const int32_t* d_rowof,
                  const int32_t* d_vv_row, double* d_sqr, double* d_sq, double* d_sums);

// normalisation + optimisation (gh_grad.cu)
int32_t normalize_dev(gh_mesh* m, const double* d_u, double* d_h);
struct AdmmResult {
  int iterations = 0;
  bool converged = false;
  double final_primal = 0, final_dual = 0;
  std::vector<double> primal, dual;
  uint64_t state_bytes = 0;
  double device_ms = 0;
};
// act_f [F] / act_e (face method: [interior edges], edge method: [E]): optional
// activity flags from admm_active_flags; elements flagged 0 provably stay +0
// through every iteration and are skipped
AdmmResult admm_face_dev(gh_mesh* m, const double* d_h, const gh_admm_config& cfg, double* d_g,
                         const uint8_t* act_f = nullptr, const uint8_t* act_e = nullptr);
AdmmResult admm_edge_dev(gh_mesh* m, const double* d_h, const gh_admm_config& cfg, double* d_x,
                         const uint8_t* act_f = nullptr, const uint8_t* act_e = nullptr);
// Zero skipping in the ADMM: the level bound below which a
// face can differ from +0 within `iterations` iterations (from the targets H:
// the largest min-vertex-level of a face with a nonzero target, + iterations
// + 1), or -1 when skipping would not pay / is switched off; and the flags.
int32_t admm_active_level(gh_levels* L, const double* d_h, int32_t iterations);
void admm_active_flags(gh_levels* L, int32_t level_bound, bool interior_edges, uint8_t* act_f, uint8_t* act_e);

// integration (gh_integrate.cu)
void integrate_face_dev(gh_levels* L, const double* d_g, double* d_d);
void integrate_edge_dev(gh_levels* L, const double* d_x, double* d_d);

// deterministic reductions (gh_mesh.cu): sum of partials[0..kReduceGrid)
void reduce_partials(gh_mesh* m, double* d_result_slot);
// the reference's left-to-right sum of n non-negative doubles, bit for bit (gh_seqsum.cu)
double sequential_sum_nonneg(const double* d_x, int64_t n, cudaStream_t s, int* launches);
// any signs: the exact path when every term is >= 0, else one thread in order
double deterministic_sum_dev(const double* d_x, int64_t n, cudaStream_t s);
// count independent left-to-right sums (any sign), sum i over d_x[i * stride + 0 .. n), into d_out[i]
void sequential_sums_group(const double* d_x, int64_t n, int64_t stride, int32_t count, double* d_out,
                           cudaStream_t s);
// the same with the per-segment sums T (count x seqsum_segments(n); any
// summation order, only a bound) already computed by the caller
int64_t seqsum_segments(int64_t n);
constexpr int kSeqsumSegment = 1024;  // terms per segment of T
void sequential_sums_from_T(const double* d_x, int64_t n, int64_t stride, int32_t count, const double* d_T,
                            double* d_out, cudaStream_t s);

// classic heat method on CG (gh_poisson.cu)
struct PoissonOut {
  int heat_iterations = 0, poisson_iterations = 0;
  double heat_residual = 0, poisson_residual = 0, heat_seconds = 0, poisson_seconds = 0;
};
PoissonOut poisson_heat_dev(gh_levels* L, double t, double tol, double* d_d);

// evaluation layer (gh_metrics.cu)
double triangulation_quality_dev(gh_mesh* m);
void subdivide_once(gh_mesh* src, gh_mesh* dst);
void copy_mesh_arrays(gh_mesh* src, gh_mesh* dst);
void analytic_dev(gh_mesh* m, int kind, const int32_t* d_src, int32_t ns, double* d_out);
void dijkstra_dev(gh_mesh* m, const int32_t* d_src, int32_t ns, double* d_out);
void errors_dev(cudaStream_t s, const double* d, const double* r, int64_t n, const int32_t* src, int32_t ns,
                double* mre, int32_t* excluded, double* e2);

}  // namespace gh

// ---------------------------------------------------------------- device helpers

namespace ghd {

struct v3 {
  double x, y, z;
};
__device__ __forceinline__ v3 mk(double x, double y, double z) { return v3{x, y, z}; }
__device__ __forceinline__ v3 ld3(const double* p, int64_t i) { return v3{p[3 * i], p[3 * i + 1], p[3 * i + 2]}; }
__device__ __forceinline__ void st3(double* p, int64_t i, v3 a) {
  p[3 * i] = a.x;
  p[3 * i + 1] = a.y;
  p[3 * i + 2] = a.z;
}
__device__ __forceinline__ v3 sub(v3 a, v3 b) { return v3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ v3 add(v3 a, v3 b) { return v3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ v3 scale(double s, v3 a) { return v3{s * a.x, s * a.y, s * a.z}; }
// n / d, IEEE round to nearest. A zero numerator (common: zero gradients,
// zero multipliers, underflowed heat) sends the inline division down its slow
// path, so that case returns the signed zero directly; the asm keeps the
// division itself under the branch instead of being computed speculatively.
__device__ __forceinline__ double ddiv(double n, double d) {
  if (n == 0.0 && d != 0.0 && d == d) return (__double_as_longlong(n) ^ __double_as_longlong(d)) < 0 ? -0.0 : 0.0;
  double q;
  asm volatile("div.rn.f64 %0, %1, %2;" : "=d"(q) : "d"(n), "d"(d));
  return q;
}
__device__ __forceinline__ v3 divs(v3 a, double s) { return v3{ddiv(a.x, s), ddiv(a.y, s), ddiv(a.z, s)}; }
// Eigen size-3 dot order: (x0*y0 + x1*y1) + x2*y2
__device__ __forceinline__ double dot(v3 a, v3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__device__ __forceinline__ double sqnorm(v3 a) { return dot(a, a); }
__device__ __forceinline__ double norm(v3 a) { return sqrt(sqnorm(a)); }
__device__ __forceinline__ v3 cross(v3 a, v3 b) {
  return v3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ v3 normalized(v3 a) {
  double n2 = sqnorm(a);
  return n2 > 0.0 ? divs(a, sqrt(n2)) : a;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier for cooperative (co-resident) launches: one monotonic
// arrival counter, zeroed before the launch; the k-th barrier (k = 0, 1, ...)
// completes at (k + 1) * gridDim.x arrivals. Cheaper than cg::grid_group::sync
// for the many short levels of BFS.
__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned k) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // release arrival (cumulative over the block's writes ordered by the
    // __syncthreads), acquire polling: no sequentially consistent fence
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
    const unsigned target = (k + 1) * gridDim.x;
    while (ld_acquire_u32(counter) < target) {
    }
  }
  __syncthreads();
}

// Block-wide sum in a fixed tree order (deterministic for a fixed blockDim).
template <int BLOCK>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[BLOCK / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = lane < BLOCK / 32 ? sh[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

}  // namespace ghd
