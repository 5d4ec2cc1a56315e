// The C ABI (include/geoheat_b200.h): handle management, host<->device
// staging, error mapping. No exception crosses this boundary: every entry
// point catches gh::Error / std::bad_alloc and returns a gh_status, with the
// message kept per thread for gh_last_error() (the reference's exception
// types map to codes as in tools/geoheat.cpp:337-349).

#include <chrono>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <new>

#include "gh_internal.cuh"
#include "gh_meshio.hpp"

namespace {

thread_local std::string g_last_error;
thread_local int g_device = -1;

gh_status set_err(int code, const std::string& msg) {
  g_last_error = msg;
  return (gh_status)code;
}

template <class F>
gh_status guarded(F&& f) {
  try {
    f();
    return GH_OK;
  } catch (const gh::Error& e) {
    return set_err(e.code, e.msg);
  } catch (const std::bad_alloc&) {
    return set_err(GH_ERR_CUDA, "host allocation failed");
  } catch (const std::exception& e) {
    return set_err(GH_ERR_INTERNAL, e.what());
  }
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void require(bool ok, const char* what) {
  if (!ok) gh::fail(GH_ERR_INVALID, what);
}

// One C-ABI call's hold on a handle: the mesh's device for the call (the
// caller's current device restored on return) and the mesh's lock, so calls
// from several host threads on one mesh (or its levels / bands) run one after
// another (gh_mesh::mtx).
struct Use {
  gh::DeviceScope dev;
  std::lock_guard<std::recursive_mutex> lock;
  explicit Use(const gh_mesh* m) : dev(m->device), lock(m->mtx) {}
};

template <class T>
void to_host(T* dst, const T* src, size_t n, cudaStream_t s) {
  const uint64_t bytes = sizeof(T) * (uint64_t)n;
  if (bytes >= (32ull << 20) && gh::host_pageable(dst)) {  // large pageable results: staged by host threads
    int dev = 0;
    GH_CUDA(cudaGetDevice(&dev));
    GH_CUDA(cudaStreamSynchronize(s));
    gh::device_to_host_staged(src, bytes, dst, dev);
    return;
  }
  if (n) GH_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
}

void fill_solver_report(gh_solver_report* r, const gh::AdmmResult& a, uint64_t formula, double wall,
                        int launches) {
  if (!r) return;
  r->iterations = a.iterations;
  r->converged = a.converged ? 1 : 0;
  r->final_primal = a.final_primal;
  r->final_dual = a.final_dual;
  for (int i = 0; i < r->history_capacity && i < (int)a.primal.size(); ++i) {
    if (r->primal_history) r->primal_history[i] = a.primal[i];
    if (r->dual_history) r->dual_history[i] = a.dual[i];
  }
  r->state_bytes_formula = formula;
  r->state_bytes_allocated = a.state_bytes;
  r->wall_seconds = wall;
  r->device_ms = a.device_ms;
  r->kernel_launches = launches;
}

uint64_t state_formula(const gh_mesh* m, int method) {
  const uint64_t nf = (uint64_t)m->nf, ne = (uint64_t)m->ne, ni = (uint64_t)m->ni;
  if (method == GH_METHOD_FACE) return (6 * nf + 15 * ni) * 8;  // grad_face.hpp:222
  return (6 * nf + 2 * ne) * 8 + 3 * nf;                        // grad_face.hpp:223
}

// Handle memory comes from the device's default stream-ordered pool. Keeping
// freed blocks cached (release threshold = max) makes repeated solves reuse
// them instead of paying cudaMalloc/cudaFree on every call.
bool pool_done[64] = {false};
bool pool_touched(int device) { return device >= 0 && device < 64 && pool_done[device]; }
void keep_pool_memory(int device) {
  bool* done = pool_done;
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  GH_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t threshold = ~0ull;
  GH_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
  done[device] = true;
}

// Two non-blocking streams per (host thread, device) — the work stream and
// one for uploads that overlap it — created on first use and kept for the
// life of the thread: creating and destroying them per mesh cost up to
// hundreds of ms per end-to-end solve.
void thread_context(int device, cudaStream_t* stream, cudaStream_t* copy_stream) {
  struct Ctx {
    cudaStream_t stream = nullptr, copy = nullptr;
  };
  thread_local Ctx ctx[64];
  if (device < 0 || device >= 64) gh::fail(GH_ERR_CUDA, "device ordinal out of range");
  Ctx& c = ctx[device];
  if (!c.stream) {
    GH_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    GH_CUDA(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
  }
  *stream = c.stream;
  if (copy_stream) *copy_stream = c.copy;
}

int take_launches(gh_mesh* m) {
  int n = m->launches;
  m->launches = 0;
  return n;
}

}  // namespace

extern "C" {

const char* gh_last_error(void) { return g_last_error.c_str(); }
const char* gh_version(void) { return "geoheat_b200 0.1 (sm_100a)"; }

gh_status gh_set_device(int32_t device) {
  return guarded([&] {
    GH_CUDA(cudaSetDevice(device));
    g_device = device;
  });
}

gh_status gh_device_count(int32_t* count) {
  return guarded([&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      n = 0;
    }
    *count = n;
  });
}

gh_status gh_host_alloc(size_t bytes, void** out) {
  return guarded([&] { GH_CUDA(cudaMallocHost(out, bytes ? bytes : 1)); });
}

gh_status gh_host_free(void* p) {
  return guarded([&] {
    if (p) GH_CUDA(cudaFreeHost(p));
  });
}

gh_status gh_set_zero_level_truncation(int32_t on) {
  return guarded([&] { gh::set_zero_level_truncation(on != 0); });
}

gh_status gh_release_cached_memory(void) {
  return guarded([&] {
    int cur = 0, ndev = 0;
    GH_CUDA(cudaGetDevice(&cur));
    GH_CUDA(cudaGetDeviceCount(&ndev));
    gh::dev_cache_flush();
    for (int d = 0; d < ndev && d < 64; ++d) {
      if (!pool_touched(d)) continue;
      GH_CUDA(cudaSetDevice(d));
      GH_CUDA(cudaDeviceSynchronize());
      cudaMemPool_t pool;
      GH_CUDA(cudaDeviceGetDefaultMemPool(&pool, d));
      GH_CUDA(cudaMemPoolTrimTo(pool, 0));
    }
    GH_CUDA(cudaSetDevice(cur));
  });
}

// A fresh handle on the selected device with the thread's stream.
static std::unique_ptr<gh_mesh> new_mesh() {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    (void)cudaGetLastError();
    gh::fail(GH_ERR_CUDA, "no CUDA device available (the geoheat_b200 path has no CPU fallback)");
  }
  std::unique_ptr<gh_mesh> m(new gh_mesh());
  if (g_device >= 0) GH_CUDA(cudaSetDevice(g_device));
  GH_CUDA(cudaGetDevice(&m->device));
  keep_pool_memory(m->device);
  thread_context(m->device, &m->stream, &m->copy_stream);
  return m;
}

gh_status gh_mesh_create(const double* positions, int32_t nv, const int32_t* faces, int32_t nf, gh_mesh** out) {
  return guarded([&] {
    require(out != nullptr, "gh_mesh_create: null output");
    require(nv >= 0 && nf >= 0, "gh_mesh_create: negative size");
    require((nv == 0 || positions) && (nf == 0 || faces), "gh_mesh_create: null input array");
    require((int64_t)nf * 3 <= 0x7fffffffLL, "gh_mesh_create: more than 2^31 halfedges");
    std::unique_ptr<gh_mesh> m = new_mesh();
    m->nv = nv;
    m->nf = nf;
    gh::mesh_build(m.get(), positions, faces);
    *out = m.release();
  });
}

// ---- mesh I/O (gh_load.cu, gh_meshio.cpp)
static gh_status load_common(gh_mesh** out, gh_load_report* report, const std::function<void(gh_mesh*)>& body) {
  return guarded([&] {
    require(out != nullptr, "gh_mesh_load: null output");
    const double t0 = now_s();
    if (report) *report = gh_load_report{};
    std::unique_ptr<gh_mesh> m = new_mesh();
    body(m.get());
    GH_CUDA(cudaStreamSynchronize(m->stream));
    if (report) {
      report->total_ms = (now_s() - t0) * 1e3;
      report->kernel_launches = take_launches(m.get());
    }
    *out = m.release();
  });
}

gh_status gh_mesh_format_from_path(const char* path, int32_t* format_out) {
  return guarded([&] {
    require(path && format_out, "gh_mesh_format_from_path: null argument");
    try {
      *format_out = (int32_t)ghio::format_from_path(path);
    } catch (const ghio::LoadError& e) {
      gh::fail(GH_ERR_MESH, e.msg);
    }
  });
}

gh_status gh_mesh_load(const char* path, gh_mesh** out, gh_load_report* report) {
  if (!path) return set_err(GH_ERR_INVALID, "gh_mesh_load: null path");
  return load_common(out, report, [&](gh_mesh* m) { gh::load_mesh_file(m, path, 0, report); });
}

gh_status gh_mesh_load_memory(const void* data, uint64_t bytes, int32_t format, gh_mesh** out,
                              gh_load_report* report) {
  if (!data && bytes) return set_err(GH_ERR_INVALID, "gh_mesh_load_memory: null data");
  if (format != GH_FORMAT_OBJ && format != GH_FORMAT_PLY)
    return set_err(GH_ERR_INVALID, "gh_mesh_load_memory: unknown format");
  return load_common(out, report, [&](gh_mesh* m) {
    gh::load_mesh_bytes(m, (const unsigned char*)data, bytes, format, 0, report);
  });
}

gh_status gh_mesh_parse_text(const void* data, uint64_t bytes, int32_t format, int32_t threads, double** positions,
                             int64_t* nv, int32_t** faces, int64_t* nf) {
  return guarded([&] {
    require((data || !bytes) && positions && nv && faces && nf, "gh_mesh_parse_text: null argument");
    require(format == GH_FORMAT_OBJ || format == GH_FORMAT_PLY, "gh_mesh_parse_text: unknown format");
    ghio::HostMesh hm;
    try {
      if (format == GH_FORMAT_OBJ) {
        ghio::parse_obj((const char*)data, bytes, threads, hm);
      } else {
        const ghio::PlyHeader h = ghio::parse_ply_header((const char*)data, bytes);
        require(!h.binary, "gh_mesh_parse_text: binary PLY records are decoded on the device (gh_mesh_load_memory)");
        ghio::parse_ply_ascii(h, (const char*)data, bytes, threads, hm);
      }
    } catch (const ghio::LoadError& e) {
      gh::fail(GH_ERR_MESH, e.msg);
    }
    double* p = (double*)std::malloc(sizeof(double) * std::max<size_t>(1, hm.pos.size()));
    int32_t* f = (int32_t*)std::malloc(sizeof(int32_t) * std::max<size_t>(1, hm.faces.size()));
    if (!p || !f) {
      std::free(p);
      std::free(f);
      throw std::bad_alloc();
    }
    std::memcpy(p, hm.pos.data(), sizeof(double) * hm.pos.size());
    std::memcpy(f, hm.faces.data(), sizeof(int32_t) * hm.faces.size());
    *positions = p;
    *faces = f;
    *nv = (int64_t)hm.pos.size() / 3;
    *nf = (int64_t)hm.faces.size() / 3;
  });
}

static void* to_malloc(const std::string& s, uint64_t* bytes) {
  void* p = std::malloc(std::max<size_t>(1, s.size()));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size());
  *bytes = s.size();
  return p;
}

static void write_file(const char* path, const std::string& s) {
  FILE* f = std::fopen(path, "wb");
  if (!f) gh::fail(GH_ERR_MESH, std::string("cannot open output file '") + path + "'");
  const size_t w = s.empty() ? 0 : std::fwrite(s.data(), 1, s.size(), f);
  const int c = std::fclose(f);
  if (w != s.size() || c != 0) gh::fail(GH_ERR_MESH, std::string("write failed for '") + path + "'");
}

gh_status gh_mesh_serialize(gh_mesh* mesh, int32_t format, const double* quality, void** data, uint64_t* bytes) {
  return guarded([&] {
    require(mesh && data && bytes, "gh_mesh_serialize: null argument");
    require(format == GH_FORMAT_OBJ || format == GH_FORMAT_PLY, "gh_mesh_serialize: unknown format");
    require(!quality || format == GH_FORMAT_PLY, "gh_mesh_serialize: quality is written by PLY only");
    Use use_(mesh);
    *data = to_malloc(gh::serialize_mesh(mesh, format, quality), bytes);
  });
}

gh_status gh_mesh_save(gh_mesh* mesh, const char* path, const double* quality) {
  return guarded([&] {
    require(mesh && path, "gh_mesh_save: null argument");
    Use use_(mesh);
    // save_mesh opens the file before it infers the format (mesh_io.hpp:321-326)
    FILE* probe = std::fopen(path, "wb");
    if (!probe) gh::fail(GH_ERR_MESH, std::string("cannot open output file '") + path + "'");
    std::fclose(probe);
    int format = 0;
    try {
      format = (int)ghio::format_from_path(path);
    } catch (const ghio::LoadError& e) {
      gh::fail(GH_ERR_MESH, e.msg);
    }
    require(!quality || format == GH_FORMAT_PLY, "gh_mesh_save: quality is written by PLY only");
    write_file(path, gh::serialize_mesh(mesh, format, quality));
  });
}

gh_status gh_format_distances(const double* d, int64_t n, int32_t format, void** data, uint64_t* bytes) {
  return guarded([&] {
    require((d || n == 0) && n >= 0 && data && bytes, "gh_format_distances: bad argument");
    require(format == GH_DISTANCES_TXT || format == GH_DISTANCES_CSV, "gh_format_distances: unknown format");
    std::string s;
    ghio::format_distances(d, n, format == GH_DISTANCES_CSV, 0, s);
    *data = to_malloc(s, bytes);
  });
}

gh_status gh_write_distances(const char* path, const double* d, int64_t n, int32_t format) {
  return guarded([&] {
    require(path && (d || n == 0) && n >= 0, "gh_write_distances: bad argument");
    require(format == GH_DISTANCES_TXT || format == GH_DISTANCES_CSV, "gh_write_distances: unknown format");
    std::string s;
    ghio::format_distances(d, n, format == GH_DISTANCES_CSV, 0, s);
    write_file(path, s);
  });
}

void gh_free(void* p) { std::free(p); }

static void free_mesh(gh_mesh* mesh) {
  gh::DeviceScope dev(mesh->device);
  cudaStreamSynchronize(mesh->stream);
  delete mesh;  // buffers return to the stream-ordered pool; stream and pinned scratch are per thread
}

gh_status gh_mesh_destroy(gh_mesh* mesh) {
  return guarded([&] {
    if (!mesh) return;
    // levels borrow the mesh: the last of them frees it (any destroy order is safe)
    if (mesh->level_refs > 0) {
      mesh->destroy_pending = true;
      return;
    }
    free_mesh(mesh);
  });
}

gh_status gh_mesh_get_info(const gh_mesh* mesh, gh_mesh_info* info) {
  return guarded([&] {
    require(mesh && info, "gh_mesh_get_info: null argument");
    info->vertices = mesh->nv;
    info->faces = mesh->nf;
    info->edges = mesh->ne;
    info->interior_edges = mesh->ni;
    info->boundary_vertices = mesh->boundary_vertices;
    info->device_bytes = mesh->device_bytes();
  });
}

gh_status gh_mesh_download(const gh_mesh* mesh, int32_t which, void* host_out, int64_t count) {
  return guarded([&] {
    require(mesh && host_out, "gh_mesh_download: null argument");
    Use use_(mesh);
    const void* src = nullptr;
    size_t n = 0, es = 0;
    const gh_mesh& m = *mesh;
    switch (which) {
#define ARR(id, buf) \
  case id:           \
    src = m.buf.p;   \
    n = m.buf.n;     \
    es = sizeof(*m.buf.p); \
    break;
      ARR(GH_POSITIONS, pos)
      ARR(GH_FACES, faces)
      ARR(GH_HALFEDGE_TWIN, he_twin)
      ARR(GH_HALFEDGE_EDGE, he_edge)
      ARR(GH_EDGE_VERTICES, edge_v)
      ARR(GH_EDGE_HALFEDGES, edge_he)
      ARR(GH_INTERIOR_EDGES, interior_edges)
      ARR(GH_INTERIOR_EDGE_INDEX, interior_edge_index)
      ARR(GH_VERTEX_ON_BOUNDARY, on_boundary)
      ARR(GH_FACE_AREA, face_area)
      ARR(GH_FACE_NORMAL, face_normal)
      ARR(GH_VERTEX_AREA, vertex_area)
      ARR(GH_HALFEDGE_COT, he_cot)
      ARR(GH_EDGE_WEIGHT, edge_weight)
      ARR(GH_VERTEX_WEIGHT_SUM, vertex_weight_sum)
      ARR(GH_VV_OFFSET, vv_offset)
      ARR(GH_VV_INDEX, vv_index)
      ARR(GH_VV_EDGE, vv_edge)
      ARR(GH_VV_WEIGHT, vv_weight)
      ARR(GH_VC_OFFSET, vc_offset)
      ARR(GH_VC_CORNER, vc_corner)
#undef ARR
      default:
        gh::fail(GH_ERR_INVALID, "gh_mesh_download: unknown array id");
    }
    require((size_t)count == n, "gh_mesh_download: count does not match the array length");
    if (n) GH_CUDA(cudaMemcpyAsync(host_out, src, n * es, cudaMemcpyDeviceToHost, m.stream));
    GH_CUDA(cudaStreamSynchronize(m.stream));
  });
}

gh_status gh_average_edge_length(gh_mesh* mesh, double* h_out) {
  return guarded([&] {
    require(mesh && h_out, "gh_average_edge_length: null argument");
    Use use_(mesh);
    *h_out = gh::mesh_average_edge_length(mesh);
  });
}

gh_status gh_diffusion_time(gh_mesh* mesh, double m, double* t_out) {
  return guarded([&] {
    require(mesh && t_out, "gh_diffusion_time: null argument");
    if (!(m > 0.0)) gh::fail(GH_ERR_INVALID, "diffusion_time: m must be positive");
    Use use_(mesh);
    const double h = gh::mesh_average_edge_length(mesh);
    *t_out = m * h * h;  // diffusion.hpp:30-31
  });
}

gh_status gh_face_gradient(gh_mesh* mesh, const double* u, double* grad_out) {
  return guarded([&] {
    require(mesh && u && grad_out, "gh_face_gradient: null argument");
    Use use_(mesh);
    cudaStream_t s = mesh->stream;
    gh::Scratch<double> du(mesh->nv, s), dg(3 * (size_t)mesh->nf, s);
    GH_CUDA(cudaMemcpyAsync(du.p, u, sizeof(double) * mesh->nv, cudaMemcpyHostToDevice, s));
    gh::face_gradient_dev(mesh, du.p, dg.p);
    to_host(grad_out, dg.p, 3 * (size_t)mesh->nf, s);
  });
}

gh_status gh_bfs_create(gh_mesh* mesh, const int32_t* sources, int32_t ns, gh_levels** out) {
  return guarded([&] {
    require(mesh && out, "gh_bfs_create: null argument");
    require(ns == 0 || sources, "gh_bfs_create: null sources");
    Use use_(mesh);
    std::unique_ptr<gh_levels> L(new gh_levels());
    L->mesh = mesh;
    gh::bfs_build(L.get(), sources, ns);
    mesh->level_refs++;
    *out = L.release();
  });
}

gh_status gh_bfs_destroy(gh_levels* levels) {
  return guarded([&] {
    if (!levels) return;
    gh_mesh* m = levels->mesh;
    gh::DeviceScope dev(m->device);
    {
      std::lock_guard<std::recursive_mutex> lock(m->mtx);
      cudaStreamSynchronize(m->stream);
      delete levels;
    }
    if (--m->level_refs == 0 && m->destroy_pending) free_mesh(m);
  });
}

gh_status gh_bfs_get_info(const gh_levels* levels, gh_levels_info* info) {
  return guarded([&] {
    require(levels && info, "gh_bfs_get_info: null argument");
    info->level_count = levels->nlev;
    info->unreachable_count = levels->unreachable;
    info->max_level_width = levels->max_width;
    info->column_bits = levels->last_col16 ? 16 : levels->u_valid ? 32 : 0;
    info->active_levels = levels->last_active_levels;
    info->diffusion_launches = levels->last_launches;
    info->diffusion_retries = levels->last_retries;
    info->layout_levels = levels->main.le;
    info->row_updates = levels->last_row_updates;
  });
}

gh_status gh_bfs_download(const gh_levels* levels, int32_t* level_of_vertex, int32_t* parent_of_vertex,
                          int32_t* order, int32_t* offsets) {
  return guarded([&] {
    require(levels != nullptr, "gh_bfs_download: null levels");
    const gh_mesh* m = levels->mesh;
    Use use_(m);
    cudaStream_t s = m->stream;
    if (level_of_vertex) to_host(level_of_vertex, levels->level.p, m->nv, s);
    if (parent_of_vertex) to_host(parent_of_vertex, levels->parent.p, m->nv, s);
    if (order) to_host(order, levels->order.p, levels->nreach, s);
    if (offsets) std::memcpy(offsets, levels->h_offsets.data(), sizeof(int32_t) * (levels->nlev + 1));
  });
}

gh_status gh_gs_diffuse(gh_levels* levels, double t, int32_t sweeps, const double* initial, double* u_out,
                        gh_solver_report* report) {
  return guarded([&] {
    require(levels != nullptr, "gh_gs_diffuse: null levels");
    gh_mesh* m = levels->mesh;
    Use use_(m);
    cudaStream_t s = m->stream;
    const double w0 = now_s();
    take_launches(m);
    gh::Scratch<double> dinit(initial ? m->nv : 0, s);
    if (initial) GH_CUDA(cudaMemcpyAsync(dinit.p, initial, sizeof(double) * m->nv, cudaMemcpyHostToDevice, s));
    const double ms = gh::diffuse_dev(levels, t, sweeps, initial ? dinit.p : nullptr);
    if (u_out) to_host(u_out, levels->u_orig.p, m->nv, s);
    else GH_CUDA(cudaStreamSynchronize(s));
    if (report) {
      report->iterations = sweeps;
      report->converged = 0;
      report->wall_seconds = now_s() - w0;
      report->device_ms = ms;
      report->kernel_launches = take_launches(m);
      report->state_bytes_allocated = levels->device_bytes();
    }
  });
}

gh_status gh_gs_diffuse_tol(gh_levels* levels, double t, int32_t sweeps, double tolerance, const double* initial,
                            double* u_out, gh_solver_report* report) {
  return guarded([&] {
    require(levels != nullptr, "gh_gs_diffuse_tol: null levels");
    gh_mesh* m = levels->mesh;
    Use use_(m);
    cudaStream_t s = m->stream;
    const double w0 = now_s();
    take_launches(m);
    // E1 is checked after every sweep (diffusion.hpp:110-117). The sweeps run
    // pipelined in groups of K per launch; the kernel also writes every
    // update into a snapshot of its sweep, so after a group each sweep's u is
    // scattered to vertex order, its E1 computed (the exact left-to-right sum)
    // and the first sweep at or below the tolerance ends the solve with that
    // sweep's u. The next group is warm-started from the group's last u (a
    // sweep depends on u only, so this is bit-identical to one long run).
    gh::Scratch<double> cur(m->nv, s);
    double ms = 0.0;
    int done = 0;
    bool converged = false;
    if (sweeps == 0 || levels->nreach == 0) {
      if (initial) GH_CUDA(cudaMemcpyAsync(cur.p, initial, sizeof(double) * m->nv, cudaMemcpyHostToDevice, s));
      ms += gh::diffuse_dev(levels, t, 0, initial ? cur.p : nullptr);
      for (int k = 0; k < sweeps; ++k) {  // nothing reachable moves: every sweep leaves u as it is
        const double e1 = gh::diffusion_residual_dev(levels, levels->u_orig.p, t);
        ++done;
        if (report && report->residual_history && k < report->history_capacity) report->residual_history[k] = e1;
        if (e1 <= tolerance) {
          converged = true;
          break;
        }
      }
    } else {
      if (!(t > 0.0)) gh::fail(GH_ERR_INVALID, "gs_diffuse: t must be positive");
      gh::main_layout_ensure(levels, levels->nlev);  // the snapshots hold every level's rows
      // per sweep of a group: its snapshot (row order) and its r^2 terms
      // (vertex order); groups of up to 256 sweeps within half the free memory
      size_t free_b = 0, total_b = 0;
      GH_CUDA(cudaMemGetInfo(&free_b, &total_b));
      const size_t nv = (size_t)m->nv, nrows = (size_t)levels->main.nrows;
      const size_t own = (size_t)levels->main.own_rows;
      const size_t per = sizeof(double) * (nrows + own + nv);
      int32_t kmax = (int32_t)std::max<size_t>(1, std::min<size_t>(256, free_b / 2 / std::max<size_t>(per, 1)));
      if (const char* e = getenv("GH_TOL_GROUP")) kmax = std::max(1, atoi(e));  // tests: small groups
      kmax = std::min(kmax, sweeps);
      gh::Scratch<double> snap((size_t)kmax * nrows, s), sqr((size_t)kmax * own, s), sq((size_t)kmax * nv, s);
      gh::Scratch<double> sums((size_t)kmax, s);
      gh::Scratch<int32_t> rowof(nv, s), vv_row(m->vv_index.n, s);
      std::vector<double> h_sums((size_t)kmax);
      // cur = the start state (u0, or the initial field) = u_orig; unreachable
      // vertices keep it through every sweep, so cur also serves as their values
      if (initial) GH_CUDA(cudaMemcpyAsync(cur.p, initial, sizeof(double) * nv, cudaMemcpyHostToDevice, s));
      gh::diffuse_dev(levels, t, 0, initial ? cur.p : nullptr);
      if (!initial)
        GH_CUDA(cudaMemcpyAsync(cur.p, levels->u_orig.p, sizeof(double) * nv, cudaMemcpyDeviceToDevice, s));
      gh::e1_setup_dev(levels, rowof.p, vv_row.p, cur.p, t, kmax, sq.p);
      const double* start = initial ? cur.p : nullptr;  // the next group's start state (nullptr: u0)
      std::vector<double> hist;
      while (done < sweeps && !converged) {
        // group size: 32 sweeps first (a stop there wastes little), then what the E1 decay predicts
        // is left to the tolerance (sweeps past the stop are wasted), at most kmax
        int32_t k = std::min(kmax, 32);
        if (hist.size() >= 8) {
          const size_t n = hist.size();
          const double a = std::log(hist[n - 8]), b = std::log(hist[n - 1]);
          const double rate = (b - a) / 7.0;
          if (rate < 0.0 && std::isfinite(rate) && hist[n - 1] > 0.0) {
            const double left = (std::log(tolerance) - b) / rate;
            k = left < (double)kmax ? std::max(8, (int32_t)std::ceil(left * 1.05) + 2) : kmax;
          } else {
            k = kmax;
          }
        }
        k = std::min(std::min(k, kmax), sweeps - done);
        ms += gh::diffuse_dev(levels, t, k, start, snap.p);
        static const bool prof = getenv("GH_E1_PROFILE") != nullptr;  // stage times on stderr (experiments)
        if (prof) {
          gh::EventTimer te(s);
          te.start();
          gh::e1_group_dev(levels, snap.p, k, t, rowof.p, vv_row.p, sqr.p, sq.p, sums.p);
          te.stop();
          fprintf(stderr, "e1_group k=%d e1_ms %.3f per_sweep_us %.1f\n", k, te.ms(), 1e3 * te.ms() / k);
        } else {
          gh::e1_group_dev(levels, snap.p, k, t, rowof.p, vv_row.p, sqr.p, sq.p, sums.p);
        }
        GH_CUDA(cudaMemcpyAsync(h_sums.data(), sums.p, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
        GH_CUDA(cudaStreamSynchronize(s));
        int32_t at = k - 1;
        for (int32_t i = 0; i < k; ++i) {
          const double e1 = std::sqrt(h_sums[i]);  // diffusion.hpp:48
          hist.push_back(e1);
          if (report && report->residual_history && done < report->history_capacity)
            report->residual_history[done] = e1;
          ++done;
          if (e1 <= tolerance) {
            converged = true;
            at = i;
            break;
          }
        }
        // cur = u after the last sweep kept (a sweep depends on u only: the next
        // group continues from it bit for bit)
        gh::snapshot_to_orig(levels, snap.p + (size_t)at * nrows, cur.p);
        start = cur.p;
      }
      GH_CUDA(cudaMemcpyAsync(levels->u_orig.p, cur.p, sizeof(double) * nv, cudaMemcpyDeviceToDevice, s));
      levels->u_sweeps = done;
    }
    if (u_out) to_host(u_out, levels->u_orig.p, m->nv, s);
    else GH_CUDA(cudaStreamSynchronize(s));
    if (report) {
      report->iterations = done;
      report->converged = converged ? 1 : 0;
      report->wall_seconds = now_s() - w0;
      report->device_ms = ms;
      report->kernel_launches = take_launches(m);
      report->state_bytes_allocated = levels->device_bytes();
    }
  });
}

gh_status gh_diffusion_residual(gh_levels* levels, const double* u, double t, double* e1_out) {
  return guarded([&] {
    require(levels && u && e1_out, "gh_diffusion_residual: null argument");
    gh_mesh* m = levels->mesh;
    Use use_(m);
    gh::Scratch<double> du(m->nv, m->stream);
    GH_CUDA(cudaMemcpyAsync(du.p, u, sizeof(double) * m->nv, cudaMemcpyHostToDevice, m->stream));
    *e1_out = gh::diffusion_residual_dev(levels, du.p, t);
  });
}

gh_status gh_normalized_target_gradients(gh_mesh* mesh, const double* u, double* h_out, int32_t* zero_count) {
  return guarded([&] {
    require(mesh && u && h_out, "gh_normalized_target_gradients: null argument");
    Use use_(mesh);
    cudaStream_t s = mesh->stream;
    gh::Scratch<double> du(mesh->nv, s), dh(3 * (size_t)mesh->nf, s);
    GH_CUDA(cudaMemcpyAsync(du.p, u, sizeof(double) * mesh->nv, cudaMemcpyHostToDevice, s));
    const int32_t z = gh::normalize_dev(mesh, du.p, dh.p);
    to_host(h_out, dh.p, 3 * (size_t)mesh->nf, s);
    if (zero_count) *zero_count = z;
  });
}

gh_status gh_admm_face_optimize(gh_mesh* mesh, const double* h, const gh_admm_config* config, double* g_out,
                                gh_solver_report* report) {
  return guarded([&] {
    require(mesh && h && config && g_out, "gh_admm_face_optimize: null argument");
    Use use_(mesh);
    cudaStream_t s = mesh->stream;
    const double w0 = now_s();
    take_launches(mesh);
    gh::Scratch<double> dh(3 * (size_t)mesh->nf, s), dg(3 * (size_t)mesh->nf, s);
    GH_CUDA(cudaMemcpyAsync(dh.p, h, sizeof(double) * 3 * mesh->nf, cudaMemcpyHostToDevice, s));
    gh::AdmmResult r = gh::admm_face_dev(mesh, dh.p, *config, dg.p);
    to_host(g_out, dg.p, 3 * (size_t)mesh->nf, s);
    fill_solver_report(report, r, state_formula(mesh, GH_METHOD_FACE), now_s() - w0, take_launches(mesh));
  });
}

gh_status gh_admm_edge_optimize(gh_mesh* mesh, const double* h, const gh_admm_config* config, double* x_out,
                                gh_solver_report* report) {
  return guarded([&] {
    require(mesh && h && config && x_out, "gh_admm_edge_optimize: null argument");
    Use use_(mesh);
    cudaStream_t s = mesh->stream;
    const double w0 = now_s();
    take_launches(mesh);
    gh::Scratch<double> dh(3 * (size_t)mesh->nf, s), dx(mesh->ne, s);
    GH_CUDA(cudaMemcpyAsync(dh.p, h, sizeof(double) * 3 * mesh->nf, cudaMemcpyHostToDevice, s));
    gh::AdmmResult r = gh::admm_edge_dev(mesh, dh.p, *config, dx.p);
    to_host(x_out, dx.p, mesh->ne, s);
    fill_solver_report(report, r, state_formula(mesh, GH_METHOD_EDGE), now_s() - w0, take_launches(mesh));
  });
}

gh_status gh_solver_state_bytes(const gh_mesh* mesh, int32_t method, uint64_t* bytes_out) {
  return guarded([&] {
    require(mesh && bytes_out, "gh_solver_state_bytes: null argument");
    *bytes_out = state_formula(mesh, method);
  });
}

gh_status gh_integrate_face_gradients(gh_levels* levels, const double* g, double* d_out) {
  return guarded([&] {
    require(levels && g && d_out, "gh_integrate_face_gradients: null argument");
    gh_mesh* m = levels->mesh;
    Use use_(m);
    cudaStream_t s = m->stream;
    gh::Scratch<double> dg(3 * (size_t)m->nf, s), dd(m->nv, s);
    GH_CUDA(cudaMemcpyAsync(dg.p, g, sizeof(double) * 3 * m->nf, cudaMemcpyHostToDevice, s));
    gh::integrate_face_dev(levels, dg.p, dd.p);
    to_host(d_out, dd.p, m->nv, s);
  });
}

gh_status gh_integrate_edge_differences(gh_levels* levels, const double* x, double* d_out) {
  return guarded([&] {
    require(levels && x && d_out, "gh_integrate_edge_differences: null argument");
    gh_mesh* m = levels->mesh;
    Use use_(m);
    cudaStream_t s = m->stream;
    gh::Scratch<double> dx(m->ne, s), dd(m->nv, s);
    GH_CUDA(cudaMemcpyAsync(dx.p, x, sizeof(double) * m->ne, cudaMemcpyHostToDevice, s));
    gh::integrate_edge_dev(levels, dx.p, dd.p);
    to_host(d_out, dd.p, m->nv, s);
  });
}

}  // extern "C"

namespace {

// the device-resident chain of run_pipeline (tools/geoheat.cpp:108-143)
void distance_on_device(gh_levels* L, const gh_pipeline_config& c, double* d_dist, gh_run_report* rep) {
  gh_mesh* m = L->mesh;
  cudaStream_t s = m->stream;
  require(c.method == GH_METHOD_FACE || c.method == GH_METHOD_EDGE || c.method == GH_METHOD_POISSON,
          "gh_distance: unknown method");
  double t = c.t;
  if (!(t > 0.0)) {
    if (!(c.m > 0.0)) gh::fail(GH_ERR_INVALID, "diffusion_time: m must be positive");
    const double h = gh::mesh_average_edge_length(m);
    t = c.m * h * h;
  }
  if (rep) rep->diffusion_e1 = -1.0;
  if (c.method == GH_METHOD_POISSON) {  // geoheat.cpp:96-103
    require(c.cg_tol > 0.0, "gh_distance: cg_tol must be positive");
    const gh::PoissonOut po = gh::poisson_heat_dev(L, t, c.cg_tol, d_dist);
    if (rep) {
      rep->t = t;
      rep->cg_iterations = po.heat_iterations + po.poisson_iterations;
      rep->final_primal = po.poisson_residual;
      rep->poisson_residual = po.poisson_residual;
      rep->diffusion_ms = po.heat_seconds * 1e3;
      rep->optimization_ms = po.poisson_seconds * 1e3;
      rep->solver_state_bytes = state_formula(m, GH_METHOD_FACE);  // geoheat.cpp:145-147
    }
    return;
  }
  gh::EventTimer tn(s), ti(s);
  const double diff_ms = (c.flags & GH_PIPE_U_READY) ? 0.0 : gh::diffuse_dev(L, t, c.sweeps, nullptr);
  if (rep && (c.flags & GH_PIPE_DIFFUSION_E1)) rep->diffusion_e1 = gh::diffusion_residual_dev(L, L->u_orig.p, t);
  gh::Scratch<double> H(3 * (size_t)m->nf, s);
  tn.start();
  const int32_t zc = gh::normalize_dev(m, L->u_orig.p, H.p);
  tn.stop();
  gh::AdmmResult r;
  // elements that provably stay +0 through the optimisation are skipped (gh_grad.cu)
  const int32_t bound = gh::admm_active_level(L, H.p, c.admm.max_iterations);
  const bool skip = bound >= 0;
  gh::Scratch<uint8_t> act_f(skip ? (size_t)m->nf : 0, s);
  // (+32: k_face_lambda_pair reads the edge flags 16 bytes at a time; the pad is zero)
  const size_t n_act_e = (size_t)(c.method == GH_METHOD_FACE ? m->ni : m->ne);
  gh::Scratch<uint8_t> act_e(skip ? n_act_e + 32 : 0, s);
  if (skip) {
    GH_CUDA(cudaMemsetAsync(act_e.p + n_act_e, 0, 32, s));
    gh::admm_active_flags(L, bound, c.method == GH_METHOD_FACE, act_f.p, act_e.p);
  }
  if (c.method == GH_METHOD_FACE) {
    gh::Scratch<double> G(3 * (size_t)m->nf, s);
    r = gh::admm_face_dev(m, H.p, c.admm, G.p, act_f.p, act_e.p);
    ti.start();
    gh::integrate_face_dev(L, G.p, d_dist);
    ti.stop();
  } else {
    gh::Scratch<double> X(m->ne, s);
    r = gh::admm_edge_dev(m, H.p, c.admm, X.p, act_f.p, act_e.p);
    ti.start();
    gh::integrate_edge_dev(L, X.p, d_dist);
    ti.stop();
  }
  if (rep) {
    rep->t = t;
    rep->gs_iterations = c.sweeps;
    rep->admm_iterations = r.iterations;
    rep->converged = r.converged ? 1 : 0;
    rep->zero_count = zc;
    rep->final_primal = r.final_primal;
    rep->final_dual = r.final_dual;
    rep->diffusion_ms = diff_ms;
    rep->diffusion_row_updates = L->last_row_updates;
    rep->diffusion_active_levels = L->last_active_levels;
    rep->diffusion_launches = L->last_launches;
    rep->normalize_ms = tn.ms();
    rep->optimization_ms = r.device_ms;
    rep->integration_ms = ti.ms();
    rep->solver_state_bytes = state_formula(m, c.method);
    rep->state_bytes_allocated = r.state_bytes;
  }
}

}  // namespace

extern "C" {

gh_status gh_distance(gh_levels* levels, const gh_pipeline_config* config, double* d_out, gh_run_report* report) {
  return guarded([&] {
    require(levels && config && d_out, "gh_distance: null argument");
    gh_mesh* m = levels->mesh;
    Use use_(m);
    cudaStream_t s = m->stream;
    take_launches(m);
    if (report) std::memset(report, 0, sizeof(*report));
    gh::EventTimer total(s), d2h(s);
    total.start();
    gh::Scratch<double> dd(m->nv, s);
    distance_on_device(levels, *config, dd.p, report);
    d2h.start();
    GH_CUDA(cudaMemcpyAsync(d_out, dd.p, sizeof(double) * m->nv, cudaMemcpyDeviceToHost, s));
    d2h.stop();
    total.stop();
    GH_CUDA(cudaStreamSynchronize(s));
    if (report) {
      report->d2h_ms = d2h.ms();
      report->d2h_bytes = sizeof(double) * (uint64_t)m->nv;
      report->total_ms = total.ms();
      report->kernel_launches = take_launches(m);
    }
  });
}

gh_status gh_distance_host(const double* positions, int32_t nv, const int32_t* faces, int32_t nf,
                           const int32_t* sources, int32_t ns, const gh_pipeline_config* config, double* d_out,
                           gh_run_report* report) {
  gh_mesh* mesh = nullptr;
  gh_levels* levels = nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  gh_status st = gh_mesh_create(positions, nv, faces, nf, &mesh);
  const auto t1 = std::chrono::steady_clock::now();
  if (st != GH_OK) return st;
  int launches = mesh->launches;
  st = gh_bfs_create(mesh, sources, ns, &levels);
  const auto t2 = std::chrono::steady_clock::now();
  launches = mesh->launches;
  if (st == GH_OK) st = gh_distance(levels, config, d_out, report);
  const auto t3 = std::chrono::steady_clock::now();
  if (st == GH_OK && report) {
    report->build_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    report->bfs_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
    report->h2d_bytes = sizeof(double) * 3 * (uint64_t)nv + sizeof(int32_t) * 3 * (uint64_t)nf + 4 * (uint64_t)ns;
    report->total_ms = std::chrono::duration<double, std::milli>(t3 - t0).count();
    report->kernel_launches += launches;
  }
  gh_status s2 = gh_bfs_destroy(levels);
  gh_status s3 = gh_mesh_destroy(mesh);
  if (st == GH_OK) st = s2 != GH_OK ? s2 : s3;
  return st;
}

gh_status gh_poisson_heat_method(gh_levels* levels, double t, double cg_tol, double* d_out, gh_poisson_report* report) {
  return guarded([&] {
    require(levels && d_out, "gh_poisson_heat_method: null argument");
    require(t > 0.0 && cg_tol > 0.0, "gh_poisson_heat_method: t and cg_tol must be positive");
    gh_mesh* m = levels->mesh;
    Use use_(m);
    take_launches(m);
    gh::Scratch<double> dd(m->nv, m->stream);
    const gh::PoissonOut po = gh::poisson_heat_dev(levels, t, cg_tol, dd.p);
    to_host(d_out, dd.p, m->nv, m->stream);
    if (report) {
      report->heat_iterations = po.heat_iterations;
      report->poisson_iterations = po.poisson_iterations;
      report->heat_residual = po.heat_residual;
      report->poisson_residual = po.poisson_residual;
      report->heat_seconds = po.heat_seconds;
      report->poisson_seconds = po.poisson_seconds;
      report->kernel_launches = take_launches(m);
      report->reserved = 0;
    }
  });
}

gh_status gh_triangulation_quality(gh_mesh* mesh, double* tau_out) {
  return guarded([&] {
    require(mesh && tau_out, "gh_triangulation_quality: null argument");
    Use use_(mesh);
    *tau_out = gh::triangulation_quality_dev(mesh);
  });
}

gh_status gh_mesh_subdivide(gh_mesh* mesh, int32_t levels, gh_mesh** out) {
  return guarded([&] {
    require(mesh && out, "gh_mesh_subdivide: null argument");
    Use use_(mesh);
    std::unique_ptr<gh_mesh> cur = new_mesh();
    if (levels <= 0) {
      gh::copy_mesh_arrays(mesh, cur.get());  // midpoint_subdivide(mesh, 0) returns the mesh
    } else {
      gh::subdivide_once(mesh, cur.get());
      for (int32_t i = 1; i < levels; ++i) {
        std::unique_ptr<gh_mesh> next = new_mesh();
        gh::subdivide_once(cur.get(), next.get());
        cur = std::move(next);
      }
    }
    GH_CUDA(cudaStreamSynchronize(cur->stream));
    *out = cur.release();
  });
}

static void check_sources(const gh_mesh* m, const int32_t* sources, int32_t ns) {
  require(ns >= 0 && (ns == 0 || sources), "null sources");
  for (int32_t i = 0; i < ns; ++i)
    if (sources[i] < 0 || sources[i] >= m->nv)
      gh::fail(GH_ERR_INVALID, "source index " + std::to_string(sources[i]) + " out of range");
}

gh_status gh_analytic_distance(gh_mesh* mesh, int32_t kind, const int32_t* sources, int32_t ns, double* d_out) {
  return guarded([&] {
    require(mesh && d_out, "gh_analytic_distance: null argument");
    require(kind == GH_SURFACE_PLANE || kind == GH_SURFACE_SPHERE, "gh_analytic_distance: unknown surface");
    check_sources(mesh, sources, ns);
    Use use_(mesh);
    cudaStream_t s = mesh->stream;
    gh::Scratch<int32_t> src(ns, s);
    gh::Scratch<double> d(mesh->nv, s);
    if (ns) GH_CUDA(cudaMemcpyAsync(src.p, sources, sizeof(int32_t) * ns, cudaMemcpyHostToDevice, s));
    gh::analytic_dev(mesh, kind, src.p, ns, d.p);
    to_host(d_out, d.p, mesh->nv, s);
  });
}

gh_status gh_dijkstra_distance(gh_mesh* mesh, const int32_t* sources, int32_t ns, double* d_out) {
  return guarded([&] {
    require(mesh && d_out, "gh_dijkstra_distance: null argument");
    check_sources(mesh, sources, ns);
    Use use_(mesh);
    cudaStream_t s = mesh->stream;
    gh::Scratch<int32_t> src(ns, s);
    gh::Scratch<double> d(mesh->nv, s);
    if (ns) GH_CUDA(cudaMemcpyAsync(src.p, sources, sizeof(int32_t) * ns, cudaMemcpyHostToDevice, s));
    gh::dijkstra_dev(mesh, src.p, ns, d.p);
    to_host(d_out, d.p, mesh->nv, s);
  });
}

gh_status gh_error_metrics(const double* d, const double* d_ref, int64_t n, const int32_t* sources, int32_t ns,
                           double* mean_rel_error, int32_t* excluded, double* e2) {
  return guarded([&] {
    require(n > 0 && d && d_ref && mean_rel_error && excluded && e2, "gh_error_metrics: bad argument");
    require(ns >= 0 && (ns == 0 || sources), "gh_error_metrics: null sources");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      (void)cudaGetLastError();
      gh::fail(GH_ERR_CUDA, "no CUDA device available (the geoheat_b200 path has no CPU fallback)");
    }
    if (g_device >= 0) GH_CUDA(cudaSetDevice(g_device));
    int dev = 0;
    GH_CUDA(cudaGetDevice(&dev));
    cudaStream_t s;
    thread_context(dev, &s, nullptr);
    gh::errors_dev(s, d, d_ref, n, sources, ns, mean_rel_error, excluded, e2);
  });
}

gh_status gh_deterministic_sum(const double* terms, int64_t n, double* sum_out) {
  return guarded([&] {
    require(sum_out && n >= 0 && (n == 0 || terms), "gh_deterministic_sum: bad argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      (void)cudaGetLastError();
      gh::fail(GH_ERR_CUDA, "no CUDA device available (the geoheat_b200 path has no CPU fallback)");
    }
    if (g_device >= 0) GH_CUDA(cudaSetDevice(g_device));
    int dev = 0;
    GH_CUDA(cudaGetDevice(&dev));
    keep_pool_memory(dev);
    cudaStream_t s;
    thread_context(dev, &s, nullptr);
    gh::Scratch<double> x(n, s);
    if (n) GH_CUDA(cudaMemcpyAsync(x.p, terms, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    *sum_out = gh::deterministic_sum_dev(x.p, n, s);
  });
}

gh_status gh_deterministic_sums(const double* terms, int64_t n, int32_t count, double* sums_out) {
  return guarded([&] {
    require(sums_out && n >= 0 && count >= 0 && (n == 0 || count == 0 || terms), "gh_deterministic_sums: bad argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      (void)cudaGetLastError();
      gh::fail(GH_ERR_CUDA, "no CUDA device available (the geoheat_b200 path has no CPU fallback)");
    }
    if (count == 0) return;
    if (g_device >= 0) GH_CUDA(cudaSetDevice(g_device));
    int dev = 0;
    GH_CUDA(cudaGetDevice(&dev));
    keep_pool_memory(dev);
    cudaStream_t s;
    thread_context(dev, &s, nullptr);
    gh::Scratch<double> x((size_t)n * count, s), out((size_t)count, s);
    if (n) GH_CUDA(cudaMemcpyAsync(x.p, terms, sizeof(double) * n * count, cudaMemcpyHostToDevice, s));
    gh::sequential_sums_group(x.p, n, n, count, out.p, s);
    GH_CUDA(cudaMemcpyAsync(sums_out, out.p, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
    GH_CUDA(cudaStreamSynchronize(s));
  });
}

uint64_t gh_field_hash(const double* values, int64_t n) {
  uint64_t h = 1469598103934665603ull;  // report.hpp:145-153
  const unsigned char* b = reinterpret_cast<const unsigned char*>(values);
  for (int64_t i = 0; i < n * (int64_t)sizeof(double); ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h;
}

}  // extern "C"

// ---------------------------------------------------------------- BFS bands (multi-GPU)

struct gh_band {
  gh_levels* levels = nullptr;
  gh::Band band;
  int32_t rank = 0, nranks = 1;
  std::vector<void*> opened;  // peer allocations mapped with cudaIpcOpenMemHandle
  // gh_band_adopt: the band's own buffers, set aside while it drives another
  // process's copies of them (restored before the band is freed)
  bool adopted = false;
  double* own_ubuf = nullptr;
  unsigned long long* own_done = nullptr;
  unsigned long long* own_gdone = nullptr;
};

namespace {

struct BandBlob {
  cudaIpcMemHandle_t ubuf;
  cudaIpcMemHandle_t done;
  cudaIpcMemHandle_t gdone;  // slices: ghost counters per (source, level)
  int32_t nslices, rank;
  int64_t nrows;
  int32_t lb, le;
  int32_t ghost_lo_row;  // row of level lb-1 inside this band, -1 without one
  int32_t ghost_hi_row;  // row of level le inside this band, -1 without one
  int32_t device, magic;
};
constexpr int32_t kBlobMagic = 0x67686264;  // "ghbd"

}  // namespace

extern "C" {

gh_status gh_plan_bands(const int32_t* offsets, int32_t nlev, int32_t nbands, int32_t* cut_out) {
  return guarded([&] {
    require(offsets && cut_out && nlev >= 1, "gh_plan_bands: bad arguments");
    const std::vector<int32_t> off(offsets, offsets + nlev + 1);
    const std::vector<int32_t> cut = gh::plan_bands(off, nbands);
    std::memcpy(cut_out, cut.data(), sizeof(int32_t) * cut.size());
  });
}

gh_status gh_gs_diffuse_bands(gh_levels* levels, int32_t nbands, double t, int32_t sweeps, const double* initial,
                              double* u_out, gh_solver_report* report) {
  return gh_gs_diffuse_partitioned(levels, nbands, GH_PARTITION_BANDS, t, sweeps, initial, u_out, report);
}

gh_status gh_gs_diffuse_partitioned(gh_levels* levels, int32_t nbands, int32_t partition, double t, int32_t sweeps,
                                    const double* initial, double* u_out, gh_solver_report* report) {
  return guarded([&] {
    require(levels != nullptr, "gh_gs_diffuse_partitioned: null levels");
    require(partition == GH_PARTITION_BANDS || partition == GH_PARTITION_SLICES,
            "gh_gs_diffuse_partitioned: unknown partition");
    gh_mesh* m = levels->mesh;
    Use use_(m);
    cudaStream_t s = m->stream;
    const double w0 = now_s();
    take_launches(m);
    std::vector<std::unique_ptr<gh::Band>> own;
    std::vector<gh::Band*> bands;
    if (partition == GH_PARTITION_SLICES) {
      require(nbands >= 1 && nbands <= gh::Band::kMaxSlices, "gh_gs_diffuse_partitioned: 1 to 8 slices");
      if (levels->nreach == 0) nbands = 1;
      for (int32_t r = 0; r < nbands; ++r) {
        own.emplace_back(new gh::Band());
        gh::slice_build(levels, own.back().get(), r, nbands);
        bands.push_back(own.back().get());
      }
      gh::slice_link(bands);
    } else {
      const std::vector<int32_t> cut = gh::plan_bands(levels->h_offsets, nbands);
      for (int32_t r = 0; r < nbands; ++r) {
        own.emplace_back(new gh::Band());
        gh::band_build(levels, own.back().get(), cut[r], cut[r + 1]);
        bands.push_back(own.back().get());
      }
      for (int32_t r = 0; r + 1 < nbands; ++r) gh::band_link(bands[r], bands[r + 1]);
    }
    gh::Scratch<double> dinit(initial ? m->nv : 0, s);
    if (initial) GH_CUDA(cudaMemcpyAsync(dinit.p, initial, sizeof(double) * m->nv, cudaMemcpyHostToDevice, s));
    const double ms = gh::diffuse_bands_dev(levels, bands, t, sweeps, initial ? dinit.p : nullptr);
    if (u_out) to_host(u_out, levels->u_orig.p, m->nv, s);
    else GH_CUDA(cudaStreamSynchronize(s));
    if (report) {
      report->iterations = sweeps;
      report->converged = 0;
      report->wall_seconds = now_s() - w0;
      report->device_ms = ms;
      report->kernel_launches = take_launches(m);
    }
  });
}

gh_status gh_band_create(gh_levels* levels, int32_t rank, int32_t nranks, gh_band** out) {
  return gh_band_create_partitioned(levels, rank, nranks, GH_PARTITION_BANDS, out);
}

gh_status gh_band_create_partitioned(gh_levels* levels, int32_t rank, int32_t nranks, int32_t partition,
                                     gh_band** out) {
  return guarded([&] {
    require(levels && out, "gh_band_create: null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "gh_band_create: bad rank");
    require(partition == GH_PARTITION_BANDS || partition == GH_PARTITION_SLICES, "gh_band_create: unknown partition");
    Use use_(levels->mesh);
    std::unique_ptr<gh_band> b(new gh_band());
    b->levels = levels;
    b->rank = rank;
    b->nranks = nranks;
    b->band.ipc = true;  // its buffers are exported to the neighbour processes
    if (partition == GH_PARTITION_SLICES) {
      require(nranks <= gh::Band::kMaxSlices, "gh_band_create: 1 to 8 slices");
      gh::slice_build(levels, &b->band, rank, nranks);
    } else {
      const std::vector<int32_t> cut = gh::plan_bands(levels->h_offsets, nranks);
      gh::band_build(levels, &b->band, cut[rank], cut[rank + 1]);
    }
    *out = b.release();
  });
}

gh_status gh_band_destroy(gh_band* band) {
  return guarded([&] {
    if (!band) return;
    Use use_(band->levels->mesh);
    cudaStreamSynchronize(band->levels->mesh->stream);
    for (void* p : band->opened) cudaIpcCloseMemHandle(p);
    if (band->adopted) {  // ~Band frees the band's own buffers, never the mapped ones
      band->band.ubuf = band->own_ubuf;
      band->band.rows_done = band->own_done;
      band->band.gdone = band->own_gdone;
    }
    delete band;
  });
}

gh_status gh_band_info(const gh_band* band, int32_t* lb, int32_t* le, int32_t* own_rows) {
  return guarded([&] {
    require(band != nullptr, "gh_band_info: null band");
    if (lb) *lb = band->band.lb;
    if (le) *le = band->band.le;
    if (own_rows) *own_rows = band->band.own_rows;
  });
}

gh_status gh_band_export(const gh_band* band, void* blob, int32_t capacity, int32_t* size) {
  return guarded([&] {
    require(band && size, "gh_band_export: null argument");
    *size = (int32_t)sizeof(BandBlob);
    if (!blob) return;
    require(capacity >= (int32_t)sizeof(BandBlob), "gh_band_export: blob buffer too small");
    const gh::Band& b = band->band;
    BandBlob x{};
    Use use_(band->levels->mesh);
    GH_CUDA(cudaIpcGetMemHandle(&x.ubuf, b.ubuf));
    GH_CUDA(cudaIpcGetMemHandle(&x.done, b.rows_done));
    if (b.gdone) GH_CUDA(cudaIpcGetMemHandle(&x.gdone, b.gdone));
    x.nslices = b.nslices;
    x.rank = b.rank;
    x.nrows = b.nrows;
    x.lb = b.lb;
    x.le = b.le;
    x.ghost_lo_row = b.lb > 0 ? b.ghost_row(b.lb - 1) : -1;
    x.ghost_hi_row = b.le < b.nlev ? b.ghost_row(b.le) : -1;
    x.device = b.device;
    x.magic = kBlobMagic;
    std::memcpy(blob, &x, sizeof(x));
  });
}

gh_status gh_band_connect(gh_band* band, const void* lower_blob, const void* upper_blob) {
  return guarded([&] {
    require(band != nullptr, "gh_band_connect: null band");
    gh::Band& b = band->band;
    require(b.nslices == 0, "gh_band_connect: slices connect to every rank (gh_band_connect_all)");
    b.peer_sys = true;  // the neighbours are other processes' GPUs
    Use use_(band->levels->mesh);
    auto open = [&](const cudaIpcMemHandle_t& h) {
      void* p = nullptr;
      GH_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      band->opened.push_back(p);
      return p;
    };
    if (lower_blob) {
      BandBlob x;
      std::memcpy(&x, lower_blob, sizeof(x));
      require(x.magic == kBlobMagic && x.le == b.lb, "gh_band_connect: lower blob is not the lower neighbour");
      b.lo_ubuf = static_cast<double*>(open(x.ubuf));
      b.lo_done = static_cast<unsigned long long*>(open(x.done));
      b.lo_nrows = x.nrows;
      b.lo_ghost = x.ghost_hi_row;  // our first level is its upper ghost
    }
    if (upper_blob) {
      BandBlob x;
      std::memcpy(&x, upper_blob, sizeof(x));
      require(x.magic == kBlobMagic && x.lb == b.le, "gh_band_connect: upper blob is not the upper neighbour");
      b.hi_ubuf = static_cast<double*>(open(x.ubuf));
      b.hi_done = static_cast<unsigned long long*>(open(x.done));
      b.hi_nrows = x.nrows;
      b.hi_ghost = x.ghost_lo_row;  // our last level is its lower ghost
    }
  });
}

gh_status gh_band_connect_all(gh_band* band, const void* const* blobs, int32_t nranks) {
  return guarded([&] {
    require(band && blobs, "gh_band_connect_all: null argument");
    gh::Band& b = band->band;
    require(b.nslices > 0, "gh_band_connect_all: not a slice (level bands connect with gh_band_connect)");
    require(nranks == b.nslices, "gh_band_connect_all: one blob per slice");
    Use use_(band->levels->mesh);
    for (int32_t d = 0; d < nranks; ++d) {
      if (d == b.rank) {
        b.peer_ubuf[d] = b.ubuf;
        b.peer_gdone[d] = b.gdone;
        continue;
      }
      require(blobs[d] != nullptr, "gh_band_connect_all: missing blob");
      BandBlob x;
      std::memcpy(&x, blobs[d], sizeof(x));
      if (!(x.magic == kBlobMagic && x.nslices == b.nslices && x.rank == d))
        gh::fail(GH_ERR_INVALID, "gh_band_connect_all: blob is not slice " + std::to_string(d) + " of this partition");
      void* p = nullptr;
      GH_CUDA(cudaIpcOpenMemHandle(&p, x.ubuf, cudaIpcMemLazyEnablePeerAccess));
      band->opened.push_back(p);
      b.peer_ubuf[d] = static_cast<double*>(p);
      GH_CUDA(cudaIpcOpenMemHandle(&p, x.gdone, cudaIpcMemLazyEnablePeerAccess));
      band->opened.push_back(p);
      b.peer_gdone[d] = static_cast<unsigned long long*>(p);
    }
    b.peer_sys = true;  // the peers are other processes' GPUs
  });
}

gh_status gh_band_adopt(gh_band* band, const void* blob) {
  return guarded([&] {
    require(band && blob, "gh_band_adopt: null argument");
    require(!band->adopted, "gh_band_adopt: band already drives another process's buffers");
    gh::Band& b = band->band;
    BandBlob x;
    std::memcpy(&x, blob, sizeof(x));
    require(x.magic == kBlobMagic, "gh_band_adopt: not a band blob");
    if (!(x.nslices == b.nslices && (b.nslices == 0 || x.rank == b.rank) && x.nrows == b.nrows && x.lb == b.lb &&
          x.le == b.le && x.device == b.device))
      gh::fail(GH_ERR_INVALID, "gh_band_adopt: the blob is not this part of this partition on this device");
    Use use_(band->levels->mesh);
    // map every buffer first: on a failure the band keeps its own buffers
    std::vector<void*> mapped;
    auto open = [&](const cudaIpcMemHandle_t& h) {
      void* p = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        for (void* q : mapped) cudaIpcCloseMemHandle(q);
        gh::fail(GH_ERR_CUDA, std::string("gh_band_adopt: cudaIpcOpenMemHandle failed: ") + cudaGetErrorString(e));
      }
      mapped.push_back(p);
      return p;
    };
    double* ubuf = static_cast<double*>(open(x.ubuf));
    unsigned long long* done = static_cast<unsigned long long*>(open(x.done));
    unsigned long long* gdone = b.gdone ? static_cast<unsigned long long*>(open(x.gdone)) : nullptr;
    band->opened.insert(band->opened.end(), mapped.begin(), mapped.end());
    band->own_ubuf = b.ubuf;
    band->own_done = b.rows_done;
    band->own_gdone = b.gdone;
    b.ubuf = ubuf;
    b.rows_done = done;
    b.gdone = gdone;
    band->adopted = true;
  });
}

gh_status gh_band_launch_group(gh_band* const* bands, int32_t n, double t, int32_t sweeps, const double* initial,
                               double* u_out, gh_solver_report* report) {
  return guarded([&] {
    require(bands && n >= 1, "gh_band_launch_group: no bands");
    gh_levels* L = bands[0] ? bands[0]->levels : nullptr;
    require(L != nullptr, "gh_band_launch_group: null band");
    std::vector<gh::Band*> v;
    bool any_adopted = false;
    for (int32_t r = 0; r < n; ++r) {
      require(bands[r] && bands[r]->levels == L, "gh_band_launch_group: bands of different BFS levels");
      require(bands[r]->rank == r && bands[r]->nranks == n,
              "gh_band_launch_group: the group must be parts 0..n-1 of one partition, in order");
      v.push_back(&bands[r]->band);
      any_adopted |= bands[r]->adopted;
    }
    const bool slices = v[0]->nslices > 0;
    for (gh::Band* b : v)
      require((b->nslices > 0) == slices, "gh_band_launch_group: slices and level bands in one group");
    gh_mesh* m = L->mesh;
    Use use_(m);
    cudaStream_t s = m->stream;
    const double w0 = now_s();
    take_launches(m);
    if (slices) {
      gh::slice_link(v);
    } else {
      for (int32_t r = 0; r + 1 < n; ++r) gh::band_link(v[r], v[r + 1]);
    }
    // buffers of other processes: system-scope releases and polls, as between GPUs
    for (gh::Band* b : v) b->peer_sys = any_adopted;
    gh::Scratch<double> dinit(initial ? m->nv : 0, s);
    if (initial) GH_CUDA(cudaMemcpyAsync(dinit.p, initial, sizeof(double) * m->nv, cudaMemcpyHostToDevice, s));
    const double ms = gh::diffuse_bands_dev(L, v, t, sweeps, initial ? dinit.p : nullptr);
    if (u_out) to_host(u_out, L->u_orig.p, m->nv, s);
    else GH_CUDA(cudaStreamSynchronize(s));
    if (report) {
      report->iterations = sweeps;
      report->converged = 0;
      report->wall_seconds = now_s() - w0;
      report->device_ms = ms;
      report->kernel_launches = take_launches(m);
    }
  });
}

gh_status gh_band_download(const gh_band* band, int32_t sweeps, double* u_out) {
  return guarded([&] {
    require(band && u_out && sweeps >= 1, "gh_band_download: bad argument");
    gh_mesh* m = band->levels->mesh;
    Use use_(m);
    cudaStream_t s = m->stream;
    gh::Scratch<double> du(m->nv, s);
    GH_CUDA(cudaMemcpyAsync(du.p, u_out, sizeof(double) * m->nv, cudaMemcpyHostToDevice, s));
    gh::band_own_u(&band->band, sweeps, du.p, s);
    to_host(u_out, du.p, m->nv, s);
  });
}

gh_status gh_levels_u_device(gh_levels* levels, double** u_dev, int64_t* n) {
  return guarded([&] {
    require(levels && u_dev, "gh_levels_u_device: null argument");
    *u_dev = levels->u_orig.p;
    if (n) *n = (int64_t)levels->u_orig.n;
  });
}

gh_status gh_band_own_mask(const gh_band* band, uint8_t* mask_out) {
  return guarded([&] {
    require(band && mask_out, "gh_band_own_mask: null argument");
    gh_mesh* m = band->levels->mesh;
    Use use_(m);
    gh::Scratch<uint8_t> d(m->nv, m->stream);
    gh::band_own_mask(&band->band, d.p, m->nv, m->stream);
    to_host(mask_out, d.p, m->nv, m->stream);
  });
}

gh_status gh_band_prepare(gh_band* band, double t, const double* initial) {
  return guarded([&] {
    require(band != nullptr, "gh_band_prepare: null band");
    if (!(t > 0.0)) gh::fail(GH_ERR_INVALID, "gs_diffuse: t must be positive");
    gh_mesh* m = band->levels->mesh;
    Use use_(m);
    cudaStream_t s = m->stream;
    gh::Scratch<double> dinit(initial ? m->nv : 0, s);
    if (initial) GH_CUDA(cudaMemcpyAsync(dinit.p, initial, sizeof(double) * m->nv, cudaMemcpyHostToDevice, s));
    std::vector<gh::Band*> one{&band->band};
    gh::bands_prepare(band->levels, one, t, initial ? dinit.p : nullptr);
    GH_CUDA(cudaStreamSynchronize(s));
  });
}

gh_status gh_band_launch(gh_band* band, double t, int32_t sweeps, double* u_out, gh_solver_report* report) {
  return guarded([&] {
    require(band != nullptr, "gh_band_launch: null band");
    require(sweeps >= 1, "gh_band_launch: sweeps must be >= 1");
    gh_mesh* m = band->levels->mesh;
    Use use_(m);
    cudaStream_t s = m->stream;
    const double w0 = now_s();
    take_launches(m);
    std::vector<gh::Band*> one{&band->band};
    const double ms = gh::bands_launch(band->levels, one, t, sweeps);
    if (u_out) to_host(u_out, band->levels->u_orig.p, m->nv, s);
    else GH_CUDA(cudaStreamSynchronize(s));
    if (report) {
      report->iterations = sweeps;
      report->wall_seconds = now_s() - w0;
      report->device_ms = ms;
      report->kernel_launches = take_launches(m);
    }
  });
}

}  // extern "C"
