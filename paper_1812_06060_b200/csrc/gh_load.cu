// Mesh load -> device build (load_mesh, mesh_io.hpp:
// 267-285). A file is memory-mapped; binary little-endian PLY is streamed to
// HBM through pinned slots by several host threads and its records are
// decoded ON THE DEVICE straight into the mesh arrays build_mesh consumes;
// text formats (OBJ, ASCII PLY) are tokenised by host threads
// (gh_meshio.cpp) and copied once. Errors match the reference's messages
// and precedence: the device decoder flags the first suspicious face record
// and the host walker re-reads exactly that record the way the reference
// would (truncation offsets, non-triangles, index range).

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <mutex>
#include <thread>

#include "gh_internal.cuh"
#include "gh_meshio.hpp"

namespace {

using gh::fail;

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

struct MemSource : ghio::ByteSource {
  const unsigned char* p;
  uint64_t n;
  MemSource(const unsigned char* data, uint64_t bytes) : p(data), n(bytes) {}
  uint64_t size() const override { return n; }
  void read(uint64_t off, uint64_t len, void* dst) const override { std::memcpy(dst, p + off, len); }
};

// Read-only mapping of a whole file.
struct Mapping {
  const unsigned char* p = nullptr;
  uint64_t n = 0;
  int fd = -1;
  explicit Mapping(const std::string& path) {
    fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
    struct stat st;
    if (fd < 0 || ::fstat(fd, &st) != 0 || !S_ISREG(st.st_mode)) {
      if (fd >= 0) ::close(fd);
      fd = -1;
      fail(GH_ERR_MESH, "cannot open mesh file '" + path + "'");
    }
    n = (uint64_t)st.st_size;
    if (n) {
      void* m = ::mmap(nullptr, n, PROT_READ, MAP_PRIVATE, fd, 0);
      if (m == MAP_FAILED) {
        ::close(fd);
        fd = -1;
        fail(GH_ERR_MESH, "cannot open mesh file '" + path + "'");
      }
      ::madvise(m, n, MADV_SEQUENTIAL);
      p = (const unsigned char*)m;
    }
  }
  ~Mapping() {
    if (p) ::munmap(const_cast<unsigned char*>(p), n);
    if (fd >= 0) ::close(fd);
  }
};

// ------------------------------------------------------- host -> device
// Process-wide pinned staging slots (grow-only, like the device pool).
constexpr uint64_t kSlot = 16ull << 20;
std::mutex g_slot_mu;
std::vector<void*> g_slots;

std::vector<void*> take_slots(size_t count) {
  std::lock_guard<std::mutex> lk(g_slot_mu);
  while (g_slots.size() < count) {
    void* p = nullptr;
    GH_CUDA(cudaMallocHost(&p, kSlot));
    g_slots.push_back(p);
  }
  std::vector<void*> out(g_slots.end() - count, g_slots.end());
  g_slots.resize(g_slots.size() - count);
  return out;
}
void give_slots(const std::vector<void*>& s) {
  std::lock_guard<std::mutex> lk(g_slot_mu);
  g_slots.insert(g_slots.end(), s.begin(), s.end());
}

// Copies host [src, src+n) to device dst: `threads` workers each fill two
// pinned slots in turn (the memcpy also faults the mapped file in) and issue
// the H2D copy of one while filling the other. Returns when the data is on
// the device.
void stage_to_device(const unsigned char* src, uint64_t n, unsigned char* dst, int threads, int device) {
  if (!n) return;
  const uint64_t chunks = (n + kSlot - 1) / kSlot;
  const int nt = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)std::max(threads, 1), chunks));
  std::vector<void*> slots = take_slots(2 * (size_t)nt);
  std::vector<std::string> errors(nt);
  auto worker = [&](int j) {
    cudaStream_t s = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    try {
      GH_CUDA(cudaSetDevice(device));
      GH_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      GH_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
      GH_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
      int k = 0;
      for (uint64_t c = (uint64_t)j; c < chunks; c += (uint64_t)nt, ++k) {
        const int b = k & 1;
        void* slot = slots[2 * j + b];
        if (k >= 2) GH_CUDA(cudaEventSynchronize(ev[b]));
        const uint64_t off = c * kSlot, len = std::min(kSlot, n - off);
        std::memcpy(slot, src + off, len);
        GH_CUDA(cudaMemcpyAsync(dst + off, slot, len, cudaMemcpyHostToDevice, s));
        GH_CUDA(cudaEventRecord(ev[b], s));
      }
      GH_CUDA(cudaStreamSynchronize(s));
    } catch (const gh::Error& e) {
      errors[j] = e.msg;
    } catch (...) {  // nothing may escape a std::thread
      errors[j] = "host->device staging failed";
    }
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  };
  std::vector<std::thread> pool;
  for (int j = 1; j < nt; ++j) pool.emplace_back(worker, j);
  worker(0);
  for (auto& t : pool) t.join();
  give_slots(slots);
  for (const std::string& e : errors)
    if (!e.empty()) fail(GH_ERR_CUDA, e);
}

// The reverse: device [src, src+n) to pageable host dst, each worker taking
// chunks through two pinned slots (H2D of one while the other is copied out).
void stage_from_device(const unsigned char* src, uint64_t n, unsigned char* dst, int threads, int device) {
  if (!n) return;
  const uint64_t chunks = (n + kSlot - 1) / kSlot;
  const int nt = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)std::max(threads, 1), chunks));
  std::vector<void*> slots = take_slots(2 * (size_t)nt);
  std::vector<std::string> errors(nt);
  auto worker = [&](int j) {
    cudaStream_t s = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    try {
      GH_CUDA(cudaSetDevice(device));
      GH_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      GH_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
      GH_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
      uint64_t pend_off[2] = {0, 0}, pend_len[2] = {0, 0};
      int k = 0;
      for (uint64_t c = (uint64_t)j;; c += (uint64_t)nt, ++k) {
        const int b = k & 1;
        if (c < chunks) {  // start chunk c into slot b
          const uint64_t off = c * kSlot, len = std::min(kSlot, n - off);
          GH_CUDA(cudaMemcpyAsync(slots[2 * j + b], src + off, len, cudaMemcpyDeviceToHost, s));
          GH_CUDA(cudaEventRecord(ev[b], s));
          pend_off[b] = off;
          pend_len[b] = len;
        }
        const int o = b ^ 1;  // finish the other slot's chunk (started last round)
        if (pend_len[o]) {
          GH_CUDA(cudaEventSynchronize(ev[o]));
          std::memcpy(dst + pend_off[o], slots[2 * j + o], pend_len[o]);
          pend_len[o] = 0;
        }
        if (c >= chunks && !pend_len[b]) break;
      }
    } catch (const gh::Error& e) {
      errors[j] = e.msg;
    } catch (...) {
      errors[j] = "device->host staging failed";
    }
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  };
  std::vector<std::thread> pool;
  for (int j = 1; j < nt; ++j) pool.emplace_back(worker, j);
  worker(0);
  for (auto& t : pool) t.join();
  give_slots(slots);
  for (const std::string& e : errors)
    if (!e.empty()) fail(GH_ERR_CUDA, e);
}

// ------------------------------------------------------- device decode
__device__ __forceinline__ double load_scalar(const unsigned char* p, int type) {
  uint64_t bits = 0;
  const int n = (type <= ghio::U8) ? 1 : (type <= ghio::U16) ? 2 : (type == ghio::F64) ? 8 : 4;
  for (int i = 0; i < n; ++i) bits |= (uint64_t)p[i] << (8 * i);
  switch (type) {
    case ghio::I8: return (double)(int8_t)bits;
    case ghio::U8: return (double)(uint8_t)bits;
    case ghio::I16: return (double)(int16_t)bits;
    case ghio::U16: return (double)(uint16_t)bits;
    case ghio::I32: return (double)(int32_t)bits;
    case ghio::U32: return (double)(uint32_t)bits;
    case ghio::F32: return (double)__uint_as_float((uint32_t)bits);
    default: return __longlong_as_double((long long)bits);
  }
}

// static_cast<long>(double) with x86-64 semantics (LONG_MIN when out of range
// or NaN), as the reference executes it on the host.
__device__ __forceinline__ long long to_long_x86(double v) {
  if (v >= -9223372036854775808.0 && v < 9223372036854775808.0) return (long long)v;
  return (long long)0x8000000000000000ull;
}

struct VertexDecode {
  int32_t stride, off[3];
  int32_t type[3];
};
struct FaceDecode {
  int32_t stride, list_off, count_type, value_type, count_size, value_size;
};

__global__ void k_decode_vertices(const unsigned char* __restrict__ raw, int64_t n, VertexDecode L,
                                  double* __restrict__ pos) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned char* r = raw + v * L.stride;
#pragma unroll
    for (int k = 0; k < 3; ++k) pos[3 * v + k] = load_scalar(r + L.off[k], L.type[k]);
  }
}

// Faces assuming list length 3; *first_bad = lowest record whose length is
// not 3 or whose index is outside [0, nv) (mesh_io.hpp:250-258).
__global__ void k_decode_faces(const unsigned char* __restrict__ raw, int64_t n, FaceDecode L, int64_t nv,
                               int32_t* __restrict__ faces, unsigned long long* first_bad) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n; f += (int64_t)gridDim.x * blockDim.x) {
    const unsigned char* r = raw + f * L.stride + L.list_off;
    bool bad = to_long_x86(load_scalar(r, L.count_type)) != 3;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const long long v = to_long_x86(load_scalar(r + L.count_size + k * L.value_size, L.value_type));
      bad |= v < 0 || v >= nv;
      faces[3 * f + k] = (int32_t)v;
    }
    if (bad) atomicMin(first_bad, (unsigned long long)f);
  }
}

void check_counts(int64_t nv, int64_t nf) {
  if (nv > 0x7fffffffLL || 3 * nf > 0x7fffffffLL)
    fail(GH_ERR_MESH, "mesh exceeds the int32 index range (" + std::to_string(nv) + " vertices, " +
                          std::to_string(nf) + " faces)");
}

void from_host(gh_mesh* m, const ghio::HostMesh& hm) {
  const int64_t nv = (int64_t)hm.pos.size() / 3, nf = (int64_t)hm.faces.size() / 3;
  check_counts(nv, nf);
  m->nv = (int32_t)nv;
  m->nf = (int32_t)nf;
  gh::mesh_build(m, hm.pos.data(), hm.faces.data());
}

// Binary PLY: device decode of the fixed layout, host walker for the rest.
void load_binary_ply(gh_mesh* m, const ghio::PlyHeader& h, const unsigned char* bytes, uint64_t n, int threads,
                     gh_load_report* rep) {
  const unsigned char* data = bytes + h.data_offset;
  const uint64_t avail = n - h.data_offset;
  MemSource src(data, avail);
  const ghio::FixedLayout L = ghio::fixed_layout(h);
  auto t0 = std::chrono::steady_clock::now();
  if (!L.ok) {
    // layouts outside the fixed-stride decoder (list properties on vertices,
    // several face lists, repeated vertex/face elements): the sequential walk
    ghio::HostMesh hm;
    ghio::walk_binary(h, src, 0, 0, 0, 0, &hm);
    if (rep) rep->parse_ms = ms_since(t0);
    auto tb = std::chrono::steady_clock::now();
    from_host(m, hm);
    if (rep) {
      GH_CUDA(cudaStreamSynchronize(m->stream));
      rep->build_ms = ms_since(tb);
    }
    return;
  }
  const uint64_t vs = (uint64_t)L.vstride, fs = (uint64_t)L.fstride;
  const uint64_t nv_full = std::min<uint64_t>((uint64_t)L.nv, avail / vs);
  if (nv_full < (uint64_t)L.nv) ghio::walk_binary(h, src, 0, (int64_t)nv_full, nv_full * vs, (int64_t)nv_full, nullptr);
  const uint64_t vbytes = (uint64_t)L.nv * vs;
  const uint64_t nf_full = std::min<uint64_t>((uint64_t)L.nf, (avail - vbytes) / fs);
  check_counts(L.nv, (int64_t)nf_full);
  const uint64_t need = vbytes + nf_full * fs;

  cudaStream_t s = m->stream;
  gh::Scratch<unsigned char> raw(need ? need : 1, s);
  GH_CUDA(cudaStreamSynchronize(s));  // the scratch exists before other streams write it
  auto tr = std::chrono::steady_clock::now();
  stage_to_device(data, need, raw.p, threads, m->device);
  if (rep) {
    rep->read_ms = ms_since(tr);
    rep->device_decoded = 1;
  }
  auto td = std::chrono::steady_clock::now();
  m->nv = (int32_t)L.nv;
  m->nf = (int32_t)nf_full;
  m->pos.alloc(3 * (size_t)L.nv, s);
  m->faces.alloc(3 * (size_t)nf_full, s);
  gh::Scratch<unsigned long long> bad(1, s);
  GH_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), s));
  if (L.nv) {
    VertexDecode vd{L.vstride, {L.voff[0], L.voff[1], L.voff[2]}, {L.vtype[0], L.vtype[1], L.vtype[2]}};
    k_decode_vertices<<<gh::grid_for(L.nv, 256, 148 * 16), 256, 0, s>>>(raw.p, L.nv, vd, m->pos.p);
    GH_LAUNCH_CHECK();
    m->launches++;
  }
  if (nf_full) {
    FaceDecode fd{L.fstride, L.list_off, L.count_type, L.value_type, ghio::type_size(L.count_type),
                  ghio::type_size(L.value_type)};
    k_decode_faces<<<gh::grid_for((int64_t)nf_full, 256, 148 * 16), 256, 0, s>>>(raw.p + vbytes, (int64_t)nf_full, fd,
                                                                                  L.nv, m->faces.p, bad.p);
    GH_LAUNCH_CHECK();
    m->launches++;
  }
  unsigned long long first_bad = ~0ull;
  GH_CUDA(cudaMemcpyAsync(&first_bad, bad.p, sizeof(first_bad), cudaMemcpyDeviceToHost, s));
  GH_CUDA(cudaStreamSynchronize(s));
  if (first_bad != ~0ull) {
    ghio::walk_binary(h, src, 1, (int64_t)first_bad, vbytes + first_bad * fs, L.nv, nullptr);
    fail(GH_ERR_INTERNAL, "binary PLY decoder flagged face " + std::to_string(first_bad) + " but it reads clean");
  }
  if (nf_full < (uint64_t)L.nf) {
    ghio::walk_binary(h, src, 1, (int64_t)nf_full, vbytes + nf_full * fs, L.nv, nullptr);
    fail(GH_ERR_INTERNAL, "binary PLY: truncated face element reads clean");
  }
  if (h.elements.size() > 2) ghio::walk_binary(h, src, 2, 0, vbytes + (uint64_t)L.nf * fs, L.nv, nullptr);
  if (rep) rep->parse_ms = ms_since(td);
  auto tb = std::chrono::steady_clock::now();
  gh::mesh_build(m, nullptr, nullptr);
  if (rep) {
    GH_CUDA(cudaStreamSynchronize(s));
    rep->build_ms = ms_since(tb);
  }
}

}  // namespace

namespace gh {

bool host_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

int staging_threads() {
  const unsigned hw = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(16u, hw ? hw : 1u));
}

void host_to_device_staged(const void* src, uint64_t n, void* dst, int device) {
  stage_to_device(static_cast<const unsigned char*>(src), n, static_cast<unsigned char*>(dst), staging_threads(),
                  device);
}

void device_to_host_staged(const void* src, uint64_t n, void* dst, int device) {
  stage_from_device(static_cast<const unsigned char*>(src), n, static_cast<unsigned char*>(dst), staging_threads(),
                    device);
}

void load_mesh_bytes(gh_mesh* m, const unsigned char* bytes, uint64_t n, int format, int threads,
                     gh_load_report* rep) {
  try {
    if (threads <= 0) threads = ghio::default_threads(n);
    if (rep) {
      rep->format = format;
      rep->bytes = n;
      rep->host_threads = threads;
    }
    auto t0 = std::chrono::steady_clock::now();
    if (format == GH_FORMAT_OBJ) {
      ghio::HostMesh hm;
      ghio::parse_obj((const char*)bytes, n, threads, hm);
      if (rep) {
        rep->parse_ms = ms_since(t0);
        rep->host_threads = hm.threads_used;
      }
      auto tb = std::chrono::steady_clock::now();
      from_host(m, hm);
      if (rep) {
        GH_CUDA(cudaStreamSynchronize(m->stream));
        rep->build_ms = ms_since(tb);
      }
      return;
    }
    const ghio::PlyHeader h = ghio::parse_ply_header((const char*)bytes, n);
    if (rep) rep->binary = h.binary ? 1 : 0;
    if (!h.binary) {
      ghio::HostMesh hm;
      ghio::parse_ply_ascii(h, (const char*)bytes, n, threads, hm);
      if (rep) {
        rep->parse_ms = ms_since(t0);
        rep->host_threads = hm.threads_used;
      }
      auto tb = std::chrono::steady_clock::now();
      from_host(m, hm);
      if (rep) {
        GH_CUDA(cudaStreamSynchronize(m->stream));
        rep->build_ms = ms_since(tb);
      }
      return;
    }
    double parse0 = ms_since(t0);
    load_binary_ply(m, h, bytes, n, threads, rep);
    if (rep) rep->parse_ms += parse0;
  } catch (const ghio::LoadError& e) {
    fail(GH_ERR_MESH, e.msg);
  }
}

void load_mesh_file(gh_mesh* m, const char* path, int threads, gh_load_report* rep) {
  int format = 0;
  try {
    format = (int)ghio::format_from_path(path);
  } catch (const ghio::LoadError& e) {
    fail(GH_ERR_MESH, e.msg);
  }
  auto t0 = std::chrono::steady_clock::now();
  Mapping map(path);
  const double map_ms = ms_since(t0);
  load_mesh_bytes(m, map.p, map.n, format, threads, rep);
  if (rep) rep->read_ms += map_ms;
}

// Device-side packing of the binary PLY body of save_ply (mesh_io.hpp:
// 297-319): vertex records (x, y, z[, quality]) as doubles, then face records
// (uchar 3, int32 x3).
__global__ void k_pack_ply(const double* __restrict__ pos, const double* __restrict__ quality, int64_t nv,
                           const int32_t* __restrict__ faces, int64_t nf, unsigned char* __restrict__ out) {
  const int64_t vstride = quality ? 32 : 24;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += stride) {
    double* o = (double*)(out + v * vstride);  // vstride is a multiple of 8 and out is aligned
    o[0] = pos[3 * v];
    o[1] = pos[3 * v + 1];
    o[2] = pos[3 * v + 2];
    if (quality) o[3] = quality[v];
  }
  unsigned char* fo = out + nv * vstride;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += stride) {
    unsigned char* r = fo + 13 * f;
    r[0] = 3;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const uint32_t v = (uint32_t)faces[3 * f + k];
#pragma unroll
      for (int b = 0; b < 4; ++b) r[1 + 4 * k + b] = (unsigned char)(v >> (8 * b));
    }
  }
}

std::string serialize_mesh(gh_mesh* m, int format, const double* quality) {
  cudaStream_t s = m->stream;
  const int64_t nv = m->nv, nf = m->nf;
  try {
    if (format == GH_FORMAT_OBJ) {
      std::vector<double> pos(3 * (size_t)nv);
      std::vector<int32_t> faces(3 * (size_t)nf);
      if (nv) GH_CUDA(cudaMemcpyAsync(pos.data(), m->pos.p, 24 * (size_t)nv, cudaMemcpyDeviceToHost, s));
      if (nf) GH_CUDA(cudaMemcpyAsync(faces.data(), m->faces.p, 12 * (size_t)nf, cudaMemcpyDeviceToHost, s));
      GH_CUDA(cudaStreamSynchronize(s));
      std::string out;
      ghio::format_obj(pos.data(), nv, faces.data(), nf, 0, out);
      return out;
    }
    std::string out = ghio::ply_header(nv, nf, quality != nullptr);
    const size_t head = out.size();
    const uint64_t body = (uint64_t)nv * (quality ? 32 : 24) + 13 * (uint64_t)nf;
    out.resize(head + body);
    if (!body) return out;
    Scratch<unsigned char> packed(body, s);
    Scratch<double> q(quality ? (size_t)nv : 0, s);
    if (quality && nv) GH_CUDA(cudaMemcpyAsync(q.p, quality, 8 * (size_t)nv, cudaMemcpyHostToDevice, s));
    k_pack_ply<<<grid_for(std::max(nv, nf), 256, 148 * 16), 256, 0, s>>>(m->pos.p, quality ? q.p : nullptr, nv,
                                                                          m->faces.p, nf, packed.p);
    GH_LAUNCH_CHECK();
    m->launches++;
    GH_CUDA(cudaMemcpyAsync(&out[head], packed.p, body, cudaMemcpyDeviceToHost, s));
    GH_CUDA(cudaStreamSynchronize(s));
    return out;
  } catch (const ghio::LoadError& e) {
    fail(GH_ERR_MESH, e.msg);
  }
}

}  // namespace gh
