// Host side of mesh I/O: PLY header parsing, the
// multi-threaded text tokenisers (OBJ, ASCII PLY), the binary-PLY record
// walker that resolves errors at exact byte offsets, and the output writers.
// Plain C++17 (compiled by g++ into libgeoheat_b200.so); the CUDA side
// (gh_load.cu) decodes binary PLY records on the device and builds the mesh.
//
// Behaviour follows reference/proj/include/geoheat/mesh_io.hpp: the same
// accepted inputs, the same values (std::istream >> double semantics for
// text), and the same error messages in the same precedence (first failing
// line / record / byte offset wins).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace ghio {

// Thrown for anything the reference reports as geoheat::MeshError (or the
// std::length_error its vector::reserve raises for a negative count).
struct LoadError {
  std::string msg;
};

enum class Format : int32_t { OBJ = 0, PLY = 1 };

// format_from_path (mesh_io.hpp:271-278).
Format format_from_path(const std::string& path);

// ---- PLY header (mesh_io.hpp:140-197)
enum PlyType : int8_t { I8, U8, I16, U16, I32, U32, F32, F64 };
int type_size(PlyType t);

struct PlyProperty {
  std::string name;
  bool is_list = false;
  PlyType count_type = U8;
  PlyType value_type = F32;
};
struct PlyElement {
  std::string name;
  long count = 0;
  std::vector<PlyProperty> props;
};
struct PlyHeader {
  bool binary = false;
  std::vector<PlyElement> elements;
  size_t data_offset = 0;  // first byte after the end_header line
  long lines = 0;          // header lines read (line numbers of ASCII records follow)
};

// Parses the header and applies the vertex-then-face check and the
// vector::reserve behaviour of mesh_io.hpp:198-204. Throws LoadError.
PlyHeader parse_ply_header(const char* data, size_t n);

// x/y/z property indices of a vertex element (last match wins, as in
// mesh_io.hpp:216-222); throws when one is missing.
void vertex_xyz(const PlyElement& el, int idx[3]);

// ---- text tokenisers: positions [3V] and faces [3F] as the reference
// builds them before build_mesh. `threads` <= 0 picks a count by size.
struct HostMesh {
  std::vector<double> pos;
  std::vector<int32_t> faces;
  int threads_used = 1;
};
void parse_obj(const char* data, size_t n, int threads, HostMesh& out);
void parse_ply_ascii(const PlyHeader& h, const char* data, size_t n, int threads, HostMesh& out);

// ---- binary PLY
// Byte source of the data section (file or memory).
struct ByteSource {
  virtual ~ByteSource() = default;
  virtual uint64_t size() const = 0;                               // bytes available after data_offset
  virtual void read(uint64_t off, uint64_t n, void* dst) const = 0;  // [off, off+n) within size()
};

// Fixed-stride layout the device decoder handles: element 0 "vertex" without
// list properties, element 1 "face" with exactly one list property whose
// count is assumed to be 3 (the decoder flags the first record where it is
// not, and the walker below resolves that record exactly).
struct FixedLayout {
  bool ok = false;
  int64_t nv = 0, nf = 0;
  int32_t vstride = 0, voff[3] = {0, 0, 0};
  PlyType vtype[3] = {F64, F64, F64};
  int32_t fstride = 0, list_off = 0;
  PlyType count_type = U8, value_type = I32;
};
FixedLayout fixed_layout(const PlyHeader& h);

// Sequential reference semantics over the binary data section from
// (element, record, byte offset) on; appends to out and throws LoadError at
// the first failure. positions_before = positions pushed by earlier records.
void walk_binary(const PlyHeader& h, const ByteSource& src, size_t element, int64_t record, uint64_t offset,
                 int64_t positions_before, HostMesh* out);

// ---- writers (mesh_io.hpp:287-344)
void format_obj(const double* pos, int64_t nv, const int32_t* faces, int64_t nf, int threads, std::string& out);
std::string ply_header(int64_t nv, int64_t nf, bool quality);
// write_distances_txt / write_distances_csv
void format_distances(const double* d, int64_t n, bool csv, int threads, std::string& out);

int default_threads(size_t bytes);

}  // namespace ghio
