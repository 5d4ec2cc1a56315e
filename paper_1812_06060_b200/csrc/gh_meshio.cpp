// Host side of mesh I/O; see gh_meshio.hpp. Every parser below restates the
// reference loader's observable behaviour (reference/proj/include/geoheat/
// mesh_io.hpp) without its per-line std::istringstream: text is split into
// line-aligned chunks that threads tokenise independently, and errors carry
// their line (or record) so the first one in file order is reported, as the
// sequential reference would report it.

#include "gh_meshio.hpp"

#include <locale.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <thread>

namespace ghio {
namespace {

[[noreturn]] void fail(const std::string& msg) { throw LoadError{msg}; }

// ---------------------------------------------------------------- threads
void parallel_for(int n, const std::function<void(int)>& body) {
  if (n <= 1) {
    if (n == 1) body(0);
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::string> errors(n);
  std::vector<char> bad(n, 0);
  pool.reserve(n - 1);
  auto run = [&](int i) {
    try {
      body(i);
    } catch (const LoadError& e) {
      errors[i] = e.msg;
      bad[i] = 1;
    } catch (const std::bad_alloc&) {
      errors[i] = "std::bad_alloc";
      bad[i] = 2;
    } catch (const std::exception& e) {  // nothing may escape a std::thread
      errors[i] = e.what();
      bad[i] = 1;
    } catch (...) {
      errors[i] = "unknown error in a mesh I/O worker";
      bad[i] = 1;
    }
  };
  for (int i = 1; i < n; ++i) pool.emplace_back(run, i);
  run(0);
  for (auto& t : pool) t.join();
  for (int i = 0; i < n; ++i) {
    if (bad[i] == 2) throw std::bad_alloc();
    if (bad[i]) fail(errors[i]);
  }
}

// ---------------------------------------------------- istream emulation
// The reference reads text through std::istringstream in the "C" locale
// (libstdc++). These helpers reproduce operator>> for std::string, long and
// double on a line held as [p, e): same whitespace set, same accepted
// characters, same failure cases.
inline bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

locale_t c_locale() {
  static locale_t loc = newlocale(LC_ALL_MASK, "C", (locale_t)0);
  return loc;
}

struct Cur {
  const char* p;
  const char* e;
};

inline void skip_ws(Cur& c) {
  while (c.p < c.e && is_space(*c.p)) ++c.p;
}

// operator>>(std::string&)
bool extract_token(Cur& c, std::string& out) {
  skip_ws(c);
  if (c.p == c.e) return false;
  const char* b = c.p;
  while (c.p < c.e && !is_space(*c.p)) ++c.p;
  out.assign(b, c.p);
  return true;
}

// operator>>(double&): libstdc++ num_get::_M_extract_float collects
// [sign] [leading zeros -> one '0'] digits [one '.'] [e|E after a mantissa
// digit [sign]], stopping at the first other character, then converts with
// strtod in the C locale; a conversion that does not consume the whole
// collected string, or that overflows to +-inf, fails.
bool extract_double(Cur& c, double& out) {
  skip_ws(c);
  if (c.p == c.e) return false;
  char small[96];
  std::string big;
  size_t n = 0;
  auto put = [&](char ch) {
    if (n + 1 < sizeof(small)) {
      small[n++] = ch;
    } else {
      if (big.empty()) big.assign(small, n);
      big.push_back(ch);
      ++n;
    }
  };
  const char* p = c.p;
  const char* e = c.e;
  if (*p == '+' || *p == '-') put(*p++);
  bool mant = false;
  while (p < e && *p == '0') {
    if (!mant) {
      put('0');
      mant = true;
    }
    ++p;
  }
  bool dec = false, sci = false;
  while (p < e) {
    const char ch = *p;
    if (ch >= '0' && ch <= '9') {
      put(ch);
      mant = true;
    } else if (ch == '.' && !dec && !sci) {
      put('.');
      dec = true;
    } else if ((ch == 'e' || ch == 'E') && !sci && mant) {
      put('e');
      sci = true;
      ++p;
      if (p < e) {
        if (*p == '+' || *p == '-') {
          put(*p);
        } else {
          continue;
        }
      } else {
        break;
      }
    } else {
      break;
    }
    ++p;
  }
  c.p = p;
  const char* s;
  if (big.empty()) {
    small[n] = 0;
    s = small;
  } else {
    s = big.c_str();
  }
  char* end = nullptr;
  const double v = strtod_l(s, &end, c_locale());
  if (end == s || *end != '\0') return false;
  if (v == HUGE_VAL || v == -HUGE_VAL) return false;
  out = v;
  return true;
}

// operator>>(long&) in base 10 (PLY element counts).
bool extract_long(Cur& c, long& out) {
  skip_ws(c);
  if (c.p == c.e) return false;
  const char* p = c.p;
  bool neg = false;
  if (*p == '+' || *p == '-') neg = (*p++ == '-');
  unsigned long v = 0;
  bool digits = false, overflow = false;
  const unsigned long lim = neg ? (unsigned long)LONG_MAX + 1ul : (unsigned long)LONG_MAX;
  while (p < c.e && *p >= '0' && *p <= '9') {
    const unsigned d = (unsigned)(*p - '0');
    if (v > (lim - d) / 10) overflow = true;
    else v = v * 10 + d;
    digits = true;
    ++p;
  }
  c.p = p;
  if (!digits || overflow) return false;
  out = neg ? (long)(0ul - v) : (long)v;
  return true;
}

// static_cast<long>(double) as x86-64 executes it (cvttsd2si): truncation,
// and the "integer indefinite" LONG_MIN for NaN and out-of-range values.
inline long to_long(double v) {
  if (v >= -9223372036854775808.0 && v < 9223372036854775808.0) return (long)v;
  return LONG_MIN;
}

// parse_obj_index (mesh_io.hpp:30-37).
bool parse_obj_index(const std::string& token, long& out) {
  std::string head = token.substr(0, token.find('/'));
  if (head.empty()) return false;
  const char* begin = head.c_str();
  char* end = nullptr;
  out = std::strtol(begin, &end, 10);
  return end != begin && *end == '\0';
}

// ------------------------------------------------------------- lines
// std::getline semantics: '\n'-terminated lines, plus a final unterminated
// non-empty line.
struct Chunk {
  size_t b = 0, e = 0;
};

std::vector<Chunk> split_lines(const char* d, size_t n, int parts) {
  std::vector<Chunk> out;
  size_t b = 0;
  for (int k = 1; k <= parts && b < n; ++k) {
    size_t cut = k == parts ? n : std::max(b, (size_t)((double)n * k / parts));
    if (cut < n) {
      const void* nl = std::memchr(d + cut, '\n', n - cut);
      cut = nl ? (size_t)((const char*)nl - d) + 1 : n;
    }
    if (cut > b) out.push_back({b, cut});
    b = cut;
  }
  return out;
}

int64_t count_lines(const char* d, size_t b, size_t e) {
  int64_t lines = 0;
  size_t p = b;
  while (p < e) {
    const void* nl = std::memchr(d + p, '\n', e - p);
    ++lines;
    if (!nl) break;
    p = (size_t)((const char*)nl - d) + 1;
  }
  return lines;
}

// First error of a chunk; `key` orders errors in file order.
struct Err {
  int64_t key = INT64_MAX;
  std::string msg;
  void set(int64_t k, std::string m) {
    if (k < key) {
      key = k;
      msg = std::move(m);
    }
  }
};

PlyType ply_type(const std::string& name) {
  if (name == "char" || name == "int8") return I8;
  if (name == "uchar" || name == "uint8") return U8;
  if (name == "short" || name == "int16") return I16;
  if (name == "ushort" || name == "uint16") return U16;
  if (name == "int" || name == "int32") return I32;
  if (name == "uint" || name == "uint32") return U32;
  if (name == "float" || name == "float32") return F32;
  if (name == "double" || name == "float64") return F64;
  fail("PLY: unsupported property type '" + name + "'");
}

inline double decode(const unsigned char* b, PlyType t) {
  switch (t) {
    case I8: return (double)(int8_t)b[0];
    case U8: return (double)b[0];
    case I16: { int16_t v; std::memcpy(&v, b, 2); return v; }
    case U16: { uint16_t v; std::memcpy(&v, b, 2); return v; }
    case I32: { int32_t v; std::memcpy(&v, b, 4); return v; }
    case U32: { uint32_t v; std::memcpy(&v, b, 4); return v; }
    case F32: { float v; std::memcpy(&v, b, 4); return v; }
    case F64: { double v; std::memcpy(&v, b, 8); return v; }
  }
  return 0.0;
}

}  // namespace

int type_size(PlyType t) {
  switch (t) {
    case I8:
    case U8: return 1;
    case I16:
    case U16: return 2;
    case I32:
    case U32:
    case F32: return 4;
    case F64: return 8;
  }
  return 0;
}

int default_threads(size_t bytes) {
  unsigned hw = std::thread::hardware_concurrency();
  int t = hw ? (int)hw : 1;
  t = std::min(t, 32);
  const int by_size = (int)std::max<size_t>(1, bytes / (4u << 20));  // >= 4 MiB per thread
  return std::max(1, std::min(t, by_size));
}

Format format_from_path(const std::string& path) {
  auto dot = path.rfind('.');
  std::string ext = dot == std::string::npos ? "" : path.substr(dot + 1);
  for (char& ch : ext) ch = (char)std::tolower((unsigned char)ch);
  if (ext == "obj") return Format::OBJ;
  if (ext == "ply") return Format::PLY;
  fail("cannot infer mesh format from path '" + path + "' (expected .obj or .ply)");
}

// ------------------------------------------------------------ PLY header
PlyHeader parse_ply_header(const char* d, size_t n) {
  PlyHeader h;
  size_t pos = 0;
  std::string line;
  auto next_line = [&](const char* what) {
    if (pos >= n) fail(std::string("PLY parse failure: unexpected end of header while reading ") + what);
    const void* nl = std::memchr(d + pos, '\n', n - pos);
    const size_t end = nl ? (size_t)((const char*)nl - d) : n;
    line.assign(d + pos, end - pos);
    pos = nl ? end + 1 : n;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    ++h.lines;
  };
  const auto at = [&] { return "PLY parse failure at line " + std::to_string(h.lines); };
  next_line("magic");
  if (line != "ply") fail("PLY parse failure at line 1: missing 'ply' magic");
  while (true) {
    next_line("header");
    Cur c{line.data(), line.data() + line.size()};
    std::string tag;
    extract_token(c, tag);
    if (tag == "comment" || tag == "obj_info") continue;
    if (tag == "format") {
      std::string fmt, version;
      if (extract_token(c, fmt)) extract_token(c, version);
      if (fmt == "ascii") h.binary = false;
      else if (fmt == "binary_little_endian") h.binary = true;
      else fail(at() + ": unsupported format '" + fmt + "'");
    } else if (tag == "element") {
      PlyElement el;
      if (!extract_token(c, el.name) || !extract_long(c, el.count)) fail(at() + ": bad element");
      h.elements.push_back(el);
    } else if (tag == "property") {
      if (h.elements.empty()) fail(at() + ": property before element");
      PlyProperty prop;
      std::string type_name;
      extract_token(c, type_name);
      if (type_name == "list") {
        std::string count_name, value_name;
        if (!extract_token(c, count_name) || !extract_token(c, value_name) || !extract_token(c, prop.name))
          fail(at() + ": bad list property");
        prop.is_list = true;
        prop.count_type = ply_type(count_name);
        prop.value_type = ply_type(value_name);
      } else {
        if (!extract_token(c, prop.name)) fail(at() + ": bad property");
        prop.value_type = ply_type(type_name);
      }
      h.elements.back().props.push_back(prop);
    } else if (tag == "end_header") {
      break;
    } else {
      fail(at() + ": unknown header line '" + line + "'");
    }
  }
  if (h.elements.size() < 2 || h.elements[0].name != "vertex" || h.elements[1].name != "face")
    fail("PLY parse failure: expected elements in vertex-then-face order");
  // positions.reserve / faces.reserve (mesh_io.hpp:202-203) throw
  // std::length_error("vector::reserve") for a negative count.
  if (h.elements[0].count < 0 || h.elements[1].count < 0) fail("vector::reserve");
  h.data_offset = pos;
  return h;
}

void vertex_xyz(const PlyElement& el, int idx[3]) {
  idx[0] = idx[1] = idx[2] = -1;
  for (size_t p = 0; p < el.props.size(); ++p) {
    if (el.props[p].name == "x") idx[0] = (int)p;
    if (el.props[p].name == "y") idx[1] = (int)p;
    if (el.props[p].name == "z") idx[2] = (int)p;
  }
  if (idx[0] < 0 || idx[1] < 0 || idx[2] < 0) fail("PLY parse failure: vertex element lacks x/y/z properties");
}

namespace {

// Static plan of a PLY body: per element its first record (= data line for
// ASCII), how many of its records exist, and where they land in the output.
struct ElementPlan {
  int kind = 0;  // 0 other, 1 vertex, 2 face
  int64_t first = 0, count = 0, avail = 0;
  int64_t out_base = 0;         // vertex or face output index of record 0
  int64_t positions_before = 0; // positions pushed before this element (faces)
  int xyz[3] = {-1, -1, -1};
  bool xyz_ok = true;
};

std::vector<ElementPlan> plan_elements(const PlyHeader& h, int64_t records_available) {
  std::vector<ElementPlan> plan(h.elements.size());
  int64_t rec = 0, nvp = 0, nfp = 0;
  for (size_t e = 0; e < h.elements.size(); ++e) {
    const PlyElement& el = h.elements[e];
    ElementPlan& p = plan[e];
    p.kind = el.name == "vertex" ? 1 : el.name == "face" ? 2 : 0;
    p.first = rec;
    p.count = std::max<long>(el.count, 0);
    p.avail = std::max<int64_t>(0, std::min(p.count, records_available - rec));
    p.positions_before = nvp;
    if (p.kind == 1) {
      p.out_base = nvp;
      nvp += p.count;
      try {
        vertex_xyz(el, p.xyz);
      } catch (const LoadError&) {
        p.xyz_ok = false;
      }
    } else if (p.kind == 2) {
      p.out_base = nfp;
      nfp += p.count;
    }
    rec = (rec > INT64_MAX - p.count) ? INT64_MAX : rec + p.count;
  }
  return plan;
}

// One PLY record's values, shared by the ASCII and binary readers.
// Only the first three list values are kept: the checks need the list
// length and, for triangles, the three indices.
struct Record {
  std::vector<double> scalars;
  int64_t list_n = 0;
  long list[3] = {0, 0, 0};
  void clear() {
    scalars.clear();
    list_n = 0;
  }
  void begin_list() { list_n = 0; }
  void push_list(long v) {
    if (list_n < 3) list[list_n] = v;
    ++list_n;
  }
};

// The checks mesh_io.hpp:246-259 apply once a record is read. Returns an
// error message or empty.
inline const char* finish_face(const Record& r, int64_t positions, int32_t* tri, std::string& msg) {
  if (r.list_n != 3) {
    msg = "PLY: non-triangle face with " + std::to_string(r.list_n) + " vertices";
    return msg.c_str();
  }
  for (int k = 0; k < 3; ++k) {
    if (r.list[k] < 0 || r.list[k] >= positions) {
      msg = "PLY: face index out of range";
      return msg.c_str();
    }
    tri[k] = (int32_t)r.list[k];
  }
  return nullptr;
}

inline const char* finish_vertex(const Record& r, const int xyz[3], double* p, std::string& msg) {
  for (int k = 0; k < 3; ++k) {
    // The reference indexes its scalar list with the property index; with a
    // list property before x/y/z that read is out of bounds (undefined), so
    // such elements are rejected here.
    if ((size_t)xyz[k] >= r.scalars.size()) {
      msg = "PLY: vertex element with list properties before x/y/z is not supported";
      return msg.c_str();
    }
    p[k] = r.scalars[xyz[k]];
  }
  return nullptr;
}

}  // namespace


// ------------------------------------------------------------- ASCII PLY
// mesh_io.hpp:205-262 with format ascii: one record per line after the
// header, every value read as a double (lists cast to long).
void parse_ply_ascii(const PlyHeader& h, const char* d0, size_t n0, int threads, HostMesh& out) {
  const char* d = d0 + h.data_offset;
  const size_t n = n0 - h.data_offset;
  if (threads <= 0) threads = default_threads(n);
  const std::vector<Chunk> chunks = split_lines(d, n, threads);
  const int nc = (int)chunks.size();
  std::vector<int64_t> lines(nc + 1, 0);
  parallel_for(nc, [&](int i) { lines[i + 1] = count_lines(d, chunks[i].b, chunks[i].e); });
  for (int i = 0; i < nc; ++i) lines[i + 1] += lines[i];
  const int64_t total_lines = lines[nc];

  const std::vector<ElementPlan> plan = plan_elements(h, total_lines);
  // Output sized by the records present: a header count larger than the
  // body fails below without allocating for it.
  int64_t nv_alloc = 0, nf_alloc = 0, records = 0;
  for (const ElementPlan& p : plan) {
    if (p.kind == 1) nv_alloc = std::max(nv_alloc, p.out_base + p.avail);
    if (p.kind == 2) nf_alloc = std::max(nf_alloc, p.out_base + p.avail);
    records = (records > INT64_MAX - p.count) ? INT64_MAX : records + p.count;
  }
  out.pos.assign(3 * nv_alloc, 0.0);
  out.faces.assign(3 * nf_alloc, 0);
  out.threads_used = std::max(nc, 1);

  // Errors are keyed 2*line+1 for a record and 2*first for an element-level
  // check that the reference runs before the element's first record.
  Err global;
  for (const ElementPlan& p : plan)
    if (p.kind == 1 && !p.xyz_ok) global.set(2 * p.first, "PLY parse failure: vertex element lacks x/y/z properties");
  if (total_lines < records) {
    size_t e = 0;
    while (e + 1 < plan.size() && total_lines >= plan[e].first + plan[e].count) ++e;
    global.set(2 * total_lines + 1,
               "PLY parse failure: unexpected end of header while reading " + h.elements[e].name);
  }

  std::vector<Err> errs(nc);
  parallel_for(nc, [&](int ci) {
    Err& err = errs[ci];
    Record rec;
    std::string msg;
    size_t p = chunks[ci].b;
    const size_t ce = chunks[ci].e;
    int64_t li = lines[ci];
    size_t ei = 0;
    while (p < ce) {
      const size_t lb = p;
      const void* nl = std::memchr(d + p, '\n', ce - p);
      size_t le = nl ? (size_t)((const char*)nl - d) : ce;
      p = nl ? le + 1 : ce;
      if (le > lb && d[le - 1] == '\r') --le;
      const int64_t line_idx = li++;
      while (ei < plan.size() && line_idx >= plan[ei].first + plan[ei].count) ++ei;
      if (ei >= plan.size()) break;  // lines after the last record are never read
      const int64_t key = 2 * line_idx + 1;
      if (key > global.key) break;
      const ElementPlan& ep = plan[ei];
      if (ep.kind == 1 && !ep.xyz_ok) break;  // the reference stops before this element
      const PlyElement& el = h.elements[ei];
      const auto at = [&] { return "PLY parse failure at line " + std::to_string(h.lines + line_idx + 1) + ": bad "; };
      Cur c{d + lb, d + le};
      rec.clear();
      bool bad = false;
      for (const PlyProperty& prop : el.props) {
        double v;
        if (prop.is_list) {
          if (!extract_double(c, v)) {
            err.set(key, at() + "list count");
            bad = true;
            break;
          }
          const long cnt = to_long(v);
          rec.begin_list();
          for (long k = 0; k < cnt; ++k) {
            if (!extract_double(c, v)) {
              err.set(key, at() + "list value");
              bad = true;
              break;
            }
            rec.push_list(to_long(v));
          }
          if (bad) break;
        } else {
          if (!extract_double(c, v)) {
            err.set(key, at() + prop.name);
            bad = true;
            break;
          }
          rec.scalars.push_back(v);
        }
      }
      if (bad) break;
      const int64_t r = line_idx - ep.first;
      if (ep.kind == 1) {
        if (finish_vertex(rec, ep.xyz, &out.pos[3 * (ep.out_base + r)], msg)) {
          err.set(key, msg);
          break;
        }
      } else if (ep.kind == 2) {
        if (finish_face(rec, ep.positions_before, &out.faces[3 * (ep.out_base + r)], msg)) {
          err.set(key, msg);
          break;
        }
      }
    }
  });
  for (const Err& e : errs) global.set(e.key, e.msg);
  if (global.key != INT64_MAX) fail(global.msg);
}

// ------------------------------------------------------------------- OBJ
// load_obj (mesh_io.hpp:39-78). Pass 1 tokenises line-aligned chunks in
// parallel; face indices are kept raw with the chunk-local vertex count of
// their line, and pass 2 applies the relative-index rule and the range
// check once every chunk's vertex offset is known.
void parse_obj(const char* d, size_t n, int threads, HostMesh& out) {
  if (threads <= 0) threads = default_threads(n);
  const std::vector<Chunk> chunks = split_lines(d, n, threads);
  const int nc = (int)chunks.size();
  std::vector<int64_t> lines(nc + 1, 0);
  parallel_for(nc, [&](int i) { lines[i + 1] = count_lines(d, chunks[i].b, chunks[i].e); });
  for (int i = 0; i < nc; ++i) lines[i + 1] += lines[i];

  struct Part {
    std::vector<double> pos;
    std::vector<int64_t> raw;    // 3 per face
    std::vector<int64_t> local;  // vertices of this chunk before the face
    Err err;
  };
  std::vector<Part> parts(nc);
  parallel_for(nc, [&](int ci) {
    Part& pt = parts[ci];
    pt.pos.reserve((chunks[ci].e - chunks[ci].b) / 40 * 3);
    std::string tag, tok;
    std::vector<long> idx;
    size_t p = chunks[ci].b;
    const size_t ce = chunks[ci].e;
    int64_t li = lines[ci];
    int64_t nverts = 0;
    while (p < ce) {
      const size_t lb = p;
      const void* nl = std::memchr(d + p, '\n', ce - p);
      const size_t le = nl ? (size_t)((const char*)nl - d) : ce;
      p = nl ? le + 1 : ce;
      const int64_t line_no = ++li;  // 1-based, as the reference counts
      Cur c{d + lb, d + le};
      if (!extract_token(c, tag) || tag[0] == '#') continue;
      const auto at = [&] { return "OBJ parse failure at line " + std::to_string(line_no) + ": "; };
      if (tag == "v") {
        double x, y, z;
        if (!extract_double(c, x) || !extract_double(c, y) || !extract_double(c, z)) {
          pt.err.set(line_no, at() + "bad vertex");
          break;
        }
        pt.pos.push_back(x);
        pt.pos.push_back(y);
        pt.pos.push_back(z);
        ++nverts;
      } else if (tag == "f") {
        idx.clear();
        bool bad = false;
        while (extract_token(c, tok)) {
          long value;
          if (!parse_obj_index(tok, value)) {
            pt.err.set(line_no, at() + "bad face entry '" + tok + "'");
            bad = true;
            break;
          }
          idx.push_back(value);
        }
        if (bad) break;
        if (idx.size() != 3) {
          pt.err.set(line_no, at() + "non-triangle face with " + std::to_string(idx.size()) + " vertices");
          break;
        }
        pt.raw.insert(pt.raw.end(), idx.begin(), idx.end());
        pt.local.push_back(nverts);
      }
    }
  });

  std::vector<int64_t> vbase(nc + 1, 0), fbase(nc + 1, 0);
  for (int i = 0; i < nc; ++i) {
    vbase[i + 1] = vbase[i] + (int64_t)parts[i].pos.size() / 3;
    fbase[i + 1] = fbase[i] + (int64_t)parts[i].local.size();
  }
  out.pos.resize(3 * vbase[nc]);
  out.faces.resize(3 * fbase[nc]);
  out.threads_used = std::max(nc, 1);
  std::vector<Err> range(nc);
  parallel_for(nc, [&](int ci) {
    Part& pt = parts[ci];
    std::copy(pt.pos.begin(), pt.pos.end(), out.pos.begin() + 3 * vbase[ci]);
    std::vector<double>().swap(pt.pos);
    int32_t* dst = out.faces.data() + 3 * fbase[ci];
    const int64_t nfc = (int64_t)pt.local.size();
    for (int64_t j = 0; j < nfc; ++j) {
      const int64_t positions = vbase[ci] + pt.local[j];
      bool ok = true;
      for (int k = 0; k < 3; ++k) {
        int64_t v = pt.raw[3 * j + k];
        if (v < 0) v = positions + 1 + v;
        if (v < 1 || v > positions) {
          ok = false;
          break;
        }
        dst[3 * j + k] = (int32_t)(v - 1);
      }
      if (ok) continue;
      // map face j of this chunk back to its line for the message
      int64_t line_no = lines[ci], seen = 0;
      size_t p = chunks[ci].b;
      std::string tag;
      while (p < chunks[ci].e) {
        const size_t lb = p;
        const void* nl = std::memchr(d + p, '\n', chunks[ci].e - p);
        const size_t le = nl ? (size_t)((const char*)nl - d) : chunks[ci].e;
        p = nl ? le + 1 : chunks[ci].e;
        ++line_no;
        Cur c{d + lb, d + le};
        if (extract_token(c, tag) && tag == "f" && seen++ == j) break;
      }
      range[ci].set(line_no, "OBJ parse failure at line " + std::to_string(line_no) + ": face index out of range");
      break;
    }
  });
  Err first;
  for (int i = 0; i < nc; ++i) {
    first.set(parts[i].err.key, parts[i].err.msg);
    first.set(range[i].key, range[i].msg);
  }
  if (first.key != INT64_MAX) fail(first.msg);
}

// ---------------------------------------------------------- binary PLY
namespace {

class BinReader {
 public:
  BinReader(const ByteSource& src, uint64_t off) : src_(src), off_(off), size_(src.size()) {}
  double scalar(PlyType t) {
    const int n = type_size(t);
    if (off_ + (uint64_t)n > size_)
      fail("PLY parse failure at byte offset " + std::to_string(off_) + ": unexpected end of data");
    if (off_ < start_ || off_ + n > start_ + len_) {
      len_ = std::min<uint64_t>(sizeof(buf_), size_ - off_);
      src_.read(off_, len_, buf_);
      start_ = off_;
    }
    const double v = decode(buf_ + (off_ - start_), t);
    off_ += (uint64_t)n;
    return v;
  }

 private:
  const ByteSource& src_;
  uint64_t off_, size_;
  uint64_t start_ = 0, len_ = 0;
  unsigned char buf_[1 << 16];
};

}  // namespace

void walk_binary(const PlyHeader& h, const ByteSource& src, size_t element, int64_t record, uint64_t offset,
                 int64_t positions_before, HostMesh* out) {
  std::unique_ptr<BinReader> r(new BinReader(src, offset));
  int64_t positions = positions_before;
  Record rec;
  std::string msg;
  for (size_t e = element; e < h.elements.size(); ++e) {
    const PlyElement& el = h.elements[e];
    const bool is_vertex = el.name == "vertex", is_face = el.name == "face";
    int xyz[3] = {-1, -1, -1};
    if (is_vertex) vertex_xyz(el, xyz);
    for (int64_t i = e == element ? record : 0; i < el.count; ++i) {
      rec.clear();
      for (const PlyProperty& prop : el.props) {
        if (prop.is_list) {
          const long cnt = to_long(r->scalar(prop.count_type));
          rec.begin_list();
          for (long k = 0; k < cnt; ++k) rec.push_list(to_long(r->scalar(prop.value_type)));
        } else {
          rec.scalars.push_back(r->scalar(prop.value_type));
        }
      }
      if (is_vertex) {
        double p[3];
        if (finish_vertex(rec, xyz, p, msg)) fail(msg);
        if (out) out->pos.insert(out->pos.end(), p, p + 3);
        ++positions;
      } else if (is_face) {
        int32_t tri[3];
        if (finish_face(rec, positions, tri, msg)) fail(msg);
        if (out) out->faces.insert(out->faces.end(), tri, tri + 3);
      }
    }
  }
}

FixedLayout fixed_layout(const PlyHeader& h) {
  FixedLayout L;
  for (size_t e = 2; e < h.elements.size(); ++e)
    if (h.elements[e].name == "vertex" || h.elements[e].name == "face") return L;  // appends: host walk
  const PlyElement& v = h.elements[0];
  int32_t off = 0;
  bool have[3] = {false, false, false};
  for (const PlyProperty& p : v.props) {
    if (p.is_list) return L;
    for (int k = 0; k < 3; ++k)
      if (p.name == (k == 0 ? "x" : k == 1 ? "y" : "z")) {
        L.voff[k] = off;
        L.vtype[k] = p.value_type;
        have[k] = true;
      }
    off += type_size(p.value_type);
  }
  if (!have[0] || !have[1] || !have[2]) return L;
  L.vstride = off;
  const PlyElement& f = h.elements[1];
  off = 0;
  int lists = 0;
  for (const PlyProperty& p : f.props) {
    if (p.is_list) {
      ++lists;
      L.list_off = off;
      L.count_type = p.count_type;
      L.value_type = p.value_type;
      off += type_size(p.count_type) + 3 * type_size(p.value_type);
    } else {
      off += type_size(p.value_type);
    }
  }
  if (lists != 1) return L;
  L.fstride = off;
  L.nv = v.count;
  L.nf = f.count;
  L.ok = true;
  return L;
}

// ---------------------------------------------------------------- writers
namespace {

// Formats items [0, n) with `fmt_one` into per-thread strings, joined in order.
void format_parallel(int64_t n, int threads, const std::function<void(int64_t, std::string&)>& fmt_one,
                     std::string& out) {
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(threads, (n + 65535) / 65536));
  std::vector<std::string> parts(nt);
  parallel_for(nt, [&](int t) {
    const int64_t b = n * t / nt, e = n * (t + 1) / nt;
    std::string& s = parts[t];
    s.reserve((size_t)(e - b) * 26);
    for (int64_t i = b; i < e; ++i) fmt_one(i, s);
  });
  size_t total = out.size();
  std::vector<size_t> at(nt);
  for (int t = 0; t < nt; ++t) {
    at[t] = total;
    total += parts[t].size();
  }
  out.resize(total);
  parallel_for(nt, [&](int t) { std::memcpy(&out[at[t]], parts[t].data(), parts[t].size()); });
}

}  // namespace

void format_obj(const double* pos, int64_t nv, const int32_t* faces, int64_t nf, int threads, std::string& out) {
  if (threads <= 0) threads = default_threads((size_t)nv * 60);
  format_parallel(
      nv, threads,
      [&](int64_t v, std::string& s) {
        char buf[128];
        const int k = std::snprintf(buf, sizeof(buf), "v %.17g %.17g %.17g\n", pos[3 * v], pos[3 * v + 1], pos[3 * v + 2]);
        s.append(buf, (size_t)k);
      },
      out);
  format_parallel(
      nf, threads,
      [&](int64_t f, std::string& s) {
        char buf[64];
        const int k =
            std::snprintf(buf, sizeof(buf), "f %d %d %d\n", faces[3 * f] + 1, faces[3 * f + 1] + 1, faces[3 * f + 2] + 1);
        s.append(buf, (size_t)k);
      },
      out);
}

std::string ply_header(int64_t nv, int64_t nf, bool quality) {
  std::string s = "ply\nformat binary_little_endian 1.0\n";
  s += "element vertex " + std::to_string(nv) + "\n";
  s += "property double x\nproperty double y\nproperty double z\n";
  if (quality) s += "property double quality\n";
  s += "element face " + std::to_string(nf) + "\n";
  s += "property list uchar int vertex_indices\n";
  s += "end_header\n";
  return s;
}

void format_distances(const double* d, int64_t n, bool csv, int threads, std::string& out) {
  if (threads <= 0) threads = default_threads((size_t)n * 24);
  if (csv) out += "vertex_index,distance\n";
  format_parallel(
      n, threads,
      [&](int64_t i, std::string& s) {
        char buf[64];
        const int k = csv ? std::snprintf(buf, sizeof(buf), "%zu,%.17g\n", (size_t)i, d[i])
                          : std::snprintf(buf, sizeof(buf), "%.17g\n", d[i]);
        s.append(buf, (size_t)k);
      },
      out);
}

}  // namespace ghio
