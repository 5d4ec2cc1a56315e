// geoheat_b200: the reference command-line tool (tools/geoheat.cpp) on the
// B200 path. Same subcommands (distance, bench, subdivide), options, output
// formats, RunReport text (report.hpp:50-135), bench CSV columns and exit
// codes (0 ok, 1 parse/IO failure, 2 invalid configuration, 3 solver
// failure); every computation goes through the C ABI of
// include/geoheat_b200.h on the GPU. `--device gpu` is accepted (and is the
// only device); `--threads` / `--seq` are echoed into the report exactly as
// the reference resolves them, without changing the (deterministic) result.

#include <sys/resource.h>

#include <chrono>
#include <cerrno>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "geoheat_b200.h"

namespace {

// ---------------------------------------------------------------- errors
struct Failure {  // -> exit code
  int code;
  std::string text;
};
struct MeshError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SolverError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void check(gh_status st) {
  if (st == GH_OK) return;
  const std::string msg = gh_last_error();
  if (st == GH_ERR_INVALID) throw std::invalid_argument(msg);
  if (st == GH_ERR_SOLVER) throw SolverError(msg);
  throw MeshError(msg);  // mesh, CUDA and internal failures report as "error:" (exit 1)
}

std::string format_double(double v) {  // report.hpp:43-47
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ---------------------------------------------------------------- options
struct PipelineOptions {  // tools/geoheat.cpp:27-38
  std::string mesh_path;
  std::string method = "face";
  std::vector<int32_t> sources;
  double m = 1.0;
  int gs_iters = 1000;
  int admm_iters = 10;
  double mu = 100.0;
  double eps = 1e-5;
  int threads = 0;
  bool sequential = false;
  std::string device = "gpu";
};

int resolve_threads(const PipelineOptions& opt) {  // tools/geoheat.cpp:40-50
  if (opt.sequential) return 1;
  if (opt.threads > 0) return opt.threads;
  if (const char* env = std::getenv("GEOHEAT_THREADS")) {
    int n = std::atoi(env);
    if (n > 0) return n;
  }
  unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}

// Minimal CLI11-style parser: --name value | --name=value, flags, required
// options, ',' lists; any misuse is a parse error (exit 2).
struct ParseError {
  std::string msg;
};
struct Help {};

class Command {
 public:
  explicit Command(std::string name, std::string about) : name_(std::move(name)), about_(std::move(about)) {}
  void opt(const std::string& flag, std::string* dst, const std::string& help, bool required = false) {
    add(flag, help, required, false, [dst](const std::string& v) { *dst = v; });
  }
  void opt(const std::string& flag, int* dst, const std::string& help) {
    add(flag, help, false, false, [dst, flag](const std::string& v) { *dst = to_int(flag, v); });
  }
  void opt(const std::string& flag, double* dst, const std::string& help) {
    add(flag, help, false, false, [dst, flag](const std::string& v) { *dst = to_double(flag, v); });
  }
  void list(const std::string& flag, std::vector<std::string>* dst, const std::string& help) {
    add(flag, help, false, false, [dst](const std::string& v) { *dst = split(v); });
  }
  void list(const std::string& flag, std::vector<int>* dst, const std::string& help) {
    add(flag, help, false, false, [dst, flag](const std::string& v) {
      dst->clear();
      for (const std::string& x : split(v)) dst->push_back(to_int(flag, x));
    });
  }
  void flag(const std::string& flag, bool* dst, const std::string& help) {
    add(flag, help, false, true, [dst](const std::string&) { *dst = true; });
  }
  void parse(const std::vector<std::string>& args) {
    std::map<std::string, int> seen;
    for (size_t i = 0; i < args.size(); ++i) {
      std::string a = args[i], value;
      if (a == "--help" || a == "-h") throw Help{};
      bool inline_value = false;
      const size_t eq = a.find('=');
      if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
        value = a.substr(eq + 1);
        a = a.substr(0, eq);
        inline_value = true;
      }
      auto it = opts_.find(a);
      if (it == opts_.end()) throw ParseError{"The following argument was not expected: " + args[i]};
      Opt& o = it->second;
      if (seen[a]++) throw ParseError{a + ": only one occurrence allowed"};
      if (o.is_flag) {
        if (inline_value) throw ParseError{a + ": flag takes no value"};
        o.set("");
        continue;
      }
      if (!inline_value) {
        if (i + 1 >= args.size()) throw ParseError{a + " requires an argument"};
        value = args[++i];
      }
      o.set(value);
    }
    for (const auto& kv : opts_)
      if (kv.second.required && !seen.count(kv.first)) throw ParseError{kv.first + " is required"};
  }
  std::string help() const {
    std::string s = name_ + ": " + about_ + "\nOptions:\n";
    for (const std::string& f : order_) s += "  " + f + (opts_.at(f).is_flag ? "" : " VALUE") + "\t" +
                                             opts_.at(f).help + (opts_.at(f).required ? " (required)" : "") + "\n";
    return s;
  }
  const std::string& name() const { return name_; }

 private:
  struct Opt {
    std::string help;
    bool required, is_flag;
    std::function<void(const std::string&)> set;
  };
  void add(const std::string& flag, const std::string& help, bool required, bool is_flag,
           std::function<void(const std::string&)> set) {
    opts_[flag] = Opt{help, required, is_flag, std::move(set)};
    order_.push_back(flag);
  }
  static std::vector<std::string> split(const std::string& v) {
    std::vector<std::string> out;
    size_t b = 0;
    while (true) {
      const size_t c = v.find(',', b);
      out.push_back(v.substr(b, c == std::string::npos ? std::string::npos : c - b));
      if (c == std::string::npos) break;
      b = c + 1;
    }
    return out;
  }
  static int to_int(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    errno = 0;
    const long x = std::strtol(v.c_str(), &end, 10);
    if (v.empty() || *end || errno || x < INT32_MIN || x > INT32_MAX)
      throw ParseError{"Could not convert: " + flag + " = " + v};
    return (int)x;
  }
  static double to_double(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    const double x = std::strtod(v.c_str(), &end);
    if (v.empty() || *end) throw ParseError{"Could not convert: " + flag + " = " + v};
    return x;
  }
  std::string name_, about_;
  std::map<std::string, Opt> opts_;
  std::vector<std::string> order_;
};

// parse_sources (tools/geoheat.cpp:183-196): ',' tokens, std::stol each
std::vector<int32_t> parse_sources(const std::string& text) {
  std::vector<int32_t> out;
  size_t b = 0;
  while (b <= text.size()) {
    size_t c = text.find(',', b);
    if (c == std::string::npos) c = text.size();
    const std::string token = text.substr(b, c - b);
    const bool last = c == text.size();
    b = c + 1;
    if (!token.empty()) {
      const char* s = token.c_str();
      char* end = nullptr;
      errno = 0;
      const long v = std::strtol(s, &end, 10);
      if (end == s || errno == ERANGE) throw std::invalid_argument("bad source index '" + token + "'");
      out.push_back(static_cast<int32_t>(v));
    }
    if (last) break;
  }
  return out;
}

// ---------------------------------------------------------------- handles
struct Mesh {
  gh_mesh* h = nullptr;
  gh_mesh_info info{};
  explicit Mesh(gh_mesh* m) : h(m) { check(gh_mesh_get_info(h, &info)); }
  ~Mesh() {
    if (h) gh_mesh_destroy(h);
  }
  Mesh(const Mesh&) = delete;
  Mesh& operator=(const Mesh&) = delete;
};

std::unique_ptr<Mesh> load(const std::string& path) {
  gh_mesh* m = nullptr;
  check(gh_mesh_load(path.c_str(), &m, nullptr));
  return std::unique_ptr<Mesh>(new Mesh(m));
}

void validate_options(const Mesh& mesh, const PipelineOptions& opt) {  // tools/geoheat.cpp:52-66
  if (opt.method != "face" && opt.method != "edge" && opt.method != "poisson")
    throw std::invalid_argument("unknown method '" + opt.method + "'");
  if (!(opt.m > 0.0)) throw std::invalid_argument("--m must be positive");
  if (opt.gs_iters < 0) throw std::invalid_argument("--gs-iters must be >= 0");
  if (opt.admm_iters < 0) throw std::invalid_argument("--admm-iters must be >= 0");
  if (!(opt.mu > 0.0)) throw std::invalid_argument("--mu must be positive");
  if (!(opt.eps > 0.0)) throw std::invalid_argument("--eps must be positive");
  if (opt.threads < 0) throw std::invalid_argument("--threads must be >= 1");
  if (opt.device != "gpu") throw std::invalid_argument("--device must be 'gpu' (this build has no CPU path)");
  if (opt.sources.empty()) throw std::invalid_argument("no source vertices given");
  for (int32_t s : opt.sources)
    if (s < 0 || s >= mesh.info.vertices)
      throw std::invalid_argument("source index " + std::to_string(s) + " out of range");
}

// RunReport (report.hpp:50-135)
struct RunReport {
  std::string method, mesh_path, reference;
  std::vector<int32_t> sources;
  int32_t vertices = 0, edges = 0, faces = 0;
  double quality_tau = 0, avg_edge_length = 0, m = 1, t = 0;
  int gs_sweeps = 0, admm_max_iterations = 0;
  double mu = 0, eps1 = 0, eps2 = 0;
  int threads = 1;
  bool sequential = false;
  double init_seconds = 0, diffusion_seconds = 0, optimization_seconds = 0, integration_seconds = 0,
         total_seconds = 0;
  uint64_t solver_state_bytes = 0, state_bytes_allocated = 0, peak_rss_bytes = 0;
  int gs_iterations = 0, admm_iterations = 0, cg_iterations = 0;
  double final_primal = 0, final_dual = 0, diffusion_e1 = -1.0;
  double mean_rel_error = -1.0;
  int32_t mre_excluded = 0;
  double e2 = -1.0;

  std::string text() const {
    std::string s;
    auto kv = [&](const char* k, const std::string& v) { s += std::string(k) + " = " + v + "\n"; };
    std::string src;
    for (size_t i = 0; i < sources.size(); ++i) src += (i ? "," : "") + std::to_string(sources[i]);
    kv("method", method);
    kv("mesh", mesh_path);
    kv("sources", src);
    kv("vertices", std::to_string(vertices));
    kv("edges", std::to_string(edges));
    kv("faces", std::to_string(faces));
    kv("tau", format_double(quality_tau));
    kv("avg_edge_length", format_double(avg_edge_length));
    kv("m", format_double(m));
    kv("t", format_double(t));
    kv("gs_iters", std::to_string(gs_sweeps));
    kv("admm_iters", std::to_string(admm_max_iterations));
    kv("mu", format_double(mu));
    kv("eps1", format_double(eps1));
    kv("eps2", format_double(eps2));
    kv("threads", std::to_string(threads));
    kv("seq", sequential ? "1" : "0");
    kv("init_seconds", format_double(init_seconds));
    kv("diffusion_seconds", format_double(diffusion_seconds));
    kv("optimization_seconds", format_double(optimization_seconds));
    kv("integration_seconds", format_double(integration_seconds));
    kv("total_seconds", format_double(total_seconds));
    kv("solver_state_bytes", std::to_string(solver_state_bytes));
    kv("state_bytes_allocated", std::to_string(state_bytes_allocated));
    if (peak_rss_bytes > 0) kv("peak_rss_bytes", std::to_string(peak_rss_bytes));
    kv("gs_iterations", std::to_string(gs_iterations));
    kv("admm_iterations", std::to_string(admm_iterations));
    kv("cg_iterations", std::to_string(cg_iterations));
    kv("final_primal", format_double(final_primal));
    kv("final_dual", format_double(final_dual));
    kv("diffusion_e1", format_double(diffusion_e1));
    if (!reference.empty()) {
      kv("reference", reference);
      kv("mean_rel_error", format_double(mean_rel_error));
      kv("mean_rel_error_excluded", std::to_string(mre_excluded));
      kv("e2", format_double(e2));
    }
    return s;
  }
};

struct PipelineResult {
  std::vector<double> distances;
  RunReport report;
};

// run_pipeline (tools/geoheat.cpp:71-161) with the solver chain on the GPU
PipelineResult run_pipeline(const Mesh& mesh, const PipelineOptions& opt) {
  PipelineResult out;
  RunReport& rep = out.report;
  rep.method = opt.method;
  rep.mesh_path = opt.mesh_path;
  rep.sources = opt.sources;
  rep.vertices = mesh.info.vertices;
  rep.edges = mesh.info.edges;
  rep.faces = mesh.info.faces;
  rep.m = opt.m;
  rep.gs_sweeps = opt.gs_iters;
  rep.admm_max_iterations = opt.admm_iters;
  rep.mu = opt.mu;
  rep.eps1 = opt.eps;
  rep.eps2 = opt.eps;
  rep.threads = resolve_threads(opt);
  rep.sequential = opt.sequential;

  const double total0 = now_s();
  check(gh_triangulation_quality(mesh.h, &rep.quality_tau));
  check(gh_average_edge_length(mesh.h, &rep.avg_edge_length));
  rep.t = opt.m * rep.avg_edge_length * rep.avg_edge_length;
  gh_levels* levels = nullptr;
  check(gh_bfs_create(mesh.h, opt.sources.data(), (int32_t)opt.sources.size(), &levels));
  struct Guard {
    gh_levels* l;
    ~Guard() { gh_bfs_destroy(l); }
  } guard{levels};
  rep.init_seconds = now_s() - total0;
  gh_levels_info li{};
  check(gh_bfs_get_info(levels, &li));
  if (li.unreachable_count > 0) std::fprintf(stderr, "warning: %d unreachable vertices\n", li.unreachable_count);

  out.distances.assign(mesh.info.vertices, 0.0);
  gh_pipeline_config cfg{};
  cfg.method = opt.method == "face" ? GH_METHOD_FACE : opt.method == "edge" ? GH_METHOD_EDGE : GH_METHOD_POISSON;
  cfg.sweeps = opt.gs_iters;
  cfg.t = rep.t;
  cfg.m = opt.m;
  cfg.admm.max_iterations = opt.admm_iters;
  cfg.admm.eps1 = opt.eps;
  cfg.admm.eps2 = opt.eps;
  cfg.admm.mu = opt.mu;
  cfg.cg_tol = opt.eps;
  cfg.flags = GH_PIPE_DIFFUSION_E1;
  gh_run_report rr{};
  check(gh_distance(levels, &cfg, out.distances.data(), &rr));
  if (cfg.method == GH_METHOD_POISSON) {
    rep.diffusion_seconds = rr.diffusion_ms * 1e-3;
    rep.optimization_seconds = rr.optimization_ms * 1e-3;
    rep.cg_iterations = rr.cg_iterations;
    rep.final_primal = rr.poisson_residual;
  } else {
    rep.diffusion_seconds = (rr.diffusion_ms + rr.normalize_ms) * 1e-3;
    rep.gs_iterations = rr.gs_iterations;
    rep.diffusion_e1 = rr.diffusion_e1;
    rep.optimization_seconds = rr.optimization_ms * 1e-3;
    rep.integration_seconds = rr.integration_ms * 1e-3;
    rep.admm_iterations = rr.admm_iterations;
    rep.final_primal = rr.final_primal;
    rep.final_dual = rr.final_dual;
    rep.solver_state_bytes = rr.solver_state_bytes;
    rep.state_bytes_allocated = rr.state_bytes_allocated;
  }
  if (rep.solver_state_bytes == 0)
    check(gh_solver_state_bytes(mesh.h, opt.method == "edge" ? GH_METHOD_EDGE : GH_METHOD_FACE,
                                &rep.solver_state_bytes));
  rep.total_seconds = now_s() - total0;
  struct rusage usage;
  if (getrusage(RUSAGE_SELF, &usage) == 0) rep.peak_rss_bytes = (uint64_t)usage.ru_maxrss * 1024;
  return out;
}

// attach_reference_metrics (tools/geoheat.cpp:164-181)
void attach_reference_metrics(const Mesh& mesh, const PipelineOptions& opt, const std::string& reference,
                              PipelineResult& result) {
  if (reference.empty()) return;
  std::vector<double> d_ref(mesh.info.vertices);
  const int32_t ns = (int32_t)opt.sources.size();
  if (reference == "euclid") check(gh_analytic_distance(mesh.h, GH_SURFACE_PLANE, opt.sources.data(), ns, d_ref.data()));
  else if (reference == "sphere")
    check(gh_analytic_distance(mesh.h, GH_SURFACE_SPHERE, opt.sources.data(), ns, d_ref.data()));
  else if (reference == "dijkstra") check(gh_dijkstra_distance(mesh.h, opt.sources.data(), ns, d_ref.data()));
  else throw std::invalid_argument("unknown reference '" + reference + "'");
  result.report.reference = reference;
  check(gh_error_metrics(result.distances.data(), d_ref.data(), (int64_t)d_ref.size(), opt.sources.data(), ns,
                         &result.report.mean_rel_error, &result.report.mre_excluded, &result.report.e2));
}

struct OutFile {
  FILE* f = nullptr;
  bool owned = false;
  ~OutFile() {
    if (owned && f) std::fclose(f);
  }
};

void write_all(FILE* f, const void* data, uint64_t n) {
  if (n && std::fwrite(data, 1, n, f) != n) throw MeshError("write failed");
}

// write_distance_output (tools/geoheat.cpp:198-212)
void write_distance_output(const Mesh& mesh, const std::vector<double>& d, const std::string& out_path,
                           const std::string& format) {
  OutFile out;
  out.f = stdout;
  if (!out_path.empty()) {
    out.f = std::fopen(out_path.c_str(), "wb");
    if (!out.f) throw MeshError("cannot open output file '" + out_path + "'");
    out.owned = true;
  }
  void* buf = nullptr;
  uint64_t n = 0;
  if (format == "txt") check(gh_format_distances(d.data(), (int64_t)d.size(), GH_DISTANCES_TXT, &buf, &n));
  else if (format == "csv") check(gh_format_distances(d.data(), (int64_t)d.size(), GH_DISTANCES_CSV, &buf, &n));
  else if (format == "ply") check(gh_mesh_serialize(mesh.h, GH_FORMAT_PLY, d.data(), &buf, &n));
  else throw std::invalid_argument("unknown output format '" + format + "'");
  try {
    write_all(out.f, buf, n);
  } catch (...) {
    gh_free(buf);
    throw;
  }
  gh_free(buf);
  std::fflush(out.f);
}

int cmd_distance(const PipelineOptions& opt, const std::string& out_path, const std::string& out_format,
                 const std::string& report_path, const std::string& reference) {
  std::unique_ptr<Mesh> mesh = load(opt.mesh_path);
  validate_options(*mesh, opt);
  PipelineResult result = run_pipeline(*mesh, opt);
  attach_reference_metrics(*mesh, opt, reference, result);
  write_distance_output(*mesh, result.distances, out_path, out_format);
  const std::string text = result.report.text();
  if (report_path.empty()) {
    std::fputs(text.c_str(), stderr);
  } else {
    FILE* f = std::fopen(report_path.c_str(), "w");
    if (!f) throw MeshError("cannot open report file '" + report_path + "'");
    std::fputs(text.c_str(), f);
    std::fclose(f);
  }
  return 0;
}

int cmd_bench(PipelineOptions opt, const std::vector<std::string>& methods, const std::vector<int>& threads_list,
              int repeats) {  // tools/geoheat.cpp:229-263
  if (repeats < 1) throw std::invalid_argument("--repeats must be >= 1");
  for (int n : threads_list)
    if (n < 1) throw std::invalid_argument("thread counts must be >= 1");
  std::unique_ptr<Mesh> mesh = load(opt.mesh_path);
  if (opt.sources.empty()) opt.sources = {0};
  validate_options(*mesh, opt);
  std::printf(
      "method,threads,repeat,vertices,edges,faces,init_seconds,diffusion_seconds,optimization_seconds,"
      "integration_seconds,total_seconds,solver_state_bytes,gs_iterations,admm_iterations,final_primal,"
      "final_dual,distance_hash\n");
  std::fflush(stdout);
  for (const std::string& method : methods) {
    for (int threads : threads_list) {
      for (int repeat = 0; repeat < repeats; ++repeat) {
        PipelineOptions run = opt;
        run.method = method;
        run.threads = threads;
        validate_options(*mesh, run);
        PipelineResult result = run_pipeline(*mesh, run);
        const RunReport& r = result.report;
        std::printf("%s,%d,%d,%d,%d,%d,%s,%s,%s,%s,%s,%llu,%d,%d,%s,%s,%llu\n", method.c_str(), threads, repeat,
                    r.vertices, r.edges, r.faces, format_double(r.init_seconds).c_str(),
                    format_double(r.diffusion_seconds).c_str(), format_double(r.optimization_seconds).c_str(),
                    format_double(r.integration_seconds).c_str(), format_double(r.total_seconds).c_str(),
                    (unsigned long long)r.solver_state_bytes, r.gs_iterations, r.admm_iterations,
                    format_double(r.final_primal).c_str(), format_double(r.final_dual).c_str(),
                    (unsigned long long)gh_field_hash(result.distances.data(), (int64_t)result.distances.size()));
        std::fflush(stdout);
      }
    }
  }
  return 0;
}

int cmd_subdivide(const std::string& mesh_path, int levels, const std::string& out_path) {  // 265-275
  if (levels < 0) throw std::invalid_argument("--levels must be >= 0");
  std::unique_ptr<Mesh> mesh = load(mesh_path);
  gh_mesh* fine_h = nullptr;
  check(gh_mesh_subdivide(mesh->h, levels, &fine_h));
  Mesh fine(fine_h);
  check(gh_mesh_save(fine.h, out_path.c_str(), nullptr));
  std::fprintf(stderr, "vertices = %d\nedges = %d\nfaces = %d\n", fine.info.vertices, fine.info.edges,
               fine.info.faces);
  return 0;
}

const char* kAbout = "geodesic distance on triangle meshes via a parallel heat-method pipeline (B200)";

}  // namespace

int main(int argc, char** argv) {
  PipelineOptions opt;
  std::string source_list = "0";
  std::string out_path, out_format = "txt", report_path, reference;

  Command distance("distance", "compute per-vertex geodesic distances");
  distance.opt("--mesh", &opt.mesh_path, "input mesh (.obj or .ply)", true);
  distance.opt("--source", &source_list, "source vertex indices, comma separated");
  distance.opt("--method", &opt.method, "face | edge | poisson");
  distance.opt("--m", &opt.m, "smoothing factor, t = m*h^2");
  distance.opt("--gs-iters", &opt.gs_iters, "Gauss-Seidel sweeps");
  distance.opt("--admm-iters", &opt.admm_iters, "max ADMM iterations");
  distance.opt("--mu", &opt.mu, "ADMM penalty");
  distance.opt("--eps", &opt.eps, "residual threshold (and CG tolerance for poisson)");
  distance.opt("--threads", &opt.threads, "thread budget echoed into the report (GPU run)");
  distance.flag("--seq", &opt.sequential, "report a sequential run (threads = 1)");
  distance.opt("--device", &opt.device, "gpu");
  distance.opt("--out", &out_path, "output path (default: stdout)");
  distance.opt("--out-format", &out_format, "txt | ply | csv");
  distance.opt("--report", &report_path, "write the run report here instead of stderr");
  distance.opt("--reference", &reference, "compare against: euclid | sphere | dijkstra");

  std::vector<std::string> methods{"face"};
  std::vector<int> threads_list{1};
  int repeats = 1;
  Command bench("bench", "benchmark methods over thread counts, CSV to stdout");
  bench.opt("--mesh", &opt.mesh_path, "input mesh (.obj or .ply)", true);
  bench.list("--methods", &methods, "methods to run");
  bench.list("--threads-list", &threads_list, "thread counts to sweep");
  bench.opt("--repeats", &repeats, "repetitions per configuration");
  bench.opt("--source", &source_list, "source vertex indices, comma separated");
  bench.opt("--m", &opt.m, "smoothing factor");
  bench.opt("--gs-iters", &opt.gs_iters, "Gauss-Seidel sweeps");
  bench.opt("--admm-iters", &opt.admm_iters, "max ADMM iterations");
  bench.opt("--mu", &opt.mu, "ADMM penalty");
  bench.opt("--eps", &opt.eps, "residual threshold");
  bench.opt("--device", &opt.device, "gpu");

  std::string sub_mesh, sub_out;
  int sub_levels = 1;
  Command subdivide("subdivide", "midpoint 1-to-4 subdivision");
  subdivide.opt("--mesh", &sub_mesh, "input mesh", true);
  subdivide.opt("--levels", &sub_levels, "subdivision levels");
  subdivide.opt("--out", &sub_out, "output mesh path", true);

  Command* cmds[] = {&distance, &bench, &subdivide};
  Command* chosen = nullptr;
  try {
    std::vector<std::string> args(argv + 1, argv + argc);
    if (!args.empty() && (args[0] == "--help" || args[0] == "-h")) throw Help{};
    if (args.empty()) throw ParseError{"A subcommand is required"};
    for (Command* c : cmds)
      if (c->name() == args[0]) chosen = c;
    if (!chosen) throw ParseError{"The following argument was not expected: " + args[0]};
    chosen->parse(std::vector<std::string>(args.begin() + 1, args.end()));
  } catch (const Help&) {
    std::printf("%s\nUsage: geoheat_b200 SUBCOMMAND [OPTIONS]\n\n", kAbout);
    for (Command* c : cmds)
      if (!chosen || c == chosen) std::printf("%s\n", c->help().c_str());
    return 0;
  } catch (const ParseError& e) {
    std::fprintf(stderr, "%s\nRun with --help for more information.\n", e.msg.c_str());
    return 2;
  }

  try {
    opt.sources = parse_sources(source_list);
    if (chosen == &distance) return cmd_distance(opt, out_path, out_format, report_path, reference);
    if (chosen == &bench) return cmd_bench(opt, methods, threads_list, repeats);
    return cmd_subdivide(sub_mesh, sub_levels, sub_out);
  } catch (const SolverError& e) {
    std::fprintf(stderr, "solver failure: %s\n", e.what());
    return 3;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "invalid configuration: %s\n", e.what());
    return 2;
  } catch (const MeshError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
