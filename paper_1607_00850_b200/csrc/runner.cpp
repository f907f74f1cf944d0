// Runner, bench harness and config files over the C ABI: the production
// driver layer that sits on top of the hot path in the reference
// (proj/core/src/runner.cpp, proj/core/src/config_file.cpp,
// proj/core/include/sdns/runner.hpp, config_file.hpp), rebuilt around the
// device pipeline. Everything numeric goes through the public entry points
// of include/sdns_cuda.h (context, fields, fused steps, stats, checkpoints);
// this file owns rank threads, hooks, timing reductions and the output files,
// whose formats are byte-identical to the reference's.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <filesystem>
#include <fstream>
#include <mutex>
#include <numbers>
#include <sstream>
#include <thread>
#include <vector>

#include "host.h"

using namespace sdns_host;

namespace sdns_host {
void ck(int rc) {
  if (rc != SDNS_OK) throw Error(rc, sdns_last_error());
}
}  // namespace sdns_host

namespace {


[[noreturn]] void io_error(const std::string& m) { throw Error(SDNS_IO_ERROR, m); }

std::string fmt(double v) {  // runner.cpp:23-27
  char buf[32];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

void copy_str(char* dst, size_t cap, const std::string& s) {
  if (!cap) return;
  const size_t n = std::min(cap - 1, s.size());
  std::memcpy(dst, s.data(), n);
  dst[n] = '\0';
}

const char* decomp_name(int d) { return d == SDNS_PENCIL ? "pencil" : "slab"; }  // config.cpp:7-9

int decomp_from_string(const std::string& s) {  // config.cpp:11-15
  if (s == "slab") return SDNS_SLAB;
  if (s == "pencil") return SDNS_PENCIL;
  config_error("unknown decomposition '" + s + "' (expected slab|pencil)");
}

// ---- config files (config_file.cpp) ---------------------------------------

std::string trim(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r\n");
  if (b == std::string::npos) return "";
  const auto e = s.find_last_not_of(" \t\r\n");
  return s.substr(b, e - b + 1);
}

int parse_int(const std::string& key, const std::string& value) {
  try {
    size_t pos = 0;
    const int v = std::stoi(value, &pos);
    if (pos != value.size()) throw std::invalid_argument(value);
    return v;
  } catch (const std::exception&) {
    config_error("key '" + key + "': expected integer, got '" + value + "'");
  }
}

double parse_double(const std::string& key, const std::string& value) {
  try {
    size_t pos = 0;
    const double v = std::stod(value, &pos);
    if (pos != value.size() || !std::isfinite(v)) throw std::invalid_argument(value);
    return v;
  } catch (const std::exception&) {
    config_error("key '" + key + "': expected number, got '" + value + "'");
  }
}

bool parse_bool(const std::string& key, const std::string& value) {
  if (value == "true" || value == "on" || value == "yes" || value == "1") return true;
  if (value == "false" || value == "off" || value == "no" || value == "0") return false;
  config_error("key '" + key + "': expected boolean, got '" + value + "'");
}

std::pair<int, int> default_pencil_grid(int n, int p) {  // config_file.cpp:43-55
  for (int p1 = static_cast<int>(std::sqrt(static_cast<double>(p))); p1 >= 1; --p1) {
    if (p % p1 != 0) continue;
    const int p2 = p / p1;
    if (n % p1 == 0 && n % p2 == 0 && p2 <= n / 2) return {p1, p2};
  }
  config_error("no valid pencil grid for n=" + std::to_string(n) + ", p=" + std::to_string(p));
}

sdns_config config_defaults() {  // config.hpp:17-28
  sdns_config c{};
  c.n = 32;
  c.decomp = SDNS_SLAB;
  c.p = c.p1 = c.p2 = 1;
  c.nu = 1.0 / 1600.0;
  c.dt = 1e-3;
  c.t_end = 0.1;
  c.dealias = 1;
  c.out_every = 10;
  return c;
}

void validate_case(const std::string& initial_case) {  // config.cpp:49
  if (initial_case.empty()) config_error("initial_case must be non-empty");
}

void parse_config(const std::string& text, const char* const* keys, const char* const* values,
                  int n_over, sdns_parsed_config* out) {  // config_file.cpp:57-136
  sdns_config cfg = config_defaults();
  std::string initial_case = "taylor_green";
  std::string notices;
  bool saw_t_end = false, saw_pencil_grid = false;
  auto apply = [&](const std::string& key, const std::string& value) {
    if (key == "n") {
      cfg.n = parse_int(key, value);
    } else if (key == "decomp") {
      cfg.decomp = decomp_from_string(value);
    } else if (key == "p") {
      cfg.p = parse_int(key, value);
    } else if (key == "p1") {
      cfg.p1 = parse_int(key, value);
      saw_pencil_grid = true;
    } else if (key == "p2") {
      cfg.p2 = parse_int(key, value);
      saw_pencil_grid = true;
    } else if (key == "nu") {
      cfg.nu = parse_double(key, value);
    } else if (key == "re") {
      const double re = parse_double(key, value);
      if (re <= 0.0) config_error("key 're': must be > 0");
      cfg.nu = 1.0 / re;
    } else if (key == "dt") {
      cfg.dt = parse_double(key, value);
    } else if (key == "t_end") {
      cfg.t_end = parse_double(key, value);
      saw_t_end = true;
    } else if (key == "dealias") {
      cfg.dealias = parse_bool(key, value) ? 1 : 0;
    } else if (key == "case") {
      initial_case = value;
    } else if (key == "out_every") {
      cfg.out_every = parse_int(key, value);
    } else {
      config_error("unknown config key '" + key + "'");
    }
  };
  std::istringstream in(text);
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (const auto hash = line.find('#'); hash != std::string::npos) line.erase(hash);
    line = trim(line);
    if (line.empty()) continue;
    const auto eq = line.find('=');
    if (eq == std::string::npos)
      config_error("line " + std::to_string(lineno) + ": expected 'key = value', got '" + line +
                   "'");
    apply(trim(line.substr(0, eq)), trim(line.substr(eq + 1)));
  }
  for (int i = 0; i < n_over; ++i) apply(keys[i] ? keys[i] : "", values[i] ? values[i] : "");
  if (!saw_t_end) notices += "t_end not specified; defaulting to " + std::to_string(cfg.t_end) + "\n";
  if (cfg.decomp == SDNS_PENCIL && !saw_pencil_grid && cfg.p > 1) {
    const auto [p1, p2] = default_pencil_grid(cfg.n, cfg.p);
    cfg.p1 = p1;
    cfg.p2 = p2;
    notices += "pencil grid not specified; using p1=" + std::to_string(p1) +
               " p2=" + std::to_string(p2) + "\n";
  }
  validate(cfg);
  validate_case(initial_case);
  if (initial_case.size() >= sizeof(out->initial_case)) config_error("initial case name too long");
  out->cfg = cfg;
  copy_str(out->initial_case, sizeof(out->initial_case), initial_case);
  copy_str(out->notices, sizeof(out->notices), notices);
}

std::string read_file(const std::string& path, const std::string& what) {
  std::ifstream in(path);
  if (!in) io_error("cannot open " + what + " '" + path + "'");
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

// ---- bench matrix (runner.cpp:249-297) -------------------------------------

std::vector<sdns_bench_entry> parse_bench_matrix(const std::string& text) {
  std::vector<sdns_bench_entry> entries;
  std::istringstream in(text);
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (const auto hash = line.find('#'); hash != std::string::npos) line.erase(hash);
    for (char& ch : line)
      if (ch == ',') ch = ' ';
    std::istringstream ls(line);
    std::string n_s, d_s, p_s, p1_s, p2_s;
    if (!(ls >> n_s)) continue;
    const std::string where = "bench matrix line " + std::to_string(lineno);
    if (!(ls >> d_s >> p_s)) config_error(where + ": expected 'n, decomp, p[, p1, p2]'");
    sdns_bench_entry e{};
    try {
      e.n = std::stoi(n_s);
      e.decomp = decomp_from_string(d_s);
      e.p = std::stoi(p_s);
      if (ls >> p1_s) {
        if (!(ls >> p2_s)) config_error(where + ": p1 given without p2");
        e.p1 = std::stoi(p1_s);
        e.p2 = std::stoi(p2_s);
      }
    } catch (const Error&) {
      throw;
    } catch (const std::exception&) {
      config_error(where + ": malformed entry '" + line + "'");
    }
    std::string extra;
    if (ls >> extra) config_error(where + ": trailing fields");
    entries.push_back(e);
  }
  return entries;
}

void put_entries(const std::vector<sdns_bench_entry>& v, sdns_bench_entry* out, int cap,
                 int* count) {
  if (out)
    for (size_t i = 0; i < v.size() && static_cast<int>(i) < cap; ++i) out[i] = v[i];
  if (count) *count = static_cast<int>(v.size());
}

// ---- output files (runner.cpp:215-247, :399-414) ---------------------------

void write_diagnostics_csv(const std::string& path, const int64_t* steps, const double* rows,
                           int64_t nrows, int shells) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) io_error("cannot open '" + path + "' for writing");
  out << "step,t,E,Z,eps,div_max";
  for (int s = 0; s < shells; ++s) out << ",shell_" << s;
  out << "\n";
  const int w = 5 + shells;
  for (int64_t r = 0; r < nrows; ++r) {
    const double* row = rows + r * w;
    out << steps[r] << ',' << fmt(row[0]) << ',' << fmt(row[1]) << ',' << fmt(row[2]) << ','
        << fmt(row[3]) << ',' << fmt(row[4]);
    for (int s = 0; s < shells; ++s) out << ',' << fmt(row[5 + s]);
    out << "\n";
  }
  if (!out) io_error("short write to '" + path + "'");
}

void write_manifest(const std::string& path, const sdns_config& cfg, const std::string& icase,
                    const sdns_run_result& r) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) io_error("cannot open '" + path + "' for writing");
  out << "format = sdns-manifest-1\n"
      << "version = " << sdns_version() << "\n"
      << "backend = " << r.backend << "\n"
      << "status = " << r.status << "\n"
      << "n = " << cfg.n << "\n"
      << "decomp = " << decomp_name(cfg.decomp) << "\n"
      << "p = " << cfg.p << "\n"
      << "p1 = " << cfg.p1 << "\n"
      << "p2 = " << cfg.p2 << "\n"
      << "nu = " << fmt(cfg.nu) << "\n"
      << "dt = " << fmt(cfg.dt) << "\n"
      << "t_end = " << fmt(cfg.t_end) << "\n"
      << "dealias = " << (cfg.dealias ? "true" : "false") << "\n"
      << "case = " << icase << "\n"
      << "out_every = " << cfg.out_every << "\n"
      << "steps = " << r.steps << "\n"
      << "step_seconds_min = " << fmt(r.step_min_s) << "\n"
      << "step_seconds_mean = " << fmt(r.step_mean_s) << "\n"
      << "step_seconds_max = " << fmt(r.step_max_s) << "\n"
      << "timed_steps = " << r.timed_steps << "\n"
      << "csv = " << r.csv_path << "\n"
      << "checkpoint = " << r.checkpoint_path << "\n";
  if (!out) io_error("short write to '" + path + "'");
}

void write_bench_csv(const std::string& path, const sdns_bench_row* rows, int count) {
  const auto dir = std::filesystem::path(path).parent_path();
  if (!dir.empty()) std::filesystem::create_directories(dir);
  std::ofstream out(path, std::ios::trunc);
  if (!out) io_error("cannot open '" + path + "' for writing");
  out << "n,decomp,p,p1,p2,nodes_per_rank,sec_per_step,status\n";
  for (int i = 0; i < count; ++i) {
    const sdns_bench_row& r = rows[i];
    std::string status = r.status;
    for (char& ch : status)
      if (ch == ',' || ch == '\n') ch = ';';
    out << r.entry.n << ',' << decomp_name(r.entry.decomp) << ',' << r.entry.p << ','
        << r.entry.p1 << ',' << r.entry.p2 << ',' << r.nodes_per_rank << ','
        << fmt(r.sec_per_step) << ',' << status << "\n";
  }
  if (!out) io_error("short write to '" + path + "'");
}


}  // namespace

namespace sdns_host {

// The rank's real block of a Taylor-Green field on physical_mesh
// (mesh.cpp:8-21): the reference's case (taylor_green_init,
// navier_stokes.cpp:7-25: cos x sin y sin z, -sin x cos y sin z, 0) or
// BASELINE configs[0]'s (sin x cos y cos z, -cos x sin y cos z, 0).
std::vector<double> tg_real_block(const sdns_layout& lo, bool reference_variant) {
  const double h = 2.0 * std::numbers::pi / static_cast<double>(lo.n);
  auto axis = [h](int64_t len, int64_t off) {
    std::vector<double> v(static_cast<size_t>(len));
    for (int64_t i = 0; i < len; ++i) v[static_cast<size_t>(i)] = h * static_cast<double>(off + i);
    return v;
  };
  const auto x = axis(lo.real_shape[0], lo.real_offset[0]);
  const auto y = axis(lo.real_shape[1], lo.real_offset[1]);
  const auto z = axis(lo.real_shape[2], lo.real_offset[2]);
  const int64_t s0 = lo.real_shape[0], s1 = lo.real_shape[1], s2 = lo.real_shape[2];
  const size_t cs = static_cast<size_t>(s0 * s1 * s2);
  std::vector<double> u(3 * cs, 0.0);
  for (int64_t i = 0; i < s0; ++i) {
    const double sx = std::sin(x[i]), cx = std::cos(x[i]);
    for (int64_t j = 0; j < s1; ++j) {
      const double sy = std::sin(y[j]), cy = std::cos(y[j]);
      for (int64_t k = 0; k < s2; ++k) {
        const size_t at = static_cast<size_t>((i * s1 + j) * s2 + k);
        if (reference_variant) {
          const double sz = std::sin(z[k]);
          u[at] = cx * sy * sz;
          u[cs + at] = -sx * cy * sz;
        } else {
          const double cz = std::cos(z[k]);
          u[at] = sx * cy * cz;
          u[cs + at] = -(cx * sy * cz);
        }
      }
    }
  }
  return u;
}

// Initial spectral state of one rank: the named case (make_initial_condition,
// navier_stokes.cpp:27-32) forward transformed and projected
// (runner.cpp:78-82), or the seeded isotropic field set in spectral space.
void initial_state(sdns_ctx* ctx, const sdns_config& cfg, const std::string& icase,
                   uint64_t seed, sdns_field* u_hat) {
  sdns_layout lo{};
  ck(sdns_ctx_layout(ctx, &lo));
  if (icase == "isotropic") {
    const int64_t count = 3 * lo.spec_shape[0] * lo.spec_shape[1] * lo.spec_shape[2] * 2;
    std::vector<double> h(static_cast<size_t>(count));
    ck(sdns_iso_init_host(cfg.n, seed, 4.0, 0.5, &lo, h.data()));
    ck(sdns_field_upload(ctx, u_hat, h.data()));
    return;
  }
  const bool ref_tg = icase == "taylor_green";
  if (!ref_tg && icase != "taylor_green_baseline")
    config_error("unknown initial case '" + icase + "'");
  const std::vector<double> u = tg_real_block(lo, ref_tg);
  sdns_field* real = nullptr;
  ck(sdns_field_alloc(ctx, SDNS_REAL, 3, &real));
  std::unique_ptr<sdns_field, int (*)(sdns_field*)> hold(real, sdns_field_free);
  ck(sdns_field_upload(ctx, real, u.data()));
  ck(sdns_fft_forward(ctx, real, u_hat));
  ck(sdns_project(ctx, u_hat));
}

}  // namespace sdns_host

namespace {

// reduce_timing (runner.cpp:42-65): first min(5, n) steps are warm-up.
void reduce_timing(const std::vector<double>& sec, sdns_comm* comm, sdns_run_result& r) {
  const size_t warm = std::min<size_t>(5, sec.size());
  r.timed_steps = static_cast<int64_t>(sec.size() - warm);
  double lo = 0.0, hi = 0.0, mean = 0.0;
  if (r.timed_steps > 0) {
    lo = hi = sec[warm];
    double sum = 0.0;
    for (size_t i = warm; i < sec.size(); ++i) {
      lo = std::min(lo, sec[i]);
      hi = std::max(hi, sec[i]);
      sum += sec[i];
    }
    mean = sum / static_cast<double>(r.timed_steps);
  }
  ck(sdns_comm_allreduce(comm, &lo, 1, 2));
  ck(sdns_comm_allreduce(comm, &hi, 1, 1));
  ck(sdns_comm_allreduce(comm, &mean, 1, 0));
  r.step_min_s = lo;
  r.step_max_s = hi;
  r.step_mean_s = r.timed_steps > 0 ? mean / static_cast<double>(sdns_comm_size(comm)) : 0.0;
}

struct Hooked {
  sdns_ctx* ctx;
  sdns_state* st;
  sdns_field* snap;
  double nu;
  int rank, shells;
  std::vector<int64_t> steps;
  std::vector<double> rows;
  std::vector<double> seconds;
  double snap_t = 0.0;
  int64_t snap_step = 0;
  int err = SDNS_OK;  // first failure inside a hook (hooks cannot throw through C)
  std::string err_msg;
};

void on_sample(int64_t step, double t, void* user) {  // runner.cpp:88-95
  auto* h = static_cast<Hooked*>(user);
  if (h->err) return;
  std::vector<double> row(static_cast<size_t>(5 + h->shells));
  int rc = sdns_collect_stats(h->ctx, sdns_state_u_hat(h->st), h->nu, t, row.data());
  if (rc == SDNS_OK) rc = sdns_fft_inverse(h->ctx, sdns_state_u_hat(h->st), h->snap);
  if (rc != SDNS_OK) {
    h->err = rc;
    h->err_msg = sdns_last_error();
    return;
  }
  h->snap_t = t;
  h->snap_step = step;
  if (h->rank == 0) {
    h->steps.push_back(step);
    h->rows.insert(h->rows.end(), row.begin(), row.end());
  }
}

void on_timing(int64_t, double s, void* user) { static_cast<Hooked*>(user)->seconds.push_back(s); }

std::string resolve_backend(const sdns_config& cfg, const std::string& name) {  // runner.cpp:29-40
  if (name == "auto") return cfg.p > 1 ? "inprocess" : "loopback";
  if (name == "loopback") {
    if (cfg.p != 1)
      config_error("loopback backend supports only p=1, got p=" + std::to_string(cfg.p));
    return "loopback";
  }
  if (name == "inprocess") return "inprocess";
  config_error("unknown backend '" + name + "' (expected auto|loopback|inprocess)");
}

struct Opts {
  std::string out_dir = "out", backend = "auto";
  double timeout_s = 30.0;
  int device = 0;
  uint64_t seed = 1607;
  sdns_ctx_options ctx{};
};

Opts read_opts(const sdns_run_options* o) {
  Opts r;
  if (!o) return r;
  if (o->out_dir && *o->out_dir) r.out_dir = o->out_dir;
  if (o->backend && *o->backend) r.backend = o->backend;
  if (o->collective_timeout_s > 0) r.timeout_s = o->collective_timeout_s;
  r.device = o->device;
  r.seed = o->seed;
  r.ctx = o->ctx;
  return r;
}

// run_worker (runner.cpp:67-146) for one rank; rank 0 alone fills `out`
// (other ranks work on a private copy) and writes the files.
void run_worker(const sdns_config& cfg, const std::string& icase, const Opts& o, int rank,
                sdns_comm* comm, int device, sdns_run_result& out) {
  sdns_run_result res = out;
  Ctx ctx;
  ck(sdns_ctx_create_ex(&cfg, rank, device, comm, nullptr, &o.ctx, &ctx.c));
  Fld u_hat, snap;
  ck(sdns_field_alloc(ctx.c, SDNS_SPECTRAL, 3, &u_hat.f));
  ck(sdns_field_alloc(ctx.c, SDNS_REAL, 3, &snap.f));
  initial_state(ctx.c, cfg, icase, o.seed, u_hat.f);
  State st;
  ck(sdns_state_create(ctx.c, &st.s));
  ck(sdns_state_set(ctx.c, st.s, u_hat.f, 0.0, 0));

  Hooked h{ctx.c, st.s, snap.f, cfg.nu, rank, sdns_spectrum_shells(cfg.n), {}, {}, {}, 0.0, 0, SDNS_OK, {}};
  const sdns_advance_hooks hooks{on_sample, on_timing, &h};
  int64_t fail_step = 0;
  const int rc = sdns_advance_hooks_run(ctx.c, st.s, &hooks, &fail_step);
  if (h.err) throw Error(h.err, h.err_msg);
  std::string div_msg;
  if (rc == SDNS_DIVERGENCE_ERROR)
    div_msg = sdns_last_error();
  else
    ck(rc);
  const bool diverged = rc == SDNS_DIVERGENCE_ERROR;

  // final (or last-good) checkpoint, collective on every path
  double ck_t = 0.0;
  int64_t ck_step = 0;
  ck(sdns_state_time(st.s, &ck_t, &ck_step));
  if (!diverged) {
    ck(sdns_fft_inverse(ctx.c, sdns_state_u_hat(st.s), snap.f));
  } else {
    ck_t = h.snap_t;
    ck_step = h.snap_step;
  }
  const std::string ckpt = o.out_dir + "/checkpoint.sdns";
  ck(sdns_checkpoint_write(ctx.c, snap.f, ckpt.c_str(), ck_t, ck_step));
  reduce_timing(h.seconds, comm, res);

  if (rank == 0) {
    int64_t steps_done = 0;
    ck(sdns_state_time(st.s, nullptr, &steps_done));
    copy_str(res.status, sizeof(res.status),
             diverged ? "diverged at step " + std::to_string(fail_step) : std::string("ok"));
    res.steps = diverged ? fail_step - 1 : steps_done;
    res.shells = h.shells;
    res.n_samples = static_cast<int64_t>(h.steps.size());
    const int w = 5 + h.shells;
    if (res.sample_steps && res.sample_rows)
      for (int64_t i = 0; i < res.n_samples && i < res.sample_cap; ++i) {
        res.sample_steps[i] = h.steps[static_cast<size_t>(i)];
        std::memcpy(res.sample_rows + i * w, h.rows.data() + i * w, sizeof(double) * w);
      }
    copy_str(res.csv_path, sizeof(res.csv_path), o.out_dir + "/diagnostics.csv");
    copy_str(res.checkpoint_path, sizeof(res.checkpoint_path), ckpt);
    copy_str(res.manifest_path, sizeof(res.manifest_path), o.out_dir + "/manifest.txt");
    write_diagnostics_csv(res.csv_path, h.steps.data(), h.rows.data(), res.n_samples, h.shells);
    write_manifest(res.manifest_path, cfg, icase, res);
    out = res;
  }
  if (diverged)
    throw Error(SDNS_DIVERGENCE_ERROR, div_msg + "; last good state (step " +
                                           std::to_string(ck_step) + ", t=" + fmt(ck_t) +
                                           ") checkpointed to " + ckpt);
}

// drive_workers (runner.cpp:151-190): one host thread per rank on one
// device; the first failure by rank is rethrown, and a non-collective
// failure poisons the group so the other ranks fail fast.
template <class Body>
void drive_workers(const sdns_config& cfg, const Opts& o, Body&& body) {
  const std::string backend = resolve_backend(cfg, o.backend);
  if (backend == "loopback") {
    sdns_comm* lb = nullptr;
    ck(sdns_comm_loopback(&lb));
    std::unique_ptr<sdns_comm, int (*)(sdns_comm*)> hold(lb, sdns_comm_destroy);
    body(0, lb);
    return;
  }
  std::vector<sdns_comm*> comms(static_cast<size_t>(cfg.p), nullptr);
  ck(sdns_comm_inprocess_group(cfg.p, o.device, o.timeout_s, comms.data()));
  std::vector<std::exception_ptr> errors(static_cast<size_t>(cfg.p));
  auto worker = [&](int rank) {
    try {
      body(rank, comms[static_cast<size_t>(rank)]);
    } catch (const Error& e) {
      errors[static_cast<size_t>(rank)] = std::current_exception();
      if (e.code != SDNS_DIVERGENCE_ERROR)  // divergence is collective by construction
        comms[static_cast<size_t>(rank)]->c->poison("rank " + std::to_string(rank) +
                                                     " failed: " + e.what());
    } catch (const std::exception& e) {
      errors[static_cast<size_t>(rank)] = std::current_exception();
      comms[static_cast<size_t>(rank)]->c->poison("rank " + std::to_string(rank) +
                                                   " failed: " + e.what());
    }
  };
  if (cfg.p == 1) {
    worker(0);
  } else {
    std::vector<std::thread> threads;
    for (int r = 0; r < cfg.p; ++r) threads.emplace_back(worker, r);
    for (auto& t : threads) t.join();
  }
  for (auto* c : comms) sdns_comm_destroy(c);
  for (auto& e : errors)
    if (e) std::rethrow_exception(e);
}

void run_all(const sdns_config& cfg, const std::string& icase, const Opts& o,
             sdns_run_result& res) {  // runner.cpp:197-213
  validate(cfg);
  validate_case(icase);
  std::filesystem::create_directories(o.out_dir);
  copy_str(res.backend, sizeof(res.backend), resolve_backend(cfg, o.backend));
  copy_str(res.status, sizeof(res.status), "ok");
  drive_workers(cfg, o, [&](int rank, sdns_comm* comm) {
    run_worker(cfg, icase, o, rank, comm, o.device, res);
  });
}

// bench_config + bench_entry_seconds (runner.cpp:301-373)
double bench_entry_seconds(const sdns_config& cfg, int steps, const Opts& o) {
  constexpr int kWarmup = 5;
  double sec = 0.0;
  std::mutex mu;
  drive_workers(cfg, o, [&](int rank, sdns_comm* comm) {
    Ctx ctx;
    ck(sdns_ctx_create_ex(&cfg, rank, o.device, comm, nullptr, &o.ctx, &ctx.c));
    Fld u_hat;
    ck(sdns_field_alloc(ctx.c, SDNS_SPECTRAL, 3, &u_hat.f));
    initial_state(ctx.c, cfg, "taylor_green", o.seed, u_hat.f);
    State st;
    ck(sdns_state_create(ctx.c, &st.s));
    ck(sdns_state_set(ctx.c, st.s, u_hat.f, 0.0, 0));
    // rk4_step + project, as the production loop (runner.cpp:356-359)
    const auto timed_step = [&] { ck(sdns_rk4_step(ctx.c, st.s, cfg.dt, 1, nullptr)); };
    for (int k = 0; k < kWarmup; ++k) timed_step();
    ck(sdns_ctx_sync(ctx.c));
    ck(sdns_comm_barrier(comm));
    const auto t0 = std::chrono::steady_clock::now();
    for (int k = 0; k < steps; ++k) timed_step();
    ck(sdns_ctx_sync(ctx.c));
    ck(sdns_comm_barrier(comm));
    const auto t1 = std::chrono::steady_clock::now();
    if (rank == 0) {
      std::lock_guard<std::mutex> lk(mu);
      sec = std::chrono::duration<double>(t1 - t0).count() / static_cast<double>(steps);
    }
  });
  return sec;
}

}  // namespace

extern "C" {

void sdns_config_defaults(sdns_config* cfg) {
  if (cfg) *cfg = config_defaults();
}

int sdns_parse_config_text(const char* text, const char* const* keys, const char* const* values,
                           int n_overrides, sdns_parsed_config* out) {
  return run_guarded([&] { parse_config(text ? text : "", keys, values, n_overrides, out); });
}

int sdns_parse_config_file(const char* path, const char* const* keys, const char* const* values,
                           int n_overrides, sdns_parsed_config* out) {
  return run_guarded([&] {
    const std::string text = read_file(path ? path : "", "config file");
    parse_config(text, keys, values, n_overrides, out);
  });
}

int sdns_default_pencil_grid(int n, int p, int* p1, int* p2) {
  return run_guarded([&] {
    const auto g = default_pencil_grid(n, p);
    *p1 = g.first;
    *p2 = g.second;
  });
}

int sdns_run(const sdns_config* cfg, const char* initial_case, const sdns_run_options* opts,
             sdns_run_result* out) {
  return run_guarded([&] {
    run_all(*cfg, initial_case ? initial_case : "taylor_green", read_opts(opts), *out);
  });
}

int sdns_run_rank(const sdns_config* cfg, const char* initial_case, const sdns_run_options* opts,
                  int rank, sdns_comm* comm, sdns_run_result* out) {
  return run_guarded([&] {
    const Opts o = read_opts(opts);
    const std::string icase = initial_case ? initial_case : "taylor_green";
    validate(*cfg);
    validate_case(icase);
    if (rank == 0) std::filesystem::create_directories(o.out_dir);
    comm->c->set_timeout(o.timeout_s);  // RunOptions::collective_timeout
    ck(sdns_comm_barrier(comm));
    copy_str(out->backend, sizeof(out->backend), comm->c->kind());
    copy_str(out->status, sizeof(out->status), "ok");
    run_worker(*cfg, icase, o, rank, comm, o.device, *out);
  });
}

int sdns_parse_bench_matrix_text(const char* text, sdns_bench_entry* out, int cap, int* count) {
  return run_guarded([&] { put_entries(parse_bench_matrix(text ? text : ""), out, cap, count); });
}

int sdns_parse_bench_matrix_file(const char* path, sdns_bench_entry* out, int cap, int* count) {
  return run_guarded([&] {
    put_entries(parse_bench_matrix(read_file(path ? path : "", "bench matrix")), out, cap, count);
  });
}

int sdns_bench(const sdns_bench_entry* entries, int count, int steps,
               const sdns_run_options* opts, sdns_bench_row* rows) {
  return run_guarded([&] {  // runner.cpp:375-397
    if (steps < 1) config_error("bench steps must be >= 1");
    const Opts o = read_opts(opts);
    for (int i = 0; i < count; ++i) {
      sdns_bench_row& row = rows[i];
      row = sdns_bench_row{};
      row.entry = entries[i];
      copy_str(row.status, sizeof(row.status), "ok");
      try {
        sdns_config cfg = config_defaults();
        const sdns_bench_entry& e = entries[i];
        cfg.n = e.n;
        cfg.decomp = e.decomp;
        cfg.p = e.p;
        if (e.decomp == SDNS_PENCIL) {
          if (e.p1 > 0 && e.p2 > 0) {
            cfg.p1 = e.p1;
            cfg.p2 = e.p2;
          } else {
            std::tie(cfg.p1, cfg.p2) = default_pencil_grid(e.n, e.p);
          }
        }
        validate(cfg);
        row.entry.p1 = cfg.p1;
        row.entry.p2 = cfg.p2;
        row.nodes_per_rank = static_cast<int64_t>(cfg.n) * cfg.n * cfg.n / cfg.p;
        row.sec_per_step = bench_entry_seconds(cfg, steps, o);
      } catch (const std::exception& ex) {
        copy_str(row.status, sizeof(row.status), ex.what());
      }
    }
  });
}

int sdns_write_bench_csv(const char* path, const sdns_bench_row* rows, int count) {
  return run_guarded([&] { write_bench_csv(path ? path : "", rows, count); });
}

int sdns_write_diagnostics_csv(const char* path, const int64_t* steps, const double* rows,
                               int64_t nrows, int shells) {
  return run_guarded([&] { write_diagnostics_csv(path ? path : "", steps, rows, nrows, shells); });
}

int sdns_write_manifest(const char* path, const sdns_config* cfg, const char* initial_case,
                        const sdns_run_result* result) {
  return run_guarded([&] {
    write_manifest(path ? path : "", *cfg, initial_case ? initial_case : "", *result);
  });
}

}  // extern "C"
