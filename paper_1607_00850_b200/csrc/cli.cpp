// sdns_cuda: command-line front end over the C ABI, a drop-in for the
// reference CLI (proj/tools/sdns.cpp:1-162): `run` a configured case,
// `bench` a scaling matrix, `verify` the acceptance criteria. Same
// subcommands, flags, console lines and exit codes (0 ok, 1 error,
// 2 divergence); the solver behind them is the device pipeline. Two flags
// are added: --device (CUDA device of the ranks) and --seed (case
// `isotropic`).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>
#include <utility>
#include <vector>

#include "../../include/sdns_cuda.h"

namespace {

struct Fail {
  int code;
  std::string msg;
};

void ck(int rc) {
  if (rc != SDNS_OK) throw Fail{rc, sdns_last_error()};
}

const char* decomp_name(int d) { return d == SDNS_PENCIL ? "pencil" : "slab"; }

// --flag VALUE or --flag=VALUE
struct Args {
  std::vector<std::string> v;
  size_t i = 0;
  bool next(std::string& flag, std::string& value, bool& has_value) {
    if (i >= v.size()) return false;
    flag = v[i++];
    has_value = false;
    const auto eq = flag.find('=');
    if (flag.rfind("--", 0) == 0 && eq != std::string::npos) {
      value = flag.substr(eq + 1);
      flag = flag.substr(0, eq);
      has_value = true;
    }
    return true;
  }
  std::string take(const std::string& flag, std::string& value, bool has_value) {
    if (has_value) return value;
    if (i >= v.size()) throw Fail{106, flag + " requires an argument"};
    return v[i++];
  }
};

int usage(int rc) {
  std::cout << "pseudo-spectral Navier-Stokes solver (Taylor-Green case), B200 pipeline\n"
               "Usage: sdns_cuda [--version] SUBCOMMAND\n"
               "  run     advance a configured case  [--config F] [--n V] [--p V] [--p1 V]\n"
               "          [--p2 V] [--decomp slab|pencil] [--re V] [--nu V] [--dt V] [--t-end V]\n"
               "          [--dealias V] [--case NAME] [--out-every V] [--backend B] [--out DIR]\n"
               "          [--device D] [--seed S]\n"
               "  bench   time a weak/strong scaling matrix  --matrix F [--steps K] [--out CSV]\n"
               "  verify  run the acceptance property suite\n";
  return rc;
}

int cmd_run(Args& a) {  // sdns.cpp:36-66
  std::string config_path, out_dir = "out", backend = "auto";
  int device = 0;
  uint64_t seed = 1607;
  std::vector<std::pair<std::string, std::string>> overrides;
  static const std::pair<const char*, const char*> kOverride[] = {
      {"--n", "n"},     {"--p", "p"},           {"--p1", "p1"},       {"--p2", "p2"},
      {"--decomp", "decomp"}, {"--re", "re"},   {"--nu", "nu"},       {"--dt", "dt"},
      {"--t-end", "t_end"}, {"--dealias", "dealias"}, {"--case", "case"},
      {"--out-every", "out_every"}};
  std::string flag, value;
  bool hv = false;
  while (a.next(flag, value, hv)) {
    bool done = false;
    for (const auto& [f, key] : kOverride)
      if (flag == f) {
        overrides.emplace_back(key, a.take(flag, value, hv));
        done = true;
      }
    if (done) continue;
    if (flag == "--config") config_path = a.take(flag, value, hv);
    else if (flag == "--out") out_dir = a.take(flag, value, hv);
    else if (flag == "--backend") backend = a.take(flag, value, hv);
    else if (flag == "--device") device = std::atoi(a.take(flag, value, hv).c_str());
    else if (flag == "--seed") seed = std::strtoull(a.take(flag, value, hv).c_str(), nullptr, 10);
    else throw Fail{109, "The following argument was not expected: " + flag};
  }
  std::vector<const char*> keys, values;
  for (const auto& kv : overrides) {
    keys.push_back(kv.first.c_str());
    values.push_back(kv.second.c_str());
  }
  sdns_parsed_config parsed{};
  if (config_path.empty())
    ck(sdns_parse_config_text("", keys.data(), values.data(), static_cast<int>(keys.size()),
                              &parsed));
  else
    ck(sdns_parse_config_file(config_path.c_str(), keys.data(), values.data(),
                              static_cast<int>(keys.size()), &parsed));
  std::string notices = parsed.notices;
  for (size_t s = 0, e; (e = notices.find('\n', s)) != std::string::npos; s = e + 1)
    std::cout << "note: " << notices.substr(s, e - s) << "\n";

  const sdns_config& cfg = parsed.cfg;
  std::cout << "running " << parsed.initial_case << ": n=" << cfg.n << " "
            << decomp_name(cfg.decomp) << " p=" << cfg.p << " nu=" << cfg.nu
            << " dt=" << cfg.dt << " t_end=" << cfg.t_end << "\n";

  const int shells = sdns_spectrum_shells(cfg.n);
  const int64_t cap = sdns_step_count(cfg.t_end, cfg.dt) / cfg.out_every + 2;
  std::vector<int64_t> steps(static_cast<size_t>(cap));
  std::vector<double> rows(static_cast<size_t>(cap * (5 + shells)));
  sdns_run_options opts{out_dir.c_str(), backend.c_str(), 30.0, device, seed, {}};
  sdns_run_result r{};
  r.sample_cap = cap;
  r.sample_steps = steps.data();
  r.sample_rows = rows.data();
  ck(sdns_run(&cfg, parsed.initial_case, &opts, &r));

  const double* last = rows.data() + (r.n_samples - 1) * (5 + shells);
  std::cout << "completed " << r.steps << " steps; E=" << last[1] << " Z=" << last[2]
            << " div_max=" << last[4] << "\n"
            << "mean step time " << r.step_mean_s << " s over " << r.timed_steps
            << " timed steps\n"
            << "wrote " << r.csv_path << ", " << r.checkpoint_path << ", " << r.manifest_path
            << "\n";
  return 0;
}

int cmd_bench(Args& a) {  // sdns.cpp:68-92
  std::string matrix, out_csv = "bench.csv";
  int steps = 10;
  int device = 0;
  std::string flag, value;
  bool hv = false;
  while (a.next(flag, value, hv)) {
    if (flag == "--matrix") matrix = a.take(flag, value, hv);
    else if (flag == "--steps") {
      steps = std::atoi(a.take(flag, value, hv).c_str());
      if (steps <= 0) throw Fail{105, "--steps: Value must be a positive number"};
    } else if (flag == "--out") out_csv = a.take(flag, value, hv);
    else if (flag == "--device") device = std::atoi(a.take(flag, value, hv).c_str());
    else throw Fail{109, "The following argument was not expected: " + flag};
  }
  if (matrix.empty()) throw Fail{106, "--matrix is required"};
  int count = 0;
  ck(sdns_parse_bench_matrix_file(matrix.c_str(), nullptr, 0, &count));
  std::vector<sdns_bench_entry> entries(static_cast<size_t>(count));
  ck(sdns_parse_bench_matrix_file(matrix.c_str(), entries.data(), count, &count));
  std::cout << "benchmarking " << entries.size() << " entries, " << steps
            << " timed steps each\n";
  std::vector<sdns_bench_row> rows(entries.size());
  sdns_run_options opts{"out", "auto", 30.0, device, 1607, {}};
  ck(sdns_bench(entries.data(), count, steps, &opts, rows.data()));
  ck(sdns_write_bench_csv(out_csv.c_str(), rows.data(), count));
  bool all_ok = true;
  for (const sdns_bench_row& r : rows) {
    std::cout << "  n=" << r.entry.n << " " << decomp_name(r.entry.decomp) << " p=" << r.entry.p;
    if (std::strcmp(r.status, "ok") == 0)
      std::cout << ": " << r.sec_per_step << " s/step\n";
    else
      std::cout << ": FAILED (" << r.status << ")\n";
    all_ok = all_ok && std::strcmp(r.status, "ok") == 0;
  }
  std::cout << "wrote " << out_csv << "\n";
  return all_ok ? 0 : 1;
}

int cmd_verify(Args& a) {  // sdns.cpp:94-100
  int device = 0;
  std::string flag, value;
  bool hv = false;
  while (a.next(flag, value, hv)) {
    if (flag == "--device") device = std::atoi(a.take(flag, value, hv).c_str());
    else throw Fail{109, "The following argument was not expected: " + flag};
  }
  std::cout << "sdns acceptance suite (" << sdns_version() << ")\n";
  int passed = 0;
  ck(sdns_acceptance_suite(device, 1, nullptr, &passed));
  std::cout << (passed ? "ALL CRITERIA PASSED" : "FAILURES PRESENT") << "\n";
  return passed ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  for (int i = 1; i < argc; ++i) a.v.emplace_back(argv[i]);
  if (a.v.empty()) {
    std::cerr << "A subcommand is required\n";
    return usage(106);
  }
  const std::string sub = a.v[a.i++];
  try {
    if (sub == "--version") {
      std::cout << sdns_version() << "\n";
      return 0;
    }
    if (sub == "-h" || sub == "--help") return usage(0);
    if (sub == "run") return cmd_run(a);
    if (sub == "bench") return cmd_bench(a);
    if (sub == "verify") return cmd_verify(a);
    std::cerr << "The following argument was not expected: " << sub << "\n";
    return usage(109);
  } catch (const Fail& f) {
    if (f.code == SDNS_DIVERGENCE_ERROR) {
      std::cerr << "error: solution diverged: " << f.msg << "\n";
      return 2;
    }
    if (f.code > 100) {  // argument errors, as CLI11 reports them
      std::cerr << f.msg << "\n";
      return f.code;
    }
    std::cerr << "error: " << f.msg << "\n";
    return 1;
  }
}
