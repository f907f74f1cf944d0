// Decomposition setup: SolverConfig::validate (proj/core/src/config.cpp:17-50),
// block rule and build_layout (proj/core/src/layout.cpp:7-76), step_count
// (proj/core/src/rk4.cpp:79-84), spectrum_shells (diagnostics.cpp:66-69).
// Host-only; needs no device.
#include <algorithm>
#include <cmath>

#include "host.h"

namespace sdns_host {

int64_t block_size(int64_t total, int parts, int index) {
  const int64_t base = total / parts;
  return base + (index < total % parts ? 1 : 0);
}

int64_t block_start(int64_t total, int parts, int index) {
  const int64_t base = total / parts;
  return index * base + std::min<int64_t>(index, total % parts);
}

void validate(const sdns_config& c) {
  const auto s = [](auto v) { return std::to_string(v); };
  if (c.n < 4) config_error("n must be >= 4, got " + s(c.n));
  if (c.n % 2 != 0) config_error("n must be even, got " + s(c.n));
  if (c.p < 1) config_error("p must be >= 1, got " + s(c.p));
  if (c.decomp == SDNS_SLAB) {
    if (c.p > c.n) config_error("slab requires p <= n, got p=" + s(c.p) + " n=" + s(c.n));
    if (c.n % c.p != 0)
      config_error("slab requires p to divide n, got p=" + s(c.p) + " n=" + s(c.n));
  } else if (c.decomp == SDNS_PENCIL) {
    if (c.p1 < 1 || c.p2 < 1) config_error("pencil requires p1 >= 1 and p2 >= 1");
    if (c.p != c.p1 * c.p2)
      config_error("pencil requires p = p1*p2, got p=" + s(c.p) + " p1=" + s(c.p1) +
                   " p2=" + s(c.p2));
    if (c.n % c.p1 != 0)
      config_error("pencil requires p1 to divide n, got p1=" + s(c.p1) + " n=" + s(c.n));
    if (c.n % c.p2 != 0)
      config_error("pencil requires p2 to divide n, got p2=" + s(c.p2) + " n=" + s(c.n));
    if (c.p2 > c.n / 2)
      config_error("pencil requires p2 <= n/2, got p2=" + s(c.p2) + " n=" + s(c.n));
  } else {
    config_error("unknown decomposition " + s(c.decomp) + " (expected slab|pencil)");
  }
  if (c.nu < 0.0) config_error("nu must be >= 0");
  if (!(c.dt > 0.0)) config_error("dt must be > 0");
  if (c.t_end < 0.0) config_error("t_end must be >= 0");
  if (c.out_every < 1) config_error("out_every must be >= 1");
}

sdns_layout build_layout(const sdns_config& cfg, int rank) {
  validate(cfg);
  if (rank < 0 || rank >= cfg.p)
    config_error("rank " + std::to_string(rank) + " out of range for p=" + std::to_string(cfg.p));
  sdns_layout lo{};
  lo.rank = rank;
  lo.p = cfg.p;
  lo.n = cfg.n;
  lo.nf = cfg.n / 2 + 1;
  const int64_t n = cfg.n;
  if (cfg.decomp == SDNS_SLAB) {
    if (cfg.p > SDNS_MAX_PEERS) config_error("p exceeds SDNS_MAX_PEERS");
    lo.p1 = cfg.p;
    lo.p2 = 1;
    lo.coord1 = rank;
    lo.coord2 = 0;
    const int64_t np = n / cfg.p;
    const int64_t rs[3] = {np, n, n}, ro[3] = {rank * np, 0, 0};
    const int64_t ss[3] = {n, np, lo.nf}, so[3] = {0, rank * np, 0};
    for (int i = 0; i < 3; ++i) {
      lo.real_shape[i] = rs[i];
      lo.real_offset[i] = ro[i];
      lo.spec_shape[i] = ss[i];
      lo.spec_offset[i] = so[i];
    }
    lo.nstages = 1;
    lo.stage_peers[0] = cfg.p;
    for (int q = 0; q < cfg.p; ++q) {
      lo.send_counts[0][q] = np * np * lo.nf;
      lo.recv_counts[0][q] = np * np * lo.nf;
    }
  } else {
    if (cfg.p1 > SDNS_MAX_PEERS || cfg.p2 > SDNS_MAX_PEERS) config_error("p1/p2 exceed SDNS_MAX_PEERS");
    lo.p1 = cfg.p1;
    lo.p2 = cfg.p2;
    lo.coord1 = rank / cfg.p2;
    lo.coord2 = rank % cfg.p2;
    const int64_t xl = n / cfg.p1, yl = n / cfg.p2, yl2 = n / cfg.p1;
    const int64_t b = block_size(lo.nf, cfg.p2, lo.coord2);
    const int64_t rs[3] = {xl, yl, n}, ro[3] = {lo.coord1 * xl, lo.coord2 * yl, 0};
    const int64_t ss[3] = {n, yl2, b};
    const int64_t so[3] = {0, lo.coord1 * yl2, block_start(lo.nf, cfg.p2, lo.coord2)};
    for (int i = 0; i < 3; ++i) {
      lo.real_shape[i] = rs[i];
      lo.real_offset[i] = ro[i];
      lo.spec_shape[i] = ss[i];
      lo.spec_offset[i] = so[i];
    }
    lo.nstages = 2;
    lo.stage_peers[0] = cfg.p2;
    lo.stage_peers[1] = cfg.p1;
    for (int q = 0; q < cfg.p2; ++q) {
      lo.send_counts[0][q] = xl * yl * block_size(lo.nf, cfg.p2, q);
      lo.recv_counts[0][q] = xl * yl * b;
    }
    for (int s = 0; s < cfg.p1; ++s) {
      lo.send_counts[1][s] = xl * yl2 * b;
      lo.recv_counts[1][s] = xl * yl2 * b;
    }
  }
  return lo;
}

int64_t step_count(double t_end, double dt) {
  if (t_end <= 0.0) return 0;
  const double q = t_end / dt;
  const auto n = static_cast<int64_t>(std::ceil(q - 1e-9));
  return n < 0 ? 0 : n;
}

int spectrum_shells(int64_t n) {
  const double half = static_cast<double>(n / 2);
  return static_cast<int>(std::llround(std::sqrt(3.0 * half * half))) + 1;
}

}  // namespace sdns_host
