// The reference-side binding a maintainer adds to proj/core (INTEGRATION.md
// §2): run_worker's step loop (proj/core/src/runner.cpp:67-111) on the B200
// path through the C ABI of include/sdns_cuda.h. Compiled by
// tests/test_integration_cpu.py against the reference's own headers
// (/root/reference/proj/core/include) and linked against libsdns_cuda.so, so
// the snippet cannot drift from either interface.
#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>

#include "sdns/diagnostics.hpp"
#include "sdns/layout.hpp"
#include "sdns/mesh.hpp"
#include "sdns/navier_stokes.hpp"
#include "sdns/types.hpp"
#include "sdns_cuda.h"

namespace sdns_gpu {

// status -> the reference's exception types (types.hpp:28-62)
inline void check(int rc) {
  if (rc == SDNS_OK) return;
  const std::string m = sdns_last_error();
  switch (rc) {
    case SDNS_CONFIG_ERROR: throw sdns::ConfigError(m);
    case SDNS_PROTOCOL_ERROR: throw sdns::ProtocolError(m);
    case SDNS_TIMEOUT_ERROR: throw sdns::TimeoutError(m);
    case SDNS_DIVERGENCE_ERROR: throw sdns::DivergenceError(0, m);
    case SDNS_IO_ERROR: throw sdns::IoError(m);
    default: throw std::runtime_error(m);
  }
}

struct Hook {
  sdns_ctx* ctx;
  sdns_state* st;
  double nu;
  int shells;
  std::vector<sdns::FlowStats>* out;
};

// AdvanceHooks::sample (rk4.hpp:45-55): collect_stats of the device state.
inline void sample(int64_t, double t, void* user) {
  auto* h = static_cast<Hook*>(user);
  std::vector<double> row(static_cast<size_t>(5 + h->shells));
  check(sdns_collect_stats(h->ctx, sdns_state_u_hat(h->st), h->nu, t, row.data()));
  sdns::FlowStats s;
  s.t = row[0];
  s.energy = row[1];
  s.enstrophy = row[2];
  s.dissipation = row[3];
  s.divergence_max = row[4];
  s.spectrum.assign(row.begin() + 5, row.end());
  h->out->push_back(std::move(s));
}

// One rank of run_worker on its GPU; nccl_id: created by rank 0
// (sdns_comm_nccl_unique_id) and distributed by the caller.
std::vector<sdns::FlowStats> run_worker_gpu(const sdns::SolverConfig& cfg, int rank, int device,
                                            const unsigned char nccl_id[128],
                                            const std::string& checkpoint_path) {
  sdns_config c{cfg.n, cfg.decomp == sdns::Decomp::Slab ? SDNS_SLAB : SDNS_PENCIL,
                cfg.p, cfg.p1, cfg.p2, cfg.nu, cfg.dt, cfg.t_end, cfg.dealias ? 1 : 0,
                cfg.out_every};
  sdns_comm* comm = nullptr;
  check(cfg.p == 1 ? sdns_comm_loopback(&comm)
                   : sdns_comm_nccl_init(nccl_id, cfg.p, rank, device, &comm));
  check(sdns_comm_set_timeout(comm, 30.0));  // RunOptions::collective_timeout
  sdns_ctx* ctx = nullptr;  // DistributedFFT + WavenumberMesh + RhsWorkspace
  check(sdns_ctx_create(&c, rank, device, comm, /*stream=*/nullptr, &ctx));

  // initial condition exactly like runner.cpp:77-82: forward + project
  const sdns::RankLayout lo = sdns::build_layout(cfg, rank);
  sdns::RealField3 u0 =
      sdns::make_initial_condition(cfg.initial_case, lo, sdns::physical_mesh(lo));
  const size_t comp = static_cast<size_t>(lo.real.shape.size());
  std::vector<double> host(3 * comp);
  for (int q = 0; q < 3; ++q)
    std::copy(u0[q].data.begin(), u0[q].data.end(), host.begin() + static_cast<long>(q * comp));
  sdns_field *ur = nullptr, *uh = nullptr;
  check(sdns_field_alloc(ctx, SDNS_REAL, 3, &ur));
  check(sdns_field_alloc(ctx, SDNS_SPECTRAL, 3, &uh));
  check(sdns_field_upload(ctx, ur, host.data()));
  check(sdns_fft_forward(ctx, ur, uh));
  check(sdns_project(ctx, uh));

  sdns_state* st = nullptr;  // Rk4State
  check(sdns_state_create(ctx, &st));
  check(sdns_state_set(ctx, st, uh, 0.0, 0));

  sdns_layout dl{};
  check(sdns_ctx_layout(ctx, &dl));
  std::vector<sdns::FlowStats> samples;
  Hook hk{ctx, st, cfg.nu, sdns_spectrum_shells(dl.n), &samples};
  int64_t fail_step = 0;
  const int rc = sdns_advance(ctx, st, sample, &hk, &fail_step);  // rk4.cpp:86-107
  if (rc == SDNS_DIVERGENCE_ERROR) throw sdns::DivergenceError(fail_step, sdns_last_error());
  check(rc);
  // final checkpoint in the reference's format (checkpoint.cpp:64-113):
  // inverse transform on the device, then the collective gather-and-write
  check(sdns_fft_inverse(ctx, sdns_state_u_hat(st), ur));
  check(sdns_checkpoint_write(ctx, ur, checkpoint_path.c_str(), cfg.t_end,
                              sdns_step_count(cfg.t_end, cfg.dt)));
  sdns_state_destroy(st);
  sdns_field_free(ur);
  sdns_field_free(uh);
  sdns_ctx_destroy(ctx);
  sdns_comm_destroy(comm);
  return samples;
}

}  // namespace sdns_gpu
