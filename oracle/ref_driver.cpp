// TEST INFRASTRUCTURE (oracle only) — a small extern "C" driver over the
// UNMODIFIED reference library (proj/core, compiled from /root/reference by
// oracle/Makefile against oracle/fftw_shim). It uses only the reference's
// public API, exactly as its own run_worker / bench / verification code does:
//   build_layout            proj/core/include/sdns/layout.hpp:48
//   wavenumbers             proj/core/include/sdns/mesh.hpp:36
//   DistributedFFT          proj/core/include/sdns/fft.hpp:26-62
//   compute_rhs / project   proj/core/include/sdns/navier_stokes.hpp:17-49
//   Rk4State / advance      proj/core/include/sdns/rk4.hpp:18-62
//   collect_stats           proj/core/include/sdns/diagnostics.hpp:36-38
//   run_group               proj/core/include/sdns/transport.hpp:103-106
//   bench                   proj/core/include/sdns/runner.hpp:73-74
//   run / write_*_csv / write_manifest   runner.hpp:44-82
//   parse_config_text       proj/core/include/sdns/config_file.hpp:24-26
// Global arrays passed across this ABI are row-major: spectral (n, n, n/2+1)
// complex as interleaved doubles, real (n, n, n); vector fields are three
// such arrays back to back (component-major).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <cmath>
#include <vector>

#include "sdns/checkpoint.hpp"
#include "sdns/config_file.hpp"
#include "sdns/diagnostics.hpp"
#include "sdns/fft.hpp"
#include "sdns/layout.hpp"
#include "sdns/mesh.hpp"
#include "sdns/navier_stokes.hpp"
#include "sdns/rk4.hpp"
#include "sdns/runner.hpp"
#include "sdns/transport.hpp"

using namespace sdns;

namespace {

thread_local std::string g_err;

SolverConfig make_cfg(int n, int decomp, int p, int p1, int p2, double nu,
                      double dt, double t_end, int dealias, int out_every) {
  SolverConfig cfg;
  cfg.n = n;
  cfg.decomp = decomp == 0 ? Decomp::Slab : Decomp::Pencil;
  cfg.p = p;
  cfg.p1 = decomp == 0 ? 1 : p1;
  cfg.p2 = decomp == 0 ? 1 : p2;
  cfg.nu = nu;
  cfg.dt = dt;
  cfg.t_end = t_end;
  cfg.dealias = dealias != 0;
  cfg.out_every = out_every < 1 ? 1 : out_every;
  cfg.validate();
  return cfg;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const ProtocolError& e) {
    g_err = e.what();
    return 2;
  } catch (const TimeoutError& e) {
    g_err = e.what();
    return 3;
  } catch (const DivergenceError& e) {
    g_err = e.what();
    return 4;
  } catch (const IoError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

void group(int p, const std::function<void(int, std::shared_ptr<Communicator>)>& body) {
  if (p == 1) {
    body(0, make_loopback());
  } else {
    run_group(p, body, std::chrono::seconds(600));
  }
}

std::int64_t spec_index(std::int64_t n, std::int64_t nf, const Extents3& ex,
                        std::int64_t i, std::int64_t j, std::int64_t k) {
  return ((ex.offset[0] + i) * n + (ex.offset[1] + j)) * nf + (ex.offset[2] + k);
}

void scatter_spec(const double* g, std::int64_t n, const Extents3& ex,
                  SpectralField3& f) {
  const std::int64_t nf = n / 2 + 1;
  const std::int64_t gsz = n * n * nf;
  for (int c = 0; c < 3; ++c)
    for (std::int64_t i = 0; i < ex.shape.n0; ++i)
      for (std::int64_t j = 0; j < ex.shape.n1; ++j)
        for (std::int64_t k = 0; k < ex.shape.n2; ++k) {
          const std::int64_t m = c * gsz + spec_index(n, nf, ex, i, j, k);
          f[c](i, j, k) = Complex(g[2 * m], g[2 * m + 1]);
        }
}

void gather_spec(const SpectralField3& f, std::int64_t n, const Extents3& ex,
                 double* g) {
  const std::int64_t nf = n / 2 + 1;
  const std::int64_t gsz = n * n * nf;
  for (int c = 0; c < 3; ++c)
    for (std::int64_t i = 0; i < ex.shape.n0; ++i)
      for (std::int64_t j = 0; j < ex.shape.n1; ++j)
        for (std::int64_t k = 0; k < ex.shape.n2; ++k) {
          const std::int64_t m = c * gsz + spec_index(n, nf, ex, i, j, k);
          const Complex v = f[c](i, j, k);
          g[2 * m] = v.real();
          g[2 * m + 1] = v.imag();
        }
}

void scatter_real(const double* g, std::int64_t n, const Extents3& ex,
                  RealField3& f) {
  const std::int64_t gsz = n * n * n;
  for (int c = 0; c < 3; ++c)
    for (std::int64_t i = 0; i < ex.shape.n0; ++i)
      for (std::int64_t j = 0; j < ex.shape.n1; ++j)
        for (std::int64_t k = 0; k < ex.shape.n2; ++k)
          f[c](i, j, k) = g[c * gsz + ((ex.offset[0] + i) * n + ex.offset[1] + j) * n +
                            ex.offset[2] + k];
}

void gather_real(const RealField3& f, std::int64_t n, const Extents3& ex,
                 double* g) {
  const std::int64_t gsz = n * n * n;
  for (int c = 0; c < 3; ++c)
    for (std::int64_t i = 0; i < ex.shape.n0; ++i)
      for (std::int64_t j = 0; j < ex.shape.n1; ++j)
        for (std::int64_t k = 0; k < ex.shape.n2; ++k)
          g[c * gsz + ((ex.offset[0] + i) * n + ex.offset[1] + j) * n + ex.offset[2] + k] =
              f[c](i, j, k);
}

// stats row: t, E, Z, eps, div_max, then `shells` spectrum values
void put_stats(const FlowStats& s, double* row) {
  row[0] = s.t;
  row[1] = s.energy;
  row[2] = s.enstrophy;
  row[3] = s.dissipation;
  row[4] = s.divergence_max;
  for (std::size_t i = 0; i < s.spectrum.size(); ++i) row[5 + i] = s.spectrum[i];
}

}  // namespace

extern "C" {

const char* sdns_ref_last_error() { return g_err.c_str(); }

int sdns_ref_spectrum_shells(int n) { return spectrum_shells(n); }

/// Distributed forward transform of a global 3-component real field.
int sdns_ref_forward(int n, int decomp, int p, int p1, int p2, const double* u,
                     double* uhat) {
  return guarded([&] {
    const SolverConfig cfg = make_cfg(n, decomp, p, p1, p2, 0.0, 1.0, 0.0, 1, 1);
    std::mutex mu;
    group(p, [&](int rank, std::shared_ptr<Communicator> comm) {
      const RankLayout lo = build_layout(cfg, rank);
      DistributedFFT fft(cfg, lo, comm);
      RealField3 f(lo.real.shape);
      scatter_real(u, n, lo.real, f);
      SpectralField3 fu(lo.spec.shape);
      fft.forward(f, fu);
      std::lock_guard lk(mu);
      gather_spec(fu, n, lo.spec, uhat);
    });
  });
}

/// Distributed inverse transform (normalised) of a global spectral field.
int sdns_ref_inverse(int n, int decomp, int p, int p1, int p2,
                     const double* uhat, double* u) {
  return guarded([&] {
    const SolverConfig cfg = make_cfg(n, decomp, p, p1, p2, 0.0, 1.0, 0.0, 1, 1);
    std::mutex mu;
    group(p, [&](int rank, std::shared_ptr<Communicator> comm) {
      const RankLayout lo = build_layout(cfg, rank);
      DistributedFFT fft(cfg, lo, comm);
      SpectralField3 fu(lo.spec.shape);
      scatter_spec(uhat, n, lo.spec, fu);
      RealField3 f(lo.real.shape);
      fft.inverse(fu, f);
      std::lock_guard lk(mu);
      gather_real(f, n, lo.real, u);
    });
  });
}

/// Distributed forward transform of `ncomp` global real components through
/// the SCALAR overload DistributedFFT::forward(const RealField&, SpectralField&)
/// (proj/core/src/fft.cpp:59-63), one component at a time; needs only one
/// component's worth of reference buffers (used for the 1024^3 pins).
int sdns_ref_forward_scalar(int n, int decomp, int p, int p1, int p2, int ncomp,
                            const double* u, double* uhat) {
  return guarded([&] {
    const SolverConfig cfg = make_cfg(n, decomp, p, p1, p2, 0.0, 1.0, 0.0, 1, 1);
    const std::int64_t nn = n, nf = n / 2 + 1;
    group(p, [&](int rank, std::shared_ptr<Communicator> comm) {
      const RankLayout lo = build_layout(cfg, rank);
      DistributedFFT fft(cfg, lo, comm);
      const Extents3& rx = lo.real;
      const Extents3& sx = lo.spec;
      RealField f(rx.shape);
      SpectralField fu(sx.shape);
      for (int c = 0; c < ncomp; ++c) {
        const double* g = u + c * nn * nn * nn;
        for (std::int64_t i = 0; i < rx.shape.n0; ++i)
          for (std::int64_t j = 0; j < rx.shape.n1; ++j)
            for (std::int64_t k = 0; k < rx.shape.n2; ++k)
              f(i, j, k) = g[((rx.offset[0] + i) * nn + rx.offset[1] + j) * nn + rx.offset[2] + k];
        fft.forward(f, fu);
        double* o = uhat + 2 * c * nn * nn * nf;
        for (std::int64_t i = 0; i < sx.shape.n0; ++i)
          for (std::int64_t j = 0; j < sx.shape.n1; ++j)
            for (std::int64_t k = 0; k < sx.shape.n2; ++k) {
              const std::int64_t m = spec_index(nn, nf, sx, i, j, k);
              o[2 * m] = fu(i, j, k).real();
              o[2 * m + 1] = fu(i, j, k).imag();
            }
      }
    });
  });
}

/// Normalised inverse of `ncomp` global spectral components through the
/// scalar overload DistributedFFT::inverse (proj/core/src/fft.cpp:65-69).
int sdns_ref_inverse_scalar(int n, int decomp, int p, int p1, int p2, int ncomp,
                            const double* uhat, double* u) {
  return guarded([&] {
    const SolverConfig cfg = make_cfg(n, decomp, p, p1, p2, 0.0, 1.0, 0.0, 1, 1);
    const std::int64_t nn = n, nf = n / 2 + 1;
    group(p, [&](int rank, std::shared_ptr<Communicator> comm) {
      const RankLayout lo = build_layout(cfg, rank);
      DistributedFFT fft(cfg, lo, comm);
      const Extents3& rx = lo.real;
      const Extents3& sx = lo.spec;
      RealField f(rx.shape);
      SpectralField fu(sx.shape);
      for (int c = 0; c < ncomp; ++c) {
        const double* g = uhat + 2 * c * nn * nn * nf;
        for (std::int64_t i = 0; i < sx.shape.n0; ++i)
          for (std::int64_t j = 0; j < sx.shape.n1; ++j)
            for (std::int64_t k = 0; k < sx.shape.n2; ++k) {
              const std::int64_t m = spec_index(nn, nf, sx, i, j, k);
              fu(i, j, k) = Complex(g[2 * m], g[2 * m + 1]);
            }
        fft.inverse(fu, f);
        double* o = u + c * nn * nn * nn;
        for (std::int64_t i = 0; i < rx.shape.n0; ++i)
          for (std::int64_t j = 0; j < rx.shape.n1; ++j)
            for (std::int64_t k = 0; k < rx.shape.n2; ++k)
              o[((rx.offset[0] + i) * nn + rx.offset[1] + j) * nn + rx.offset[2] + k] = f(i, j, k);
      }
    });
  });
}

/// Oracle restatement of the seeded isotropic initial field (BASELINE
/// configs 2-4), GLOBAL array (3, n, n, n/2+1).
/// The reference has no such case, so the construction is restated here from
/// the survey's recipe, independently of the product's csrc/iso_init.cpp, and
/// a CPU test pins the two bit for bit: counter-based Box-Muller Gaussians
/// keyed by (seed, component, global index), E(k) = k^4 exp(-2 (k/k0)^2)
/// amplitudes, zero DC / Nyquist, Hermitian kz = 0 plane (the lexicographically
/// smaller of (i, j) and (-i, -j) is drawn, the other is its conjugate), the
/// reference project() per mode (navier_stokes.cpp:85-102), energy scaled to
/// `energy` with the Hermitian weights (diagnostics.cpp:41-48), per-x-plane
/// sums added in x order.
int sdns_ref_iso_init(int n, unsigned long long seed, double k0, double energy,
                      double* out) {
  return guarded([&] {
    const std::int64_t N = n, nf = n / 2 + 1, h = n / 2;
    auto mix = [](std::uint64_t x) {
      x += 0x9E3779B97F4A7C15ULL;
      x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
      x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
      return x ^ (x >> 31);
    };
    auto kw = [&](std::int64_t j) { return static_cast<double>(j < h ? j : j - N); };
    const std::uint64_t key = mix(seed);
    // value of global mode (i, j, k), projected, before the energy scale
    auto mode = [&](std::int64_t i, std::int64_t j, std::int64_t k, Complex v[3]) {
      for (int c = 0; c < 3; ++c) v[c] = Complex(0.0, 0.0);
      if ((i | j | k) == 0 || i == h || j == h || k == h) return;
      bool flip = false;
      if (k == 0) {
        const std::int64_t mi = (N - i) % N, mj = (N - j) % N;
        if (mi * N + mj < i * N + j) {
          i = mi;
          j = mj;
          flip = true;
        }
      }
      const double kx = kw(i), ky = kw(j), kz = static_cast<double>(k);
      const double k2 = kx * kx + ky * ky + kz * kz;
      const double kk = std::sqrt(k2);
      const double amp = std::sqrt(k2 * k2 * std::exp(-2.0 * (kk / k0) * (kk / k0)) /
                                   (4.0 * M_PI * k2));
      const std::uint64_t g = static_cast<std::uint64_t>((i * N + j) * nf + k);
      for (int c = 0; c < 3; ++c) {
        const std::uint64_t ctr = (g * 3 + static_cast<std::uint64_t>(c)) * 2;
        const double a = (static_cast<double>(mix(key ^ mix(ctr)) >> 11) + 1.0) * 0x1.0p-53;
        const double b = (static_cast<double>(mix(key ^ mix(ctr + 1)) >> 11) + 1.0) * 0x1.0p-53;
        const double r = std::sqrt(-2.0 * std::log(a));
        v[c] = Complex(amp * r * std::cos(2.0 * M_PI * b), amp * r * std::sin(2.0 * M_PI * b));
      }
      const double inv = k2 > 0.0 ? 1.0 / k2 : 0.0;
      const double ko[3] = {kx * inv, ky * inv, kz * inv};
      const double dr = kx * v[0].real() + ky * v[1].real() + kz * v[2].real();
      const double di = kx * v[0].imag() + ky * v[1].imag() + kz * v[2].imag();
      for (int c = 0; c < 3; ++c) {
        const double re = v[c].real() - ko[c] * dr;
        const double im = v[c].imag() - ko[c] * di;
        v[c] = Complex(re, flip ? -im : im);
      }
    };
    unsigned nth = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    std::vector<double> plane(static_cast<std::size_t>(N), 0.0);
    const std::int64_t comp = N * N * nf;
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < nth; ++w)
      pool.emplace_back([&, w] {
        Complex v[3];
        for (std::int64_t i = w; i < N; i += nth) {
          double acc = 0.0;
          for (std::int64_t j = 0; j < N; ++j)
            for (std::int64_t k = 0; k < nf; ++k) {
              mode(i, j, k, v);
              const double e = std::norm(v[0]) + std::norm(v[1]) + std::norm(v[2]);
              acc += (k == 0 || k == h ? 1.0 : 2.0) * e;
              const std::int64_t m = (i * N + j) * nf + k;
              for (int c = 0; c < 3; ++c) {
                out[2 * (c * comp + m)] = v[c].real();
                out[2 * (c * comp + m) + 1] = v[c].imag();
              }
            }
          plane[static_cast<std::size_t>(i)] = acc;
        }
      });
    for (auto& t : pool) t.join();
    double sum = 0.0;
    for (double v : plane) sum += v;
    const double n3 = static_cast<double>(N) * static_cast<double>(N) * static_cast<double>(N);
    const double e0 = 0.5 * sum / (n3 * n3);
    const double scale = e0 > 0.0 ? std::sqrt(energy / e0) : 0.0;
    pool.clear();
    for (unsigned w = 0; w < nth; ++w)
      pool.emplace_back([&, w] {
        for (std::int64_t q = std::int64_t{w} * 4096; q < 6 * comp; q += std::int64_t{nth} * 4096)
          for (std::int64_t r = q; r < std::min<std::int64_t>(q + 4096, 6 * comp); ++r)
            out[r] *= scale;
      });
    for (auto& t : pool) t.join();
  });
}

/// compute_rhs on a global spectral state.
int sdns_ref_compute_rhs(int n, int decomp, int p, int p1, int p2, double nu,
                         int dealias, const double* uhat, double* du) {
  return guarded([&] {
    const SolverConfig cfg = make_cfg(n, decomp, p, p1, p2, nu, 1.0, 0.0, dealias, 1);
    std::mutex mu;
    group(p, [&](int rank, std::shared_ptr<Communicator> comm) {
      const RankLayout lo = build_layout(cfg, rank);
      const WavenumberMesh wm = wavenumbers(cfg, lo);
      DistributedFFT fft(cfg, lo, comm);
      RhsWorkspace ws(lo);
      SpectralField3 u(lo.spec.shape), d(lo.spec.shape);
      scatter_spec(uhat, n, lo.spec, u);
      compute_rhs(u, wm, fft, ws, nu, d);
      std::lock_guard lk(mu);
      gather_spec(d, n, lo.spec, du);
    });
  });
}

/// Pointwise ops on a global spectral field (p = 1 semantics).
///   op 0: curl_hat(in) -> out        op 1: project(in) -> out
///   op 2: pressure_hat(in) -> out (component 0 only)
int sdns_ref_spectral_op(int n, int op, int dealias, const double* in, double* out) {
  return guarded([&] {
    const SolverConfig cfg = make_cfg(n, 0, 1, 1, 1, 0.0, 1.0, 0.0, dealias, 1);
    const RankLayout lo = build_layout(cfg, 0);
    const WavenumberMesh wm = wavenumbers(cfg, lo);
    SpectralField3 u(lo.spec.shape), o(lo.spec.shape);
    scatter_spec(in, n, lo.spec, u);
    if (op == 0) {
      curl_hat(u, wm, o);
    } else if (op == 1) {
      o = u;
      project(o, wm);
    } else if (op == 2) {
      pressure_hat(u, wm, o[0]);
    } else {
      throw ConfigError("unknown op");
    }
    gather_spec(o, n, lo.spec, out);
  });
}

/// cross(a, b) on flat 3-component real arrays of `count` points each.
int sdns_ref_cross(std::int64_t count, const double* a, const double* b, double* out) {
  return guarded([&] {
    RealField3 fa(Shape3{1, 1, count}), fb(Shape3{1, 1, count}), fo(Shape3{1, 1, count});
    for (int c = 0; c < 3; ++c) {
      std::memcpy(fa[c].data.data(), a + c * count, sizeof(double) * count);
      std::memcpy(fb[c].data.data(), b + c * count, sizeof(double) * count);
    }
    cross(fa, fb, fo);
    for (int c = 0; c < 3; ++c)
      std::memcpy(out + c * count, fo[c].data.data(), sizeof(double) * count);
  });
}

/// collect_stats of a global spectral state; row = t,E,Z,eps,div,spectrum.
int sdns_ref_collect_stats(int n, int decomp, int p, int p1, int p2, double nu,
                           const double* uhat, double* row) {
  return guarded([&] {
    const SolverConfig cfg = make_cfg(n, decomp, p, p1, p2, nu, 1.0, 0.0, 1, 1);
    std::mutex mu;
    group(p, [&](int rank, std::shared_ptr<Communicator> comm) {
      const RankLayout lo = build_layout(cfg, rank);
      const WavenumberMesh wm = wavenumbers(cfg, lo);
      SpectralField3 u(lo.spec.shape);
      scatter_spec(uhat, n, lo.spec, u);
      const FlowStats s = collect_stats(0.0, u, wm, nu, *comm);
      if (rank == 0) {
        std::lock_guard lk(mu);
        put_stats(s, row);
      }
    });
  });
}

/// A production-style run (mirrors run_worker, proj/core/src/runner.cpp:67-111):
/// state = uhat0 (optionally projected first), advance() to t_end = steps*dt
/// with post_step = project and a collect_stats sample every out_every
/// steps. `stats` receives one row per sample (step 0 included) of
/// 5 + shells doubles; *n_samples is set. uhat_final receives the final
/// global state.
int sdns_ref_run(int n, int decomp, int p, int p1, int p2, double nu, double dt,
                 int steps, int out_every, int dealias, int init_project,
                 const double* uhat0, double* stats, int* n_samples,
                 double* uhat_final) {
  return guarded([&] {
    const SolverConfig cfg = make_cfg(n, decomp, p, p1, p2, nu, dt,
                                      static_cast<double>(steps) * dt, dealias, out_every);
    const int shells = spectrum_shells(n);
    std::mutex mu;
    int count = 0;
    group(p, [&](int rank, std::shared_ptr<Communicator> comm) {
      const RankLayout lo = build_layout(cfg, rank);
      const WavenumberMesh wm = wavenumbers(cfg, lo);
      DistributedFFT fft(cfg, lo, comm);
      RhsWorkspace ws(lo);
      Rk4State st(lo.spec.shape);
      scatter_spec(uhat0, n, lo.spec, st.u_hat);
      if (init_project) project(st.u_hat, wm);
      RhsFn rhs = [&](const SpectralField3& uh, SpectralField3& du) {
        compute_rhs(uh, wm, fft, ws, cfg.nu, du);
      };
      AdvanceHooks hooks;
      hooks.post_step = [&] { project(st.u_hat, wm); };
      int local = 0;
      hooks.sample = [&](std::int64_t, double t) {
        const FlowStats s = collect_stats(t, st.u_hat, wm, cfg.nu, *comm);
        if (rank == 0 && stats) put_stats(s, stats + static_cast<std::size_t>(local) * (5 + shells));
        ++local;
      };
      advance(st, cfg, rhs, *comm, hooks);
      std::lock_guard lk(mu);
      if (rank == 0) count = local;
      if (uhat_final) gather_spec(st.u_hat, n, lo.spec, uhat_final);
    });
    if (n_samples) *n_samples = count;
  });
}

/// One classical RK4 step with a fixed dt (rk4_step_finite), optionally
/// followed by project (the bench loop, proj/core/src/runner.cpp:356-359).
/// The Neumaier carry starts at zero.
int sdns_ref_rk4_steps(int n, int decomp, int p, int p1, int p2, double nu,
                       double dt, int steps, int post_project, double* uhat) {
  return guarded([&] {
    const SolverConfig cfg = make_cfg(n, decomp, p, p1, p2, nu, dt, dt, 1, 1);
    std::mutex mu;
    group(p, [&](int rank, std::shared_ptr<Communicator> comm) {
      const RankLayout lo = build_layout(cfg, rank);
      const WavenumberMesh wm = wavenumbers(cfg, lo);
      DistributedFFT fft(cfg, lo, comm);
      RhsWorkspace ws(lo);
      Rk4State st(lo.spec.shape);
      scatter_spec(uhat, n, lo.spec, st.u_hat);
      RhsFn rhs = [&](const SpectralField3& uh, SpectralField3& du) {
        compute_rhs(uh, wm, fft, ws, cfg.nu, du);
      };
      for (int s = 0; s < steps; ++s) {
        rk4_step(st, dt, rhs);
        if (post_project) project(st.u_hat, wm);
      }
      std::lock_guard lk(mu);
      gather_spec(st.u_hat, n, lo.spec, uhat);
    });
  });
}

/// bench_entry_seconds (proj/core/src/runner.cpp:336-373) with a
/// configurable warm-up and an optional initial spectral state (NULL: the
/// reference's own Taylor-Green init + forward + project). unit 0 times
/// rk4_step + project (the reference's step), unit 1 times one compute_rhs
/// (a quarter-step sample). Returns mean seconds per unit from rank 0.
int sdns_ref_time_units(int n, int decomp, int p, int p1, int p2, double nu, double dt,
                        int warmup, int units, int unit, const double* uhat0,
                        double* seconds) {
  return guarded([&] {
    const SolverConfig cfg = make_cfg(n, decomp, p, p1, p2, nu, dt, dt, 1, 1);
    double sec = 0.0;
    std::mutex mu;
    group(p, [&](int rank, std::shared_ptr<Communicator> comm) {
      const RankLayout lo = build_layout(cfg, rank);
      const PhysicalMesh mesh = physical_mesh(lo);
      const WavenumberMesh wm = wavenumbers(cfg, lo);
      DistributedFFT fft(cfg, lo, comm);
      RhsWorkspace ws(lo);
      Rk4State st(lo.spec.shape);
      if (uhat0) {
        scatter_spec(uhat0, n, lo.spec, st.u_hat);
      } else {
        RealField3 u = make_initial_condition("taylor_green", lo, mesh);
        fft.forward(u, st.u_hat);
        project(st.u_hat, wm);
      }
      RhsFn rhs = [&](const SpectralField3& uh, SpectralField3& du) {
        compute_rhs(uh, wm, fft, ws, cfg.nu, du);
      };
      const auto one = [&] {
        if (unit == 0) {
          rk4_step(st, dt, rhs);
          project(st.u_hat, wm);
        } else {
          compute_rhs(st.u_hat, wm, fft, ws, cfg.nu, st.rhs);
        }
      };
      for (int k = 0; k < warmup; ++k) one();
      comm->barrier();
      const auto t0 = std::chrono::steady_clock::now();
      for (int k = 0; k < units; ++k) one();
      comm->barrier();
      const auto t1 = std::chrono::steady_clock::now();
      if (rank == 0) {
        std::lock_guard lk(mu);
        sec = std::chrono::duration<double>(t1 - t0).count() / static_cast<double>(units);
      }
    });
    *seconds = sec;
  });
}

/// The reference's own bench harness (proj/core/src/runner.cpp:336-397):
/// 5 warm-up steps, then `steps` timed rk4_step + project between
/// barriers; returns mean seconds per step from rank 0.
int sdns_ref_bench(int n, int decomp, int p, int p1, int p2, int steps,
                   double* sec_per_step) {
  return guarded([&] {
    BenchEntry e;
    e.n = n;
    e.decomp = decomp == 0 ? Decomp::Slab : Decomp::Pencil;
    e.p = p;
    e.p1 = p1;
    e.p2 = p2;
    RunOptions opts;
    opts.backend = p == 1 ? "loopback" : "inprocess";
    opts.collective_timeout = std::chrono::milliseconds(3600 * 1000);
    const auto rows = bench({e}, steps, opts);
    if (rows.empty() || rows[0].status != "ok")
      throw ConfigError(rows.empty() ? "bench produced no rows" : rows[0].status);
    *sec_per_step = rows[0].sec_per_step;
  });
}

// write_checkpoint / read_checkpoint (checkpoint.hpp:24-33) of the global
// real field u (3, n, n, n), decomposed like the given config.
int sdns_ref_checkpoint_write(int n, int decomp, int p, int p1, int p2, const double* u,
                              const char* path, double t, std::int64_t step) {
  return guarded([&] {
    const SolverConfig cfg = make_cfg(n, decomp, p, p1, p2, 0.0, 1.0, 1.0, 1, 1);
    group(p, [&](int rank, std::shared_ptr<Communicator> comm) {
      const RankLayout lo = build_layout(cfg, rank);
      RealField3 f(lo.real.shape);
      scatter_real(u, n, lo.real, f);
      write_checkpoint(path, cfg, lo, *comm, f, t, step);
    });
  });
}

int sdns_ref_checkpoint_read(int n, int decomp, int p, int p1, int p2, const char* path,
                             double* u, double* t, std::int64_t* step) {
  return guarded([&] {
    const SolverConfig cfg = make_cfg(n, decomp, p, p1, p2, 0.0, 1.0, 1.0, 1, 1);
    group(p, [&](int rank, std::shared_ptr<Communicator> comm) {
      const RankLayout lo = build_layout(cfg, rank);
      RealField3 f(lo.real.shape);
      const CheckpointInfo info = read_checkpoint(path, cfg, lo, *comm, f);
      gather_real(f, n, lo.real, u);  // disjoint blocks
      if (rank == 0) {
        *t = info.t;
        *step = info.step;
      }
    });
  });
}


// --- runner layer (host-only pieces and the full run) ------------------------

void put_cstr(char* dst, int cap, const std::string& s) {
  if (cap <= 0) return;
  const std::size_t n = std::min<std::size_t>(static_cast<std::size_t>(cap - 1), s.size());
  std::memcpy(dst, s.data(), n);
  dst[n] = '\0';
}

/// parse_config_text (config_file.cpp:57-136). iout = [n, decomp, p, p1, p2,
/// dealias, out_every], dout = [nu, dt, t_end]; notices '\n'-terminated.
int sdns_ref_parse_config(const char* text, const char* const* keys, const char* const* values,
                          int n_over, int* iout, double* dout, char* icase, int case_cap,
                          char* notes, int notes_cap) {
  return guarded([&] {
    ConfigOverrides ov;
    for (int i = 0; i < n_over; ++i) ov.emplace_back(keys[i], values[i]);
    const ParsedConfig pc = parse_config_text(text, ov);
    const SolverConfig& c = pc.cfg;
    const int iv[7] = {c.n, c.decomp == Decomp::Slab ? 0 : 1, c.p, c.p1, c.p2,
                       c.dealias ? 1 : 0, c.out_every};
    std::memcpy(iout, iv, sizeof(iv));
    dout[0] = c.nu;
    dout[1] = c.dt;
    dout[2] = c.t_end;
    put_cstr(icase, case_cap, c.initial_case);
    std::string all;
    for (const auto& s : pc.notices) all += s + "\n";
    put_cstr(notes, notes_cap, all);
  });
}

/// parse_bench_matrix_text (runner.cpp:249-289): 5 ints per entry.
int sdns_ref_parse_bench_matrix(const char* text, int* out, int cap, int* count) {
  return guarded([&] {
    const auto es = parse_bench_matrix_text(text);
    for (std::size_t i = 0; i < es.size() && static_cast<int>(i) < cap; ++i) {
      out[5 * i + 0] = es[i].n;
      out[5 * i + 1] = es[i].decomp == Decomp::Slab ? 0 : 1;
      out[5 * i + 2] = es[i].p;
      out[5 * i + 3] = es[i].p1;
      out[5 * i + 4] = es[i].p2;
    }
    *count = static_cast<int>(es.size());
  });
}

/// write_diagnostics_csv (runner.cpp:215-231); rows of 5 + shells doubles.
int sdns_ref_write_diagnostics_csv(const char* path, const std::int64_t* steps,
                                   const double* rows, std::int64_t nrows, int shells) {
  return guarded([&] {
    std::vector<SampleRow> samples;
    for (std::int64_t r = 0; r < nrows; ++r) {
      const double* x = rows + r * (5 + shells);
      SampleRow row;
      row.step = steps[r];
      row.stats.t = x[0];
      row.stats.energy = x[1];
      row.stats.enstrophy = x[2];
      row.stats.dissipation = x[3];
      row.stats.divergence_max = x[4];
      row.stats.spectrum.assign(x + 5, x + 5 + shells);
      samples.push_back(row);
    }
    write_diagnostics_csv(path, samples, shells);
  });
}

/// write_bench_csv (runner.cpp:399-414); entries 5 ints each.
int sdns_ref_write_bench_csv(const char* path, const int* ent, const std::int64_t* nodes,
                             const double* secs, const char* const* statuses, int count) {
  return guarded([&] {
    std::vector<BenchRow> rows;
    for (int i = 0; i < count; ++i) {
      BenchRow r;
      r.entry.n = ent[5 * i];
      r.entry.decomp = ent[5 * i + 1] == 0 ? Decomp::Slab : Decomp::Pencil;
      r.entry.p = ent[5 * i + 2];
      r.entry.p1 = ent[5 * i + 3];
      r.entry.p2 = ent[5 * i + 4];
      r.nodes_per_rank = nodes[i];
      r.sec_per_step = secs[i];
      r.status = statuses[i];
      rows.push_back(r);
    }
    write_bench_csv(path, rows);
  });
}

/// write_manifest (runner.cpp:233-247). iin = [n, decomp, p, p1, p2,
/// dealias, out_every]; din = [nu, dt, t_end, min_s, mean_s, max_s].
int sdns_ref_write_manifest(const char* path, const int* iin, const double* din,
                            const char* icase, const char* backend, const char* status,
                            std::int64_t steps, std::int64_t timed_steps, const char* csv,
                            const char* ckpt) {
  return guarded([&] {
    RunResult r;
    r.cfg.n = iin[0];
    r.cfg.decomp = iin[1] == 0 ? Decomp::Slab : Decomp::Pencil;
    r.cfg.p = iin[2];
    r.cfg.p1 = iin[3];
    r.cfg.p2 = iin[4];
    r.cfg.dealias = iin[5] != 0;
    r.cfg.out_every = iin[6];
    r.cfg.nu = din[0];
    r.cfg.dt = din[1];
    r.cfg.t_end = din[2];
    r.cfg.initial_case = icase;
    r.backend = backend;
    r.status = status;
    r.steps = steps;
    r.timing.min_s = din[3];
    r.timing.mean_s = din[4];
    r.timing.max_s = din[5];
    r.timing.timed_steps = timed_steps;
    r.csv_path = csv;
    r.checkpoint_path = ckpt;
    write_manifest(path, r);
  });
}

/// run() (runner.cpp:197-213) of a config text into out_dir: writes the
/// reference's diagnostics.csv, checkpoint.sdns and manifest.txt.
int sdns_ref_run_files(const char* config_text, const char* out_dir, char* status, int cap) {
  return guarded([&] {
    const ParsedConfig pc = parse_config_text(config_text);
    RunOptions opts;
    opts.out_dir = out_dir;
    opts.collective_timeout = std::chrono::milliseconds(600 * 1000);
    const RunResult r = run(pc.cfg, opts);
    put_cstr(status, cap, r.status);
  });
}

}  // extern "C"
