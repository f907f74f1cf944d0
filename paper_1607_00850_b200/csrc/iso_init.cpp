// Seeded isotropic initial field for BASELINE configs 2-4.
// The reference has no such case (only "taylor_green",
// proj/core/src/navier_stokes.cpp:27-32), so it is defined here once and fed
// bit-identically to the oracle and to the device path:
//   1. three complex Gaussians per global half-spectrum mode from a
//      counter-based generator keyed by (seed, component, global index);
//   2. amplitude sqrt(E(k)/(4 pi k^2)), E(k) = k^4 exp(-2 (k/k0)^2);
//   3. k = 0 and the Nyquist indices (kx or ky = -n/2, kz = n/2) are zero;
//   4. Hermitian symmetry on kz = 0: u(-kx,-ky,0) = conj u(kx,ky,0);
//   5. the reference project() formula (navier_stokes.cpp:85-102);
//   6. scaled to the requested energy with the reference energy formula
//      (diagnostics.cpp:41-48, :84), summed in global index order so every
//      decomposition gets bit-identical values.
#include <cmath>
#include <thread>

#include "host.h"

namespace sdns_host {

namespace {

inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// uniform in (0, 1]
inline double unit(uint64_t h) { return (static_cast<double>(h >> 11) + 1.0) * 0x1.0p-53; }

struct C3 {
  double re[3], im[3];
};

inline int64_t wavenum(int64_t j, int64_t n) { return j <= n / 2 - 1 ? j : j - n; }

// Raw (unprojected) Gaussian amplitudes at global mode (i, j, k).
C3 raw_mode(int64_t n, uint64_t seed, double k0, int64_t i, int64_t j, int64_t k) {
  C3 r{};
  const int64_t nf = n / 2 + 1;
  const double kx = static_cast<double>(wavenum(i, n));
  const double ky = static_cast<double>(wavenum(j, n));
  const double kz = static_cast<double>(k);
  const double k2 = kx * kx + ky * ky + kz * kz;
  const double kk = std::sqrt(k2);
  const double ek = k2 * k2 * std::exp(-2.0 * (kk / k0) * (kk / k0));
  const double amp = std::sqrt(ek / (4.0 * M_PI * k2));
  const uint64_t gidx = static_cast<uint64_t>((i * n + j) * nf + k);
  const uint64_t key = splitmix64(seed);
  for (int c = 0; c < 3; ++c) {
    const uint64_t ctr = (gidx * 3 + static_cast<uint64_t>(c)) * 2;
    const double u1 = unit(splitmix64(key ^ splitmix64(ctr)));
    const double u2 = unit(splitmix64(key ^ splitmix64(ctr + 1)));
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * M_PI * u2;
    r.re[c] = amp * rad * std::cos(th);
    r.im[c] = amp * rad * std::sin(th);
  }
  return r;
}

// Projected, Hermitian-consistent value at a global mode (before scaling).
C3 iso_mode(int64_t n, uint64_t seed, double k0, int64_t i, int64_t j, int64_t k) {
  C3 z{};
  const int64_t h = n / 2;
  if ((i == 0 && j == 0 && k == 0) || i == h || j == h || k == h) return z;
  int64_t si = i, sj = j;
  bool conj = false;
  if (k == 0) {
    const int64_t pi = (n - i) % n, pj = (n - j) % n;
    if (pi * n + pj < i * n + j) {
      si = pi;
      sj = pj;
      conj = true;
    }
  }
  C3 r = raw_mode(n, seed, k0, si, sj, k);
  // project() at the canonical mode, navier_stokes.cpp:85-102
  const double kx = static_cast<double>(wavenum(si, n));
  const double ky = static_cast<double>(wavenum(sj, n));
  const double kz = static_cast<double>(k);
  const double k2 = kx * kx + ky * ky + kz * kz;
  const double inv = k2 > 0.0 ? 1.0 / k2 : 0.0;
  const double ko[3] = {kx * inv, ky * inv, kz * inv};
  const double kdr = kx * r.re[0] + ky * r.re[1] + kz * r.re[2];
  const double kdi = kx * r.im[0] + ky * r.im[1] + kz * r.im[2];
  for (int c = 0; c < 3; ++c) {
    r.re[c] = r.re[c] - ko[c] * kdr;
    r.im[c] = r.im[c] - ko[c] * kdi;
    if (conj) r.im[c] = -r.im[c];
  }
  return r;
}

}  // namespace

void iso_init(int64_t n, uint64_t seed, double k0, double energy, const sdns_layout& lo,
              double* out) {
  const int64_t nf = n / 2 + 1;
  // Global energy, in global index order, chunked by kx plane (fixed order).
  unsigned nth = std::thread::hardware_concurrency();
  if (nth == 0) nth = 1;
  if (nth > 64) nth = 64;
  std::vector<double> plane(static_cast<size_t>(n), 0.0);
  {
    std::vector<std::thread> th;
    for (unsigned w = 0; w < nth; ++w) {
      th.emplace_back([&, w] {
        for (int64_t i = w; i < n; i += nth) {
          double acc = 0.0;
          for (int64_t j = 0; j < n; ++j)
            for (int64_t k = 0; k < nf; ++k) {
              const C3 v = iso_mode(n, seed, k0, i, j, k);
              const double wgt = (k == 0 || k == n / 2) ? 1.0 : 2.0;
              const double e = (v.re[0] * v.re[0] + v.im[0] * v.im[0]) +
                               (v.re[1] * v.re[1] + v.im[1] * v.im[1]) +
                               (v.re[2] * v.re[2] + v.im[2] * v.im[2]);
              acc += wgt * e;
            }
          plane[static_cast<size_t>(i)] = acc;
        }
      });
    }
    for (auto& t : th) t.join();
  }
  double sum = 0.0;
  for (double v : plane) sum += v;
  const double n3 = static_cast<double>(n) * static_cast<double>(n) * static_cast<double>(n);
  const double e0 = 0.5 * sum / (n3 * n3);
  const double scale = e0 > 0.0 ? std::sqrt(energy / e0) : 0.0;

  const int64_t s0 = lo.spec_shape[0], s1 = lo.spec_shape[1], s2 = lo.spec_shape[2];
  const int64_t o0 = lo.spec_offset[0], o1 = lo.spec_offset[1], o2 = lo.spec_offset[2];
  const int64_t comp = s0 * s1 * s2;
  std::vector<std::thread> th;
  for (unsigned w = 0; w < nth; ++w) {
    th.emplace_back([&, w] {
      for (int64_t a = w; a < s0; a += nth)
        for (int64_t b = 0; b < s1; ++b)
          for (int64_t c = 0; c < s2; ++c) {
            const C3 v = iso_mode(n, seed, k0, o0 + a, o1 + b, o2 + c);
            const int64_t m = (a * s1 + b) * s2 + c;
            for (int q = 0; q < 3; ++q) {
              out[2 * (q * comp + m)] = v.re[q] * scale;
              out[2 * (q * comp + m) + 1] = v.im[q] * scale;
            }
          }
    });
  }
  for (auto& t : th) t.join();
}

}  // namespace sdns_host
