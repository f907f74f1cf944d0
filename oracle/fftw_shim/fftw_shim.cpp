// TEST INFRASTRUCTURE (oracle only) — never linked into the product library.
//
// Self-written implementation of the FFTW3 guru64 subset declared in
// fftw3.h, so that the UNMODIFIED reference sources (proj/core/src/*.cpp)
// compile and run as the CPU oracle and CPU baseline. Algorithm: mixed-radix
// Stockham autosort (radices 4, 2, 3, 5 and a generic O(p^2) prime
// butterfly) on contiguous line buffers; even-length r2c/c2r through the
// classic half-length complex transform plus a twiddle post/pre-pass. No FFTW
// source was consulted or copied; only FFTW's documented semantics are
// restated (see fftw3.h).
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

namespace {

using cd = std::complex<double>;

// ---------------------------------------------------------------------------
// 1-D complex engine of one length and sign.
struct Engine {
  std::int64_t n = 1;
  int sign = -1;
  std::vector<int> radix;                    // stage radices, product = n
  std::vector<std::vector<cd>> tw;           // per stage: Ns*(R-1) twiddles
  std::vector<std::vector<cd>> roots;        // per stage: R roots (generic)

  static cd unit(long double num, long double den, int sign) {
    const long double a = 2.0L * 3.141592653589793238462643383279502884L * num / den;
    return cd(static_cast<double>(std::cos(a)),
              static_cast<double>(sign * std::sin(a)));
  }

  Engine(std::int64_t len, int sgn) : n(len), sign(sgn) {
    std::int64_t m = n;
    while (m % 4 == 0) { radix.push_back(4); m /= 4; }
    while (m % 2 == 0) { radix.push_back(2); m /= 2; }
    for (std::int64_t f = 3; m > 1;) {
      if (m % f == 0) { radix.push_back(static_cast<int>(f)); m /= f; }
      else f += 2;
    }
    std::int64_t ns = 1;
    for (int r : radix) {
      std::vector<cd> t(static_cast<std::size_t>(ns * (r - 1)));
      for (std::int64_t k = 0; k < ns; ++k)
        for (int q = 1; q < r; ++q)
          t[static_cast<std::size_t>(k * (r - 1) + q - 1)] =
              unit(static_cast<long double>((k * q) % (ns * r)),
                   static_cast<long double>(ns * r), sign);
      tw.push_back(std::move(t));
      std::vector<cd> ro(static_cast<std::size_t>(r));
      for (int q = 0; q < r; ++q) ro[static_cast<std::size_t>(q)] = unit(q, r, sign);
      roots.push_back(std::move(ro));
      ns *= r;
    }
  }

  // Runs the transform of `a` in place; `b` is scratch of n elements.
  void run(cd* a, cd* b) const {
    cd* in = a;
    cd* out = b;
    std::int64_t ns = 1;
    for (std::size_t s = 0; s < radix.size(); ++s) {
      const int r = radix[s];
      const std::int64_t m = n / r;
      const cd* t = tw[s].data();
      switch (r) {
        case 4: stage4(in, out, m, ns, t); break;
        case 2: stage2(in, out, m, ns, t); break;
        default: stage_generic(in, out, m, ns, r, t, roots[s].data()); break;
      }
      std::swap(in, out);
      ns *= r;
    }
    if (in != a) std::memcpy(a, in, static_cast<std::size_t>(n) * sizeof(cd));
  }

  static inline cd mul(cd x, cd w) {
    return cd(x.real() * w.real() - x.imag() * w.imag(),
              x.real() * w.imag() + x.imag() * w.real());
  }

  void stage2(const cd* in, cd* out, std::int64_t m, std::int64_t ns,
              const cd* t) const {
    for (std::int64_t j = 0; j < m; ++j) {
      const std::int64_t k = j % ns;
      const cd v0 = in[j];
      const cd v1 = k ? mul(in[j + m], t[k]) : in[j + m];
      const std::int64_t base = (j - k) * 2 + k;
      out[base] = v0 + v1;
      out[base + ns] = v0 - v1;
    }
  }

  void stage4(const cd* in, cd* out, std::int64_t m, std::int64_t ns,
              const cd* t) const {
    for (std::int64_t j = 0; j < m; ++j) {
      const std::int64_t k = j % ns;
      cd v0 = in[j], v1 = in[j + m], v2 = in[j + 2 * m], v3 = in[j + 3 * m];
      if (k) {
        const cd* w = t + 3 * k;
        v1 = mul(v1, w[0]);
        v2 = mul(v2, w[1]);
        v3 = mul(v3, w[2]);
      }
      const cd s02 = v0 + v2, d02 = v0 - v2;
      const cd s13 = v1 + v3, d13 = v1 - v3;
      // multiply d13 by sign*i: forward (sign=-1) gives -i.
      const cd jd13 = sign < 0 ? cd(d13.imag(), -d13.real())
                               : cd(-d13.imag(), d13.real());
      const std::int64_t base = (j - k) * 4 + k;
      out[base] = s02 + s13;
      out[base + ns] = d02 + jd13;
      out[base + 2 * ns] = s02 - s13;
      out[base + 3 * ns] = d02 - jd13;
    }
  }

  void stage_generic(const cd* in, cd* out, std::int64_t m, std::int64_t ns,
                     int r, const cd* t, const cd* ro) const {
    cd v[64];
    std::vector<cd> big;
    cd* vp = v;
    if (r > 64) { big.resize(static_cast<std::size_t>(r)); vp = big.data(); }
    for (std::int64_t j = 0; j < m; ++j) {
      const std::int64_t k = j % ns;
      for (int q = 0; q < r; ++q) {
        cd x = in[j + q * m];
        if (k && q) x = mul(x, t[k * (r - 1) + q - 1]);
        vp[q] = x;
      }
      const std::int64_t base = (j - k) * r + k;
      for (int o = 0; o < r; ++o) {
        cd acc(0.0, 0.0);
        for (int q = 0; q < r; ++q) acc += mul(vp[q], ro[(static_cast<std::int64_t>(o) * q) % r]);
        out[base + o * ns] = acc;
      }
    }
  }
};

std::mutex g_engine_mu;
std::map<std::pair<std::int64_t, int>, std::shared_ptr<const Engine>> g_engines;

std::shared_ptr<const Engine> engine(std::int64_t n, int sign) {
  std::lock_guard<std::mutex> lk(g_engine_mu);
  auto key = std::make_pair(n, sign);
  auto it = g_engines.find(key);
  if (it != g_engines.end()) return it->second;
  auto e = std::make_shared<const Engine>(n, sign);
  g_engines.emplace(key, e);
  return e;
}

// Per-thread scratch (plans may execute concurrently from several threads).
struct Scratch {
  std::vector<cd> a, b, c;
};
thread_local Scratch t_scratch;

cd* grow(std::vector<cd>& v, std::size_t n) {
  if (v.size() < n) v.resize(n);
  return v.data();
}

struct Dim {
  std::int64_t n, is, os;
};

// Calls f(in_off, out_off) for every multi-index of `loops`, except that the
// last loop (if any) is visited in chunks: f receives (in_off, out_off, cnt)
// with the last loop's element stride available as loops.back().
template <class F>
void for_each_chunk(const std::vector<Dim>& loops, std::int64_t chunk, F&& f) {
  if (loops.empty()) { f(0, 0, 1); return; }
  const std::size_t nl = loops.size();
  std::vector<std::int64_t> idx(nl, 0);
  const Dim& last = loops.back();
  for (;;) {
    std::int64_t io = 0, oo = 0;
    for (std::size_t d = 0; d + 1 < nl; ++d) { io += idx[d] * loops[d].is; oo += idx[d] * loops[d].os; }
    for (std::int64_t c = 0; c < last.n; c += chunk) {
      const std::int64_t cnt = std::min<std::int64_t>(chunk, last.n - c);
      f(io + c * last.is, oo + c * last.os, cnt);
    }
    // advance the outer indices (all but last) as an odometer
    std::int64_t d = static_cast<std::int64_t>(nl) - 2;
    while (d >= 0) {
      if (++idx[static_cast<std::size_t>(d)] < loops[static_cast<std::size_t>(d)].n) break;
      idx[static_cast<std::size_t>(d)] = 0;
      --d;
    }
    if (d < 0) return;
  }
}

constexpr std::int64_t kChunk = 8;

// Complex lines along one axis. `in` may equal `out` (in-place).
void c2c_axis(const Engine& e, const cd* in, cd* out, std::int64_t is_line,
              std::int64_t os_line, const std::vector<Dim>& loops) {
  const std::int64_t n = e.n;
  const std::int64_t lstride_i = loops.empty() ? 0 : loops.back().is;
  const std::int64_t lstride_o = loops.empty() ? 0 : loops.back().os;
  cd* buf = grow(t_scratch.a, static_cast<std::size_t>(n * kChunk));
  cd* scr = grow(t_scratch.b, static_cast<std::size_t>(n));
  for_each_chunk(loops, kChunk, [&](std::int64_t io, std::int64_t oo, std::int64_t cnt) {
    for (std::int64_t x = 0; x < n; ++x)
      for (std::int64_t c = 0; c < cnt; ++c)
        buf[c * n + x] = in[io + c * lstride_i + x * is_line];
    for (std::int64_t c = 0; c < cnt; ++c) e.run(buf + c * n, scr);
    for (std::int64_t x = 0; x < n; ++x)
      for (std::int64_t c = 0; c < cnt; ++c)
        out[oo + c * lstride_o + x * os_line] = buf[c * n + x];
  });
}

// Real-to-complex along one axis of logical length n.
void r2c_axis(std::int64_t n, const double* in, cd* out, std::int64_t is_line,
              std::int64_t os_line, const std::vector<Dim>& loops) {
  const std::int64_t nf = n / 2 + 1;
  const std::int64_t lstride_i = loops.empty() ? 0 : loops.back().is;
  const std::int64_t lstride_o = loops.empty() ? 0 : loops.back().os;
  if (n % 2 == 0) {
    const std::int64_t h = n / 2;
    auto eh = engine(h, FFTW_FORWARD);
    std::vector<cd> w(static_cast<std::size_t>(h + 1));
    for (std::int64_t k = 0; k <= h; ++k) w[static_cast<std::size_t>(k)] = Engine::unit(k, n, -1);
    cd* buf = grow(t_scratch.a, static_cast<std::size_t>(h * kChunk));
    cd* scr = grow(t_scratch.b, static_cast<std::size_t>(h));
    cd* res = grow(t_scratch.c, static_cast<std::size_t>(nf * kChunk));
    for_each_chunk(loops, kChunk, [&](std::int64_t io, std::int64_t oo, std::int64_t cnt) {
      for (std::int64_t c = 0; c < cnt; ++c) {
        const double* src = in + io + c * lstride_i;
        cd* z = buf + c * h;
        for (std::int64_t m = 0; m < h; ++m)
          z[m] = cd(src[(2 * m) * is_line], src[(2 * m + 1) * is_line]);
        eh->run(z, scr);
        cd* X = res + c * nf;
        for (std::int64_t k = 0; k <= h; ++k) {
          const cd zk = z[k % h];
          const cd zc = std::conj(z[(h - k) % h]);
          const cd ze = 0.5 * (zk + zc);
          const cd d = zk - zc;                       // = 2i * Zo
          const cd zo(0.5 * d.imag(), -0.5 * d.real());  // d / (2i)
          X[k] = ze + Engine::mul(zo, w[static_cast<std::size_t>(k)]);
        }
      }
      for (std::int64_t k = 0; k < nf; ++k)
        for (std::int64_t c = 0; c < cnt; ++c)
          out[oo + c * lstride_o + k * os_line] = res[c * nf + k];
    });
  } else {
    auto e = engine(n, FFTW_FORWARD);
    cd* buf = grow(t_scratch.a, static_cast<std::size_t>(n));
    cd* scr = grow(t_scratch.b, static_cast<std::size_t>(n));
    for_each_chunk(loops, 1, [&](std::int64_t io, std::int64_t oo, std::int64_t) {
      for (std::int64_t x = 0; x < n; ++x) buf[x] = cd(in[io + x * is_line], 0.0);
      e->run(buf, scr);
      for (std::int64_t k = 0; k < nf; ++k) out[oo + k * os_line] = buf[k];
    });
  }
}

// Complex-to-real along one axis of logical length n (Hermitian input,
// imaginary parts of DC and Nyquist ignored). Does not modify `in`.
void c2r_axis(std::int64_t n, const cd* in, double* out, std::int64_t is_line,
              std::int64_t os_line, const std::vector<Dim>& loops) {
  const std::int64_t nf = n / 2 + 1;
  const std::int64_t lstride_i = loops.empty() ? 0 : loops.back().is;
  const std::int64_t lstride_o = loops.empty() ? 0 : loops.back().os;
  if (n % 2 == 0) {
    const std::int64_t h = n / 2;
    auto eh = engine(h, FFTW_BACKWARD);
    std::vector<cd> w(static_cast<std::size_t>(h));
    for (std::int64_t k = 0; k < h; ++k) w[static_cast<std::size_t>(k)] = Engine::unit(k, n, +1);
    cd* X = grow(t_scratch.c, static_cast<std::size_t>(nf * kChunk));
    cd* z = grow(t_scratch.a, static_cast<std::size_t>(h));
    cd* scr = grow(t_scratch.b, static_cast<std::size_t>(h));
    for_each_chunk(loops, kChunk, [&](std::int64_t io, std::int64_t oo, std::int64_t cnt) {
      for (std::int64_t k = 0; k < nf; ++k)
        for (std::int64_t c = 0; c < cnt; ++c)
          X[c * nf + k] = in[io + c * lstride_i + k * is_line];
      for (std::int64_t c = 0; c < cnt; ++c) {
        cd* Xc = X + c * nf;
        Xc[0] = cd(Xc[0].real(), 0.0);
        Xc[h] = cd(Xc[h].real(), 0.0);
        for (std::int64_t k = 0; k < h; ++k) {
          const cd a = Xc[k];
          const cd b = std::conj(Xc[h - k]);
          const cd xe = a + b;
          const cd xo = Engine::mul(a - b, w[static_cast<std::size_t>(k)]);
          z[k] = cd(xe.real() - xo.imag(), xe.imag() + xo.real());  // xe + i*xo
        }
        eh->run(z, scr);
        double* dst = out + oo + c * lstride_o;
        for (std::int64_t m = 0; m < h; ++m) {
          dst[(2 * m) * os_line] = z[m].real();
          dst[(2 * m + 1) * os_line] = z[m].imag();
        }
      }
    });
  } else {
    auto e = engine(n, FFTW_BACKWARD);
    cd* buf = grow(t_scratch.a, static_cast<std::size_t>(n));
    cd* scr = grow(t_scratch.b, static_cast<std::size_t>(n));
    for_each_chunk(loops, 1, [&](std::int64_t io, std::int64_t oo, std::int64_t) {
      buf[0] = cd(in[io].real(), 0.0);
      for (std::int64_t k = 1; k < nf; ++k) {
        buf[k] = in[io + k * is_line];
        buf[n - k] = std::conj(buf[k]);
      }
      e->run(buf, scr);
      for (std::int64_t x = 0; x < n; ++x) out[oo + x * os_line] = buf[x].real();
    });
  }
}

enum class Kind { C2C, R2C, C2R };

}  // namespace

struct fftw_plan_s {
  Kind kind;
  int sign;
  std::vector<Dim> dims, howmany;
};

namespace {

fftw_plan make_plan(Kind k, int sign, int rank, const fftw_iodim64* dims,
                    int hr, const fftw_iodim64* hd) {
  auto* p = new fftw_plan_s;
  p->kind = k;
  p->sign = sign;
  for (int i = 0; i < rank; ++i) p->dims.push_back({dims[i].n, dims[i].is, dims[i].os});
  for (int i = 0; i < hr; ++i) p->howmany.push_back({hd[i].n, hd[i].is, hd[i].os});
  // Pre-build engines so execution never plans.
  for (int i = 0; i < rank; ++i) {
    const std::int64_t n = dims[i].n;
    const bool last = i == rank - 1;
    if (k == Kind::C2C || !last) {
      engine(n, k == Kind::C2C ? sign : (k == Kind::R2C ? FFTW_FORWARD : FFTW_BACKWARD));
    } else {
      engine(n % 2 == 0 ? n / 2 : n, k == Kind::R2C ? FFTW_FORWARD : FFTW_BACKWARD);
    }
  }
  return p;
}

// Loops for a pass along axis `a`: howmany dims plus every other transform
// dim, with the given (in, out) stride selectors. `last_n` overrides the
// extent of the last transform dim (the n/2+1 complex half axis).
std::vector<Dim> pass_loops(const fftw_plan_s& p, int a, bool in_is, bool out_os,
                            std::int64_t last_n) {
  std::vector<Dim> loops;
  auto sel = [&](const Dim& d, std::int64_t n) {
    return Dim{n, in_is ? d.is : d.os, out_os ? d.os : d.is};
  };
  for (const Dim& d : p.howmany) loops.push_back(sel(d, d.n));
  const int r = static_cast<int>(p.dims.size());
  for (int i = 0; i < r; ++i) {
    if (i == a) continue;
    const std::int64_t n = (i == r - 1 && last_n > 0) ? last_n : p.dims[static_cast<std::size_t>(i)].n;
    loops.push_back(sel(p.dims[static_cast<std::size_t>(i)], n));
  }
  // Keep a unit-stride loop innermost when one exists (chunked gathers).
  for (std::size_t i = 0; i + 1 < loops.size(); ++i) {
    if (loops[i].is == 1 && loops[i].n > 1 && loops.back().is != 1) {
      std::swap(loops[i], loops.back());
      break;
    }
  }
  return loops;
}

}  // namespace

extern "C" {

fftw_plan fftw_plan_guru64_dft(int rank, const fftw_iodim64* dims, int hr,
                               const fftw_iodim64* hd, fftw_complex*,
                               fftw_complex*, int sign, unsigned) {
  return make_plan(Kind::C2C, sign, rank, dims, hr, hd);
}

fftw_plan fftw_plan_guru64_dft_r2c(int rank, const fftw_iodim64* dims, int hr,
                                   const fftw_iodim64* hd, double*,
                                   fftw_complex*, unsigned) {
  return make_plan(Kind::R2C, FFTW_FORWARD, rank, dims, hr, hd);
}

fftw_plan fftw_plan_guru64_dft_c2r(int rank, const fftw_iodim64* dims, int hr,
                                   const fftw_iodim64* hd, fftw_complex*,
                                   double*, unsigned) {
  return make_plan(Kind::C2R, FFTW_BACKWARD, rank, dims, hr, hd);
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
  auto* ci = reinterpret_cast<cd*>(in);
  auto* co = reinterpret_cast<cd*>(out);
  const int r = static_cast<int>(p->dims.size());
  for (int a = r - 1; a >= 0; --a) {
    const bool first = a == r - 1;
    const Dim& d = p->dims[static_cast<std::size_t>(a)];
    auto loops = pass_loops(*p, a, first, true, 0);
    c2c_axis(*engine(d.n, p->sign), first ? ci : co, co, first ? d.is : d.os, d.os, loops);
  }
}

void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out) {
  auto* co = reinterpret_cast<cd*>(out);
  const int r = static_cast<int>(p->dims.size());
  const Dim& dl = p->dims[static_cast<std::size_t>(r - 1)];
  r2c_axis(dl.n, in, co, dl.is, dl.os, pass_loops(*p, r - 1, true, true, 0));
  const std::int64_t nf = dl.n / 2 + 1;
  for (int a = r - 2; a >= 0; --a) {
    const Dim& d = p->dims[static_cast<std::size_t>(a)];
    c2c_axis(*engine(d.n, FFTW_FORWARD), co, co, d.os, d.os,
             pass_loops(*p, a, false, true, nf));
  }
}

void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out) {
  auto* ci = reinterpret_cast<cd*>(in);
  const int r = static_cast<int>(p->dims.size());
  const Dim& dl = p->dims[static_cast<std::size_t>(r - 1)];
  const std::int64_t nf = dl.n / 2 + 1;
  // Leading axes: in place on the input (FFTW may destroy c2r input).
  for (int a = 0; a < r - 1; ++a) {
    const Dim& d = p->dims[static_cast<std::size_t>(a)];
    c2c_axis(*engine(d.n, FFTW_BACKWARD), ci, ci, d.is, d.is,
             pass_loops(*p, a, true, false, nf));
  }
  c2r_axis(dl.n, ci, out, dl.is, dl.os, pass_loops(*p, r - 1, true, true, 0));
}

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
