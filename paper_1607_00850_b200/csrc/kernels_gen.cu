// Generic-length kernels: every pass of the RHS pipeline for even n that is
// not a power of two in [4, 1024] (the reference accepts any even n >= 4,
// proj/core/src/config.cpp:17-19, and its FFTW plans any length,
// proj/core/src/serial_fft.cpp:57-125). They sit behind the same launchers,
// ColGeom / RowMap geometries and transposes as the tuned radix-8/16
// kernels, so the slab, pencil, all-to-all and peer-direct paths are
// unchanged; only the transforms differ:
//   - a length-n transform is a mixed-radix Stockham sequence over the prime
//     factors of n, staged in shared memory (two ping-pong line buffers);
//     each output of a stage is computed directly as its radix-R sum with
//     table twiddles exp(-2 pi i q / n) (one table, any n), so no radix needs
//     a hand-written butterfly and arbitrary primes work;
//   - column passes move tiles of TC consecutive kz columns (coalesced along
//     kz) through shared memory and run an item list per tile (the P1 / P2
//     curl splits are items with pre/post operations);
//   - z passes run one z line per CTA: c2r as complex inverse transforms of
//     Hermitian-extended pairs (imaginary parts of the kz = 0 and n/2 bins
//     ignored, as FFTW's c2r), 1/n^3, u x omega, and r2c of the products.
// They are correct-first kernels: the BASELINE configs all use tuned lengths.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "fft_core.cuh"
#include "kernels.cuh"
#include "rowmap.cuh"

namespace sdns_dev {

namespace {

constexpr int kGThreads = 256;
constexpr int kMaxStages = 24;

// Stockham stage radices of n: 8s, then a 4 or a 2 for the rest of the
// power of two, then the odd prime factors smallest first.
struct GPlan {
  int nst = 0;
  int rad[kMaxStages] = {};
};

GPlan plan_of(int n) {
  GPlan p;
  int m = n;
  while (m % 8 == 0 && p.nst < kMaxStages) {
    p.rad[p.nst++] = 8;
    m /= 8;
  }
  if (m % 4 == 0) {
    p.rad[p.nst++] = 4;
    m /= 4;
  }
  if (m % 2 == 0) {
    p.rad[p.nst++] = 2;
    m /= 2;
  }
  for (int f = 3; m > 1 && p.nst < kMaxStages; f += 2) {
    while (m % f == 0 && p.nst < kMaxStages) {
      p.rad[p.nst++] = f;
      m /= f;
    }
    if (f * f > m && m > 1) {  // the remainder is prime
      p.rad[p.nst++] = m;
      m = 1;
    }
  }
  return p;
}

__device__ __forceinline__ double2 gmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ double gwave(int j, int n) {
  return static_cast<double>(j <= n / 2 - 1 ? j : j - n);
}

__device__ __forceinline__ double2 gtw(const double2* __restrict__ tw, int q, int dir) {
  double2 w = __ldg(tw + q);
  if (dir > 0) w.y = -w.y;
  return w;
}

// One butterfly of a radix-R Stockham stage held in registers: x[r] =
// input j + r m (twiddled by W_n^{r k span}), outputs (j - k) R + k + q ns.
// R = 2, 4, 8 use the tuned DFTs of fft_core.cuh; other radices sum
// directly with the table's R-th roots of unity.
template <int R>
__device__ __forceinline__ void gbfly(const double2* __restrict__ x, double2* __restrict__ y,
                                      int j, int k, int m, int ns, int span, int n,
                                      const double2* __restrict__ tw, int dir) {
  double2 v[R];
  v[0] = x[j];
  int qq = 0;
  const int step = k * span;
#pragma unroll
  for (int r = 1; r < R; ++r) {
    qq += step;
    if (qq >= n) qq -= n;
    const double2 a = x[j + r * m];
    v[r] = step ? gmul(a, gtw(tw, qq, dir)) : a;
  }
  if constexpr (R == 2 || R == 4 || R == 8) {
    if (dir < 0) Dft<R, -1>::run(v);
    else Dft<R, +1>::run(v);
  } else {
    double2 o[R];
    const int root = n / R;  // W_R = W_n^root
#pragma unroll
    for (int q = 0; q < R; ++q) {
      double2 acc = v[0];
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const int e = (r * q) % R;
        const double2 t = e ? gmul(v[r], gtw(tw, e * root, dir)) : v[r];
        acc.x += t.x;
        acc.y += t.y;
      }
      o[q] = acc;
    }
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = o[q];
  }
  const int base = (j - k) * R + k;
#pragma unroll
  for (int q = 0; q < R; ++q) y[base + q * ns] = v[q];
}

// In-place (ping-pong) transform of `nl` lines of length n stored at
// a + l*n; returns the buffer holding the result (a or b). dir -1 forward,
// +1 inverse (conjugate twiddles); unnormalised. Every thread of the CTA
// calls it; it begins and ends with a barrier. A thread runs whole
// butterflies (each element read and written once per stage); radices
// without a register butterfly (primes > 7) sum each output directly.
__device__ double2* gfft(double2* a, double2* b, int nl, int n, const GPlan& pl,
                         const double2* __restrict__ tw, int dir) {
  __syncthreads();
  int ns = 1;
  for (int st = 0; st < pl.nst; ++st) {
    const int R = pl.rad[st];
    const int m = n / R;            // butterflies per line
    const int span = n / (ns * R);  // twiddle stride of this stage
    if (R <= 8 && R != 6) {
      for (int idx = threadIdx.x; idx < nl * m; idx += blockDim.x) {
        const int l = idx / m, j = idx - l * m;
        const int k = j % ns;
        const double2* x = a + l * n;
        double2* y = b + l * n;
        switch (R) {
          case 2: gbfly<2>(x, y, j, k, m, ns, span, n, tw, dir); break;
          case 3: gbfly<3>(x, y, j, k, m, ns, span, n, tw, dir); break;
          case 4: gbfly<4>(x, y, j, k, m, ns, span, n, tw, dir); break;
          case 5: gbfly<5>(x, y, j, k, m, ns, span, n, tw, dir); break;
          case 7: gbfly<7>(x, y, j, k, m, ns, span, n, tw, dir); break;
          default: gbfly<8>(x, y, j, k, m, ns, span, n, tw, dir); break;
        }
      }
    } else {
      for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
        const int l = idx / n, o = idx - l * n;
        // output o = (j / ns) * ns * R + k + q * ns, j = (o / (ns R)) ns + k
        const int blk = o / (ns * R), rem = o - blk * ns * R;
        const int q = rem / ns, k = rem - q * ns;
        const int j = blk * ns + k;
        // y[o] = sum_r x[j + r m] W_n^{r (k span + q m)}
        const int step = (k * span + q * m) % n;
        const double2* x = a + l * n + j;
        double2 acc = x[0];
        int qq = 0;
        for (int r = 1; r < R; ++r) {
          qq += step;
          if (qq >= n) qq -= n;
          const double2 v = gmul(x[r * m], gtw(tw, qq, dir));
          acc.x += v.x;
          acc.y += v.y;
        }
        b[l * n + o] = acc;
      }
    }
    __syncthreads();
    double2* t = a;
    a = b;
    b = t;
    ns *= R;
  }
  return a;
}

// Element offset of position pos along a column pass's transformed axis.
__device__ __forceinline__ long long gpos(const ColGeom& g, int pos) {
  if (g.pblk > 0) {
    const int q = pos / g.pblk;
    return static_cast<long long>(q) * g.ps1 + static_cast<long long>(pos - q * g.pblk) * g.ps0;
  }
  return static_cast<long long>(pos) * g.ps0;
}

struct GColArgs {
  const double2* in;
  double2* out;
  long long in_cs, out_cs;
  ColGeom g, go;
  int n, dir, tc, nitems, ntiles;
  GItem it[8];
  GPlan pl;
  const double2* tw;
};

__global__ void __launch_bounds__(kGThreads) k_gen_col(const __grid_constant__ GColArgs a) {
  extern __shared__ __align__(16) double2 gsm[];
  const int n = a.n, tc = a.tc;
  double2* b0 = gsm;
  double2* b1 = gsm + tc * n;
  const ColGeom& g = a.g;
  const ColGeom& go = a.go;
  const int tiles_per_row = g.pitch / tc;
  for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const int re = tile / tiles_per_row;
    const int kz0 = (tile - re * tiles_per_row) * tc;
    const int row = re < g.seg_a ? re + g.off0 : re - g.seg_a + g.off1;
    const double krow = gwave(g.row_off + row, n);
    for (int it = 0; it < a.nitems; ++it) {
      const GItem I = a.it[it];
      const double2* src = a.in + I.fin * a.in_cs;
      for (int idx = threadIdx.x; idx < tc * n; idx += blockDim.x) {
        const int c = idx % tc, pos = idx / tc;
        const int kz = kz0 + c;
        double2 v = make_double2(0.0, 0.0);
        if (kz < g.n2) {
          const long long e = static_cast<long long>(row) * g.rs +
                              static_cast<long long>(kz >> 3) * g.kcs + (kz & 7) + gpos(g, pos);
          v = src[e];
          const double k = gwave(pos, n);
          if (I.pre == G_K) v = make_double2(k * v.x, k * v.y);
          else if (I.pre == G_IK) v = make_double2(-(k * v.y), k * v.x);
          else if (I.pre == G_MI) v = make_double2(v.y, -v.x);
        }
        b0[c * n + pos] = v;
      }
      const double2* r = gfft(b0, b1, tc, n, a.pl, a.tw, a.dir);
      double2* dst = a.out + I.fout * a.out_cs;
      const double2* u0 = a.out;  // G_W2: U0 = output field 0, same geometry
      for (int idx = threadIdx.x; idx < tc * n; idx += blockDim.x) {
        const int c = idx % tc, pos = idx / tc;
        const int kz = kz0 + c;
        if (kz >= g.n2) continue;
        if (go.keep_k >= 0 && pos > go.keep_k && pos < n - go.keep_k) continue;
        long long e = static_cast<long long>(row) * go.rs +
                      static_cast<long long>(kz >> 3) * go.kcs + (kz & 7) + gpos(go, pos);
        if (go.seg) e += __ldg(go.seg + (go.pblk > 0 ? pos / go.pblk : 0));
        double2 v = r[c * n + pos];
        if (I.post == G_W2) {
          const double2 w = u0[e];
          const double2 d = make_double2(v.x - krow * w.x, v.y - krow * w.y);
          v = make_double2(-d.y, d.x);
        }
        dst[e] = v;
      }
      __syncthreads();  // U0 stores visible to the W2 item; buffers reused
    }
  }
  if (go.seg) __threadfence_system();  // peers read after a stream barrier
}

// --- z lines -------------------------------------------------------------------

struct GZArgs {
  double2* rows;       // z_fused: 6 fields; c2r: spectral source
  long long cs;
  RowMap rm;
  double2* out;        // z_fused_to / r2c: destination (with rmo)
  RowMap rmo;
  int po;              // outputs through rmo (peer-direct / segmented)
  const double* real;  // r2c source
  double* real_out;    // c2r destination
  int field;           // r2c_to: component
  double norm;
  int n;
  GPlan pl;
  const double2* tw;
};

// Hermitian extension of a half spectrum H (n/2+1 entries) at position pos,
// with the imaginary parts of the DC and Nyquist bins dropped (FFTW c2r).
__device__ __forceinline__ double2 hext(const double2* H, int pos, int n) {
  if (pos == 0 || pos == n / 2) return make_double2(H[pos].x, 0.0);
  if (pos < n / 2) return H[pos];
  const double2 v = H[n - pos];
  return make_double2(v.x, -v.y);
}

// Loads half-row `k` range of line ri of field f into H.
__device__ __forceinline__ void load_half(double2* H, const double2* base, const RowMap& rm,
                                          long long ro, int ri, int nf) {
  for (int k = threadIdx.x; k < nf; k += blockDim.x) H[k] = base[zel(rm, ro, ri, k)];
}

// Stores the r2c result Z (an n-point forward transform of a + i b) as the
// half spectra of a (component fa) and b (component fb, if fb >= 0) for kz <
// min(n/2+1, kz_keep).
__device__ __forceinline__ void store_pair(const GZArgs& a, const double2* Z, int ri, long long ro,
                                           int fa, int fb) {
  const int n = a.n, nf = n / 2 + 1;
  const int kk = min(nf, a.rm.kz_keep);
  for (int k = threadIdx.x; k < kk; k += blockDim.x) {
    const double2 d = Z[k];
    const double2 m = Z[(n - k) % n];
    const double2 e = make_double2(m.x, -m.y);  // conj Z[n-k]
    const double2 A = make_double2(0.5 * (d.x + e.x), 0.5 * (d.y + e.y));
    const double2 dd = make_double2(d.x - e.x, d.y - e.y);
    const double2 B = make_double2(0.5 * dd.y, -0.5 * dd.x);
    if (a.po) {
      const ZDst z = zdst(a.rmo, ri, k);
      a.out[z.el + fa * z.cs] = A;
      if (fb >= 0) a.out[z.el + fb * z.cs] = B;
    } else {
      const long long el = zel(a.rm, ro, ri, k);
      a.out[fa * a.cs + el] = A;
      if (fb >= 0) a.out[fb * a.cs + el] = B;
    }
  }
}

// Fused z pass for one line per CTA (k_z_fused's arithmetic): fields 0..5 =
// u0, u1, u2, w0', w1', w2; w0 = w0' - i kz u1, w1 = w1' + i kz u0.
__global__ void __launch_bounds__(kGThreads) k_gen_z_fused(const __grid_constant__ GZArgs a) {
  extern __shared__ __align__(16) double2 gsm[];
  const int n = a.n, nf = n / 2 + 1;
  const int hp = (nf + 1) & ~1;
  double2* H = gsm;              // 6 half rows
  double2* P = H + 6 * hp;       // 3 complex lines: the pair results
  double2* X = P + 3 * n;        // transform buffers
  double2* Y = X + n;
  const int ri = blockIdx.x;
  const RowMap& rm = a.rm;
  const long long ro = rm.nseg ? 0 : zrow_off(rm, ri);
  for (int f = 0; f < 6; ++f) load_half(H + f * hp, a.rows + f * a.cs, rm, ro, ri, nf);
  __syncthreads();
  // z part of the curl
  for (int k = threadIdx.x; k < nf; k += blockDim.x) {
    const double kz = static_cast<double>(k);
    const double2 u0 = H[k], u1 = H[hp + k];
    const double2 w0 = H[3 * hp + k], w1 = H[4 * hp + k];
    H[3 * hp + k] = make_double2(w0.x + kz * u1.y, w0.y - kz * u1.x);
    H[4 * hp + k] = make_double2(w1.x - kz * u0.y, w1.y + kz * u0.x);
  }
  // pairs (u0, u1), (u2, w0), (w1, w2) -> A + iB, inverse transform
  for (int pr = 0; pr < 3; ++pr) {
    const double2* A = H + (2 * pr) * hp;
    const double2* B = H + (2 * pr + 1) * hp;
    __syncthreads();
    for (int pos = threadIdx.x; pos < n; pos += blockDim.x) {
      const double2 x = hext(A, pos, n), y = hext(B, pos, n);
      X[pos] = make_double2(x.x - y.y, x.y + y.x);
    }
    const double2* r = gfft(X, Y, 1, n, a.pl, a.tw, +1);
    for (int pos = threadIdx.x; pos < n; pos += blockDim.x) P[pr * n + pos] = r[pos];
  }
  __syncthreads();
  // 1/n^3 (fft.cpp:125) and u x omega (navier_stokes.cpp:45-49); n0 + i n1 in
  // X, n2 in Y's partner line
  double2* X2 = Y;  // reuse: X <- n0 + i n1, then n2 separately
  for (int pos = threadIdx.x; pos < n; pos += blockDim.x) {
    const double2 p0 = P[pos], p1 = P[n + pos], p2 = P[2 * n + pos];
    const double u0 = __dmul_rn(p0.x, a.norm), u1 = __dmul_rn(p0.y, a.norm);
    const double u2 = __dmul_rn(p1.x, a.norm), w0 = __dmul_rn(p1.y, a.norm);
    const double w1 = __dmul_rn(p2.x, a.norm), w2 = __dmul_rn(p2.y, a.norm);
    const double n0 = __dsub_rn(__dmul_rn(u1, w2), __dmul_rn(u2, w1));
    const double n1 = __dsub_rn(__dmul_rn(u2, w0), __dmul_rn(u0, w2));
    const double n2 = __dsub_rn(__dmul_rn(u0, w1), __dmul_rn(u1, w0));
    X[pos] = make_double2(n0, n1);
    P[pos] = make_double2(n2, 0.0);  // pair 0 line is free now
  }
  const double2* z01 = gfft(X, X2, 1, n, a.pl, a.tw, -1);
  double2* Z01 = P + n;  // keep the (n0, n1) spectrum
  for (int pos = threadIdx.x; pos < n; pos += blockDim.x) Z01[pos] = z01[pos];
  __syncthreads();
  const GZArgs& g = a;
  store_pair(g, Z01, ri, ro, 0, 1);
  // n2 alone
  for (int pos = threadIdx.x; pos < n; pos += blockDim.x) X[pos] = P[pos];
  const double2* z2 = gfft(X, X2, 1, n, a.pl, a.tw, -1);
  store_pair(g, z2, ri, ro, 2, -1);
  if (a.po) __threadfence_system();
}

// Standalone c2r of one z line per CTA (DistributedFFT::inverse tail).
__global__ void __launch_bounds__(kGThreads) k_gen_z_c2r(const __grid_constant__ GZArgs a) {
  extern __shared__ __align__(16) double2 gsm[];
  const int n = a.n, nf = n / 2 + 1;
  const int hp = (nf + 1) & ~1;
  double2* H = gsm;
  double2* X = H + hp;
  double2* Y = X + n;
  const int ri = blockIdx.x;
  const long long ro = a.rm.nseg ? 0 : zrow_off(a.rm, ri);
  load_half(H, a.rows, a.rm, ro, ri, nf);
  __syncthreads();
  for (int pos = threadIdx.x; pos < n; pos += blockDim.x) X[pos] = hext(H, pos, n);
  const double2* r = gfft(X, Y, 1, n, a.pl, a.tw, +1);
  double* o = a.real_out + static_cast<long long>(ri) * n;
  for (int pos = threadIdx.x; pos < n; pos += blockDim.x) o[pos] = __dmul_rn(r[pos].x, a.norm);
}

// Standalone r2c of one z line per CTA (DistributedFFT::forward head).
__global__ void __launch_bounds__(kGThreads) k_gen_z_r2c(const __grid_constant__ GZArgs a) {
  extern __shared__ __align__(16) double2 gsm[];
  const int n = a.n, nf = n / 2 + 1;
  double2* X = gsm;
  double2* Y = X + n;
  const int ri = blockIdx.x;
  const double* src = a.real + static_cast<long long>(ri) * n;
  for (int pos = threadIdx.x; pos < n; pos += blockDim.x) X[pos] = make_double2(src[pos], 0.0);
  const double2* r = gfft(X, Y, 1, n, a.pl, a.tw, -1);
  const long long ro = a.rm.nseg ? 0 : zrow_off(a.rm, ri);
  for (int k = threadIdx.x; k < nf; k += blockDim.x) {
    if (a.po) {
      const ZDst z = zdst(a.rmo, ri, k);
      a.out[z.el + a.field * z.cs] = r[k];
    } else {
      a.out[zel(a.rm, ro, ri, k)] = r[k];
    }
  }
  if (a.po) __threadfence_system();
}

__global__ void k_twiddles_plain(int n, double2* tw) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  double s, c;
  sincospi(-2.0 * static_cast<double>(q) / static_cast<double>(n), &s, &c);
  tw[q] = make_double2(c, s);
}

int num_sms_gen() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

void set_smem(const void* k, size_t bytes) {
  if (bytes > 48 * 1024)
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

size_t z_fused_bytes(int n) {
  const int nf = n / 2 + 1, hp = (nf + 1) & ~1;
  return sizeof(double2) * (6 * static_cast<size_t>(hp) + 5 * static_cast<size_t>(n));
}

}  // namespace

void make_twiddles_plain(int n, double2* d_tw, cudaStream_t s) {
  k_twiddles_plain<<<(n + 255) / 256, 256, 0, s>>>(n, d_tw);
}

size_t gen_z_smem(int n) { return tuned_length(n) ? 0 : z_fused_bytes(n); }

void gen_col(int n, int dir, const double2* in, double2* out, long long in_cs, long long out_cs,
             int nitems, const GItem* it, const ColGeom& g, const ColGeom& go, const double2* tw,
             cudaStream_t s) {
  if (nitems <= 0 || g.nrows <= 0 || g.n2 <= 0) return;
  GColArgs a{};
  a.in = in;
  a.out = out;
  a.in_cs = in_cs;
  a.out_cs = out_cs;
  a.g = g;
  a.go = go;
  a.n = n;
  a.dir = dir;
  // kz columns per tile: 8 (128 B rows) while two line buffers fit 96 KB
  int tc = 8;
  while (tc > 1 && static_cast<size_t>(2 * tc) * n * sizeof(double2) > 96 * 1024) tc /= 2;
  a.tc = tc;
  a.nitems = nitems;
  for (int i = 0; i < nitems; ++i) a.it[i] = it[i];
  a.pl = plan_of(n);
  a.tw = tw;
  const long long tiles = static_cast<long long>(g.nrows) * (g.pitch / tc);
  a.ntiles = static_cast<int>(tiles);
  const size_t smem = static_cast<size_t>(2 * tc) * n * sizeof(double2);
  set_smem(reinterpret_cast<const void*>(k_gen_col), smem);
  const long long grid = std::min<long long>(tiles, 8LL * num_sms_gen());
  k_gen_col<<<static_cast<unsigned>(grid), kGThreads, smem, s>>>(a);
}

void gen_z_fused(int n, double2* rows, long long cs, const RowMap& rm, double2* out,
                 const RowMap* rmo, double norm, const double2* tw, cudaStream_t s) {
  if (rm.nrows <= 0) return;
  GZArgs a{};
  a.rows = rows;
  a.cs = cs;
  a.rm = rm;
  a.out = rmo ? out : rows;
  if (rmo) a.rmo = *rmo;
  a.po = rmo ? 1 : 0;
  a.norm = norm;
  a.n = n;
  a.pl = plan_of(n);
  a.tw = tw;
  const size_t smem = z_fused_bytes(n);
  set_smem(reinterpret_cast<const void*>(k_gen_z_fused), smem);
  k_gen_z_fused<<<static_cast<unsigned>(rm.nrows), kGThreads, smem, s>>>(a);
}

void gen_z_c2r(int n, const double2* spec, double* real, const RowMap& rm, double norm,
               const double2* tw, cudaStream_t s) {
  if (rm.nrows <= 0) return;
  GZArgs a{};
  a.rows = const_cast<double2*>(spec);
  a.rm = rm;
  a.real_out = real;
  a.norm = norm;
  a.n = n;
  a.pl = plan_of(n);
  a.tw = tw;
  const int nf = n / 2 + 1, hp = (nf + 1) & ~1;
  const size_t smem = sizeof(double2) * (static_cast<size_t>(hp) + 2 * static_cast<size_t>(n));
  set_smem(reinterpret_cast<const void*>(k_gen_z_c2r), smem);
  k_gen_z_c2r<<<static_cast<unsigned>(rm.nrows), kGThreads, smem, s>>>(a);
}

void gen_z_r2c(int n, const double* real, double2* spec, const RowMap& rm, const RowMap* rmo,
               int field, const double2* tw, cudaStream_t s) {
  if (rm.nrows <= 0) return;
  GZArgs a{};
  a.real = real;
  a.out = spec;
  a.rm = rm;
  if (rmo) a.rmo = *rmo;
  a.po = rmo ? 1 : 0;
  a.field = field;
  a.n = n;
  a.pl = plan_of(n);
  a.tw = tw;
  const size_t smem = sizeof(double2) * 2 * static_cast<size_t>(n);
  set_smem(reinterpret_cast<const void*>(k_gen_z_r2c), smem);
  k_gen_z_r2c<<<static_cast<unsigned>(rm.nrows), kGThreads, smem, s>>>(a);
}

}  // namespace sdns_dev
