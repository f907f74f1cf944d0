// sm_100a kernels of the spectral-DNS right-hand-side pipeline.
//
// Pass structure of one RHS evaluation (reference
// compute_rhs, proj/core/src/navier_stokes.cpp:104-139, and DistributedFFT,
// proj/core/src/fft.cpp:81-126):
//   P1 k_pipe_xinv    x-axis inverse c2c of u_hat (+ kx u_hat for the curl)
//   P2 k_pipe_yinv    y-axis inverse c2c, completing the x/y parts of the curl
//   P3 k_z_fused      z-axis c2r of the 6 fields (+ the kz part of the curl),
//                     1/n^3, u x omega, z r2c of 3
//   P4 k_pipe_plain   y-axis forward c2c of the 3 fields (in place)
//   P5a k_pipe_plain  x-axis forward c2c of the 3 fields (in place)
// (P1, P2, P4, P5a live in kernels_col.cu.)
//   P5b k_rk_update   dealias mask + projection + viscous term + RK4 stage
//                     update (+ Neumaier carry, projection, finite flag);
//                     k_rk3_stats also accumulates the sampled diagnostics
// Pointwise parts follow the reference operation order with explicit
// round-to-nearest intrinsics (no FMA contraction), so the standalone
// pointwise kernels are bitwise equal to the reference CPU functions.
#include <cstdio>
#include <cstring>
#include <cudaTypedefs.h>
#include <type_traits>
#include <vector>

#include "fft_core.cuh"
#include "kernels.cuh"
#include "rowmap.cuh"

namespace sdns_dev {

// Opt in to >48 KB dynamic shared memory once per kernel instantiation (the
// call sites below are templates, so each static flag is per kernel).
#define SDNS_SET_SMEM(kernel, bytes)                                              \
  do {                                                                           \
    static bool sdns_smem_done_ = false;                                          \
    if (!sdns_smem_done_) {                                                       \
      if ((bytes) > 48 * 1024)                                                    \
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             static_cast<int>(bytes));                            \
      cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, \
                           100);                                                  \
      sdns_smem_done_ = true;                                                     \
    }                                                                            \
  } while (0)

namespace {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// axis_wavenumber, proj/core/include/sdns/mesh.hpp:19-21
__device__ __forceinline__ double wavenum(int j, int n) {
  return static_cast<double>(j <= n / 2 - 1 ? j : j - n);
}

// i * (a*x - b*y) for complex x, y and real a, b (curl component).
__device__ __forceinline__ double2 i_cross(double a, double2 x, double b, double2 y) {
  const double re = dsub(dmul(a, x.x), dmul(b, y.x));
  const double im = dsub(dmul(a, x.y), dmul(b, y.y));
  return make_double2(-im, re);
}

}  // namespace

// ---------------------------------------------------------------------------
// Twiddles

// Stage-ordered table (fft_core.cuh tw_stage_off): entry (NS, r, k) holds
// W_{NS*R}^{k r} = exp(-2 pi i q / n), q = k r n / (NS R).
__global__ void k_twiddles(int n, int e, double2* tw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int off = 0;
  for (int ns = 1; ns < n;) {
    const int rem = n / ns;
    const int r = rem >= e ? e : rem;
    if (ns > 1) {
      const int cnt = ns * (r - 1);
      if (i >= off && i < off + cnt) {
        const int rr = (i - off) / ns + 1, k = (i - off) % ns;
        const int q = k * rr * (n / (ns * r));
        double s, c;
        // sincospi is accurate to ~1 ulp and exact at the symmetry points
        sincospi(-2.0 * static_cast<double>(q) / static_cast<double>(n), &s, &c);
        tw[i] = make_double2(c, s);
        return;
      }
      off += cnt;
    }
    ns *= r;
  }
}

void make_twiddles_plain(int n, double2* d_tw, cudaStream_t s);  // kernels_gen.cu
void make_twiddles(int n, double2* d_tw, cudaStream_t s) {
  if (!tuned_length(n)) {
    make_twiddles_plain(n, d_tw, s);
    return;
  }
  const int total = tw_stage_total(n);
  if (total > 0) k_twiddles<<<(total + 255) / 256, 256, 0, s>>>(n, fft_elems(n), d_tw);
}

// ---------------------------------------------------------------------------
// P5: x-axis forward transform of the 3 nonlinear components, then per mode
// the compute_rhs tail (navier_stokes.cpp:114-138) and the RK4 stage update
// (rk4.cpp:44-65), the post-step projection (runner.cpp:107) and the finite
// check (rk4.cpp:13-18, evaluated before the projection like the reference).

__device__ __forceinline__ double two_sum_err(double a, double b, double s) {
  // Neumaier branch of TwoSum, rk4.cpp:21-23
  return fabs(a) >= fabs(b) ? dadd(dsub(a, s), b) : dadd(dsub(b, s), a);
}

// P5b: the per-mode tail as a streaming kernel over the x layout, after the
// x-axis forward FFT of the nonlinear term has run in place (P5a,
// k_pipe_plain): dealias mask, projection, viscous term and the RK4 stage
// update (+ Neumaier carry, post-step projection, finite flag). Bitwise the
// reference operation order.
// One mode of P5b: the compute_rhs tail and the stage update at element e
// = (i, j, k) of the local spectral block. un receives the new state
// (XF_RK3). Explicit round-to-nearest operations: the result does not depend
// on the kernel it is inlined into.
// The loads of one mode of P5b (split from the arithmetic so that a thread
// can have the loads of several modes in flight, k_rk_update).
struct RkIn {
  double2 c0, c1, c2;
  double2 uq[3], bq[3], sq[3], cr[3];
};

template <int MODE>
__device__ __forceinline__ void rk_load(const XfArgs& a, const SpecGeom& g, long long e, int i,
                                        int j, int k, RkIn& in) {
  const double kmax = static_cast<double>(g.n) / 3.0;
  const double ubdt = a.dts ? a.dts[0] : a.ubdt;
  const double kx = wavenum(g.o0 + i, g.n), ky = wavenum(g.o1 + j, g.n);
  const double kzd = static_cast<double>(g.o2 + k);
  // dealias mask (navier_stokes.cpp:123-125): masked modes of the nonlinear
  // term are zero and were never computed by the pruned forward passes
  const bool keep = !a.dealias || (fabs(kx) < kmax && fabs(ky) < kmax && fabs(kzd) < kmax);
  in.c0 = make_double2(0.0, 0.0);
  in.c1 = in.c0;
  in.c2 = in.c0;
  if (keep) {
    in.c0 = a.nl[e];
    in.c1 = a.nl[a.nl_cs + e];
    in.c2 = a.nl[2 * a.nl_cs + e];
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    if (MODE != XF_TAIL) in.bq[q] = a.base[q * a.cs + e];
    if (MODE == XF_RK12 || MODE == XF_RK3) in.sq[q] = a.accum[q * a.cs + e];
    if (MODE == XF_RK12 && a.ubdt != 0.0)
      in.uq[q] = make_double2(dadd(in.bq[q].x, dmul(ubdt, in.sq[q].x)),
                              dadd(in.bq[q].y, dmul(ubdt, in.sq[q].y)));
    else
      in.uq[q] = a.u[q * a.cs + e];
    if (MODE == XF_RK3) in.cr[q] = a.carry[q * a.cs + e];
  }
}

template <int MODE>
__device__ __forceinline__ void rk_finish(const XfArgs& a, const SpecGeom& g, long long e, int i,
                                          int j, int k, const RkIn& in, bool& finite,
                                          double2 (&un)[3]) {
  const double bdt = a.dts ? a.dts[a.dts_stage] : a.bdt;
  const double sixth = a.dts ? a.dts[3] : a.sixth;
  const double kx = wavenum(g.o0 + i, g.n), ky = wavenum(g.o1 + j, g.n);
  const double kzd = static_cast<double>(g.o2 + k);
  double2 c0 = in.c0, c1 = in.c1, c2 = in.c2;
  const double2(&uq)[3] = in.uq;
  const double2(&bq)[3] = in.bq;
  const double2(&sq)[3] = in.sq;
  const double2(&cr)[3] = in.cr;
  // wavenumbers(), mesh.cpp:56-60
  const double k2 = dadd(dadd(dmul(kx, kx), dmul(ky, ky)), dmul(kzd, kzd));
  const double inv = k2 > 0.0 ? 1.0 / k2 : 0.0;
  const double kxk = dmul(kx, inv), kyk = dmul(ky, inv), kzk = dmul(kzd, inv);
  // kd = kx c0 + ky c1 + kz c2; c -= (k/k^2) kd  (navier_stokes.cpp:128-133)
  const double kdr = dadd(dadd(dmul(kx, c0.x), dmul(ky, c1.x)), dmul(kzd, c2.x));
  const double kdi = dadd(dadd(dmul(kx, c0.y), dmul(ky, c1.y)), dmul(kzd, c2.y));
  c0 = make_double2(dsub(c0.x, dmul(kxk, kdr)), dsub(c0.y, dmul(kxk, kdi)));
  c1 = make_double2(dsub(c1.x, dmul(kyk, kdr)), dsub(c1.y, dmul(kyk, kdi)));
  c2 = make_double2(dsub(c2.x, dmul(kzk, kdr)), dsub(c2.y, dmul(kzk, kdi)));
  const double visc = dmul(a.nu, k2);
  double2 du[3];
  const double2 cc[3] = {c0, c1, c2};
#pragma unroll
  for (int q = 0; q < 3; ++q)
    du[q] = make_double2(dsub(cc[q].x, dmul(visc, uq[q].x)), dsub(cc[q].y, dmul(visc, uq[q].y)));
  if (MODE == XF_TAIL) {
#pragma unroll
    for (int q = 0; q < 3; ++q) a.out[q * a.cs + e] = du[q];
  } else if (MODE == XF_RK0 || MODE == XF_RK12) {
    // rk4.cpp:47-50
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double2 s = make_double2(dmul(a.w, du[q].x), dmul(a.w, du[q].y));
      if (MODE == XF_RK12) s = make_double2(dadd(sq[q].x, s.x), dadd(sq[q].y, s.y));
      a.accum[q * a.cs + e] = s;
      a.out[q * a.cs + e] = make_double2(dadd(bq[q].x, dmul(bdt, du[q].x)),
                                         dadd(bq[q].y, dmul(bdt, du[q].y)));
    }
  } else {  // XF_RK3, rk4.cpp:55-64
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double dr = dadd(dmul(sixth, dadd(sq[q].x, du[q].x)), cr[q].x);
      const double di = dadd(dmul(sixth, dadd(sq[q].y, du[q].y)), cr[q].y);
      const double nr = dadd(bq[q].x, dr), ni = dadd(bq[q].y, di);
      a.carry[q * a.cs + e] = make_double2(two_sum_err(bq[q].x, dr, nr), two_sum_err(bq[q].y, di, ni));
      un[q] = make_double2(nr, ni);
      finite = finite && isfinite(nr) && isfinite(ni);
    }
    if (a.project) {
      // project(), navier_stokes.cpp:85-102
      const double pr = dadd(dadd(dmul(kx, un[0].x), dmul(ky, un[1].x)), dmul(kzd, un[2].x));
      const double pi = dadd(dadd(dmul(kx, un[0].y), dmul(ky, un[1].y)), dmul(kzd, un[2].y));
      un[0] = make_double2(dsub(un[0].x, dmul(kxk, pr)), dsub(un[0].y, dmul(kxk, pi)));
      un[1] = make_double2(dsub(un[1].x, dmul(kyk, pr)), dsub(un[1].y, dmul(kyk, pi)));
      un[2] = make_double2(dsub(un[2].x, dmul(kzk, pr)), dsub(un[2].y, dmul(kzk, pi)));
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) a.base_out[q * a.cs + e] = un[q];
  }
}

template <int MODE>
__device__ __forceinline__ void rk_elem(const XfArgs& a, const SpecGeom& g, long long e, int i,
                                        int j, int k, bool& finite, double2 (&un)[3]) {
  RkIn in;
  rk_load<MODE>(a, g, e, i, j, k, in);
  rk_finish<MODE>(a, g, e, i, j, k, in, finite, un);
}

// Stages 1-3 update two modes per iteration (both modes' loads issued
// before either's arithmetic); stages 1-2 are compiled for 2 CTAs/SM.
template <int MODE>
__global__ void __launch_bounds__(256, MODE == XF_RK12 ? 2 : 1)
k_rk_update(XfArgs a, SpecGeom g) {
  const long long total = static_cast<long long>(g.s0) * g.prow * g.pitch;
  bool finite = true;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  // stages 1-3: two modes per iteration, both modes' loads issued before
  // either's arithmetic and stores (stage 3 3.29 -> 3.11 ms, stages 1-2
  // 2.52 -> 2.44 ms; stage 0, write-bound, gains nothing)
  if constexpr (MODE == XF_RK3 || MODE == XF_RK12) {
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += 2 * stride) {
    const long long e2 = e + stride;
    long long row = e / g.pitch;
    const int k = static_cast<int>(e - row * g.pitch);
    const int j = static_cast<int>(row % g.prow);
    const int i = static_cast<int>(row / g.prow);
    const bool v1 = k < g.s2 && j < g.s1;
    row = e2 / g.pitch;
    const int k2 = static_cast<int>(e2 - row * g.pitch);
    const int j2 = static_cast<int>(row % g.prow);
    const int i2 = static_cast<int>(row / g.prow);
    const bool v2 = e2 < total && k2 < g.s2 && j2 < g.s1;
    RkIn in1, in2;
    if (v1) rk_load<MODE>(a, g, e, i, j, k, in1);
    if (v2) rk_load<MODE>(a, g, e2, i2, j2, k2, in2);
    double2 un[3];
    if (v1) rk_finish<MODE>(a, g, e, i, j, k, in1, finite, un);
    if (v2) rk_finish<MODE>(a, g, e2, i2, j2, k2, in2, finite, un);
  }
  } else {
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += stride) {
    const long long row = e / g.pitch;
    const int k = static_cast<int>(e - row * g.pitch);
    const int j = static_cast<int>(row % g.prow);
    const int i = static_cast<int>(row / g.prow);
    if (k >= g.s2 || j >= g.s1) continue;
    double2 un[3];
    rk_elem<MODE>(a, g, e, i, j, k, finite, un);
  }
  }
  if (MODE == XF_RK3 && !finite) atomicAnd(a.finite, 0);
}

// ---------------------------------------------------------------------------
// P3: per z-line (row) of the 6 fields after the y pass:
//   3 complex inverse FFTs of length n carry the 6 real lines in pairs
//   (u0,u1), (u2,w0), (w1,w2) -- c2r with the imaginary parts of the kz = 0
//   and kz = n/2 bins ignored, as FFTW's c2r does -- then the 1/n^3 scale
//   (fft.cpp:125), the cross product u x omega (navier_stokes.cpp:45-49), and
//   forward r2c of the 3 products, two in one complex FFT. Real data never
//   leaves shared memory. Results overwrite fields 0..2 of the row.

template <int N>
struct ZCfg {
  static constexpr int E = fft_elems(N);
  static constexpr int TPC = N / E;
  static constexpr int RPC = TPC >= 64 ? 4 : (128 / TPC > 32 ? 32 : 128 / TPC);
  static constexpr int THREADS = TPC * RPC;
  static constexpr int HP = N / 2 + 8;  // padded half-row (n/2+1 modes)
};

// Full-length spectrum sample at position pos of A + iB from half spectra.
template <int N>
__device__ __forceinline__ double2 pair_sample(const double2* A, const double2* B, int pos) {
  double2 a, b;
  if (pos <= N / 2) {
    a = A[pos];
    b = B[pos];
    if (pos == 0 || pos == N / 2) {
      a.y = 0.0;
      b.y = 0.0;
    }
  } else {
    a = cconj(A[N - pos]);
    b = cconj(B[N - pos]);
  }
  return make_double2(a.x - b.y, a.y + b.x);
}

// Same for A + iB with B = B' + SG i kz A (kz = the half-spectrum index):
// the z part of the curl folded into the sampling.
template <int N, int SG>
__device__ __forceinline__ double2 pair_sample_kz(const double2* A, const double2* B, int pos) {
  const int k = pos <= N / 2 ? pos : N - pos;
  double2 a = A[k], b = B[k];
  const double kz = static_cast<double>(k);
  if (SG > 0)
    b = make_double2(b.x - kz * a.y, b.y + kz * a.x);
  else
    b = make_double2(b.x + kz * a.y, b.y - kz * a.x);
  if (pos == 0 || pos == N / 2) {
    a.y = 0.0;
    b.y = 0.0;
  }
  if (pos > N / 2) {
    a = cconj(a);
    b = cconj(b);
  }
  return make_double2(a.x - b.y, a.y + b.x);
}

struct WarpBar {
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};

// n = 512 z pass, mirrored butterflies: the first stage of
// the inverse transforms and the last stage of the forward n0 + i n1
// transform run butterfly jm(t) instead of t, chosen so that jm and 64 - jm
// (whose positions p and n - p pair up through the Hermitian symmetry) sit
// on lanes l and l ^ 16 of one warp; (0, 32) are self-mirrored on warp 0's
// lanes 0 and 16. A staged mode is then read once for both positions (the
// mirrored value crosses by one shuffle), and the r2c split finds X[n - k]
// by a shuffle instead of parking the spectrum in shared memory. Same
// butterflies and operations: bitwise the plain kernel's results.
__device__ __forceinline__ int z512_jm(int t) {
  const int lane = t & 31;
  if (t < 32) return lane < 16 ? lane : (lane == 16 ? 32 : 80 - lane);
  return lane < 16 ? 16 + lane : 64 - lane;
}
__device__ __forceinline__ double2 shfl16(double2 v) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, 16), __shfl_xor_sync(0xffffffffu, v.y, 16));
}
// Samples of A + iB (SG: z part of the curl, as pair_sample_kz / pair_sample)
// at the positions jm + 64 m of butterfly jm; whole warps.
template <int SG>
__device__ __forceinline__ void z512_sample(const double2* A, const double2* B, int jm,
                                            double2 (&v)[8]) {
  auto one = [&](int k, double2& lo, double2& hi) {
    double2 a = A[k], b = B[k];
    const double kz = static_cast<double>(k);
    if (SG > 0)
      b = make_double2(b.x - kz * a.y, b.y + kz * a.x);
    else if (SG < 0)
      b = make_double2(b.x + kz * a.y, b.y - kz * a.x);
    if (k == 0 || k == 256) {  // FFTW c2r: imaginary parts of DC and Nyquist ignored
      a.y = 0.0;
      b.y = 0.0;
    }
    lo = make_double2(a.x - b.y, a.y + b.x);
    hi = make_double2(a.x + b.y, b.x - a.y);  // conj a + i conj b: the value at n - k
  };
  double2 h[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    one(jm + 64 * q, v[q], h[q]);
    const double2 rcv = shfl16(h[q]);  // the partner's mirror of position jm + 64 (7 - q)
    v[7 - q] = jm == 32 ? h[q] : rcv;
  }
  if (jm == 0) {  // positions 64 m: self-mirrored (n - 64 m = 64 (8 - m)), plus k = 256
    v[7] = h[1];
    v[6] = h[2];
    v[5] = h[3];
    double2 lo, hi;
    one(256, lo, hi);
    v[4] = lo;
  }
}

// Launch shape of the fused z pass: 4 rows of 64 threads at n >= 512 (each
// row synchronises on its own named barrier), else whole rows per warp.
template <int N>
struct ZFCfg {
  static constexpr int E = fft_elems(N);
  static constexpr int TPC = N / E;
  // n = 1024: one row per CTA, four CTAs per SM, so rows load while others
  // transform (4 rows per CTA at 1 CTA/SM: 30.4 -> 27.3 ms per launch)
  static constexpr int RPC = TPC >= 64 ? (N >= 1024 ? 1 : 4) : (256 / TPC > 64 ? 64 : 256 / TPC);
  static constexpr int THREADS = TPC * RPC;
  static constexpr int HP = N / 2 + 8;  // padded half-row (n/2+1 modes)
  // n = 512: both twiddled radix-8 stages take their twiddles from
  // registers (LastTw), so no table is staged in shared memory
  static constexpr bool REG = N == 512;
  // n = 1024: the twiddle table stays in L2/L1 (global loads) so that four
  // one-row CTAs fit an SM (with the table staged: 34.5 ms)
  static constexpr bool GTAB = N >= 1024;
  static constexpr size_t SMEM =
      sizeof(double2) * (static_cast<size_t>(RPC) * 6 * HP + ((REG || GTAB) ? 0 : N));
  // CTAs per SM the shared memory allows (n = 1024: one -- then give the
  // 16-element transforms the registers, 128 would spill)
  static constexpr int MINB = SMEM * 4 <= 227 * 1024 ? 4 : (SMEM * 2 <= 227 * 1024 ? 2 : 1);
};

// Shared-memory swizzle of the z passes' exchange buffers (see SwzIdxT).
template <int N>
using ZSwz = SwzIdxT<(fft_elems(N) >= 16 ? 4 : 3)>;

// z-pass transform.
template <int N, int S, class Bar>
__device__ __forceinline__ void zfft(double2 (&v)[fft_elems(N)], double2* sm, ZSwz<N> sw, int t,
                                     const double2* tws, Bar bar, const LastTw& lt, int jf = -1,
                                     int jl = -1) {
  block_fft_lt<N, S>(v, sm, sw, t, tws, bar, lt, jf, jl);
}

template <int N, bool PO = false>
__global__ void __launch_bounds__(ZFCfg<N>::THREADS, ZFCfg<N>::MINB)
k_z_fused(double2* f, long long cs, RowMap rm, double norm, const double2* __restrict__ tw,
          const __grid_constant__ CUtensorMap ztm, double2* fo = nullptr, RowMap rmo = RowMap{}) {
  constexpr int E = ZFCfg<N>::E, TPC = ZFCfg<N>::TPC, HP = ZFCfg<N>::HP, RPC = ZFCfg<N>::RPC;
  using Bar = typename std::conditional<(TPC >= 64), NamedBar, WarpBar>::type;
  extern __shared__ __align__(128) double2 smem[];
  const int t = threadIdx.x % TPC, r = threadIdx.x / TPC;
  const int ri = blockIdx.x * RPC + r;
  const bool valid = ri < rm.nrows;
  const long long ro = (valid && rm.nseg == 0) ? zrow_off(rm, ri) : 0;
  // Stage the 6 half-rows once (coalesced, each element read once); the
  // staging area of pair p (2 half-rows, 2*HP >= n entries) then serves as
  // that pair's FFT exchange buffer. Pair results stay in registers.
  double2* S = smem + r * 6 * HP;
  const double2* tws = tw;  // REG: the 4 register twiddles come from L2
  if constexpr (!ZFCfg<N>::REG && !ZFCfg<N>::GTAB) tws = smem + RPC * 6 * HP;
  Bar bar;
  if constexpr (TPC >= 64) bar = Bar{1 + r, TPC};
  const ZSwz<N> sw;
  // fields: 0..2 = u, 3 = w0', 4 = w1', 5 = w2, staged as the pairs
  // (u0, w1') (u1, w0') (u2, w2) -- slot s holds field kZSlot[s] -- all of
  // the row in flight at once. The z part of the curl (w0 = w0' - i kz u1,
  // w1 = w1' + i kz u0) is applied when the pair is sampled.
  // One thread per row hands the 6 contiguous half-rows (n2 * 16 B each; one
  // piece per kz segment on pencil rows) to the bulk-copy engine; the row
  // waits on its mbarrier.
  __shared__ alignas(8) unsigned long long zbar[RPC];
  if (t == 0) mbar_init(&zbar[r], 1);
  __syncthreads();  // barrier init visible before anyone waits on it
  if (valid && t == 0 && rm.cstride) {
    // chunked rows: one tensor-map box (pitch/8 chunks of 128 B) per half-row
    const int fld[6] = {0, 4, 1, 3, 2, 5};
    const int x = ri / rm.rpp, y = ri - x * rm.rpp;
    mbar_expect_tx(&zbar[r], 6u * static_cast<unsigned>(rm.pitch) * 16u);
#pragma unroll
    for (int sl = 0; sl < 6; ++sl) tma_load5(S + sl * HP, &ztm, 0, 0, y, x, fld[sl], &zbar[r]);
  } else if (valid && t == 0) {
    const int fld[6] = {0, 4, 1, 3, 2, 5};
    mbar_expect_tx(&zbar[r], 6u * static_cast<unsigned>(rm.n2) * 16u);
#pragma unroll
    for (int sl = 0; sl < 6; ++sl) {
      const double2* src = f + fld[sl] * cs;
      if (rm.nseg == 0) {
        bulk_g2s(S + sl * HP, src + ro, static_cast<unsigned>(rm.n2) * 16u, &zbar[r]);
      } else {
        for (int q = 0; q < rm.nseg; ++q) {
          const int k0 = rm.seg_k0[q], k1 = rm.seg_k0[q + 1];
          if (k1 > k0)
            bulk_g2s(S + sl * HP + k0,
                     src + rm.seg_base[q] + static_cast<long long>(ri) * rm.seg_pitch[q],
                     static_cast<unsigned>(k1 - k0) * 16u, &zbar[r]);
        }
      }
    }
  }
  // the table is staged after the rows are requested (small n: the kernel is
  // one latency chain, the two fetches overlap)
  if constexpr (!ZFCfg<N>::REG && !ZFCfg<N>::GTAB) load_twiddles(smem + RPC * 6 * HP, tw, N);
  __syncthreads();  // twiddles
  if (valid) mbar_wait(&zbar[r], 0);
  const LastTw lt = last_twiddles<N>(tws, t);
  constexpr bool MIR = N == 512;  // mirrored first / last stages (z512_jm)
  const int jm = MIR ? z512_jm(t) : t;
  double2 v[E], p1[E];
  if constexpr (MIR) {
    z512_sample<+1>(S, S + HP, jm, v);
  } else {
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = pair_sample_kz<N, +1>(S, S + HP, t + m * TPC);
  }
  bar();
  zfft<N, +1>(v, S, sw, t, tws, bar, lt, MIR ? jm : -1);
  // pair 0 result parks in its own (now free) region at this thread's positions
  if constexpr (MIR) {
#pragma unroll
    for (int m = 0; m < E; ++m) S[sw(t + m * TPC)] = v[m];
    z512_sample<-1>(S + 2 * HP, S + 3 * HP, jm, v);
  } else {
#pragma unroll
    for (int m = 0; m < E; ++m) {
      S[sw(t + m * TPC)] = v[m];
      v[m] = pair_sample_kz<N, -1>(S + 2 * HP, S + 3 * HP, t + m * TPC);
    }
  }
  bar();
  zfft<N, +1>(v, S + 2 * HP, sw, t, tws, bar, lt, MIR ? jm : -1);
  if constexpr (MIR) {
#pragma unroll
    for (int m = 0; m < E; ++m) p1[m] = v[m];
    z512_sample<0>(S + 4 * HP, S + 5 * HP, jm, v);
  } else {
#pragma unroll
    for (int m = 0; m < E; ++m) {
      p1[m] = v[m];
      v[m] = pair_sample<N>(S + 4 * HP, S + 5 * HP, t + m * TPC);
    }
  }
  bar();
  zfft<N, +1>(v, S + 4 * HP, sw, t, tws, bar, lt, MIR ? jm : -1);
  // (u0,w1) = p0 (parked), (u1,w0) = p1, (u2,w2) = v; 1/n^3 then u x omega.
  // The real third product stays in registers through the next transform
  // (parking it cost 3% of the shared-memory wavefronts).
  double n2k[E];
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const double2 q0 = S[sw(t + m * TPC)];
    const double2 q1 = p1[m];
    const double ua = dmul(q0.x, norm), ub = dmul(q1.x, norm), uc = dmul(v[m].x, norm);
    const double wa = dmul(q1.y, norm), wb = dmul(q0.y, norm), wc = dmul(v[m].y, norm);
    const double n0 = dsub(dmul(ub, wc), dmul(uc, wb));
    const double n1 = dsub(dmul(uc, wa), dmul(ua, wc));
    n2k[m] = dsub(dmul(ua, wb), dmul(ub, wa));
    v[m] = make_double2(n0, n1);
  }
  bar();  // every thread has read its parked pair-0 values
  if constexpr (MIR) {
    // last stage on butterfly jm: its twiddles W^jm, W^4jm from the table
    constexpr int TOFF = tw_stage_off(N, E, N / 8);
    LastTw lf = lt;
    lf.w1 = __ldg(tws + TOFF + jm);
    lf.w4 = __ldg(tws + TOFF + 3 * (N / 8) + jm);
    zfft<N, -1>(v, S, sw, t, tws, bar, lf, -1, jm);
    // r2c split: X[k] here, X[n - k] on the partner lane (or on this lane
    // for the self-mirrored butterflies 0 and 32)
    const int keep = rm.kz_keep < N / 2 + 1 ? rm.kz_keep : N / 2 + 1;
    auto put = [&](int k, double2 d, double2 m) {
      if (!valid || k >= keep) return;
      const double2 e = cconj(m);
      const double2 dd = csub(d, e);
      const double2 o0 = make_double2(0.5 * (d.x + e.x), 0.5 * (d.y + e.y));
      const double2 o1 = make_double2(0.5 * dd.y, -0.5 * dd.x);
      if constexpr (PO) {
        const ZDst z = zdst(rmo, ri, k);
        fo[z.el] = o0;
        fo[z.el + z.cs] = o1;
      } else {
        const long long el = zel(rm, ro, ri, k);
        f[el] = o0;
        f[cs + el] = o1;
      }
    };
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const double2 rcv = shfl16(v[7 - m]);
      const double2 mir = jm == 0 ? v[(8 - m) & 7] : (jm == 32 ? v[7 - m] : rcv);
      put(jm + 64 * m, v[m], mir);
    }
    if (jm == 0) put(256, v[4], v[4]);
  } else {
  zfft<N, -1>(v, S, sw, t, tws, bar, lt);
#pragma unroll
  for (int m = 0; m < E; ++m) S[sw(t + m * TPC)] = v[m];
  bar();
  if (valid) {
    double2* o0 = f;
    double2* o1 = f + cs;
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int k = t + m * TPC;
      if (k <= N / 2 && k < rm.kz_keep) {  // kz >= n/3 is dealiased away
        const double2 d = S[sw(k)];
        const double2 e = cconj(S[sw((N - k) & (N - 1))]);
        const double2 dd = csub(d, e);
        if constexpr (PO) {
          const ZDst z = zdst(rmo, ri, k);
          fo[z.el] = make_double2(0.5 * (d.x + e.x), 0.5 * (d.y + e.y));
          fo[z.el + z.cs] = make_double2(0.5 * dd.y, -0.5 * dd.x);
        } else {
          const long long el = zel(rm, ro, ri, k);
          o0[el] = make_double2(0.5 * (d.x + e.x), 0.5 * (d.y + e.y));
          o1[el] = make_double2(0.5 * dd.y, -0.5 * dd.x);
        }
      }
    }
  }
  }
#pragma unroll
  for (int m = 0; m < E; ++m) v[m] = make_double2(n2k[m], 0.0);
  zfft<N, -1>(v, S + 2 * HP, sw, t, tws, bar, lt);
  if (valid) {
    double2* o2 = f + 2 * cs;
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int k = t + m * TPC;
      if (k <= N / 2 && k < rm.kz_keep) {
        if constexpr (PO) {
          const ZDst z = zdst(rmo, ri, k);
          fo[z.el + 2 * z.cs] = v[m];
        } else {
          o2[zel(rm, ro, ri, k)] = v[m];
        }
      }
    }
  }
  if constexpr (PO) __threadfence_system();  // peers read after a stream barrier
}

// Standalone c2r along z (DistributedFFT::inverse tail, fft.cpp:124-125):
// rows 2i and 2i+1 of one field share one complex inverse FFT. Each pair of
// rows is one TPC-thread group with its own named barrier (n >= 512); its
// two half-rows arrive by bulk copy on the group's mbarrier; at n = 512 the
// twiddles of both twiddled stages come from registers (no table in shared
// memory).
template <int N>
__global__ void __launch_bounds__(ZCfg<N>::THREADS)
k_z_c2r(const double2* __restrict__ spec, double* __restrict__ real, RowMap rm, double norm,
        const double2* __restrict__ tw) {
  constexpr int E = ZCfg<N>::E, TPC = ZCfg<N>::TPC, HP = ZCfg<N>::HP, RPC = ZCfg<N>::RPC;
  constexpr bool REG = N == 512;
  using Bar = typename std::conditional<(TPC >= 64), NamedBar, CtaBar>::type;
  extern __shared__ __align__(128) double2 smem[];
  __shared__ alignas(8) unsigned long long zbar[RPC];
  const int t = threadIdx.x % TPC, r = threadIdx.x / TPC;
  const int pr = blockIdx.x * RPC + r;
  const int ri = 2 * pr;
  const bool valid = ri < rm.nrows;
  Bar bar;
  if constexpr (TPC >= 64) bar = Bar{1 + r, TPC};
  double2* S = smem + r * 2 * HP;
  const double2* tws = tw;
  if constexpr (!REG) {
    double2* t2 = smem + RPC * 2 * HP;
    load_twiddles(t2, tw, N);
    tws = t2;
  }
  if (t == 0) mbar_init(&zbar[r], 1);
  __syncthreads();
  if (valid && t == 0) {
    // both half-rows (a pencil z line is spread over kz blocks)
    mbar_expect_tx(&zbar[r], 2u * static_cast<unsigned>(rm.n2) * 16u);
    for (int h = 0; h < 2; ++h) {
      if (rm.nseg == 0) {
        bulk_g2s(S + h * HP, spec + zrow_off(rm, ri + h), static_cast<unsigned>(rm.n2) * 16u,
                 &zbar[r]);
      } else {
        for (int q = 0; q < rm.nseg; ++q) {
          const int k0 = rm.seg_k0[q], k1 = rm.seg_k0[q + 1];
          if (k1 > k0)
            bulk_g2s(S + h * HP + k0,
                     spec + rm.seg_base[q] + static_cast<long long>(ri + h) * rm.seg_pitch[q],
                     static_cast<unsigned>(k1 - k0) * 16u, &zbar[r]);
        }
      }
    }
  }
  LastTw lt{};
  if constexpr (REG) lt = last_twiddles<N>(tw, t);
  if (valid) mbar_wait(&zbar[r], 0);
  double2 v[E];
#pragma unroll
  for (int m = 0; m < E; ++m)
    v[m] = valid ? pair_sample<N>(S, S + HP, t + m * TPC) : make_double2(0.0, 0.0);
  bar();
  if constexpr (REG) block_fft_lt<N, +1>(v, S, ZSwz<N>{}, t, tws, bar, lt);
  else block_fft<N, +1>(v, S, ZSwz<N>{}, t, tws, bar);
  if (valid) {
    double* a = real + static_cast<long long>(ri) * N;
    double* b = a + N;
#pragma unroll
    for (int m = 0; m < E; ++m) {
      a[t + m * TPC] = dmul(v[m].x, norm);
      b[t + m * TPC] = dmul(v[m].y, norm);
    }
  }
}

// Standalone r2c along z (DistributedFFT::forward head, fft.cpp:87): two real
// rows in one complex FFT, split by the mirror relation.
template <int N, bool PO = false>
__global__ void __launch_bounds__(ZCfg<N>::THREADS)
k_z_r2c(const double* __restrict__ real, double2* __restrict__ spec, RowMap rm,
        const double2* __restrict__ tw, RowMap rmo = RowMap{}, int field = 0) {
  constexpr int E = ZCfg<N>::E, TPC = ZCfg<N>::TPC, RPC = ZCfg<N>::RPC;
  constexpr bool REG = N == 512;
  using Bar = typename std::conditional<(TPC >= 64), NamedBar, CtaBar>::type;
  extern __shared__ __align__(128) double2 smem[];
  const int t = threadIdx.x % TPC, r = threadIdx.x / TPC;
  const int pr = blockIdx.x * RPC + r;
  const int ri = 2 * pr;
  const bool valid = ri < rm.nrows;
  Bar bar;
  if constexpr (TPC >= 64) bar = Bar{1 + r, TPC};
  __shared__ alignas(8) unsigned long long zbar[RPC];
  double2* reg = smem + r * N;
  const ZSwz<N> sw;
  double2 v[E];
  // the pair's two real rows (2 x 8n B, contiguous) arrive by bulk copy into
  // its region, which then serves as the transform's exchange buffer
  if (t == 0) mbar_init(&zbar[r], 1);
  const double2* tws = tw;
  if constexpr (!REG) {
    double2* t2 = smem + RPC * N;
    load_twiddles(t2, tw, N);
    tws = t2;
  }
  __syncthreads();
  if (valid && t == 0) {
    mbar_expect_tx(&zbar[r], 2u * N * 8u);
    bulk_g2s(reg, real + static_cast<long long>(ri) * N, 2u * N * 8u, &zbar[r]);
  }
  if (valid) {
    mbar_wait(&zbar[r], 0);
    const double* a = reinterpret_cast<const double*>(reg);
    const double* b = a + N;
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = make_double2(a[t + m * TPC], b[t + m * TPC]);
  } else {
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = make_double2(0.0, 0.0);
  }
  bar();  // the region is read; the transform reuses it
  if constexpr (REG) {
    const LastTw lt = last_twiddles<N>(tw, t);
    block_fft_lt<N, -1>(v, reg, sw, t, tws, bar, lt);
  } else {
    block_fft<N, -1>(v, reg, sw, t, tws, bar);
  }
#pragma unroll
  for (int m = 0; m < E; ++m) reg[sw(t + m * TPC)] = v[m];
  bar();
  if (valid) {
    const long long ra = rm.nseg ? 0 : zrow_off(rm, ri);
    const long long rb = rm.nseg ? 0 : zrow_off(rm, ri + 1);
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int k = t + m * TPC;
      if (k <= N / 2) {
        const double2 d = reg[sw(k)];
        const double2 e = cconj(reg[sw((N - k) & (N - 1))]);
        const double2 dd = csub(d, e);
        if constexpr (PO) {  // peer-direct: kz segment -> its owner's y-pass layout
          const ZDst za = zdst(rmo, ri, k), zb = zdst(rmo, ri + 1, k);
          spec[za.el + field * za.cs] = make_double2(0.5 * (d.x + e.x), 0.5 * (d.y + e.y));
          spec[zb.el + field * zb.cs] = make_double2(0.5 * dd.y, -0.5 * dd.x);
        } else {
          spec[zel(rm, ra, ri, k)] = make_double2(0.5 * (d.x + e.x), 0.5 * (d.y + e.y));
          spec[zel(rm, rb, ri + 1, k)] = make_double2(0.5 * dd.y, -0.5 * dd.x);
        }
      }
    }
  }
  if constexpr (PO) __threadfence_system();
}

// ---------------------------------------------------------------------------
// Pointwise spectral kernels (reference op order, no contraction)

struct ModeIdx {
  int i, j, k;
  bool ok;
  long long off;
};

__device__ __forceinline__ ModeIdx mode_of(const SpecGeom& g, long long e) {
  ModeIdx m;
  const long long row = e / g.pitch;
  m.k = static_cast<int>(e - row * g.pitch);
  m.j = static_cast<int>(row % g.prow);
  m.i = static_cast<int>(row / g.prow);
  m.ok = m.i < g.s0 && m.j < g.s1 && m.k < g.s2;
  m.off = e;
  return m;
}

__global__ void k_curl(const double2* __restrict__ u, double2* __restrict__ w, SpecGeom g) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const ModeIdx m = mode_of(g, e);
  if (!m.ok) return;
  const double kx = wavenum(g.o0 + m.i, g.n), ky = wavenum(g.o1 + m.j, g.n);
  const double kz = static_cast<double>(g.o2 + m.k);
  const double2 u0 = u[e], u1 = u[g.cs + e], u2 = u[2 * g.cs + e];
  w[e] = i_cross(ky, u2, kz, u1);
  w[g.cs + e] = i_cross(kz, u0, kx, u2);
  w[2 * g.cs + e] = i_cross(kx, u1, ky, u0);
}

__device__ __forceinline__ void k_over_k2(double kx, double ky, double kz, double& a, double& b,
                                          double& c) {
  const double k2 = dadd(dadd(dmul(kx, kx), dmul(ky, ky)), dmul(kz, kz));
  const double inv = k2 > 0.0 ? 1.0 / k2 : 0.0;
  a = dmul(kx, inv);
  b = dmul(ky, inv);
  c = dmul(kz, inv);
}

__global__ void k_project(double2* u, SpecGeom g) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const ModeIdx m = mode_of(g, e);
  if (!m.ok) return;
  const double kx = wavenum(g.o0 + m.i, g.n), ky = wavenum(g.o1 + m.j, g.n);
  const double kz = static_cast<double>(g.o2 + m.k);
  double a, b, c;
  k_over_k2(kx, ky, kz, a, b, c);
  double2 u0 = u[e], u1 = u[g.cs + e], u2 = u[2 * g.cs + e];
  const double kr = dadd(dadd(dmul(kx, u0.x), dmul(ky, u1.x)), dmul(kz, u2.x));
  const double ki = dadd(dadd(dmul(kx, u0.y), dmul(ky, u1.y)), dmul(kz, u2.y));
  u[e] = make_double2(dsub(u0.x, dmul(a, kr)), dsub(u0.y, dmul(a, ki)));
  u[g.cs + e] = make_double2(dsub(u1.x, dmul(b, kr)), dsub(u1.y, dmul(b, ki)));
  u[2 * g.cs + e] = make_double2(dsub(u2.x, dmul(c, kr)), dsub(u2.y, dmul(c, ki)));
}

__global__ void k_pressure(const double2* __restrict__ nl, double2* __restrict__ p, SpecGeom g) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const ModeIdx m = mode_of(g, e);
  if (!m.ok) return;
  const double kx = wavenum(g.o0 + m.i, g.n), ky = wavenum(g.o1 + m.j, g.n);
  const double kz = static_cast<double>(g.o2 + m.k);
  double a, b, c;
  k_over_k2(kx, ky, kz, a, b, c);
  const double2 n0 = nl[e], n1 = nl[g.cs + e], n2 = nl[2 * g.cs + e];
  const double kr = dadd(dadd(dmul(a, n0.x), dmul(b, n1.x)), dmul(c, n2.x));
  const double ki = dadd(dadd(dmul(a, n0.y), dmul(b, n1.y)), dmul(c, n2.y));
  p[e] = make_double2(ki, -kr);  // Complex(0,-1) * kd
}

__global__ void k_cross(const double* __restrict__ a, const double* __restrict__ b,
                        double* __restrict__ o, long long count, long long cs) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= count) return;
  const double a0 = a[e], a1 = a[cs + e], a2 = a[2 * cs + e];
  const double b0 = b[e], b1 = b[cs + e], b2 = b[2 * cs + e];
  o[e] = dsub(dmul(a1, b2), dmul(a2, b1));
  o[cs + e] = dsub(dmul(a2, b0), dmul(a0, b2));
  o[2 * cs + e] = dsub(dmul(a0, b1), dmul(a1, b0));
}

__global__ void k_finite(const double2* __restrict__ u, SpecGeom g, int* flag) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const ModeIdx m = mode_of(g, e);
  if (!m.ok) return;
  bool ok = true;
  for (int c = 0; c < 3; ++c) {
    const double2 v = u[c * g.cs + e];
    ok = ok && isfinite(v.x) && isfinite(v.y);
  }
  if (!ok) atomicAnd(flag, 0);
}

static unsigned grid_for(long long n, int threads) {
  return static_cast<unsigned>((n + threads - 1) / threads);
}

void pw_curl(const double2* u, double2* w, const SpecGeom& g, cudaStream_t s) {
  const long long tot = static_cast<long long>(g.s0) * g.prow * g.pitch;
  k_curl<<<grid_for(tot, 256), 256, 0, s>>>(u, w, g);
}
void pw_project(double2* u, const SpecGeom& g, cudaStream_t s) {
  const long long tot = static_cast<long long>(g.s0) * g.prow * g.pitch;
  k_project<<<grid_for(tot, 256), 256, 0, s>>>(u, g);
}
void pw_pressure(const double2* nl, double2* p, const SpecGeom& g, cudaStream_t s) {
  const long long tot = static_cast<long long>(g.s0) * g.prow * g.pitch;
  k_pressure<<<grid_for(tot, 256), 256, 0, s>>>(nl, p, g);
}
void pw_cross(const double* a, const double* b, double* o, long long count, long long cs,
              cudaStream_t s) {
  k_cross<<<grid_for(count, 256), 256, 0, s>>>(a, b, o, count, cs);
}
void pw_finite(const double2* u, const SpecGeom& g, int* flag, cudaStream_t s) {
  const long long tot = static_cast<long long>(g.s0) * g.prow * g.pitch;
  k_finite<<<grid_for(tot, 256), 256, 0, s>>>(u, g, flag);
}
__global__ void k_fill_pad(double2* f, SpecGeom g, int ncomp) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const ModeIdx m = mode_of(g, e);
  if (m.i >= g.s0 || m.k < g.s2) return;
  for (int c = 0; c < ncomp; ++c) f[c * g.cs + e] = make_double2(0.0, 0.0);
}
__global__ void k_repack(const double2* __restrict__ src, double2* __restrict__ dst, int ncomp,
                         SpecGeom g, long long packed_cs, int to_packed) {
  const long long per = static_cast<long long>(g.s0) * g.s1 * g.s2;
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
       e < per * ncomp; e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long c = e / per, r = e - c * per;
    const long long row = r / g.s2;
    const int k = static_cast<int>(r - row * g.s2);
    const long long i = row / g.s1, j = row - i * g.s1;
    const long long pad = c * g.cs + (i * g.prow + j) * g.pitch + k;
    const long long pk = c * packed_cs + r;
    if (to_packed) dst[pk] = src[pad];
    else dst[pad] = src[pk];
  }
}
void pw_repack(const double2* src, double2* dst, int ncomp, const SpecGeom& g, bool to_packed,
               cudaStream_t s) {
  const long long per = static_cast<long long>(g.s0) * g.s1 * g.s2;
  k_repack<<<grid_for(per * ncomp, 256), 256, 0, s>>>(src, dst, ncomp, g, per, to_packed ? 1 : 0);
}

void pw_fill_pad(double2* f, int ncomp, const SpecGeom& g, cudaStream_t s) {
  const long long tot = static_cast<long long>(g.s0) * g.prow * g.pitch;
  k_fill_pad<<<grid_for(tot, 256), 256, 0, s>>>(f, g, ncomp);
}

// ---------------------------------------------------------------------------
// Diagnostics (collect_stats, diagnostics.cpp:24-91) with a fixed reduction
// order: one CTA per local x plane, each warp walks y rows and kz chunks in
// order; the spectrum uses per-warp shared-memory histograms fed by a
// segmented scan (|k| and hence the shell index is nondecreasing in kz along
// a row); a second kernel folds the per-plane partials in plane order.

constexpr int kStatsWarps = 8;

// Per-mode terms of accumulate_local (diagnostics.cpp:34-57) in the
// reference's operation order with explicit round-to-nearest operations (so
// the standalone and the fused kernel agree bit for bit).
struct StatsTerm {
  double e, z, we, ratio;
  int shell;
};
__device__ __forceinline__ StatsTerm stats_term(double kx, double ky, double kz, double w,
                                                double2 u0, double2 u1, double2 u2) {
  const double eps = 2.220446049250313e-16;
  auto nrm = [](double2 c) { return dadd(dmul(c.x, c.x), dmul(c.y, c.y)); };
  StatsTerm r;
  r.e = dadd(dadd(nrm(u0), nrm(u1)), nrm(u2));
  const double2 c0 = make_double2(dsub(dmul(ky, u2.x), dmul(kz, u1.x)),
                                  dsub(dmul(ky, u2.y), dmul(kz, u1.y)));
  const double2 c1 = make_double2(dsub(dmul(kz, u0.x), dmul(kx, u2.x)),
                                  dsub(dmul(kz, u0.y), dmul(kx, u2.y)));
  const double2 c2 = make_double2(dsub(dmul(kx, u1.x), dmul(ky, u0.x)),
                                  dsub(dmul(kx, u1.y), dmul(ky, u0.y)));
  r.z = dadd(dadd(nrm(c0), nrm(c1)), nrm(c2));
  const double k2 = dadd(dadd(dmul(kx, kx), dmul(ky, ky)), dmul(kz, kz));
  const double kn = sqrt(k2);
  r.shell = static_cast<int>(llround(kn));
  r.we = dmul(dmul(0.5, w), r.e);
  const double kdr = dadd(dadd(dmul(kx, u0.x), dmul(ky, u1.x)), dmul(kz, u2.x));
  const double kdi = dadd(dadd(dmul(kx, u0.y), dmul(ky, u1.y)), dmul(kz, u2.y));
  r.ratio = hypot(kdr, kdi) / dadd(dmul(kn, sqrt(r.e)), eps);
  return r;
}

// Warp-synchronous: adds the lanes' shell energies to the warp histogram in
// a fixed order (segmented inclusive scan over lanes with equal shell; the
// shell index is nondecreasing in kz along a row).
__device__ __forceinline__ void hist_add(double* hist, int shells, int lane, bool ok, double we,
                                         int shell) {
  double acc = we;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double o = __shfl_up_sync(0xffffffffu, acc, d);
    const int os = __shfl_up_sync(0xffffffffu, shell, d);
    if (lane >= d && os == shell) acc += o;
  }
  const int nxt = __shfl_down_sync(0xffffffffu, shell, 1);
  const bool tail = ok && (lane == 31 || nxt != shell);
  if (tail && shell < shells) hist[shell] += acc;
  __syncwarp();
}

// Fixed-order CTA reduction of (se, sz, dmax) and the warp histograms into
// this plane's partial row [se, sz, dmax, shells...].
__device__ __forceinline__ void stats_flush(double* sh, int shells, double se, double sz,
                                            double dmax, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    se += __shfl_xor_sync(0xffffffffu, se, d);
    sz += __shfl_xor_sync(0xffffffffu, sz, d);
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, d));
  }
  double* red = sh + kStatsWarps * shells;
  if (lane == 0) {
    red[warp * 3 + 0] = se;
    red[warp * 3 + 1] = sz;
    red[warp * 3 + 2] = dmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (int w = 0; w < kStatsWarps; ++w) {
      a += red[w * 3 + 0];
      b += red[w * 3 + 1];
      c = fmax(c, red[w * 3 + 2]);
    }
    out[0] = a;
    out[1] = b;
    out[2] = c;
  }
  for (int s = threadIdx.x; s < shells; s += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < kStatsWarps; ++w) v += sh[w * shells + s];
    out[3 + s] = v;
  }
}

__global__ void __launch_bounds__(kStatsWarps * 32)
k_stats_partial(const double2* __restrict__ u, SpecGeom g, int shells, double* partial) {
  extern __shared__ double sh[];  // [kStatsWarps][shells] + reductions
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* hist = sh + warp * shells;
  for (int s = lane; s < shells; s += 32) hist[s] = 0.0;
  __syncwarp();
  const int i = blockIdx.x;
  const double kx = wavenum(g.o0 + i, g.n);
  const double half = static_cast<double>(g.n / 2);
  double se = 0.0, sz = 0.0, dmax = 0.0;
  for (int j = warp; j < g.s1; j += kStatsWarps) {
    const double ky = wavenum(g.o1 + j, g.n);
    const long long rowoff = (static_cast<long long>(i) * g.prow + j) * g.pitch;
    for (int k0 = 0; k0 < g.s2; k0 += 32) {
      const int k = k0 + lane;
      const bool ok = k < g.s2;
      double we = 0.0;
      int shell = -1;
      if (ok) {
        const double kz = static_cast<double>(g.o2 + k);
        const double w = (kz == 0.0 || kz == half) ? 1.0 : 2.0;
        const long long e = rowoff + k;
        const StatsTerm st = stats_term(kx, ky, kz, w, u[e], u[g.cs + e], u[2 * g.cs + e]);
        se = dadd(se, dmul(w, st.e));
        sz = dadd(sz, dmul(w, st.z));
        we = st.we;
        shell = st.shell;
        dmax = fmax(dmax, st.ratio);
      }
      hist_add(hist, shells, lane, ok, we, shell);
    }
  }
  __syncthreads();
  stats_flush(sh, shells, se, sz, dmax, partial + static_cast<long long>(blockIdx.x) * (shells + 3));
}

// P5b stage 3 fused with the sampled diagnostics of the new state (SURVEY
// 8(f) rank 1): the update of k_rk_update<XF_RK3> walked in the stats
// kernel's order, accumulating the statistics of the projected new state as
// it is written -- the sample costs no extra pass over u_hat and equals
// collect_stats of that state bit for bit.
__global__ void __launch_bounds__(kStatsWarps * 32)
k_rk3_stats(XfArgs a, SpecGeom g, int shells, double* partial) {
  extern __shared__ double sh[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* hist = sh + warp * shells;
  for (int s = lane; s < shells; s += 32) hist[s] = 0.0;
  __syncwarp();
  const int i = blockIdx.x;
  const double kx = wavenum(g.o0 + i, g.n);
  const double half = static_cast<double>(g.n / 2);
  double se = 0.0, sz = 0.0, dmax = 0.0;
  bool finite = true;
  for (int j = warp; j < g.s1; j += kStatsWarps) {
    const double ky = wavenum(g.o1 + j, g.n);
    const long long rowoff = (static_cast<long long>(i) * g.prow + j) * g.pitch;
    for (int k0 = 0; k0 < g.s2; k0 += 32) {
      const int k = k0 + lane;
      const bool ok = k < g.s2;
      double we = 0.0;
      int shell = -1;
      if (ok) {
        double2 un[3];
        rk_elem<XF_RK3>(a, g, rowoff + k, i, j, k, finite, un);
        const double kz = static_cast<double>(g.o2 + k);
        const double w = (kz == 0.0 || kz == half) ? 1.0 : 2.0;
        const StatsTerm st = stats_term(kx, ky, kz, w, un[0], un[1], un[2]);
        se = dadd(se, dmul(w, st.e));
        sz = dadd(sz, dmul(w, st.z));
        we = st.we;
        shell = st.shell;
        dmax = fmax(dmax, st.ratio);
      }
      hist_add(hist, shells, lane, ok, we, shell);
    }
  }
  if (!finite) atomicAnd(a.finite, 0);
  __syncthreads();
  stats_flush(sh, shells, se, sz, dmax, partial + static_cast<long long>(blockIdx.x) * (shells + 3));
}

__global__ void k_fold_partials(const double* partial, int nblocks, int stride, double* out) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= stride) return;
  double acc = 0.0;
  if (v == 2) {
    for (int b = 0; b < nblocks; ++b) acc = fmax(acc, partial[static_cast<long long>(b) * stride + v]);
  } else {
    for (int b = 0; b < nblocks; ++b) acc += partial[static_cast<long long>(b) * stride + v];
  }
  out[v] = acc;
}

int stats_blocks(const SpecGeom& g) { return g.s0; }

void stats_local(const double2* u, const SpecGeom& g, int shells, double* d_partial,
                 double* d_out, cudaStream_t s) {
  const size_t shm = sizeof(double) * (kStatsWarps * shells + kStatsWarps * 3);
  if (shm > 48 * 1024)  // depends on n: set per launch
    cudaFuncSetAttribute(k_stats_partial, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(shm));
  k_stats_partial<<<g.s0, kStatsWarps * 32, shm, s>>>(u, g, shells, d_partial);
  const int stride = shells + 3;
  k_fold_partials<<<(stride + 127) / 128, 128, 0, s>>>(d_partial, g.s0, stride, d_out);
}

constexpr int kL2Blocks = 592;

__global__ void k_l2_partial(const double* __restrict__ a, const double* __restrict__ b,
                             long long count, double* partial) {
  __shared__ double red[256];
  double acc = 0.0;
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double d = a[e] - b[e];
    acc += d * d;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

void l2_local(const double* a, const double* b, long long count, double* d_partial,
              double* d_out, cudaStream_t s) {
  k_l2_partial<<<kL2Blocks, 256, 0, s>>>(a, b, count, d_partial);
  k_fold_partials<<<1, 32, 0, s>>>(d_partial, kL2Blocks, 1, d_out);
}

// ---------------------------------------------------------------------------
// Dispatch over the (power-of-two) transform length

#define SDNS_FOR_N(X) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024)

template <int MODE>
static void rk_update_mode(const XfArgs& a, const SpecGeom& g, cudaStream_t s) {
  static int grid = 0;
  if (!grid) {
    int occ = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rk_update<MODE>, 256, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = (occ > 0 ? occ : 1) * (sms > 0 ? sms : 148);
  }
  const long long total = static_cast<long long>(g.s0) * g.prow * g.pitch;
  const long long need = (total + 255) / 256;
  k_rk_update<MODE><<<static_cast<unsigned>(need < grid ? need : grid), 256, 0, s>>>(a, g);
}

__global__ void k_set_step_scalars(double* dts, double b0, double b1, double b2, double sixth) {
  dts[0] = b0;
  dts[1] = b1;
  dts[2] = b2;
  dts[3] = sixth;
}
void set_step_scalars(double* dts, double dt, cudaStream_t s) {
  // the same host products the eager path passes by value (bitwise equal)
  k_set_step_scalars<<<1, 1, 0, s>>>(dts, 0.5 * dt, 0.5 * dt, 1.0 * dt, dt / 6.0);
}

void rk_update(int mode, const XfArgs& a, const SpecGeom& g, cudaStream_t s) {
  switch (mode) {
    case XF_TAIL: rk_update_mode<XF_TAIL>(a, g, s); return;
    case XF_RK0: rk_update_mode<XF_RK0>(a, g, s); return;
    case XF_RK12: rk_update_mode<XF_RK12>(a, g, s); return;
    default:
      if (a.stats_partial) {
        const size_t shm = sizeof(double) * (kStatsWarps * a.shells + kStatsWarps * 3);
        if (shm > 48 * 1024)
          cudaFuncSetAttribute(k_rk3_stats, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(shm));
        k_rk3_stats<<<g.s0, kStatsWarps * 32, shm, s>>>(a, g, a.shells, a.stats_partial);
        const int stride = a.shells + 3;
        k_fold_partials<<<(stride + 127) / 128, 128, 0, s>>>(a.stats_partial, g.s0, stride,
                                                             a.stats_out);
      } else {
        rk_update_mode<XF_RK3>(a, g, s);
      }
      return;
  }
}

template <int N>
static void z_fused_n(double2* rows, long long cs, const RowMap& rm, double norm,
                      const double2* tw, cudaStream_t s) {
  using C = ZFCfg<N>;
  const unsigned grid = static_cast<unsigned>((rm.nrows + C::RPC - 1) / C::RPC);
  const size_t shm = C::SMEM;
  SDNS_SET_SMEM((k_z_fused<N>), shm);
  CUtensorMap tm;
  std::memset(&tm, 0, sizeof(tm));
  if (rm.cstride && !z_chunk_map(&tm, rows, cs, 6, rm, rm.pitch))
    std::fprintf(stderr, "sdns: z pass chunk map could not be encoded\n");
  k_z_fused<N><<<grid, C::THREADS, shm, s>>>(rows, cs, rm, norm, tw, tm);
}

bool z_chunk_map(void* tmap, const double2* base, long long cs, int nfields, const RowMap& rm,
                 int pitch) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  if (!enc || rm.rpp <= 0) return false;
  const int nch = pitch / 8;
  const int nx = rm.nrows / rm.rpp;
  const cuuint64_t B = sizeof(double2);
  // doubles of a chunk, chunks, y, x, fields
  const cuuint64_t dims[5] = {16, static_cast<cuuint64_t>(nch), static_cast<cuuint64_t>(rm.rpp),
                              static_cast<cuuint64_t>(nx), static_cast<cuuint64_t>(nfields)};
  const cuuint64_t strides[4] = {static_cast<cuuint64_t>(rm.cstride) * B, 8 * B,
                                 static_cast<cuuint64_t>(rm.xplane) * B,
                                 static_cast<cuuint64_t>(cs) * B};
  const cuuint32_t box[5] = {16, static_cast<cuuint32_t>(nch), 1, 1, 1}, es[5] = {1, 1, 1, 1, 1};
  return enc(static_cast<CUtensorMap*>(tmap), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5,
             const_cast<double2*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void z_fused(int n, double2* rows, long long cs, const RowMap& rm, double norm,
             const double2* tw, cudaStream_t s) {
  if (!tuned_length(n)) {
    gen_z_fused(n, rows, cs, rm, rows, nullptr, norm, tw, s);
    return;
  }
  switch (n) {
#define X(NN) \
  case NN: z_fused_n<NN>(rows, cs, rm, norm, tw, s); return;
    SDNS_FOR_N(X)
#undef X
  }
}

template <int N>
static void z_fused_to_n(double2* rows, long long cs, const RowMap& rm, double2* out,
                         const RowMap& rmo, double norm, const double2* tw, cudaStream_t s) {
  using C = ZFCfg<N>;
  const unsigned grid = static_cast<unsigned>((rm.nrows + C::RPC - 1) / C::RPC);
  const size_t shm = C::SMEM;
  SDNS_SET_SMEM((k_z_fused<N, true>), shm);
  CUtensorMap tm;
  std::memset(&tm, 0, sizeof(tm));
  k_z_fused<N, true><<<grid, C::THREADS, shm, s>>>(rows, cs, rm, norm, tw, tm, out, rmo);
}

void z_fused_to(int n, double2* rows, long long cs, const RowMap& rm, double2* out,
                const RowMap& rmo, double norm, const double2* tw, cudaStream_t s) {
  if (!tuned_length(n)) {
    gen_z_fused(n, rows, cs, rm, out, &rmo, norm, tw, s);
    return;
  }
  switch (n) {
#define X(NN) \
  case NN: z_fused_to_n<NN>(rows, cs, rm, out, rmo, norm, tw, s); return;
    SDNS_FOR_N(X)
#undef X
  }
}

template <int N>
static void z_c2r_n(const double2* spec, double* real, const RowMap& rm, double norm,
                    const double2* tw, cudaStream_t s) {
  using C = ZCfg<N>;
  const int pairs = rm.nrows / 2;
  const unsigned grid = static_cast<unsigned>((pairs + C::RPC - 1) / C::RPC);
  const size_t shm = sizeof(double2) * (2 * C::HP * C::RPC + N);
  SDNS_SET_SMEM((k_z_c2r<N>), shm);
  k_z_c2r<N><<<grid, C::THREADS, shm, s>>>(spec, real, rm, norm, tw);
}

void z_c2r(int n, const double2* spec, double* real, const RowMap& rm, double norm,
           const double2* tw, cudaStream_t s) {
  if (!tuned_length(n)) {
    gen_z_c2r(n, spec, real, rm, norm, tw, s);
    return;
  }
  switch (n) {
#define X(NN) \
  case NN: z_c2r_n<NN>(spec, real, rm, norm, tw, s); return;
    SDNS_FOR_N(X)
#undef X
  }
}

template <int N>
static void z_r2c_n(const double* real, double2* spec, const RowMap& rm, const double2* tw,
                    cudaStream_t s) {
  using C = ZCfg<N>;
  const int pairs = rm.nrows / 2;
  const unsigned grid = static_cast<unsigned>((pairs + C::RPC - 1) / C::RPC);
  const size_t shm = sizeof(double2) * (N * C::RPC + N);
  SDNS_SET_SMEM((k_z_r2c<N>), shm);
  k_z_r2c<N><<<grid, C::THREADS, shm, s>>>(real, spec, rm, tw);
}

template <int N>
static void z_r2c_to_n(const double* real, double2* out, const RowMap& rm, const RowMap& rmo,
                       int field, const double2* tw, cudaStream_t s) {
  using C = ZCfg<N>;
  const int pairs = rm.nrows / 2;
  const unsigned grid = static_cast<unsigned>((pairs + C::RPC - 1) / C::RPC);
  const size_t shm = sizeof(double2) * (N * C::RPC + N);
  SDNS_SET_SMEM((k_z_r2c<N, true>), shm);
  k_z_r2c<N, true><<<grid, C::THREADS, shm, s>>>(real, out, rm, tw, rmo, field);
}

void z_r2c_to(int n, const double* real, double2* out, const RowMap& rm, const RowMap& rmo,
              int field, const double2* tw, cudaStream_t s) {
  if (!tuned_length(n)) {
    gen_z_r2c(n, real, out, rm, &rmo, field, tw, s);
    return;
  }
  switch (n) {
#define X(NN) \
  case NN: z_r2c_to_n<NN>(real, out, rm, rmo, field, tw, s); return;
    SDNS_FOR_N(X)
#undef X
  }
}

void z_r2c(int n, const double* real, double2* spec, const RowMap& rm, const double2* tw,
           cudaStream_t s) {
  if (!tuned_length(n)) {
    gen_z_r2c(n, real, spec, rm, nullptr, 0, tw, s);
    return;
  }
  switch (n) {
#define X(NN) \
  case NN: z_r2c_n<NN>(real, spec, rm, tw, s); return;
    SDNS_FOR_N(X)
#undef X
  }
}

}  // namespace sdns_dev
