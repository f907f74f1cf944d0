// Device-side fp64 FFT building blocks for sm_100a.
//
// A length-N complex transform of one "column" is computed cooperatively by
// TPC = N/E threads, each holding E elements in registers. Thread t holds
// element m at position t + m*TPC both on entry and on exit (natural order),
// so the first stage reads and the last stage writes in exactly the pattern a
// coalesced global load/store wants. Between stages the data is exchanged
// through shared memory with a Stockham autosort step (no bit reversal):
//   stage radix R, sub-length NS: butterfly j in [0, N/R) reads positions
//   j + r*N/R, twiddles by W_{NS*R}^{(j mod NS)*r}, and writes
//   (j/NS)*NS*R + (j mod NS) + r*NS.
// Radices are E (8 or 16) until the remainder, which is a smaller power of
// two. Twiddles come from a per-length table tw[q] = exp(-2*pi*i*q/N) that
// each CTA copies to shared memory once, conjugated for the inverse.
// Unnormalised in both directions (FFTW convention, SerialFFT,
// proj/core/include/sdns/serial_fft.hpp:13-14).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

namespace sdns_dev {

// LDGSTS: 16-byte global->shared copy (zero-filled when !valid).
__device__ __forceinline__ void cp_async16(double2* dst, const double2* src, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
// Bulk-copy engine (TMA, SASS UBLKCP) global->shared copies completing on an
// mbarrier transaction count.
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// One 5-D tensor-map box into shared memory, completing on `bar`.
__device__ __forceinline__ void tma_load5(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                          int c3, int c4, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(smem_addr(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  }
}

// Orders this thread's generic-proxy shared-memory accesses before later
// async-proxy (bulk copy / TMA) accesses to the same addresses.
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void cp_wait2() { asm volatile("cp.async.wait_group 2;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }



__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by S*i (S = -1 forward, +1 inverse)
template <int S>
__device__ __forceinline__ double2 mul_si(double2 a) {
  return S < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

template <int S>
__device__ __forceinline__ double2 twiddle(const double2* __restrict__ tw, int q) {
  // tw is the shared-memory copy of the table (LDS, no LSU global traffic)
  const double2 w = tw[q];
  return S < 0 ? w : make_double2(w.x, -w.y);
}

// In-place DFT of R register values, output in natural order.
template <int R, int S>
struct Dft;

template <int S>
struct Dft<1, S> {
  __device__ __forceinline__ static void run(double2*) {}
};

template <int S>
struct Dft<2, S> {
  __device__ __forceinline__ static void run(double2* a) {
    const double2 t = a[1];
    a[1] = csub(a[0], t);
    a[0] = cadd(a[0], t);
  }
};

template <int S>
struct Dft<4, S> {
  __device__ __forceinline__ static void run(double2* a) {
    const double2 s02 = cadd(a[0], a[2]), d02 = csub(a[0], a[2]);
    const double2 s13 = cadd(a[1], a[3]), d13 = mul_si<S>(csub(a[1], a[3]));
    a[0] = cadd(s02, s13);
    a[2] = csub(s02, s13);
    a[1] = cadd(d02, d13);
    a[3] = csub(d02, d13);
  }
};

template <int S>
struct Dft<8, S> {
  __device__ __forceinline__ static void run(double2* a) {
    constexpr double H = 0.70710678118654752440;  // sqrt(1/2)
    double2 e[4] = {a[0], a[2], a[4], a[6]};
    double2 o[4] = {a[1], a[3], a[5], a[7]};
    Dft<4, S>::run(e);
    Dft<4, S>::run(o);
    // W8^1 = H(1 + S i), W8^2 = S i, W8^3 = H(-1 + S i)
    const double2 o1 = make_double2(H * (o[1].x - S * o[1].y), H * (o[1].y + S * o[1].x));
    const double2 o2 = mul_si<S>(o[2]);
    const double2 o3 = make_double2(H * (-o[3].x - S * o[3].y), H * (-o[3].y + S * o[3].x));
    a[0] = cadd(e[0], o[0]);
    a[4] = csub(e[0], o[0]);
    a[1] = cadd(e[1], o1);
    a[5] = csub(e[1], o1);
    a[2] = cadd(e[2], o2);
    a[6] = csub(e[2], o2);
    a[3] = cadd(e[3], o3);
    a[7] = csub(e[3], o3);
  }
};

template <int S>
struct Dft<16, S> {
  __device__ __forceinline__ static void run(double2* a) {
    // 16 = 2 x 8 decimation in time with W16^k = exp(S*2*pi*i*k/16).
    constexpr double C1 = 0.92387953251128675613;  // cos(pi/8)
    constexpr double S1 = 0.38268343236508977173;  // sin(pi/8)
    constexpr double H = 0.70710678118654752440;
    double2 e[8], o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      e[i] = a[2 * i];
      o[i] = a[2 * i + 1];
    }
    Dft<8, S>::run(e);
    Dft<8, S>::run(o);
    const double wr[8] = {1.0, C1, H, S1, 0.0, -S1, -H, -C1};
    const double wi[8] = {0.0, S1, H, C1, 1.0, C1, H, S1};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double2 w = make_double2(wr[k], S * wi[k]);
      const double2 t = (k == 0) ? o[0] : cmul(o[k], w);
      a[k] = cadd(e[k], t);
      a[k + 8] = csub(e[k], t);
    }
  }
};

// Elements held per thread for a transform of length N.
__host__ __device__ constexpr int fft_elems(int n) { return n >= 1024 ? 16 : (n >= 8 ? 8 : n); }

// Stage-ordered twiddle table. Stage NS (> 1) of radix R stores
// W_{NS*R}^{k*r} at off(NS) + (r-1)*NS + k, k in [0, NS), r in [1, R), so the
// lanes of a warp read consecutive (or identical) 16-byte entries: no bank
// conflicts, unlike strided reads of a single exp(-2 pi i q / n) table.
__host__ __device__ constexpr int tw_stage_off(int n, int e, int ns_target) {
  int off = 0;
  for (int ns = 1; ns < ns_target;) {
    const int rem = n / ns;
    const int r = rem >= e ? e : rem;
    if (ns > 1) off += ns * (r - 1);
    ns *= r;
  }
  return off;
}
__host__ __device__ constexpr int tw_stage_total(int n) {
  return tw_stage_off(n, fft_elems(n), n);
}

// Shared-memory placement of a column: element x at sm[x * cs].
struct ColIdx {
  int cs;
  __device__ __forceinline__ int operator()(int x) const { return x * cs; }
};
// Placement of a contiguous line with an XOR swizzle on 16-byte slots so the
// stride-R writes of the first Stockham stage do not serialise on one bank.
// SH = log2 of the elements per thread: the first stage of E-element threads
// writes positions E*j + r, so lanes j must land in distinct 16 B slots (the
// shift of 3 alone left the radix-16 stages of n = 1024 2-way conflicted).
template <int SH = 3>
struct SwzIdxT {
  __device__ __forceinline__ int operator()(int x) const { return x ^ ((x >> SH) & 7); }
};
using SwzIdx = SwzIdxT<3>;

// Barrier policies: the whole CTA, or a named barrier over the threads that
// own one transform (lets independent transforms in a CTA drift apart).
struct CtaBar {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct NamedBar {
  int id, nthreads;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
  }
};

// One Stockham stage (and the rest, recursively). `sm` points at this
// column's element 0 in shared memory; element x lives at sm[idx(x)].
// The stage with register twiddles besides the last: the radix-8 stage at
// NS = 8 of the 8-element transforms (n = 128, 256, 512; at 512 it is also
// the one before the last).
__host__ __device__ constexpr int mid_ns(int n) { return n >= 128 ? 8 : 1; }

// Stage twiddles held in registers by kernels that run several transforms
// per thread (the z pass): W^k and W^{4k} of the radix-8 stages with NS =
// N/64 (m*) and NS = N/8 (w*) (k = the thread's butterfly index, forward
// sign); the other powers follow by complex products (at most three
// roundings), replacing seven 128-bit shared-memory reads -- four wavefronts
// each, whatever the address overlap -- per butterfly.
struct LastTw {
  double2 w1, w4;  // last stage
  double2 m1, m4;  // middle stage
};

template <int S>
__device__ __forceinline__ void apply_tw8(double2* a, double2 w1, double2 w4) {
  if (S > 0) {
    w1.y = -w1.y;
    w4.y = -w4.y;
  }
  const double2 w2 = cmul(w1, w1), w3 = cmul(w2, w1);
  a[1] = cmul(a[1], w1);
  a[2] = cmul(a[2], w2);
  a[3] = cmul(a[3], w3);
  a[4] = cmul(a[4], w4);
  a[5] = cmul(a[5], cmul(w4, w1));
  a[6] = cmul(a[6], cmul(w4, w2));
  a[7] = cmul(a[7], cmul(w4, w3));
}

// jf / jl: butterfly index this thread runs in the first / last stage
// (default t; the z pass remaps them so mirrored butterflies share a warp).
template <int N, int E, int S, int NS, class IDX, class BAR = CtaBar, bool LREG = false>
__device__ __forceinline__ void fft_stages(double2 (&v)[E], double2* sm, IDX idx, int t,
                                           const double2* __restrict__ tw, BAR bar = BAR{},
                                           LastTw lt = LastTw{}, int jf = -1, int jl = -1) {
  constexpr int REM = N / NS;
  constexpr int R = REM >= E ? E : REM;
  constexpr int NB = E / R;
  constexpr int TPC = N / E;
  constexpr bool LAST = (NS * R == N);
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    double2 a[R];
    const int j = (NS == 1 && jf >= 0 ? jf : (LAST && jl >= 0 ? jl : t)) + b * TPC;
    const int k = j & (NS - 1);
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = v[b + r * NB];
    if constexpr (LREG && LAST && NS > 1 && R == 8 && NB == 1) {
      apply_tw8<S>(a, lt.w1, lt.w4);
    } else if constexpr (LREG && !LAST && NS == mid_ns(N) && NS > 1 && R == 8 &&
                         NB == 1) {
      apply_tw8<S>(a, lt.m1, lt.m4);
    } else if (NS > 1) {
      constexpr int TOFF = tw_stage_off(N, E, NS);
#pragma unroll
      for (int r = 1; r < R; ++r) a[r] = cmul(a[r], twiddle<S>(tw, TOFF + (r - 1) * NS + k));
    }
    Dft<R, S>::run(a);
    if (LAST) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[b + r * NB] = a[r];
    } else {
      const int base = (j - k) * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) sm[idx(base + r * NS)] = a[r];
    }
  }
  if constexpr (!LAST) {
    constexpr int NS2 = NS * R, REM2 = N / NS2, R2 = REM2 >= E ? E : REM2;
    const int tn = (NS2 * R2 == N && jl >= 0) ? jl : t;  // the next stage's butterfly
    bar();
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = sm[idx(tn + m * TPC)];
    bar();
    fft_stages<N, E, S, NS * R, IDX, BAR, LREG>(v, sm, idx, t, tw, bar, lt, jf, jl);
  }
}

// Full transform: v[m] = x[t + m*TPC] on entry, X[t + m*TPC] on exit.
// Must be called by every thread the barrier policy covers.
template <int N, int S, class IDX, class BAR = CtaBar>
__device__ __forceinline__ void block_fft(double2 (&v)[fft_elems(N)], double2* sm, IDX idx, int t,
                                          const double2* __restrict__ tw, BAR bar = BAR{}) {
  fft_stages<N, fft_elems(N), S, 1, IDX, BAR>(v, sm, idx, t, tw, bar);
}

// Same with the final-stage twiddles from registers (see LastTw).
template <int N, int S, class IDX, class BAR>
__device__ __forceinline__ void block_fft_lt(double2 (&v)[fft_elems(N)], double2* sm, IDX idx,
                                             int t, const double2* __restrict__ tw, BAR bar,
                                             const LastTw& lt, int jf = -1, int jl = -1) {
  fft_stages<N, fft_elems(N), S, 1, IDX, BAR, true>(v, sm, idx, t, tw, bar, lt, jf, jl);
}

// LastTw of thread t for length-N transforms whose last stage is radix 8
// with one butterfly per thread (tw = the stage-ordered table).
template <int N>
__device__ __forceinline__ LastTw last_twiddles(const double2* tw, int t) {
  constexpr int NS = N / 8, MS = mid_ns(N);
  constexpr int TOFF = tw_stage_off(N, fft_elems(N), NS);
  constexpr int MOFF = tw_stage_off(N, fft_elems(N), MS);
  const int k = t & (NS - 1), km = t & (MS - 1);
  return LastTw{tw[TOFF + k], tw[TOFF + 3 * NS + k], tw[MOFF + km], tw[MOFF + 3 * MS + km]};
}

// Copies the stage-ordered twiddle table of length-n transforms to shared
// memory (tw_stage_total(n) <= n entries; caller syncs).
__device__ __forceinline__ void load_twiddles(double2* dst, const double2* __restrict__ src, int n) {
  const int total = tw_stage_total(n);
  for (int i = threadIdx.x; i < total; i += blockDim.x) dst[i] = __ldg(src + i);
}

}  // namespace sdns_dev
