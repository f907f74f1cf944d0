// The fused z pass at n = 512 with ONE WARP PER Z LINE (P3):
// z part of the curl, c2r of the six fields, 1/n^3, u x omega, r2c of the
// three products -- the arithmetic of k_z_fused (kernels.cu), laid out so
// that the shared-memory pipe, which bounds that kernel, carries ~30% fewer
// wavefronts per line:
//   - each lane holds 16 elements (two radix-8 butterflies per Stockham
//     stage, 512 = 8 x 8 x 8), so a line's three transforms stages exchange
//     within one warp (__syncwarp instead of 64-thread named barriers);
//   - the first stage of the inverse transforms runs the butterflies j and
//     64 - j (j = 0 with 32) on one lane: positions p and n - p of a
//     half-spectrum pair land on the same lane, so every staged mode is read
//     ONCE (the two-warp kernel reads the mirrored half twice);
//   - the last stage of the forward transform of n0 + i n1 runs the same
//     mirrored pairs, so the r2c split X[k], conj X[n-k] happens in
//     registers (no parking of the spectrum in shared memory);
//   - the three inverse results stay in registers through the products (no
//     parking of pair 0 or of the third product).
// Twiddles: W_64^k / W_64^4k and W_512^t / W_512^4t of each lane from the
// stage-ordered table (L2), the other butterflies' by one complex product
// with a constant (W^{t+32} = W^t W^32, W^{64-t} = W^64 conj W^t) and exact
// sign/swap operations for the fourth powers.
#include <cuda.h>

#include "fft_core.cuh"
#include "kernels.cuh"
#include "rowmap.cuh"

namespace sdns_dev {

namespace {

constexpr int ZN = 512;
constexpr int ZHP = ZN / 2 + 8;  // padded half row
#ifndef SDNS_Z512RPC
#define SDNS_Z512RPC 4
#endif
#ifndef SDNS_Z512PF  // L2 prefetch of the lines the CTA SDNS_Z512PF SM-waves ahead will stage
#define SDNS_Z512PF 0
#endif
constexpr int ZRPC = SDNS_Z512RPC;  // lines (warps) per CTA

__device__ __forceinline__ double zmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double zsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ int zsw(int x) { return x ^ ((x >> 3) & 7); }

// A + iB at position k (<= n/2) and at n - k from ONE read of the two half
// spectra; SG = +1: B += i kz A, -1: B -= i kz A (the z part of the curl),
// 0: none (k_z_fused's pair_sample_kz / pair_sample, same operations).
template <int SG>
__device__ __forceinline__ void zpair(const double2* A, const double2* B, int k, double2& lo,
                                      double2& hi) {
  const double2 a = A[k];
  double2 b = B[k];
  const double kz = static_cast<double>(k);
  if (SG > 0)
    b = make_double2(b.x - kz * a.y, b.y + kz * a.x);
  else if (SG < 0)
    b = make_double2(b.x + kz * a.y, b.y - kz * a.x);
  lo = make_double2(a.x - b.y, a.y + b.x);
  hi = make_double2(a.x + b.y, b.x - a.y);  // conj a + i conj b
}
// The self-mirrored bins k = 0 and n/2: imaginary parts dropped (FFTW c2r).
template <int SG>
__device__ __forceinline__ double2 zedge(const double2* A, const double2* B, int k) {
  const double2 a = A[k];
  const double2 b = B[k];  // kz a.y and kz a.x terms only reach b.y / b.x:
  double bx = b.x;         // at k = 0 they vanish; at k = n/2, b.x picks up
  const double kz = static_cast<double>(k);  // -+ kz a.y before a.y is dropped
  if (SG > 0) bx = b.x - kz * a.y;
  else if (SG < 0) bx = b.x + kz * a.y;
  return make_double2(a.x - 0.0, 0.0 + bx);  // as pair_sample_kz: a.y = b.y = 0
}

// Mirrored first-stage elements of lane t: x[0..7] = butterfly j1 = t
// (positions t + 64 r), x[8..15] = butterfly j2 = 64 - t (t = 0: 32).
template <int SG>
__device__ __forceinline__ void zsample(const double2* A, const double2* B, int t,
                                        double2 (&x)[16]) {
  if (t != 0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) zpair<SG>(A, B, t + 64 * r, x[r], x[8 + 7 - r]);
#pragma unroll
    for (int r = 0; r < 4; ++r) zpair<SG>(A, B, 64 - t + 64 * r, x[8 + r], x[7 - r]);
  } else {
    x[0] = zedge<SG>(A, B, 0);
    x[4] = zedge<SG>(A, B, 256);
#pragma unroll
    for (int r = 1; r < 4; ++r) zpair<SG>(A, B, 64 * r, x[r], x[8 - r]);
#pragma unroll
    for (int r = 0; r < 4; ++r) zpair<SG>(A, B, 32 + 64 * r, x[8 + r], x[8 + 7 - r]);
  }
}

struct ZTw {
  double2 m1, m4;  // W_64^(t&7), W_64^(4(t&7))
  double2 w1, w4;  // W_512^t, W_512^4t
};

// Twiddles of the last-stage butterflies t + 32 and 64 - t (t = 0: 32).
__device__ __forceinline__ void tw_plus32(const ZTw& z, double2& w1, double2& w4) {
  const double2 c = make_double2(0.92387953251128675613, -0.38268343236508977173);  // W^32
  w1 = cmul(z.w1, c);
  w4 = make_double2(z.w4.y, -z.w4.x);  // W^4t * W^128 = W^4t * (-i)
}
__device__ __forceinline__ void tw_mirror(const ZTw& z, int t, double2& w1, double2& w4) {
  if (t == 0) {
    tw_plus32(z, w1, w4);
    return;
  }
  const double2 c = make_double2(0.70710678118654752440, -0.70710678118654752440);  // W^64
  w1 = cmul(c, cconj(z.w1));
  w4 = make_double2(-z.w4.x, z.w4.y);  // W^256 conj W^4t = -conj W^4t
}

// Stockham radix-8 stages of a 512-point line held by one warp (lane t).
// Stage A (NS = 1): butterflies j of x[0..7], x[8..15]; writes y[8j + r].
template <int S>
__device__ __forceinline__ void zstage_a(double2 (&x)[16], double2* sm, int j1, int j2) {
  Dft<8, S>::run(&x[0]);
  Dft<8, S>::run(&x[8]);
#pragma unroll
  for (int r = 0; r < 8; ++r) sm[zsw(8 * j1 + r)] = x[r];
#pragma unroll
  for (int r = 0; r < 8; ++r) sm[zsw(8 * j2 + r)] = x[8 + r];
  __syncwarp();
}
// Stage B (NS = 8): butterflies t and t + 32 (same k = t & 7 twiddles).
template <int S>
__device__ __forceinline__ void zstage_b(double2 (&x)[16], double2* sm, int t, const ZTw& z) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    x[r] = sm[zsw(t + 64 * r)];
    x[8 + r] = sm[zsw(t + 32 + 64 * r)];
  }
  __syncwarp();  // every lane has read before anyone overwrites
  apply_tw8<S>(&x[0], z.m1, z.m4);
  apply_tw8<S>(&x[8], z.m1, z.m4);
  Dft<8, S>::run(&x[0]);
  Dft<8, S>::run(&x[8]);
  const int k = t & 7;
  const int b1 = (t >> 3) * 64 + k, b2 = ((t + 32) >> 3) * 64 + k;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    sm[zsw(b1 + 8 * r)] = x[r];
    sm[zsw(b2 + 8 * r)] = x[8 + r];
  }
  __syncwarp();
}
// Stage C (NS = 64): butterflies j1, j2 with twiddles (w1a, w4a), (w1b,
// w4b); results x[0..7] at positions j1 + 64 r, x[8..15] at j2 + 64 r.
template <int S>
__device__ __forceinline__ void zstage_c(double2 (&x)[16], const double2* sm, int j1, int j2,
                                         double2 w1a, double2 w4a, double2 w1b, double2 w4b) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    x[r] = sm[zsw(j1 + 64 * r)];
    x[8 + r] = sm[zsw(j2 + 64 * r)];
  }
  apply_tw8<S>(&x[0], w1a, w4a);
  apply_tw8<S>(&x[8], w1b, w4b);
  Dft<8, S>::run(&x[0]);
  Dft<8, S>::run(&x[8]);
}

// Inverse transform of the pair staged at A, B (exchange buffer: A's and
// B's regions, 2 * ZHP >= 512 entries): results at positions t + 64 r
// (x[0..7]) and t + 32 + 64 r (x[8..15]).
template <int SG>
__device__ __forceinline__ void zinverse(double2 (&x)[16], double2* A, double2* B, int t,
                                         const ZTw& z) {
  zsample<SG>(A, B, t, x);
  __syncwarp();  // the staging area becomes the exchange buffer
  const int j2 = t ? 64 - t : 32;
  zstage_a<+1>(x, A, t, j2);
  zstage_b<+1>(x, A, t, z);
  double2 w1b, w4b;
  tw_plus32(z, w1b, w4b);
  zstage_c<+1>(x, A, t, t + 32, z.w1, z.w4, w1b, w4b);
}

}  // namespace

template <bool PO>
__global__ void __launch_bounds__(32 * ZRPC, 8 / ZRPC)
k_z512w(double2* f, long long cs, RowMap rm, double norm, const double2* __restrict__ tw,
        const __grid_constant__ CUtensorMap ztm, double2* fo, RowMap rmo) {
  extern __shared__ __align__(128) double2 smem[];
  __shared__ alignas(8) unsigned long long zbar[ZRPC];
  const int t = threadIdx.x & 31, r = threadIdx.x >> 5;
  const int ri = blockIdx.x * ZRPC + r;
  const bool valid = ri < rm.nrows;
  const long long ro = (valid && rm.nseg == 0) ? zrow_off(rm, ri) : 0;
  double2* S = smem + r * 6 * ZHP;
  // Stage the 6 half-rows by the bulk-copy engine (k_z_fused's staging):
  // slot s holds field {0, 4, 1, 3, 2, 5}[s], i.e. the pairs (u0, w1'),
  // (u1, w0'), (u2, w2).
  if (t == 0) mbar_init(&zbar[r], 1);
  __syncwarp();
  if (valid && t == 0) {
    const int fld[6] = {0, 4, 1, 3, 2, 5};
    if (rm.cstride) {  // chunked rows: one tensor-map box per half-row
      const int x = ri / rm.rpp, y = ri - x * rm.rpp;
      mbar_expect_tx(&zbar[r], 6u * static_cast<unsigned>(rm.pitch) * 16u);
#pragma unroll
      for (int sl = 0; sl < 6; ++sl) tma_load5(S + sl * ZHP, &ztm, 0, 0, y, x, fld[sl], &zbar[r]);
    } else {
      mbar_expect_tx(&zbar[r], 6u * static_cast<unsigned>(rm.n2) * 16u);
#pragma unroll
      for (int sl = 0; sl < 6; ++sl) {
        const double2* src = f + fld[sl] * cs;
        if (rm.nseg == 0) {
          bulk_g2s(S + sl * ZHP, src + ro, static_cast<unsigned>(rm.n2) * 16u, &zbar[r]);
        } else {
          for (int q = 0; q < rm.nseg; ++q) {
            const int k0 = rm.seg_k0[q], k1 = rm.seg_k0[q + 1];
            if (k1 > k0)
              bulk_g2s(S + sl * ZHP + k0,
                       src + rm.seg_base[q] + static_cast<long long>(ri) * rm.seg_pitch[q],
                       static_cast<unsigned>(k1 - k0) * 16u, &zbar[r]);
          }
        }
      }
    }
  }
  if constexpr (SDNS_Z512PF > 0) {  // warm L2 for the line a later CTA on this SM stages
    const int rf = ri + SDNS_Z512PF * static_cast<int>(gridDim.x > 0 ? 0 : 0) +
                   SDNS_Z512PF * ZRPC * 148 * (8 / ZRPC);
    if (t < 6 && rf < rm.nrows && rm.cstride) {
      const int fl[6] = {0, 4, 1, 3, 2, 5};
      const int xf = rf / rm.rpp, yf = rf - xf * rm.rpp;
      asm volatile(
          "cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];\n" ::"l"(&ztm),
          "r"(0), "r"(0), "r"(yf), "r"(xf), "r"(fl[t])
          : "memory");
    }
  }
  // register twiddles (from L2) while the line arrives
  constexpr int TOFF = tw_stage_off(ZN, 8, 64), MOFF = tw_stage_off(ZN, 8, 8);
  ZTw z;
  z.m1 = __ldg(tw + MOFF + (t & 7));
  z.m4 = __ldg(tw + MOFF + 3 * 8 + (t & 7));
  z.w1 = __ldg(tw + TOFF + t);
  z.w4 = __ldg(tw + TOFF + 3 * 64 + t);
  if (!valid) return;  // whole warps: no later warp-collective needs this one
  mbar_wait(&zbar[r], 0);

  double2 p0[16], p1[16], x[16];
  zinverse<+1>(p0, S, S + ZHP, t, z);                // u0 + i w1
  zinverse<-1>(p1, S + 2 * ZHP, S + 3 * ZHP, t, z);  // u1 + i w0
  // u2 + i w2: stages A and B, then stage C one butterfly at a time fused
  // with 1/n^3 (fft.cpp:125) and u x omega (navier_stokes.cpp:45-49) in
  // k_z_fused's operation order (fewer live registers): n0 + i n1 -> x,
  // n2 -> p0
  {
    double2* A = S + 4 * ZHP;
    zsample<0>(A, S + 5 * ZHP, t, x);
    __syncwarp();
    zstage_a<+1>(x, A, t, t ? 64 - t : 32);
    zstage_b<+1>(x, A, t, z);
    double2 w1b, w4b;
    tw_plus32(z, w1b, w4b);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double2 a[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = A[zsw(t + 32 * h + 64 * q)];
      apply_tw8<+1>(a, h ? w1b : z.w1, h ? w4b : z.w4);
      Dft<8, +1>::run(a);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int m = 8 * h + q;
        const double ua = zmul(p0[m].x, norm), ub = zmul(p1[m].x, norm), uc = zmul(a[q].x, norm);
        const double wa = zmul(p1[m].y, norm), wb = zmul(p0[m].y, norm), wc = zmul(a[q].y, norm);
        const double n0 = zsub(zmul(ub, wc), zmul(uc, wb));
        const double n1 = zsub(zmul(uc, wa), zmul(ua, wc));
        p0[m] = make_double2(zsub(zmul(ua, wb), zmul(ub, wa)), 0.0);
        x[m] = make_double2(n0, n1);
      }
    }
  }
  // forward transform of n0 + i n1 (input positions are the inverse
  // results' t + 64 r, t + 32 + 64 r); last stage on the mirrored pairs
  double2* E0 = S;  // regions 0-1 are free again
  __syncwarp();
  zstage_a<-1>(x, E0, t, t + 32);
  zstage_b<-1>(x, E0, t, z);
  const int j2 = t ? 64 - t : 32;
  double2 w1b, w4b;
  tw_mirror(z, t, w1b, w4b);
  zstage_c<-1>(x, E0, t, j2, z.w1, z.w4, w1b, w4b);
  // r2c split in registers: X[k], conj X[n - k] -> N0[k], N1[k], k <= n/2
  const int keep = rm.kz_keep < ZN / 2 + 1 ? rm.kz_keep : ZN / 2 + 1;
  auto put01 = [&](int k, double2 d, double2 m) {
    if (k >= keep) return;
    const double2 e = cconj(m);
    const double2 dd = csub(d, e);
    const double2 o0 = make_double2(0.5 * (d.x + e.x), 0.5 * (d.y + e.y));
    const double2 o1 = make_double2(0.5 * dd.y, -0.5 * dd.x);
    if constexpr (PO) {
      const ZDst q = zdst(rmo, ri, k);
      fo[q.el] = o0;
      fo[q.el + q.cs] = o1;
    } else {
      const long long el = zel(rm, ro, ri, k);
      f[el] = o0;
      f[cs + el] = o1;
    }
  };
  if (t != 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      put01(t + 64 * q, x[q], x[8 + 7 - q]);            // k = t + 64 q, n - k = j2 + 64 (7 - q)
      put01(64 - t + 64 * q, x[8 + q], x[7 - q]);       // k = 64 - t + 64 q
    }
  } else {
    put01(0, x[0], x[0]);
    put01(256, x[4], x[4]);
#pragma unroll
    for (int q = 1; q < 4; ++q) put01(64 * q, x[q], x[8 - q]);
#pragma unroll
    for (int q = 0; q < 4; ++q) put01(32 + 64 * q, x[8 + q], x[8 + 7 - q]);
  }
  // n2 alone: forward transform, outputs k <= n/2 on the standard lanes
  double2* E1 = S + 2 * ZHP;
  zstage_a<-1>(p0, E1, t, t + 32);
  zstage_b<-1>(p0, E1, t, z);
  tw_plus32(z, w1b, w4b);
  zstage_c<-1>(p0, E1, t, t + 32, z.w1, z.w4, w1b, w4b);
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int k = (m < 8 ? t : t + 32) + 64 * (m & 7);
    if (k <= ZN / 2 && k < keep) {
      if constexpr (PO) {
        const ZDst q = zdst(rmo, ri, k);
        fo[q.el + 2 * q.cs] = p0[m];
      } else {
        f[2 * cs + zel(rm, ro, ri, k)] = p0[m];
      }
    }
  }
  if constexpr (PO) __threadfence_system();  // peers read after a stream barrier
}

size_t z512w_smem() { return sizeof(double2) * static_cast<size_t>(ZRPC) * 6 * ZHP; }

void z512w_launch(double2* rows, long long cs, const RowMap& rm, double norm, const double2* tw,
                  const CUtensorMap& tm, double2* out, const RowMap* rmo, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>((rm.nrows + ZRPC - 1) / ZRPC);
  const size_t shm = z512w_smem();
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_z512w<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(shm));
    cudaFuncSetAttribute(k_z512w<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(shm));
    cudaFuncSetAttribute(k_z512w<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_z512w<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    init = true;
  }
  if (rmo)
    k_z512w<true><<<grid, 32 * ZRPC, shm, s>>>(rows, cs, rm, norm, tw, tm, out, *rmo);
  else
    k_z512w<false><<<grid, 32 * ZRPC, shm, s>>>(rows, cs, rm, norm, tw, tm, rows, RowMap{});
}

}  // namespace sdns_dev
