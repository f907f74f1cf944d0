// Column passes (FFTs along x or y) as persistent tile pipelines for sm_100a.
//
// A tile is CS consecutive kz columns of one row (CS*16 B contiguous per
// position) over all N positions of the transformed axis. Each CTA walks a
// strided list of (tile, item) work; tiles arrive in shared memory through a
// ring of buffers -- by TMA tensor-map box loads completing on per-slot
// mbarriers where the source is a plain (kz, rows, positions) block, by
// cp.async (LDGSTS, zero-filled outside the valid kz range) otherwise -- so
// items i+1.. load while item i is transformed in place. Results leave with
// coalesced 16-byte stores (P2: TMA tensor stores from a staging tile).
// Every item reads exactly one input tile, which is what the linearity
// restructuring of the curl allows:
//   P1 x inverse:  U_c = F_x^-1(u_c),  K2 = F_x^-1(kx u2),
//                  w2' = i (F_x^-1(kx u1) - ky U0)
//   P2 y inverse:  u_c = F_y^-1(U_c),  w0' = F_y^-1(i ky U2),
//                  w1' = F_y^-1(-i K2), w2 = F_y^-1(w2')
//   P3 (z pass) then completes w0 = w0' - i kz u1 and w1 = w1' + i kz u0,
// which is omega_hat = i k x u_hat (curl_hat, navier_stokes.cpp:52-72)
// distributed over the three axes.
//
// Tile shapes and ring depths are per pass variant (PipeCfg, measured on
// B200): 8-column / 128 B tiles at n = 512, a three-deep ring
// for the plain and y-inverse-input passes, two plus a scratch tile for P1,
// two plus a store-staging tile for P2, single 128 KB buffers at n = 1024.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "fft_core.cuh"
#include "kernels.cuh"

namespace sdns_dev {

namespace {

// Pass variants of PipeCfg: 0 = plain y/x passes below n = 1024, 8 = P1
// (ring of two + scratch tile), 9 = plain passes at n = 1024 (single 128 KB
// buffer), 10 = P2 (ring of two + TMA-store staging tile).
enum : int { VX = 0, VY = 0, VYI = 10, VXI = 8 };

template <int N, int V>
struct PipeCfg {
  static constexpr int E = fft_elems(N);
  static constexpr int TPC = N / E;
  static constexpr int CSW = (V == 1 || V == 2) ? 4 : 8;  // columns at TPC >= 64
  // n < 512: threads per CTA (measured at n = 64/128/256: small CTAs win
  // except for the two-transform inverse passes at 256)
  static constexpr int ST = (N >= 256 && (V == 8 || V == 10)) ? 512 : 64;
  static constexpr int CS0 = TPC >= 64 ? CSW : (ST / TPC > 64 ? 64 : (ST / TPC < 8 ? 8 : ST / TPC));
  // n = 1024: 4-column tiles fit two buffers; V = 9 (plain passes) keeps
  // 128 B rows with a single 128 KB buffer (measured 2x faster on the x axis)
  static constexpr int CS = (N >= 1024 && V != 9) ? 4 : CS0;
  static constexpr int THREADS = TPC * CS;
  static constexpr int NBUF = (V == 2 || V == 3 || V == 4 || V == 9) ? 1
                             : (V == 0 && N == 512) ? 3 : 2;
  static constexpr int MINB = V == 1 ? 3 : (V == 2 ? 4 : (V == 3 ? 2 : 1));
  // V = 8: one extra tile-sized exchange buffer (the x inverse pass runs its
  // first transform there and re-reads the input tile for the second)
  // V = 10: one extra tile buffer staging the y inverse pass's outputs for
  // TMA tensor stores (input ring of two)
  static constexpr int SCR = (V == 8 || V == 10) ? 1 : 0;
  static constexpr int TILE = N * CS;  // complex elements per tile buffer
  // tile buffers + scratch + the twiddle table
  static constexpr size_t SMEM = sizeof(double2) * ((NBUF + SCR) * TILE + N);
};

__device__ __forceinline__ double wavenum(int j, int n) {
  return static_cast<double>(j <= n / 2 - 1 ? j : j - n);
}

struct Tile {
  long long base;  // row*rs + kz of this thread's column
  int row, kz;
  bool valid;
};

// Shared-memory placement of a tile: position x of column c at
// tpos(x)*CS + c. With 4-column (64 B) rows, positions are swizzled in pairs
// of 8 so that the stride-8 writes of the first Stockham stage alternate
// between the two 64 B halves of a bank row.
template <int CS>
struct TileIdx {
  __device__ __forceinline__ int operator()(int x) const {
    return x * CS;
  }
};

// Shared-memory index of (position x, column col) of a tile buffer.
template <int CS>
struct CIdx {
  static constexpr int kCS = CS;
  int col;
  __device__ __forceinline__ int operator()(int x) const { return TileIdx<CS>{}(x) + col; }
};

// Placement of the Stockham exchanges inside a tile buffer. A phase of a
// 128-bit access is 8 lanes = 8 / CS positions x CS columns; with 4-column
// tiles and 16-element threads (n = 1024) the first stage's writes (positions
// 16 j + r) put the two positions of a phase on the same banks. Flipping the
// position's low bit with its bit 4 separates them (exchanges only: tiles
// arrive and leave in the linear TileIdx layout).
template <int N, int CS>
struct XIdx {
  int col;
  __device__ __forceinline__ int operator()(int x) const {
    if constexpr (CS == 4 && fft_elems(N) == 16) x ^= (x >> 4) & 1;
    return TileIdx<CS>{}(x) + col;
  }
};

template <int CS>
__device__ __forceinline__ Tile tile_of(int tile, int col, const ColGeom& g) {
  const int gc = tile * CS + col;
  // gc / pitch through a float reciprocal and one correction step (exact
  // for gc < 2^24, far above any tile count here): the 32-bit integer
  // division sequence showed up in the column passes' stall samples
  int re = __float2int_rz(__int2float_rn(gc) * __frcp_rn(__int2float_rn(g.pitch)));
  int kz = gc - re * g.pitch;
  if (kz < 0) {
    --re;
    kz += g.pitch;
  } else if (kz >= g.pitch) {
    ++re;
    kz -= g.pitch;
  }
  const int row = re < g.seg_a ? re + g.off0 : re - g.seg_a + g.off1;
  Tile t;
  t.valid = re < g.nrows && kz < g.n2;
  t.row = row;
  t.kz = kz;
  t.base = static_cast<long long>(row) * g.rs + static_cast<long long>(kz >> 3) * g.kcs + (kz & 7);
  return t;
}

// Per-thread element offsets of positions t + m*TPC, evaluated on use (a
// few integer ops) rather than held in E registers: the two-transform
// inverse passes sit at the 128-register limit.
template <int N>
struct PosOff {
  int t, ps0, ps1, shift;
  __device__ __forceinline__ PosOff(const ColGeom& g, int t_)
      : t(t_), ps0(static_cast<int>(g.ps0)), ps1(static_cast<int>(g.ps1)), shift(g.pb_shift) {}
  // A copy whose strides the compiler cannot trace back: the offsets derived
  // from it are recomputed where they are used instead of being hoisted out
  // of the item loop. In the 16-element kernels at the 128-register limit
  // (n = 1024) the hoisted offsets were spilled, and every store then waited
  // for local-memory reloads (L1 is carved down to almost nothing here): 25%
  // of the x inverse pass's stall samples (P1 at 1024: 22.0 -> 21.5 ms).
  __device__ __forceinline__ PosOff fresh() const {
    PosOff q = *this;
    asm volatile("" : "+r"(q.ps0), "+r"(q.ps1), "+r"(q.t));
    return q;
  }
  __device__ __forceinline__ int o(int m) const {
    const int pos = t + m * (N / fft_elems(N));
    return (pos >> shift) * ps1 + (pos & ((1 << shift) - 1)) * ps0;
  }
};

template <int N, class IDX>
__device__ __forceinline__ void issue_tile(double2* buf, const double2* src, const Tile& tl,
                                           const PosOff<N>& po, IDX idx, int t) {
  constexpr int E = fft_elems(N), TPC = N / E;
  const double2* b = src + tl.base;
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int pos = t + m * TPC;
    cp_async16(buf + idx(pos), tl.valid ? b + po.o(m) : src, tl.valid);
  }
}

template <int N, class IDX>
__device__ __forceinline__ void read_own(double2 (&v)[fft_elems(N)], const double2* buf, IDX idx,
                                         int t) {
  constexpr int E = fft_elems(N), TPC = N / E;
#pragma unroll
  for (int m = 0; m < E; ++m) v[m] = buf[idx(t + m * TPC)];
}

template <int N, bool PEER = false>
__device__ __forceinline__ void store_own(double2* dst, const double2 (&v)[fft_elems(N)],
                                          const ColGeom& g, const Tile& tl, const PosOff<N>& po,
                                          int t) {
  constexpr int E = fft_elems(N), TPC = N / E;
  if (!tl.valid) return;
  double2* b = dst + tl.base;
  const PosOff<N> q = E >= 16 ? po.fresh() : po;
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int pos = t + m * TPC;
    if (g.keep_k >= 0 && pos > g.keep_k && pos < N - g.keep_k) continue;  // masked mode
    if constexpr (PEER)
      b[q.o(m) + __ldg(g.seg + (pos >> g.pb_shift))] = v[m];
    else
      b[q.o(m)] = v[m];
  }
}

// Output placement: the input geometry (in-place passes, SEP 0), a separate
// one (SEP 1: pencil y passes write the next transpose's send layout
// directly) or a separate one whose position segments are other ranks'
// buffers (SEP 2: peer-direct slab transposes, ColGeom::seg).
template <int N, int SEP>
struct OutSel;
template <int N>
struct OutSel<N, 0> {
  __device__ __forceinline__ OutSel(const ColGeom&, int) {}
  __device__ __forceinline__ Tile tile(const Tile& t, const ColGeom&) const { return t; }
  __device__ __forceinline__ const PosOff<N>& po(const PosOff<N>& in) const { return in; }
};
template <int N>
struct OutSel<N, 1> {
  PosOff<N> p;
  __device__ __forceinline__ OutSel(const ColGeom& go, int t) : p(go, t) {}
  __device__ __forceinline__ Tile tile(const Tile& t, const ColGeom& go) const {
    Tile o = t;
    o.base = static_cast<long long>(t.row) * go.rs + static_cast<long long>(t.kz >> 3) * go.kcs +
             (t.kz & 7);
    return o;
  }
  __device__ __forceinline__ const PosOff<N>& po(const PosOff<N>&) const { return p; }
};
template <int N>
struct OutSel<N, 2> : OutSel<N, 1> {
  using OutSel<N, 1>::OutSel;
};

// Stores of a peer-direct pass must be visible to the peers' next pass,
// which starts after a stream barrier across the ranks.
template <int SEP>
__device__ __forceinline__ void peer_fence() {
  if constexpr (SEP == 2) __threadfence_system();
}

// Column transform. At n = 512 both twiddled radix-8 stages take their
// twiddles from registers (LastTw: 4 table reads instead of 14 per transform).
template <int N, int S, class IDX, class BAR>
__device__ __forceinline__ void col_fft(double2 (&v)[fft_elems(N)], double2* sm, IDX idx, int t,
                                        const double2* __restrict__ tw, BAR bar) {
  const XIdx<N, IDX::kCS> xi{idx.col};
  if constexpr (N == 512)
    block_fft_lt<N, S>(v, sm, xi, t, tw, bar, last_twiddles<N>(tw, t));
  else
    block_fft<N, S>(v, sm, xi, t, tw, bar);
}
// Same with the register twiddles held by the caller (read once per kernel).
template <int N, int S, class IDX, class BAR>
__device__ __forceinline__ void col_fft_lt(double2 (&v)[fft_elems(N)], double2* sm, IDX idx, int t,
                                           const double2* __restrict__ tw, BAR bar,
                                           const LastTw& lt) {
  const XIdx<N, IDX::kCS> xi{idx.col};
  if constexpr (N == 512)
    block_fft_lt<N, S>(v, sm, xi, t, tw, bar, lt);
  else
    block_fft<N, S>(v, sm, xi, t, tw, bar);
}

// Lane roles: column-minor (col = tid % CS, t = tid / CS), so a warp's
// global accesses are 32/CS positions x CS*16 B along kz. (Measured: warps
// covering 8 positions x 64 B -- two independent half-CTAs of 4 columns each
// -- are ~1.5x slower on both axes than 4 positions x 128 B.)
template <int N, int V>
struct Lanes {
  using C = PipeCfg<N, V>;
  int col, t;
  CIdx<C::CS> idx;
  CtaBar bar;
  __device__ __forceinline__ Lanes() {
    col = threadIdx.x % C::CS;
    t = threadIdx.x / C::CS;
    idx.col = col;
  }
};

__device__ __forceinline__ double2 times_i(double2 a) { return make_double2(-a.y, a.x); }
__device__ __forceinline__ double2 times_mi(double2 a) { return make_double2(a.y, -a.x); }

// Tile source by the tensor-memory accelerator: two (N <= 256: one) box
// loads of 2*CS doubles x 256 positions from a 5-D tensor map (doubles of a
// kz chunk, kz chunks, rows, positions, fields), completing on the slot's
// mbarrier. The box lands position-major, CS complex per position --
// TileIdx<8>. Issued by thread 0 (its tile coordinates are column 0's).
// (tma_load5: fft_core.cuh)

template <int N, int CS>
__device__ __forceinline__ void tma_tile(double2* buf, const CUtensorMap* tm, const ColGeom& g,
                                         const Tile& tl, int field, unsigned long long* bar) {
  constexpr int BP = N < 256 ? N : 256;
  mbar_expect_tx(bar, static_cast<unsigned>(N * CS * sizeof(double2)));
#pragma unroll
  for (int h = 0; h < N / BP; ++h)
    tma_load5(buf + h * BP * CS, tm, 2 * (tl.kz & 7), tl.kz >> 3, tl.row, h * BP, field, bar);
}

// Tile stores by the tensor-memory accelerator from a dedicated staging
// buffer (V = 10): the transformed tile is written there in the tile layout
// and thread 0 issues two box stores that drain while the CTA transforms the
// next item; the buffer is rewritten only after the previous stores have
// read it (one transform later, normally without waiting).
__device__ __forceinline__ void tma_store5(const CUtensorMap* tm, const void* src, int c0, int c1,
                                           int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];\n" ::"l"(
          tm),
      "r"(smem_addr(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

template <int N, int CS, class IDX>
__device__ __forceinline__ void tma_put(const CUtensorMap* tm, const double2 (&v)[fft_elems(N)],
                                        double2* out, IDX idx, int t, const Tile& tl, int field) {
  constexpr int E = fft_elems(N), TPC = N / E, BP = N < 256 ? N : 256;
  if (threadIdx.x == 0) bulk_wait_read0();
  __syncthreads();
#pragma unroll
  for (int m = 0; m < E; ++m) out[idx(t + m * TPC)] = v[m];
  fence_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int h = 0; h < N / BP; ++h)
      tma_store5(tm, out + h * BP * CS, 2 * (tl.kz & 7), tl.kz >> 3, tl.row, h * BP, field);
    bulk_commit();
  }
}

// Generic persistent pipeline driver: `items` items per tile; src(f) gives
// the input field of item f (fld(f) its index in the tensor map tm when
// g.tma != 0); body(f, buf, tile, pos_offsets, lanes, twiddles) transforms.
template <int N, int V, class SrcF, class FldF, class BodyF>
__device__ __forceinline__ void pipeline(int ntiles, int f_lo, int items, const ColGeom& g, SrcF src,
                                         FldF fld, const CUtensorMap* tm,
                                         const double2* __restrict__ tw_global, BodyF body) {
  extern __shared__ __align__(128) double2 smem[];
  __shared__ alignas(8) unsigned long long tbar[3];
  constexpr int CS = PipeCfg<N, V>::CS, NBUF = PipeCfg<N, V>::NBUF;
  const Lanes<N, V> ln;
  const int col = ln.col, t = ln.t;
  const PosOff<N> po(g, t);
  const bool tma = g.tma != 0;
  double2* tws = smem + (NBUF + PipeCfg<N, V>::SCR) * N * CS;
  if (tma && threadIdx.x == 0)
    for (int j = 0; j < NBUF; ++j) mbar_init(&tbar[j], 1);
  // The twiddle table is staged after the first tiles are requested (they
  // depend only on thread 0's barrier init or on nothing, LDGSTS): at small n
  // a kernel is one latency chain and the two fetches then overlap.
  auto stage_twiddles = [&] {
    load_twiddles(tws, tw_global, N);
    __syncthreads();  // table and barrier init visible to every thread
  };
  // ring slot j at smem + j*N*CS (arithmetic, not a pointer array: that
  // would live in local memory)
  auto ring = [&](int j) { return smem + j * (N * CS); };
  auto issue = [&](int slot, int f, const Tile& tl) {
    if (tma) {
      if (threadIdx.x == 0) tma_tile<N, CS>(ring(slot), tm, g, tl, fld(f), &tbar[slot]);
    } else {
      issue_tile<N>(ring(slot), src(f), tl, po, ln.idx, t);
    }
  };
  // A slot is refilled only after the barrier that ends its last transform
  // (block_fft's trailing barrier follows its last shared-memory access; the
  // single-buffer path has an explicit one): the same release the mbarrier
  // empty/full pipelines of TMA producers rely on.
  const int G = gridDim.x;
  // items f_lo .. f_lo + items - 1 of every tile
  const int f_hi = f_lo + items;
  int f = f_lo, tile = blockIdx.x;
  auto no_release = [] {};
  if (NBUF == 1 && tma) {
    // single buffer fed by TMA: the body calls release() once its transform
    // has finished with the buffer (the trailing barrier of block_fft), and
    // the next tile loads while this one is stored from registers
    Tile tl = tile_of<CS>(tile, col, g);
    if (tile < ntiles) issue(0, f, tl);
    stage_twiddles();
    for (int i = 0; tile < ntiles; ++i) {
      int fn = f + 1, tn = tile;
      if (fn == f_hi) {
        fn = f_lo;
        tn += G;
      }
      const Tile tln = tile_of<CS>(tn, col, g);
      mbar_wait(&tbar[0], i & 1);
      bool issued = false;
      auto release = [&] {
        if (tn < ntiles) issue(0, fn, tln);
        issued = true;
      };
      body(f, smem, tl, po, ln, static_cast<const double2*>(tws), release);
      if (!issued) {
        ln.bar();
        release();
      }
      f = fn;
      tile = tn;
      tl = tln;
    }
    return;
  }
  if (NBUF == 1) {
    stage_twiddles();
    for (int i = 0; tile < ntiles; ++i) {
      const Tile tl = tile_of<CS>(tile, col, g);
      issue(0, f, tl);
      cp_commit();
      cp_wait0();
      ln.bar();
      body(f, smem, tl, po, ln, static_cast<const double2*>(tws), no_release);
      ln.bar();
      if (++f == f_hi) {
        f = f_lo;
        tile += G;
      }
    }
    return;
  }
  // NBUF-deep ring: items i+1 .. i+NBUF-1 are in flight while item i is
  // transformed. The buffer refilled at step i is the one item i-1 used;
  // block_fft ends with a barrier after its last shared-memory read, so no
  // thread still reads it. Items run field-inner: the tiles in flight are one
  // kz chunk of consecutive fields, and at any time the grid covers one
  // contiguous range of tiles (measured better on the x axis than walking
  // groups of adjacent tiles per CTA).
  // n = 1024 (4-column, 64 B tile rows): a CTA walks tile PAIRS and
  // interleaves their items -- (2j, f) then (2j+1, f) -- so both 64 B halves
  // of every 128 B row are requested one item apart and the second is served
  // by L2 (measured: walking single tiles, persistent CTAs drift apart and
  // DRAM delivers every 128 B line twice). Items of one tile keep their order.
  constexpr bool PAIR = CS == 4 && N >= 1024;
  constexpr int TS = PAIR ? 2 : 1;
  struct Item {
    int t0, f, h;  // pair base (PAIR) or tile, item, half
  };
  const bool split = !PAIR && g.split;  // unit u = tile * items + (f - f_lo)
  auto adv = [&](Item it) {
    if (split) {
      const int u = it.t0 * items + (it.f - f_lo) + G;
      it.t0 = u / items;
      it.f = f_lo + (u - it.t0 * items);
      return it;
    }
    if constexpr (PAIR) {
      if (it.h == 0) {
        it.h = 1;
        return it;
      }
      it.h = 0;
    }
    if (++it.f == f_hi) {
      it.f = f_lo;
      it.t0 += G * TS;
    }
    return it;
  };
  auto tile_at = [&](const Item& it) { return tile_of<CS>(it.t0 + it.h, col, g); };
  Item cur{static_cast<int>(blockIdx.x) * TS, f_lo, 0};
  if (split) {
    cur.t0 = static_cast<int>(blockIdx.x) / items;
    cur.f = f_lo + static_cast<int>(blockIdx.x) - cur.t0 * items;
  }
  Tile tc = tile_at(cur);
  if (cur.t0 < ntiles) issue(0, cur.f, tc);
  cp_commit();
  Item n1 = adv(cur);
  Tile tn1 = tile_at(n1);
  if (NBUF > 2) {
    if (n1.t0 < ntiles) issue(1, n1.f, tn1);
    cp_commit();
  }
  stage_twiddles();
  for (int i = 0; cur.t0 < ntiles; ++i) {
    if (NBUF > 2) {
      const Item n2 = adv(n1);
      const Tile tn2 = tile_at(n2);
      if (n2.t0 < ntiles) issue((i + 2) % 3, n2.f, tn2);
      if (tma) {
        mbar_wait(&tbar[i % 3], (i / 3) & 1);
      } else {
        cp_commit();
        cp_wait2();
        ln.bar();
      }
      body(cur.f, ring(i % 3), tc, po, ln, static_cast<const double2*>(tws), no_release);
      cur = n1;
      tc = tn1;
      n1 = n2;
      tn1 = tn2;
    } else {
      if (n1.t0 < ntiles) issue((i + 1) & 1, n1.f, tn1);
      if (tma) {
        mbar_wait(&tbar[i & 1], (i >> 1) & 1);
      } else {
        cp_commit();
        cp_wait1();
        ln.bar();
      }
      body(cur.f, ring(i & 1), tc, po, ln, static_cast<const double2*>(tws), no_release);
      cur = n1;
      tc = tn1;
      n1 = adv(n1);
      tn1 = tile_at(n1);
    }
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// Plain multi-field column transform (y passes, x-forward, API passes).

template <int N, int S, int V, int SEP>
__global__ void __launch_bounds__(PipeCfg<N, V>::THREADS, PipeCfg<N, V>::MINB)
k_pipe_plain(const double2* in, double2* out, long long in_cs, long long out_cs, int nfields,
             ColGeom g, ColGeom go, int ntiles, const double2* __restrict__ tw,
             const __grid_constant__ CUtensorMap tm) {
  const OutSel<N, SEP> os(go, Lanes<N, V>().t);
  // one read of the register twiddles per kernel (from L2), not per item
  LastTw lt{};
  if constexpr (N == 512) lt = last_twiddles<N>(tw, Lanes<N, V>().t);
  pipeline<N, V>(ntiles, 0, nfields, g, [&](int f) { return in + f * in_cs; },
                 [](int f) { return f; }, &tm, tw,
                 [&](int f, double2* buf, const Tile& tl, const PosOff<N>& po,
                     const Lanes<N, V>& ln, const double2* tws, auto&& release) {
                   const int t = ln.t;
                   double2 v[fft_elems(N)];
                   read_own<N>(v, buf, ln.idx, t);
                   ln.bar();
                   col_fft_lt<N, S>(v, buf, ln.idx, t, tws, ln.bar, lt);
                   release();  // buffer no longer read: the next tile may load
                   store_own<N, SEP == 2>(out + f * out_cs, v, go, os.tile(tl, go), os.po(po), t);
                 });
  peer_fence<SEP>();
}

// ---------------------------------------------------------------------------
// P1: x inverse of u_hat -> [U0, U1, U2, w2', K2] (fields 0..4 of `out`),
// w2' = i (F(kx u1) - ky U0).

template <int N, int V, int SEP>
__global__ void __launch_bounds__(PipeCfg<N, V>::THREADS, PipeCfg<N, V>::MINB)
k_pipe_xinv(const double2* u, long long u_cs, double2* out, long long out_cs, ColGeom g,
            ColGeom go, int ntiles, int f_lo, int f_cnt, const double2* __restrict__ tw,
            const __grid_constant__ CUtensorMap tm) {
  constexpr int E = fft_elems(N), TPC = N / E;
  constexpr bool SCR = PipeCfg<N, V>::SCR > 0;
  extern __shared__ __align__(128) double2 smem[];
  const OutSel<N, SEP> os(go, Lanes<N, V>().t);
  double2* const scr = smem + PipeCfg<N, V>::NBUF * N * PipeCfg<N, V>::CS;
  pipeline<N, V>(ntiles, f_lo, f_cnt, g, [&](int f) { return u + f * u_cs; },
                 [](int f) { return f; },
                 &tm, tw,
                 [&](int f, double2* buf, const Tile& tl, const PosOff<N>& po,
                     const Lanes<N, V>& ln, const double2* tws, auto&&) {
                   const int t = ln.t;
                   double2 v[E], vin[SCR ? 1 : E];
                   (void)vin;
                   read_own<N>(v, buf, ln.idx, t);
                   if constexpr (!SCR) {
#pragma unroll
                     for (int m = 0; m < E; ++m) vin[m] = v[m];
                   }
                   if (f > 0) {
                     if constexpr (!SCR) ln.bar();  // the transform below reuses buf
                     // n <= 64: small grids walk (tile, component) units on
                     // separate CTAs (split_units), where U0 of this tile may
                     // not exist yet, so w2' = i F(kx u1 - ky u0) by linearity
                     // with u0 read directly (at every p and transpose mode,
                     // so all of them agree bit for bit)
                     const bool lin = N <= 64 && f == 1 && tl.valid;
                     const double ky = wavenum(g.row_off + tl.row, N);
#pragma unroll
                     for (int m = 0; m < E; ++m) {
                       const double kx = wavenum(t + m * TPC, N);
                       v[m] = make_double2(kx * v[m].x, kx * v[m].y);
                       if (lin) {
                         const double2 a = u[tl.base + po.o(m)];
                         v[m] = make_double2(v[m].x - ky * a.x, v[m].y - ky * a.y);
                       }
                     }
                     col_fft<N, +1>(v, SCR ? scr : buf, ln.idx, t, tws, ln.bar);
                     if (lin) {
#pragma unroll
                       for (int m = 0; m < E; ++m) v[m] = times_i(v[m]);
                     } else if (f == 1) {
                       // w2' = i (K1 - ky U0): ky is constant along an x column and
                       // U0 of this tile was stored by item 0 (L2-resident)
                       if (tl.valid) {
                         const Tile to = os.tile(tl, go);
                         const PosOff<N>& pout = os.po(po);
                         const double2* u0 = out + to.base;
#pragma unroll
                         for (int m = 0; m < E; ++m) {
                           long long at = pout.o(m);
                           if constexpr (SEP == 2) at += __ldg(go.seg + ((t + m * TPC) >> go.pb_shift));
                           const double2 a = u0[at];
                           v[m] = times_i(make_double2(v[m].x - ky * a.x, v[m].y - ky * a.y));
                         }
                       }
                     }
                     store_own<N, SEP == 2>(out + (2 + f) * out_cs, v, go, os.tile(tl, go), os.po(po), t);
                     if constexpr (SCR) {
                       read_own<N>(v, buf, ln.idx, t);
                     } else {
#pragma unroll
                       for (int m = 0; m < E; ++m) v[m] = vin[m];
                     }
                   }
                   if (SCR || f == 0) ln.bar();  // buf is read; the transform reuses it
                   col_fft<N, +1>(v, buf, ln.idx, t, tws, ln.bar);
                   store_own<N, SEP == 2>(out + f * out_cs, v, go, os.tile(tl, go), os.po(po), t);
                 });
  peer_fence<SEP>();
}

// P1 with one transform per item on a single 8-column tile buffer (n = 1024,
// where two 128 B-row tiles plus a scratch tile do not fit): items
//   0: U0 = F(u0)   1: w2' = i (F(kx u1) - ky U0)   2: U1 = F(u1)
//   3: K2 = F(kx u2)   4: U2 = F(u2)
// The second item of a component reloads its tile (from L2: the same CTA
// loaded it one item earlier). Same transforms and operations as k_pipe_xinv.
template <int N, int V, int SEP>
__global__ void __launch_bounds__(PipeCfg<N, V>::THREADS, PipeCfg<N, V>::MINB)
k_pipe_xinv1(const double2* u, long long u_cs, double2* out, long long out_cs, ColGeom g,
             ColGeom go, int ntiles, int it_lo, int it_cnt, const double2* __restrict__ tw,
             const __grid_constant__ CUtensorMap tm) {
  constexpr int E = fft_elems(N), TPC = N / E;
  const OutSel<N, SEP> os(go, Lanes<N, V>().t);
  auto comp = [](int it) { return (it + 1) >> 1; };
  pipeline<N, V>(ntiles, it_lo, it_cnt, g, [&](int it) { return u + comp(it) * u_cs; }, comp, &tm,
                 tw,
                 [&](int it, double2* buf, const Tile& tl, const PosOff<N>& po,
                     const Lanes<N, V>& ln, const double2* tws, auto&& release) {
                   const int t = ln.t;
                   const bool kxm = it & 1;
                   double2 v[E];
                   read_own<N>(v, buf, ln.idx, t);
                   if (kxm) {
#pragma unroll
                     for (int m = 0; m < E; ++m) {
                       const double kx = wavenum(t + m * TPC, N);
                       v[m] = make_double2(kx * v[m].x, kx * v[m].y);
                     }
                   }
                   ln.bar();
                   col_fft<N, +1>(v, buf, ln.idx, t, tws, ln.bar);
                   release();  // buffer no longer read: the next tile may load
                   const Tile to = os.tile(tl, go);
                   const PosOff<N> pout = E >= 16 ? os.po(po).fresh() : os.po(po);
                   if (it == 1 && tl.valid) {
                     const double ky = wavenum(g.row_off + tl.row, N);
                     const double2* u0 = out + to.base;
#pragma unroll
                     for (int m = 0; m < E; ++m) {
                       long long at = pout.o(m);
                       if constexpr (SEP == 2) at += __ldg(go.seg + ((t + m * TPC) >> go.pb_shift));
                       const double2 a = u0[at];
                       v[m] = times_i(make_double2(v[m].x - ky * a.x, v[m].y - ky * a.y));
                     }
                   }
                   const int of = kxm ? 2 + comp(it) : comp(it);
                   store_own<N, SEP == 2>(out + of * out_cs, v, go, to, pout, t);
                 });
  peer_fence<SEP>();
}

// ---------------------------------------------------------------------------
// P2: y inverse of fields 0..4 = [U0, U1, U2, w2', K2] of `fin`, producing
// [u0, u1, u2, w0', w1', w2] in fields 0..5 of `f` (in place for the slab
// layouts). Items per tile in the order U0, U1, w2', U2, K2: field 3 (w2') is
// consumed before the U2 item writes w0' over it.

template <int N, int V, int SEP>
__global__ void __launch_bounds__(PipeCfg<N, V>::THREADS, PipeCfg<N, V>::MINB)
k_pipe_yinv(const double2* fin, double2* f, long long cs_in, long long cs, ColGeom g, ColGeom go,
            int ntiles, int f_lo, int f_cnt, const double2* __restrict__ tw,
            const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmo) {
  constexpr int E = fft_elems(N), TPC = N / E;
  // field of item it: 0, 1, 3, 2, 4
  auto order = [](int it) { return it ^ ((it >> 1) & ~(it >> 2) & 1); };
  LastTw lt{};  // register twiddles read once per kernel
  if constexpr (N == 512) lt = last_twiddles<N>(tw, Lanes<N, V>().t);
  const OutSel<N, SEP> os(go, Lanes<N, V>().t);
  extern __shared__ __align__(128) double2 smem[];
  double2* const stage = smem + PipeCfg<N, V>::NBUF * N * PipeCfg<N, V>::CS;
  // peer-direct output (SEP 2) has one destination per position segment:
  // LSU stores; otherwise TMA tensor stores where an output map exists
  const bool tst = SEP != 2 && PipeCfg<N, V>::SCR > 0 && go.tma != 0;
  auto put = [&](int field, const double2(&r)[E], const Tile& tl, const PosOff<N>& po, int t) {
    if (tst)
      tma_put<N, PipeCfg<N, V>::CS>(&tmo, r, stage, CIdx<PipeCfg<N, V>::CS>{Lanes<N, V>().col}, t,
                                    tl, field);
    else
      store_own<N, SEP == 2>(f + field * cs, r, go, os.tile(tl, go), os.po(po), t);
  };
  pipeline<N, V>(ntiles, f_lo, f_cnt, g, [&](int it) { return fin + order(it) * cs_in; }, order,
                 &tm, tw,
                 [&](int it, double2* buf, const Tile& tl, const PosOff<N>& po,
                     const Lanes<N, V>& ln, const double2* tws, auto&&) {
                   const int t = ln.t;
                   double2 vin[E], v[E];
                   read_own<N>(vin, buf, ln.idx, t);
                   ln.bar();
                   if (it == 3) {  // U2 -> w0' = F(i ky U2) (and u2 below)
#pragma unroll
                     for (int m = 0; m < E; ++m) {
                       const double ky = wavenum(t + m * TPC, N);
                       v[m] = times_i(make_double2(ky * vin[m].x, ky * vin[m].y));
                     }
                     col_fft_lt<N, +1>(v, buf, ln.idx, t, tws, ln.bar, lt);
                     put(3, v, tl, po, t);
                   }
                   if (it == 2) {  // w2' -> w2 = F(w2')
                     col_fft_lt<N, +1>(vin, buf, ln.idx, t, tws, ln.bar, lt);
                     put(5, vin, tl, po, t);
                   } else if (it == 4) {  // K2 -> w1' = F(-i K2)
#pragma unroll
                     for (int m = 0; m < E; ++m) v[m] = times_mi(vin[m]);
                     col_fft_lt<N, +1>(v, buf, ln.idx, t, tws, ln.bar, lt);
                     put(4, v, tl, po, t);
                   } else {  // U0, U1, U2 -> u_c
                     col_fft_lt<N, +1>(vin, buf, ln.idx, t, tws, ln.bar, lt);
                     put(order(it), vin, tl, po, t);
                   }
                 });
  if (tst && threadIdx.x == 0) bulk_wait0();
  peer_fence<SEP>();
}

// ---------------------------------------------------------------------------
// Launchers

#define SDNS_FOR_N(X) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024)

static int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <class K>
static unsigned persistent_grid(K kernel, int threads, size_t smem, long long ntiles,
                                int* cache) {
  if (*cache == 0) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    *cache = occ > 0 ? occ : 1;
  }
  const long long g = static_cast<long long>(*cache) * num_sms();
  return static_cast<unsigned>(ntiles < g ? ntiles : g);
}

// Work units of a column pass: tiles, or tile pairs where the pipeline
// walks pairs (n = 1024, 4-column tiles).
template <int N, int V>
constexpr int NBUF_RING() {
  return PipeCfg<N, V>::NBUF;
}

template <int N, int V>
static long long work_units(long long ntiles) {
  return (PipeCfg<N, V>::CS == 4 && N >= 1024) ? (ntiles + 1) / 2 : ntiles;
}

// Fields of a tile are independent items in the plain passes and in P2
// with separate input and output buffers: when the tiles alone cannot fill
// the GPU (small n), the CTAs walk (tile, item) units so more of them run
// shorter chains (the ring pipeline is unchanged).
template <int N, int V>
static void split_units(ColGeom& g, long long nt, int items, int occ, unsigned& grid) {
  constexpr bool PAIR = PipeCfg<N, V>::CS == 4 && N >= 1024;
  const long long cap = static_cast<long long>(occ) * num_sms();
  // (measured: 64^3 step 0.170 -> 0.156 ms, bitwise equal; no gain at 128)
  if (N > 64 || PAIR || items <= 1 || nt >= cap || NBUF_RING<N, V>() < 2) return;
  g.split = 1;
  const long long units = nt * items;
  grid = static_cast<unsigned>(units < cap ? units : cap);
}

template <int N, int V>
static long long ntiles_of(const ColGeom& g) {
  const long long cols = static_cast<long long>(g.nrows) * g.pitch;
  return (cols + PipeCfg<N, V>::CS - 1) / PipeCfg<N, V>::CS;
}

// Tensor map of a column pass's tile source, or false (LDGSTS path) when the
// layout is not a plain (kz, rows, positions) block: split position strides
// (slab receive layouts), no memory pitch recorded, or tiles narrower than
// the TileIdx<8> rows a box lands in.
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// L2 promotion of the tile loads: a tile row is exactly one 128 B line; a
// 256 B promotion drags in the neighbouring line, which belongs to another
// tile and is often evicted before that tile runs (64 / 256 B / none
// measured no better).
constexpr CUtensorMapL2promotion kTilePromotion = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;

template <int N, int CS>
static ColGeom with_tile_map(const ColGeom& g, const double2* base, long long fcs, int nfields,
                             CUtensorMap* tm) {
  ColGeom r = g;
  r.tma = 0;
  std::memset(tm, 0, sizeof(*tm));
  if ((CS != 8 && CS != 4) || g.mpitch <= 0 || g.mrows <= 0 || ((N - 1) >> g.pb_shift) != 0)
    return r;
  const auto enc = tmap_encoder();
  if (!enc) return r;
  constexpr cuuint32_t BP = N < 256 ? N : 256;
  const cuuint64_t B = sizeof(double2);
  const cuuint64_t dims[5] = {16, static_cast<cuuint64_t>(g.mpitch / 8),
                              static_cast<cuuint64_t>(g.mrows), N,
                              static_cast<cuuint64_t>(nfields)};
  const cuuint64_t strides[4] = {static_cast<cuuint64_t>(g.kcs) * B,
                                 static_cast<cuuint64_t>(g.rs) * B,
                                 static_cast<cuuint64_t>(g.ps0) * B,
                                 static_cast<cuuint64_t>(fcs) * B};
  const cuuint32_t box[5] = {2 * CS, 1, 1, BP, 1}, es[5] = {1, 1, 1, 1, 1};
  const CUresult e = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double2*>(base), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, kTilePromotion,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (e == CUDA_SUCCESS) r.tma = 1;  // else: LDGSTS tiles (same results)
  return r;
}

template <int N, int S, int V, int SEP>
static void plain_launch(const double2* in, double2* out, long long in_cs, long long out_cs,
                         int nfields, const ColGeom& g, const ColGeom& go, const double2* tw,
                         cudaStream_t s) {
  using C = PipeCfg<N, V>;
  const long long nt = ntiles_of<N, V>(g);
  if (nt <= 0) return;
  static int occ = 0;
  unsigned grid =
      persistent_grid(k_pipe_plain<N, S, V, SEP>, C::THREADS, C::SMEM, work_units<N, V>(nt), &occ);
  CUtensorMap tm;
  ColGeom gt = with_tile_map<N, C::CS>(g, in, in_cs, nfields, &tm);
  split_units<N, V>(gt, nt, nfields, occ, grid);
  k_pipe_plain<N, S, V, SEP><<<grid, C::THREADS, C::SMEM, s>>>(in, out, in_cs, out_cs, nfields,
                                                               gt, go, static_cast<int>(nt), tw, tm);
}

template <int N>
static void col_plain_n(int dir, bool xaxis, const double2* in, double2* out, long long in_cs,
                        long long out_cs, int nfields, const ColGeom& g, const ColGeom* go,
                        const double2* tw, cudaStream_t s) {
  constexpr int VX = N >= 1024 ? 9 : sdns_dev::VX, VY = sdns_dev::VY;
  if (go && go->seg) {  // peer-direct output (slab transposes fused into the pass)
    if (xaxis) {
      if (dir < 0) plain_launch<N, -1, VX, 2>(in, out, in_cs, out_cs, nfields, g, *go, tw, s);
      else plain_launch<N, +1, VX, 2>(in, out, in_cs, out_cs, nfields, g, *go, tw, s);
    } else {
      if (dir < 0) plain_launch<N, -1, VY, 2>(in, out, in_cs, out_cs, nfields, g, *go, tw, s);
      else plain_launch<N, +1, VY, 2>(in, out, in_cs, out_cs, nfields, g, *go, tw, s);
    }
    return;
  }
  if (go) {  // separate output layout (pencil y passes; the chunked x forward)
    if (xaxis) {
      if (dir < 0) plain_launch<N, -1, VX, 1>(in, out, in_cs, out_cs, nfields, g, *go, tw, s);
      else plain_launch<N, +1, VX, 1>(in, out, in_cs, out_cs, nfields, g, *go, tw, s);
    } else {
      if (dir < 0) plain_launch<N, -1, VY, 1>(in, out, in_cs, out_cs, nfields, g, *go, tw, s);
      else plain_launch<N, +1, VY, 1>(in, out, in_cs, out_cs, nfields, g, *go, tw, s);
    }
    return;
  }
  if (dir < 0) {
    if (xaxis) plain_launch<N, -1, VX, 0>(in, out, in_cs, out_cs, nfields, g, g, tw, s);
    else plain_launch<N, -1, VY, 0>(in, out, in_cs, out_cs, nfields, g, g, tw, s);
  } else {
    if (xaxis) plain_launch<N, +1, VX, 0>(in, out, in_cs, out_cs, nfields, g, g, tw, s);
    else plain_launch<N, +1, VY, 0>(in, out, in_cs, out_cs, nfields, g, g, tw, s);
  }
}

// Generic-length items (kernels_gen.cu): the plain pass, P1's components
// and P2's items in the tuned kernels' order.
static void gen_plain(int n, int dir, const double2* in, double2* out, long long in_cs,
                      long long out_cs, int nfields, const ColGeom& g, const ColGeom& go,
                      const double2* tw, cudaStream_t s) {
  GItem it[8];
  for (int f = 0; f < nfields; ++f) it[f] = GItem{f, f, G_NONE, G_PLAIN};
  for (int f0 = 0; f0 < nfields; f0 += 8)
    gen_col(n, dir, in + f0 * in_cs, out + f0 * out_cs, in_cs, out_cs, std::min(8, nfields - f0),
            it, g, go, tw, s);
}

void col_plain(int n, int dir, bool xaxis, const double2* in, double2* out, long long in_cs,
               long long out_cs, int nfields, const ColGeom& g, const double2* tw,
               cudaStream_t s) {
  if (!tuned_length(n)) {
    gen_plain(n, dir, in, out, in_cs, out_cs, nfields, g, g, tw, s);
    return;
  }
  switch (n) {
#define X(NN) \
  case NN: col_plain_n<NN>(dir, xaxis, in, out, in_cs, out_cs, nfields, g, nullptr, tw, s); return;
    SDNS_FOR_N(X)
#undef X
  }
}

void col_plain_to(int n, int dir, const double2* in, double2* out, long long in_cs,
                  long long out_cs, int nfields, const ColGeom& g, const ColGeom& go,
                  const double2* tw, cudaStream_t s, bool xaxis) {
  if (!tuned_length(n)) {
    gen_plain(n, dir, in, out, in_cs, out_cs, nfields, g, go, tw, s);
    return;
  }
  switch (n) {
#define X(NN) \
  case NN: col_plain_n<NN>(dir, xaxis, in, out, in_cs, out_cs, nfields, g, &go, tw, s); return;
    SDNS_FOR_N(X)
#undef X
  }
}

// P1 as five single-transform items (k_pipe_xinv1): the default at n = 1024
// (single 8-column tile buffer); selectable at n >= 128 (ColGeom::single).
template <int N>
static void x_inv1_n(const double2* u, long long u_cs, double2* out, long long out_cs,
                     const ColGeom& g, const ColGeom* go, int f_lo, int f_cnt, const double2* tw,
                     cudaStream_t s) {
  constexpr int V = N >= 1024 ? 9 : 0;
  using C = PipeCfg<N, V>;
  const long long nt = ntiles_of<N, V>(g);
  if (nt <= 0) return;
  // components [f_lo, f_lo + f_cnt) -> items: component 0 is item 0,
  // component c > 0 items 2c - 1 and 2c
  const int it_lo = f_lo == 0 ? 0 : 2 * f_lo - 1, it_hi = 2 * (f_lo + f_cnt) - 1;
  CUtensorMap tm;
  const ColGeom gt = with_tile_map<N, C::CS>(g, u, u_cs, 3, &tm);
  const int ntl = static_cast<int>(nt);
  if (go && go->seg) {
    static int occ = 0;
    const unsigned grid = persistent_grid(k_pipe_xinv1<N, V, 2>, C::THREADS, C::SMEM, nt, &occ);
    k_pipe_xinv1<N, V, 2><<<grid, C::THREADS, C::SMEM, s>>>(u, u_cs, out, out_cs, gt, *go, ntl,
                                                            it_lo, it_hi - it_lo, tw, tm);
  } else if (go) {
    static int occ = 0;
    const unsigned grid = persistent_grid(k_pipe_xinv1<N, V, 1>, C::THREADS, C::SMEM, nt, &occ);
    k_pipe_xinv1<N, V, 1><<<grid, C::THREADS, C::SMEM, s>>>(u, u_cs, out, out_cs, gt, *go, ntl,
                                                            it_lo, it_hi - it_lo, tw, tm);
  } else {
    static int occ = 0;
    const unsigned grid = persistent_grid(k_pipe_xinv1<N, V, 0>, C::THREADS, C::SMEM, nt, &occ);
    k_pipe_xinv1<N, V, 0><<<grid, C::THREADS, C::SMEM, s>>>(u, u_cs, out, out_cs, gt, gt, ntl,
                                                            it_lo, it_hi - it_lo, tw, tm);
  }
}

template <int N>
static void x_inv_n(const double2* u, long long u_cs, double2* out, long long out_cs,
                    const ColGeom& g, const ColGeom* go, int f_lo, int f_cnt, const double2* tw,
                    cudaStream_t s) {
  if constexpr (N >= 128) {
    if (g.single) {
      x_inv1_n<N>(u, u_cs, out, out_cs, g, go, f_lo, f_cnt, tw, s);
      return;
    }
  }
  using C = PipeCfg<N, VXI>;
  const long long nt = ntiles_of<N, VXI>(g);
  CUtensorMap tm;
  const ColGeom gt = with_tile_map<N, C::CS>(g, u, u_cs, 3, &tm);
  if (go && go->seg) {  // peer-direct output (slab x inverse into the peers' receive layouts)
    static int occ = 0;
    unsigned grid = persistent_grid(k_pipe_xinv<N, VXI, 2>, C::THREADS, C::SMEM, work_units<N, VXI>(nt), &occ);
    ColGeom gs = gt;
    split_units<N, VXI>(gs, nt, f_cnt, occ, grid);
    k_pipe_xinv<N, VXI, 2><<<grid, C::THREADS, C::SMEM, s>>>(
        u, u_cs, out, out_cs, gs, *go, static_cast<int>(nt), f_lo, f_cnt, tw, tm);
  } else if (go) {
    static int occ = 0;
    unsigned grid = persistent_grid(k_pipe_xinv<N, VXI, 1>, C::THREADS, C::SMEM, work_units<N, VXI>(nt), &occ);
    ColGeom gs = gt;
    split_units<N, VXI>(gs, nt, f_cnt, occ, grid);
    k_pipe_xinv<N, VXI, 1><<<grid, C::THREADS, C::SMEM, s>>>(
        u, u_cs, out, out_cs, gs, *go, static_cast<int>(nt), f_lo, f_cnt, tw, tm);
  } else {
    static int occ = 0;
    unsigned grid =
        persistent_grid(k_pipe_xinv<N, VXI, 0>, C::THREADS, C::SMEM, work_units<N, VXI>(nt), &occ);
    ColGeom gs = gt;
    split_units<N, VXI>(gs, nt, f_cnt, occ, grid);
    k_pipe_xinv<N, VXI, 0><<<grid, C::THREADS, C::SMEM, s>>>(
        u, u_cs, out, out_cs, gs, gt, static_cast<int>(nt), f_lo, f_cnt, tw, tm);
  }
}

void x_inverse_split(int n, const double2* u, long long u_cs, double2* out, long long out_cs,
                     const ColGeom& g, const ColGeom* go, const double2* tw, cudaStream_t s,
                     int comp_lo, int comp_cnt) {
  if (!tuned_length(n)) {
    // component c: U_c (field c); c = 1 also w2' = i(F(kx u1) - ky U0)
    // (field 3), c = 2 also K2 = F(kx u2) (field 4)
    GItem it[8];
    int ni = 0;
    for (int c = comp_lo; c < comp_lo + comp_cnt; ++c) {
      it[ni++] = GItem{c, c, G_NONE, G_PLAIN};
      if (c == 1) it[ni++] = GItem{1, 3, G_K, G_W2};
      if (c == 2) it[ni++] = GItem{2, 4, G_K, G_PLAIN};
    }
    gen_col(n, +1, u, out, u_cs, out_cs, ni, it, g, go ? *go : g, tw, s);
    return;
  }
  switch (n) {
#define X(NN) \
  case NN: x_inv_n<NN>(u, u_cs, out, out_cs, g, go, comp_lo, comp_cnt, tw, s); return;
    SDNS_FOR_N(X)
#undef X
  }
}

template <int N>
static void y_inv_n(const double2* fin, double2* f, long long cs_in, long long cs,
                    const ColGeom& g, const ColGeom* go, int f_lo, int f_cnt, const double2* tw,
                    cudaStream_t s) {
  using C = PipeCfg<N, VYI>;
  const long long nt = ntiles_of<N, VYI>(g);
  if (go && go->seg) {  // peer-direct output (pencil y inverse into the row peers' z lines)
    static int occ = 0;
    const unsigned grid =
        persistent_grid(k_pipe_yinv<N, VYI, 2>, C::THREADS, C::SMEM, work_units<N, VYI>(nt), &occ);
    CUtensorMap tm;
    const ColGeom gt = with_tile_map<N, C::CS>(g, fin, cs_in, 5, &tm);
    CUtensorMap tmo;
    std::memset(&tmo, 0, sizeof(tmo));
    ColGeom got = *go;
    got.tma = 0;
    k_pipe_yinv<N, VYI, 2><<<grid, C::THREADS, C::SMEM, s>>>(
        fin, f, cs_in, cs, gt, got, static_cast<int>(nt), f_lo, f_cnt, tw, tm, tmo);
  } else if (go) {  // separate input and output buffers: items independent
    static int occ = 0;
    unsigned grid =
        persistent_grid(k_pipe_yinv<N, VYI, 1>, C::THREADS, C::SMEM, work_units<N, VYI>(nt), &occ);
    CUtensorMap tm;
    ColGeom gt = with_tile_map<N, C::CS>(g, fin, cs_in, 5, &tm);
    split_units<N, VYI>(gt, nt, f_cnt, occ, grid);
    CUtensorMap tmo;
    const ColGeom got = with_tile_map<N, C::CS>(*go, f, cs, 6, &tmo);
    k_pipe_yinv<N, VYI, 1><<<grid, C::THREADS, C::SMEM, s>>>(
        fin, f, cs_in, cs, gt, got, static_cast<int>(nt), f_lo, f_cnt, tw, tm, tmo);
  } else {
    static int occ = 0;
    const unsigned grid =
        persistent_grid(k_pipe_yinv<N, VYI, 0>, C::THREADS, C::SMEM, work_units<N, VYI>(nt), &occ);
    CUtensorMap tm;
    const ColGeom gt = with_tile_map<N, C::CS>(g, fin, cs_in, 5, &tm);
    CUtensorMap tmo;
    std::memset(&tmo, 0, sizeof(tmo));
    ColGeom go = gt;
    go.tma = 0;  // in place: LSU stores
    k_pipe_yinv<N, VYI, 0><<<grid, C::THREADS, C::SMEM, s>>>(
        fin, f, cs_in, cs, gt, go, static_cast<int>(nt), f_lo, f_cnt, tw, tm, tmo);
  }
}

// P2 items 0..4 (U0, U1, w2', U2, K2) as generic items.
static int gen_yinv_items(int item_lo, int item_cnt, GItem* it) {
  int ni = 0;
  for (int i = item_lo; i < item_lo + item_cnt; ++i) {
    if (i == 0) it[ni++] = GItem{0, 0, G_NONE, G_PLAIN};
    if (i == 1) it[ni++] = GItem{1, 1, G_NONE, G_PLAIN};
    if (i == 2) it[ni++] = GItem{3, 5, G_NONE, G_PLAIN};  // w2 = F(w2')
    if (i == 3) {
      it[ni++] = GItem{2, 3, G_IK, G_PLAIN};  // w0' = F(i ky U2)
      it[ni++] = GItem{2, 2, G_NONE, G_PLAIN};
    }
    if (i == 4) it[ni++] = GItem{4, 4, G_MI, G_PLAIN};  // w1' = F(-i K2)
  }
  return ni;
}

void y_inverse_curl(int n, double2* f, long long cs, const ColGeom& g, const double2* tw,
                    cudaStream_t s, int item_lo, int item_cnt) {
  if (!tuned_length(n)) {
    GItem it[8];
    const int ni = gen_yinv_items(item_lo, item_cnt, it);
    gen_col(n, +1, f, f, cs, cs, ni, it, g, g, tw, s);
    return;
  }
  switch (n) {
#define X(NN) \
  case NN: y_inv_n<NN>(f, f, cs, cs, g, nullptr, item_lo, item_cnt, tw, s); return;
    SDNS_FOR_N(X)
#undef X
  }
}

void y_inverse_curl_to(int n, const double2* fin, double2* fout, long long cs_in, long long cs_out,
                       const ColGeom& g, const ColGeom& go, const double2* tw, cudaStream_t s) {
  if (!tuned_length(n)) {
    GItem it[8];
    const int ni = gen_yinv_items(0, 5, it);
    gen_col(n, +1, fin, fout, cs_in, cs_out, ni, it, g, go, tw, s);
    return;
  }
  switch (n) {
#define X(NN) \
  case NN: y_inv_n<NN>(fin, fout, cs_in, cs_out, g, &go, 0, 5, tw, s); return;
    SDNS_FOR_N(X)
#undef X
  }
}

}  // namespace sdns_dev
