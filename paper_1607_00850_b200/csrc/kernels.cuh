// Kernel launch interface shared by the host orchestration (context.cu) and
// the kernel translation unit (kernels.cu). All device fields use the
// padded spectral layout described in DESIGN.md §3:
//   spectral component: rows of `pitch` complex (pitch = kz extent rounded
//   up to a multiple of 8), only the first `n2` entries of a row are modes;
//   real component: rows of n doubles, unpadded.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sdns_dev {

// Addressing of the FFT columns of a column pass (x or y axis). The element
// at (row, pos, kz) lives at row*rs + (pos >> pb_shift)*ps1 +
// (pos & ((1<<pb_shift)-1))*ps0 + kz. This covers the natural layouts and the
// slab receive layout [peer][x_l][y_l][kz] with one formula.
//
// Work enumeration (forward dealias pruning): tiles walk
// `nrows` enumerated rows x `pitch` kz slots, of which the first n2 are
// transformed; enumerated row r maps to storage row r + off0 for r < seg_a,
// else r - seg_a + off1 (the two kept |k| < n/3 bands). keep_k >= 0 limits
// the stored output positions to |wavenumber| <= keep_k.
struct ColGeom {
  long long rs = 0, ps0 = 0, ps1 = 0;
  long long kcs = 8;  // stride of 8-column kz chunks: 8 = plain rows; larger
                      // for chunk-major layouts ((kz>>3)*kcs + (kz&7))
  int pb_shift = 30;
  // position block size of the same split (pos / pblk, pos % pblk) for the
  // generic-length kernels, whose blocks need not be powers of two; 0: no
  // split (pb_shift = 30)
  int pblk = 0;
  int nrows = 0;
  int n2 = 0;     // transformed kz entries per row
  int pitch = 0;  // kz slots per enumerated row (multiple of the tile width)
  int seg_a = 1 << 30, off0 = 0, off1 = 0;
  int keep_k = -1;
  int row_off = 0;  // global index of storage row 0 (x pass: the y offset)
  // Tensor-map tile loads (launcher-set): memory row pitch (complex; 8 *
  // the number of kz chunks) and storage-row extent of the source; tma = 1:
  // tiles come from the tensor map, 0: LDGSTS path.
  int mpitch = 0, mrows = 0, tma = 0;
  // Launcher-set: the CTAs walk (tile, item) units instead of whole tiles
  // (small grids: more CTAs, each a shorter chain; only where items of a
  // tile are independent)
  int split = 0;
  // x inverse pass (P1): five single-transform items on one tile buffer
  // (k_pipe_xinv1) instead of three items with a scratch tile
  int single = 0;
  // Peer-direct output (slab transposes fused into the producing pass,
  // DESIGN.md §5): element offset of segment pos >> pb_shift's destination
  // block from the output base -- another rank's buffer on this device or
  // mapped over NVLink. Device array; nullptr: plain output.
  const long long* seg = nullptr;
};

// Wavenumbers of a column pass: which physical axis the transform runs
// along and the global offsets of the other two.
struct WaveGeom {
  int n = 0;
  int row_is_y = 1;  // x-pass: rows are local y; y-pass: rows are local x
  int row_off = 0;   // global offset of the row index (y offset for x-pass)
  int kz_off = 0;    // global kz offset of kz index 0
};

constexpr int kMaxSeg = 16;  // max pencil p2

// Row mapping for the z passes. Spectral rows live in planes of `prow`
// rows (the last row of each plane is padding, so that the plane stride is
// an odd multiple of 128 B and strided x-pass accesses spread over all HBM
// channels). Memory order (blk == 0): row ri = (plane ri / rpp, ri % rpp).
// By (x_l, y) (blk = np): ri = x_l*ny + y lives in plane (y/np)*np + x_l,
// row y % np -- the slab receive layout; at p = 1 simply plane x, row y.
struct RowMap {
  int nrows = 0;     // number of rows
  int rpp = 0;       // real rows per plane (memory order)
  int ny = 0;        // real y extent (by-(x_l, y) order)
  int blk = 0;       // 0: memory order; else slab block np
  int prow = 0;      // rows per plane including the pad row
  int pitch = 0;     // spectral row pitch (complex)
  int n2 = 0;        // valid kz entries (n/2+1 for a full z line)
  int kz_keep = 1 << 30;  // forward outputs stored only for kz < kz_keep
  // Chunked rows (p = 1 work layout [x][kz chunk][y][8]): row
  // ri = x*rpp + y starts at x*xplane + y*8 and kz chunk c lies cstride
  // complex further per chunk. cstride == 0: the row maps above.
  int cstride = 0;
  long long xplane = 0;
  // Pencil: a z line is assembled from nseg kz blocks (one per row peer,
  // fft.cpp:141-160); block q holds rows ri at seg_base[q] + ri*seg_pitch[q]
  // for kz in [seg_k0[q], seg_k0[q+1]). nseg == 0: the row maps above.
  int nseg = 0;
  long long seg_base[kMaxSeg] = {};
  int seg_pitch[kMaxSeg] = {};
  int seg_k0[kMaxSeg + 1] = {};
  // Output maps of a peer-direct z pass (z_fused_to): component stride of
  // each segment's destination (segments then live in different buffers).
  long long seg_cs[kMaxSeg] = {};
};

// Fused x-pass forward epilogue variants.
enum XfMode : int {
  XF_TAIL = 0,  // du = P[mask*FFT(nl)] - nu k^2 u            (compute_rhs)
  XF_RK0 = 1,   // stage 0: accum = du; ustage = u0 + b dt du
  XF_RK12 = 2,  // stages 1,2: accum += w du; ustage = u0 + b dt du
  XF_RK3 = 3,   // stage 3: Neumaier final update (+ optional projection)
};

struct XfArgs {
  const double2* nl;   // 3 comps, FFT input (x-layout)
  long long nl_cs;     // component stride of nl
  const double2* u;    // stage input u_hat (viscous term)
  double2* out;        // XF_TAIL: du; XF_RK0/12: new stage value
  const double2* base; // u0
  double2* base_out;   // XF_RK3: new state (may alias base)
  double2* accum;
  double2* carry;
  long long cs;        // component stride of u/out/base/accum/carry
  double nu;
  double w;            // accum weight
  double bdt;          // stage offset * dt
  double ubdt;         // XF_RK12: != 0 -> u = base + ubdt * accum (stage 1: u_1
                       // rebuilt bitwise from accum = du_0, saving the read of u)
  // When set, the dt-dependent scalars come from device memory instead
  // (captured steps replay with any dt): dts = [b0 dt, b1 dt, b2 dt, dt/6],
  // bdt = dts[dts_stage], ubdt = dts[0] (if ubdt != 0), sixth = dts[3].
  const double* dts = nullptr;
  int dts_stage = 0;
  double sixth;        // dt/6 (stage 3)
  int dealias;
  int project;         // stage 3: post-step projection
  int* finite;         // stage 3: cleared to 0 on a non-finite value
  // stage 3: when set, the sampled diagnostics of the new state are
  // accumulated in the same pass (per-plane partials, folded into stats_out)
  double* stats_partial = nullptr;
  double* stats_out = nullptr;
  int shells = 0;
};

// twiddle table of length-n transforms: the stage-ordered table of the
// radix-8/16 kernels (power-of-two n <= 1024), else exp(-2 pi i q / n),
// q in [0, n), for the generic-length kernels
void make_twiddles(int n, double2* d_tw, cudaStream_t s);

// Power-of-two n in [4, 1024] run the tuned kernels; every other even n runs
// the generic mixed-radix kernels of kernels_gen.cu behind the same
// launchers and geometries (the reference accepts any even n >= 4,
// config.cpp:17-19).
inline bool tuned_length(int n) { return n >= 4 && n <= 1024 && (n & (n - 1)) == 0; }
// Shared memory the generic z pass needs at length n (0 if n is tuned).
size_t gen_z_smem(int n);

// Generic-length column pass: `nitems` items per tile, item i reads field
// it[i].fin of `in` (geometry g), applies the pre-op, transforms (dir -1
// forward, +1 inverse), applies the post-op and stores field it[i].fout of
// `out` (geometry go; go.seg: peer-direct). Items of a tile run in order,
// so an in-place pass may overwrite a field an earlier item consumed.
enum GPre : int { G_NONE = 0, G_K = 1, G_IK = 2, G_MI = 3 };  // x, k x, i k x, -i x
enum GPost : int { G_PLAIN = 0, G_W2 = 1 };  // w2' = i (v - k_row U0), U0 = out field 0
struct GItem {
  int fin, fout, pre, post;
};
void gen_col(int n, int dir, const double2* in, double2* out, long long in_cs, long long out_cs,
             int nitems, const GItem* it, const ColGeom& g, const ColGeom& go, const double2* tw,
             cudaStream_t s);
void gen_z_fused(int n, double2* rows, long long cs, const RowMap& rm, double2* out,
                 const RowMap* rmo, double norm, const double2* tw, cudaStream_t s);
void gen_z_c2r(int n, const double2* spec, double* real, const RowMap& rm, double norm,
               const double2* tw, cudaStream_t s);
void gen_z_r2c(int n, const double* real, double2* spec, const RowMap& rm, const RowMap* rmo,
               int field, const double2* tw, cudaStream_t s);

// xaxis selects the tile shape tuned for the large-stride (x) axis.
void col_plain(int n, int dir, bool xaxis, const double2* in, double2* out, long long in_cs,
               long long out_cs, int nfields, const ColGeom& g, const double2* tw,
               cudaStream_t s);
// P1: u_hat (3 comps) -> [U0, U1, U2, w2', K2] (5 comps of `out`), written
// in geometry go (the input geometry g when go is NULL)
// comp_lo/comp_cnt: input components (items) to run; component c writes
// fields c and (c > 0) 2 + c.
void x_inverse_split(int n, const double2* u, long long u_cs, double2* out, long long out_cs,
                     const ColGeom& g, const ColGeom* go, const double2* tw, cudaStream_t s,
                     int comp_lo = 0, int comp_cnt = 3);
// P2: in place, fields [U0, U1, U2, K1, K2] -> [u0, u1, u2, w0', w1', w2]
// items item_lo .. item_lo+item_cnt-1 of the order U0, U1, w2', U2, K2
// (fields 0, 1, 3, 2, 4)
void y_inverse_curl(int n, double2* f, long long cs, const ColGeom& g, const double2* tw,
                    cudaStream_t s, int item_lo = 0, int item_cnt = 5);
// Same, reading geometry g of `fin` and writing geometry go of `fout`
// (pencil: col-receive layout in, row-send layout out).
void y_inverse_curl_to(int n, const double2* fin, double2* fout, long long cs_in, long long cs_out,
                       const ColGeom& g, const ColGeom& go, const double2* tw, cudaStream_t s);
// Plain column transform with a separate output geometry (pencil y passes;
// with go.seg, the peer-direct slab transposes -- xaxis picks the x tiles).
void col_plain_to(int n, int dir, const double2* in, double2* out, long long in_cs,
                  long long out_cs, int nfields, const ColGeom& g, const ColGeom& go,
                  const double2* tw, cudaStream_t s, bool xaxis = false);
struct SpecGeom;
// P5b: mask + projection + viscous + RK4 stage update, streaming over the
// x layout (a.nl holds the x-forward-transformed nonlinear term).
void rk_update(int mode, const XfArgs& a, const SpecGeom& g, cudaStream_t s);
// dts[0..3] = b dt (b = 1/2, 1/2, 1), dt/6 for the next captured step
void set_step_scalars(double* dts, double dt, cudaStream_t s);

void z_fused(int n, double2* rows, long long cs, const RowMap& rm, double norm,
             const double2* tw, cudaStream_t s);
// Encodes the tensor map the z pass stages chunked rows with (rm.cstride):
// one box of pitch/8 chunks x 128 B per half-row. False if unavailable.
bool z_chunk_map(void* tmap, const double2* base, long long cs, int nfields, const RowMap& rm,
                 int pitch);
// Same, storing the 3 outputs through the segmented output map `rmo`
// (element (ri, kz) of component c at out + seg_base + c*seg_cs +
// ri*seg_pitch + kz - seg_k0 of kz's segment): the pencil forward row
// transpose fused into the z pass (peer-direct).
void z_fused_to(int n, double2* rows, long long cs, const RowMap& rm, double2* out,
                const RowMap& rmo, double norm, const double2* tw, cudaStream_t s);
void z_c2r(int n, const double2* spec, double* real, const RowMap& rm, double norm,
           const double2* tw, cudaStream_t s);
void z_r2c(int n, const double* real, double2* spec, const RowMap& rm, const double2* tw,
           cudaStream_t s);
// Same, storing component `field` through the segmented output map `rmo`
// (see z_fused_to): the pencil forward row transpose fused into the z pass.
void z_r2c_to(int n, const double* real, double2* out, const RowMap& rm, const RowMap& rmo,
              int field, const double2* tw, cudaStream_t s);

// Spectral-layout geometry for pointwise kernels.
struct SpecGeom {
  int n = 0;
  int s0 = 0, s1 = 0, s2 = 0;    // local shape
  int o0 = 0, o1 = 0, o2 = 0;    // global offsets
  int pitch = 0;
  int prow = 0;                  // rows per x plane incl. the pad row (s1 + 1)
  long long cs = 0;              // component stride (s0*prow*pitch)
};

void pw_curl(const double2* u, double2* w, const SpecGeom& g, cudaStream_t s);
void pw_project(double2* u, const SpecGeom& g, cudaStream_t s);
void pw_pressure(const double2* nl, double2* p, const SpecGeom& g, cudaStream_t s);
void pw_cross(const double* a, const double* b, double* o, long long count, long long cs,
              cudaStream_t s);
void pw_fill_pad(double2* f, int ncomp, const SpecGeom& g, cudaStream_t s);
// ncomp spectral components between the padded device layout and the packed
// RankLayout block order (to_packed: padded -> packed)
void pw_repack(const double2* src, double2* dst, int ncomp, const SpecGeom& g, bool to_packed,
               cudaStream_t s);
void pw_finite(const double2* u, const SpecGeom& g, int* flag, cudaStream_t s);

// Deterministic diagnostics partials: per x-plane block sums, then a fixed
// order fold. out = [sum_we, sum_wz, shells...] and divmax.
void stats_local(const double2* u, const SpecGeom& g, int shells, double* d_partial,
                 double* d_out, cudaStream_t s);
int stats_blocks(const SpecGeom& g);
// sum over all components of (a-b)^2 on real fields
void l2_local(const double* a, const double* b, long long count, double* d_partial,
              double* d_out, cudaStream_t s);

}  // namespace sdns_dev
