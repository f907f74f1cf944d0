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
struct ColGeom {
  long long rs = 0, ps0 = 0, ps1 = 0;
  int pb_shift = 30;
  int nrows = 0;
  int n2 = 0;     // valid kz entries per row
  int pitch = 0;  // padded kz entries per row (multiple of 8)
};

// Wavenumbers of a column pass: which physical axis the transform runs
// along and the global offsets of the other two.
struct WaveGeom {
  int n = 0;
  int row_is_y = 1;  // x-pass: rows are local y; y-pass: rows are local x
  int row_off = 0;   // global offset of the row index (y offset for x-pass)
  int kz_off = 0;    // global kz offset of kz index 0
};

// Row mapping for the z passes: real row ri = (x_l, y) -> spectral row.
struct RowMap {
  int nrows = 0;     // number of (x_l, y) rows
  int ny = 0;        // real y extent
  int blk = 0;       // 0: spectral row = ri; else slab recv layout block (np)
  int pitch = 0;     // spectral row pitch
  int n2 = 0;        // valid kz entries (n/2+1 for a full z line)
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
  double sixth;        // dt/6 (stage 3)
  int dealias;
  int project;         // stage 3: post-step projection
  int* finite;         // stage 3: cleared to 0 on a non-finite value
};

// twiddle table exp(-2 pi i q / n), q in [0, n)
void make_twiddles(int n, double2* d_tw, cudaStream_t s);

void col_plain(int n, int dir, const double2* in, double2* out, long long in_cs,
               long long out_cs, int nfields, const ColGeom& g, const double2* tw,
               cudaStream_t s);
void x_inverse_curl(int n, const double2* u, long long u_cs, double2* out, long long out_cs,
                    const ColGeom& g, const WaveGeom& w, const double2* tw, cudaStream_t s);
void x_forward_fused(int n, int mode, const XfArgs& a, const ColGeom& g, const WaveGeom& w,
                     const double2* tw, cudaStream_t s);

void z_fused(int n, double2* rows, long long cs, const RowMap& rm, double norm,
             const double2* tw, cudaStream_t s);
void z_c2r(int n, const double2* spec, double* real, const RowMap& rm, double norm,
           const double2* tw, cudaStream_t s);
void z_r2c(int n, const double* real, double2* spec, const RowMap& rm, const double2* tw,
           cudaStream_t s);

// Spectral-layout geometry for pointwise kernels.
struct SpecGeom {
  int n = 0;
  int s0 = 0, s1 = 0, s2 = 0;    // local shape
  int o0 = 0, o1 = 0, o2 = 0;    // global offsets
  int pitch = 0;
  long long cs = 0;              // component stride (s0*s1*pitch)
};

void pw_curl(const double2* u, double2* w, const SpecGeom& g, cudaStream_t s);
void pw_project(double2* u, const SpecGeom& g, cudaStream_t s);
void pw_pressure(const double2* nl, double2* p, const SpecGeom& g, cudaStream_t s);
void pw_cross(const double* a, const double* b, double* o, long long count, long long cs,
              cudaStream_t s);
void pw_fill_pad(double2* f, int ncomp, const SpecGeom& g, cudaStream_t s);
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
