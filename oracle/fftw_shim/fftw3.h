/*
 * TEST INFRASTRUCTURE (oracle only) — never linked into the product library.
 *
 * Self-written stand-in for the subset of the FFTW3 (double) guru64 API that
 * the reference's SerialFFT adapter calls:
 *   fftw_plan_guru64_dft          reference proj/core/src/serial_fft.cpp:119
 *   fftw_plan_guru64_dft_r2c      :63, :88
 *   fftw_plan_guru64_dft_c2r      :76, :100
 *   fftw_execute_dft{,_r2c,_c2r}  :66, :80, :91, :104, :123
 *   fftw_destroy_plan             :41
 * FFTW itself is absent from this image and has no pinned version in the
 * reference (proj/cmake/FindFFTW3.cmake:4-22), so the published FFTW
 * semantics are restated here: unnormalised transforms, forward sign -1,
 * r2c keeps n/2+1 outputs along the last dimension, c2r takes the logical
 * real length, ignores the imaginary parts of the DC and Nyquist bins and
 * may clobber its input, arbitrary howmany loops with arbitrary strides,
 * any transform length.
 */
#ifndef SDNS_ORACLE_FFTW3_SHIM_H
#define SDNS_ORACLE_FFTW3_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

typedef struct fftw_iodim64_do_not_use_me {
  ptrdiff_t n;
  ptrdiff_t is;
  ptrdiff_t os;
} fftw_iodim64;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_DESTROY_INPUT (1U << 0)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_PRESERVE_INPUT (1U << 4)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_guru64_dft(int rank, const fftw_iodim64* dims,
                               int howmany_rank,
                               const fftw_iodim64* howmany_dims,
                               fftw_complex* in, fftw_complex* out, int sign,
                               unsigned flags);
fftw_plan fftw_plan_guru64_dft_r2c(int rank, const fftw_iodim64* dims,
                                   int howmany_rank,
                                   const fftw_iodim64* howmany_dims,
                                   double* in, fftw_complex* out,
                                   unsigned flags);
fftw_plan fftw_plan_guru64_dft_c2r(int rank, const fftw_iodim64* dims,
                                   int howmany_rank,
                                   const fftw_iodim64* howmany_dims,
                                   fftw_complex* in, double* out,
                                   unsigned flags);

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out);
void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
