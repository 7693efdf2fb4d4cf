/*
 * TEST INFRASTRUCTURE ONLY (oracle/): never linked into the product library.
 *
 * Minimal declaration of the three FFTW3 entry points the reference front-end
 * calls (/root/reference/proj/src/pipeline.cpp:179-188):
 *   fftw_plan_dft_r2c_1d(n, in, out, FFTW_ESTIMATE), fftw_execute, fftw_destroy_plan.
 * FFTW3 itself is not installed in this image and is unpinned by the reference
 * build (proj/CMakeLists.txt:13: find_library(FFTW3_LIB fftw3 REQUIRED)), so the
 * arithmetic behind these calls is provided by oracle/fftw_shim/fft_provider.c,
 * which restates FFTW's published contract for a 1-D real-to-complex forward
 * transform: out[k] = sum_j in[j] * exp(-2*pi*i*j*k/n), k = 0..n/2, unnormalised.
 */
#ifndef UWB_ORACLE_FFTW3_SHIM_H
#define UWB_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct uwb_fftw_plan_s* fftw_plan;

#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_r2c_1d(int n, double* in, fftw_complex* out, unsigned flags);
void fftw_execute(const fftw_plan plan);
void fftw_destroy_plan(fftw_plan plan);

#ifdef __cplusplus
}
#endif

#endif
