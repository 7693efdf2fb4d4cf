/*
 * TEST INFRASTRUCTURE ONLY (oracle/): the CPU provider of the FFTW3 r2c API
 * used when compiling the reference front-end (pipeline.cpp:179-188) into
 * oracle/_ref/. Never linked into the product library.
 *
 * FFTW3 is a third-party dependency that is absent from this image and from
 * /root/reference, and its version is unpinned (proj/CMakeLists.txt:13). Its
 * published contract for fftw_plan_dft_r2c_1d is the unnormalised forward DFT
 *     X[k] = sum_{j<n} x[j] * exp(-2*pi*i*j*k/n),   k = 0 .. n/2
 * which this file restates with two algorithms:
 *   - n a power of two: iterative radix-2 decimation-in-time complex FFT of
 *     (x, 0) after a bit-reversal permutation;
 *   - any other n: the direct O(n^2) DFT sum, j ascending.
 * Twiddles are W[k] = (cos(2*pi*k/n), -sin(2*pi*k/n)) from libm, evaluated with
 * the exact expression documented in include/uwbvital_b200.h, so that the GPU
 * front-end (paper_2012_11077_b200/csrc/frontend.cu) performs the identical
 * sequence of IEEE operations and reproduces this provider bit for bit.
 * Compile with -ffp-contract=off (no FMA contraction).
 *
 * Parity against FFTW itself is tolerance based and pinned by the reference's
 * own FFT tests (test_pipeline.cpp:202-252: on-bin cosine, zero input, direct
 * DFT + Parseval at 1e-9), which tests/test_oracle.py re-runs against this
 * provider.
 */
#include "fftw3.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

struct uwb_fftw_plan_s {
    int n;
    double* in;
    double (*out)[2];
    double* wr; /* twiddle real part, n entries */
    double* wi; /* twiddle imag part, n entries */
    double* re; /* scratch */
    double* im;
};

void uwb_fft_twiddles(size_t n, double* wr, double* wi) {
    for (size_t k = 0; k < n; ++k) {
        const double angle = (2.0 * M_PI * (double)k) / (double)n;
        wr[k] = cos(angle);
        wi[k] = -sin(angle);
    }
}

static int is_pow2(size_t n) { return n != 0 && (n & (n - 1)) == 0; }

/* In-place radix-2 DIT on (re, im), length n (power of two). */
void uwb_fft_pow2(double* re, double* im, size_t n, const double* wr, const double* wi) {
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            double t = re[i]; re[i] = re[j]; re[j] = t;
            t = im[i]; im[i] = im[j]; im[j] = t;
        }
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len >> 1;
        const size_t step = n / len;
        for (size_t base = 0; base < n; base += len) {
            for (size_t j = 0; j < half; ++j) {
                const double w_r = wr[j * step];
                const double w_i = wi[j * step];
                const size_t p = base + j;
                const size_t q = p + half;
                const double br = re[q], bi = im[q];
                const double tr = w_r * br - w_i * bi;
                const double ti = w_r * bi + w_i * br;
                const double ur = re[p], ui = im[p];
                re[p] = ur + tr;
                im[p] = ui + ti;
                re[q] = ur - tr;
                im[q] = ui - ti;
            }
        }
    }
}

/* Direct DFT of a real sequence x[0..n) for bins 0..n/2. */
void uwb_dft_real(const double* x, size_t n, const double* wr, const double* wi,
                  double* out_re, double* out_im) {
    for (size_t k = 0; k <= n / 2; ++k) {
        double acc_r = 0.0, acc_i = 0.0;
        for (size_t j = 0; j < n; ++j) {
            const size_t m = (j * k) % n;
            acc_r = acc_r + x[j] * wr[m];
            acc_i = acc_i + x[j] * wi[m];
        }
        out_re[k] = acc_r;
        out_im[k] = acc_i;
    }
}

/* r2c forward transform of x[0..n) into bins 0..n/2 (shared by the shim and
 * by oracle/uwb_oracle.c). */
void uwb_rfft(const double* x, size_t n, const double* wr, const double* wi, double* re,
              double* im, double* out_re, double* out_im) {
    if (is_pow2(n)) {
        for (size_t j = 0; j < n; ++j) { re[j] = x[j]; im[j] = 0.0; }
        uwb_fft_pow2(re, im, n, wr, wi);
        for (size_t k = 0; k <= n / 2; ++k) { out_re[k] = re[k]; out_im[k] = im[k]; }
    } else {
        uwb_dft_real(x, n, wr, wi, out_re, out_im);
    }
}

fftw_plan fftw_plan_dft_r2c_1d(int n, double* in, fftw_complex* out, unsigned flags) {
    (void)flags;
    if (n <= 0) return NULL;
    fftw_plan p = (fftw_plan)calloc(1, sizeof(*p));
    p->n = n;
    p->in = in;
    p->out = out;
    p->wr = (double*)malloc(sizeof(double) * (size_t)n);
    p->wi = (double*)malloc(sizeof(double) * (size_t)n);
    p->re = (double*)malloc(sizeof(double) * (size_t)n);
    p->im = (double*)malloc(sizeof(double) * (size_t)n);
    uwb_fft_twiddles((size_t)n, p->wr, p->wi);
    return p;
}

void fftw_execute(const fftw_plan p) {
    const size_t n = (size_t)p->n;
    const size_t bins = n / 2 + 1;
    double* ore = (double*)malloc(sizeof(double) * bins);
    double* oim = (double*)malloc(sizeof(double) * bins);
    uwb_rfft(p->in, n, p->wr, p->wi, p->re, p->im, ore, oim);
    for (size_t k = 0; k < bins; ++k) {
        p->out[k][0] = ore[k];
        p->out[k][1] = oim[k];
    }
    free(ore);
    free(oim);
}

void fftw_destroy_plan(fftw_plan p) {
    if (!p) return;
    free(p->wr);
    free(p->wi);
    free(p->re);
    free(p->im);
    free(p);
}
