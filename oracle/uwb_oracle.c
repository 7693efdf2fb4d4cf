/*
 * TEST INFRASTRUCTURE ONLY (oracle/). See uwb_oracle.h for scope and pinning.
 * Compiled with -ffp-contract=off so every sum/product below is one IEEE op in
 * the written order, exactly as the reference's x86-64 build evaluates it.
 */
#include "uwb_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* fft_provider.c */
void uwb_fft_twiddles(size_t n, double* wr, double* wi);
void uwb_rfft(const double* x, size_t n, const double* wr, const double* wi, double* re,
              double* im, double* out_re, double* out_im);

/* ------------------------------------------------------------------ SAT --- */

/* sat.cpp:10-37: (rows+1) x (cols+1) table, row 0 / col 0 zero, recurrence
 * out[c+1] = v + above[c+1] + out[c] - above[c] evaluated left to right. */
int uwbo_build_sat(const double* src, size_t rows, size_t cols, double* table, int64_t* bad_row,
                   int64_t* bad_col) {
    if (rows == 0 || cols == 0) return UWBO_DIMENSION;
    const size_t w = cols + 1;
    memset(table, 0, sizeof(double) * (rows + 1) * w);
    for (size_t r = 0; r < rows; ++r) {
        const double* s = src + r * cols;
        const double* above = table + r * w;
        double* out = table + (r + 1) * w;
        for (size_t c = 0; c < cols; ++c) {
            const double v = s[c];
            if (!isfinite(v)) {
                if (bad_row) *bad_row = (int64_t)r;
                if (bad_col) *bad_col = (int64_t)c;
                return UWBO_INPUT;
            }
            out[c + 1] = v + above[c + 1] + out[c] - above[c];
        }
    }
    return UWBO_OK;
}

/* sat.hpp:28-34: exactly four reads, (A + D) - (B + C). */
static double region_sum(const double* t, size_t w, size_t r0, size_t r1, size_t c0, size_t c1) {
    return t[r0 * w + c0] + t[(r1 + 1) * w + (c1 + 1)] - (t[r0 * w + (c1 + 1)] + t[(r1 + 1) * w + c0]);
}

/* ----------------------------------------------------------------- CFAR --- */

/* cfar.cpp:34-43 */
double uwbo_alpha(size_t n_train, double pfa) {
    const double n = (double)n_train;
    return n * (pow(pfa, -1.0 / n) - 1.0);
}

/* cfar.cpp:28-32, per axis */
size_t uwbo_interior_train_count(const uwbo_params* p) {
    const size_t orr = 2 * (size_t)(p->guard_rows + p->background_rows) + 1;
    const size_t oc = 2 * (size_t)(p->guard_cols + p->background_cols) + 1;
    const size_t gr = 2 * (size_t)p->guard_rows + 1;
    const size_t gc = 2 * (size_t)p->guard_cols + 1;
    return orr * oc - gr * gc;
}

/* cfar.cpp:47-55 */
static size_t clamp_low(size_t center, int radius) {
    const long long lo = (long long)center - radius;
    return lo < 0 ? 0 : (size_t)lo;
}
static size_t clamp_high(size_t center, int radius, size_t dim) {
    const size_t hi = center + (size_t)radius;
    return hi >= dim ? dim - 1 : hi;
}

typedef struct {
    size_t r0, r1, c0, c1;
} rect;
static size_t area(rect a) { return (a.r1 - a.r0 + 1) * (a.c1 - a.c0 + 1); }

static int cmp_det(const void* pa, const void* pb) {
    /* cfar.cpp:170-173: value descending, then row, col ascending */
    const uwbo_detection* a = (const uwbo_detection*)pa;
    const uwbo_detection* b = (const uwbo_detection*)pb;
    if (b->value < a->value) return -1;
    if (a->value < b->value) return 1;
    if (a->row != b->row) return a->row < b->row ? -1 : 1;
    if (a->col != b->col) return a->col < b->col ? -1 : 1;
    return 0;
}

int uwbo_cfar(const double* map, size_t rows, size_t cols, const uwbo_params* p, int backend,
              size_t row_begin, size_t row_end, int slab_local, uint8_t* mask, double* thr,
              uwbo_detection* dets, size_t det_cap, size_t* n_det, int64_t* bad_row,
              int64_t* bad_col) {
    *n_det = 0;
    const int hr = p->guard_rows + p->background_rows;
    const int hc = p->guard_cols + p->background_cols;
    double* table = NULL;
    size_t t_row0 = 0; /* global row of the table's first source row */
    size_t t_rows = rows;

    /* cfar2d_integral builds its table before run_cfar validates anything
     * (cfar.cpp:218-227), so empty / non-finite are reported first. */
    if (backend == 1) {
        if (rows == 0 || cols == 0) return UWBO_DIMENSION;
        if (slab_local) {
            t_row0 = row_begin > (size_t)hr ? row_begin - (size_t)hr : 0;
            size_t hi = row_end + (size_t)hr;
            if (hi > rows) hi = rows;
            t_rows = hi - t_row0;
        }
        /* finiteness is checked over the whole map in row-major order */
        for (size_t i = 0; i < rows * cols; ++i) {
            if (!isfinite(map[i])) {
                *bad_row = (int64_t)(i / cols);
                *bad_col = (int64_t)(i % cols);
                return UWBO_INPUT;
            }
        }
        table = (double*)malloc(sizeof(double) * (t_rows + 1) * (cols + 1));
        int64_t br, bc;
        uwbo_build_sat(map + t_row0 * cols, t_rows, cols, table, &br, &bc);
    }
    /* cfar.cpp:14-26 */
    if (p->guard_rows < 0 || p->guard_cols < 0 || p->background_rows < 1 ||
        p->background_cols < 1 || !(p->pfa > 0.0) || !(p->pfa < 1.0)) {
        free(table);
        return UWBO_PARAMETER;
    }
    /* cfar.cpp:81-94 */
    if (rows == 0 || cols == 0) {
        free(table);
        return UWBO_DIMENSION;
    }
    for (size_t i = 0; i < rows * cols; ++i) {
        if (!isfinite(map[i]) || map[i] < 0.0) {
            *bad_row = (int64_t)(i / cols);
            *bad_col = (int64_t)(i % cols);
            free(table);
            return UWBO_INPUT;
        }
    }
    /* cfar.cpp:99-107, per axis */
    if (rows <= 2 * (size_t)p->guard_rows + 1 && cols <= 2 * (size_t)p->guard_cols + 1) {
        free(table);
        return UWBO_CONFIGURATION;
    }

    /* cfar.cpp:65-79: alpha memoised per distinct n_train */
    const size_t n_int = uwbo_interior_train_count(p);
    double* alpha = (double*)malloc(sizeof(double) * (n_int + 1));
    for (size_t i = 0; i <= n_int; ++i) alpha[i] = -1.0;

    const size_t w = cols + 1;
    size_t found = 0;
    for (size_t r = row_begin; r < row_end; ++r) {
        for (size_t c = 0; c < cols; ++c) {
            /* cfar.cpp:115-127 */
            rect outer = {clamp_low(r, hr), clamp_high(r, hr, rows), clamp_low(c, hc),
                          clamp_high(c, hc, cols)};
            rect guard = {clamp_low(r, p->guard_rows), clamp_high(r, p->guard_rows, rows),
                          clamp_low(c, p->guard_cols), clamp_high(c, p->guard_cols, cols)};
            const size_t n_train = area(outer) - area(guard);
            double sum;
            if (backend == 1) {
                /* cfar.cpp:221-224 on the (possibly slab-local) table */
                sum = region_sum(table, w, outer.r0 - t_row0, outer.r1 - t_row0, outer.c0, outer.c1) -
                      region_sum(table, w, guard.r0 - t_row0, guard.r1 - t_row0, guard.c0, guard.c1);
            } else {
                /* cfar.cpp:201-214: ring loop, row-major accumulation */
                sum = 0.0;
                for (size_t rr = outer.r0; rr <= outer.r1; ++rr) {
                    const double* row = map + rr * cols;
                    const int guard_row = rr >= guard.r0 && rr <= guard.r1;
                    for (size_t cc = outer.c0; cc <= outer.c1; ++cc) {
                        if (guard_row && cc >= guard.c0 && cc <= guard.c1) continue;
                        sum += row[cc];
                    }
                }
            }
            const double mean = sum / (double)n_train;
            if (alpha[n_train] < 0.0) alpha[n_train] = uwbo_alpha(n_train, p->pfa);
            const double t = alpha[n_train] * mean;
            const double v = map[r * cols + c];
            if (thr) thr[r * cols + c] = t;
            const int hit = v > t; /* ties resolve to H0 */
            if (mask) mask[r * cols + c] = (uint8_t)hit;
            if (hit) ++found;
        }
    }
    free(table);

    /* cfar.cpp:163-173: collect in row-major order, then sort */
    uwbo_detection* all = (uwbo_detection*)malloc(sizeof(uwbo_detection) * (found ? found : 1));
    size_t k = 0;
    for (size_t r = row_begin; r < row_end && thr; ++r) {
        for (size_t c = 0; c < cols; ++c) {
            const double v = map[r * cols + c];
            const double t = thr[r * cols + c];
            if (v > t) {
                all[k].row = r;
                all[k].col = c;
                all[k].value = v;
                all[k].threshold = t;
                ++k;
            }
        }
    }
    qsort(all, k, sizeof(uwbo_detection), cmp_det);
    *n_det = k;
    if (dets) memcpy(dets, all, sizeof(uwbo_detection) * (k < det_cap ? k : det_cap));
    free(all);
    free(alpha);
    return UWBO_OK;
}

/* ------------------------------------------------------------ front-end --- */

/* pipeline.cpp:58-69 */
int uwbo_remove_dc(const double* in, size_t m, size_t n, double* out) {
    for (size_t c = 0; c < n; ++c) {
        double sum = 0.0;
        for (size_t r = 0; r < m; ++r) sum += in[r * n + c];
        const double mean = sum / (double)m;
        for (size_t r = 0; r < m; ++r) out[r * n + c] = in[r * n + c] - mean;
    }
    return UWBO_OK;
}

/* pipeline.cpp:71-98 */
int uwbo_detrend_linear(const double* in, size_t m, size_t n, double* out) {
    const double dm = (double)m;
    const double sum_r = dm * (dm - 1.0) / 2.0;
    const double sum_rr = (dm - 1.0) * dm * (2.0 * dm - 1.0) / 6.0;
    const double det = dm * sum_rr - sum_r * sum_r;
    for (size_t c = 0; c < n; ++c) {
        double sum_x = 0.0, sum_rx = 0.0;
        for (size_t r = 0; r < m; ++r) {
            const double v = in[r * n + c];
            sum_x += v;
            sum_rx += (double)r * v;
        }
        const double slope = (dm * sum_rx - sum_r * sum_x) / det;
        const double intercept = (sum_x - slope * sum_r) / dm;
        for (size_t r = 0; r < m; ++r)
            out[r * n + c] = in[r * n + c] - (intercept + slope * (double)r);
    }
    return UWBO_OK;
}

/* pipeline.cpp:100-122 */
int uwbo_mean_filter_slow(const double* in, size_t m, size_t n, size_t window, double* out) {
    if (window == 0 || window % 2 == 0 || window > n) return UWBO_PARAMETER;
    if (window == 1) {
        memcpy(out, in, sizeof(double) * m * n);
        return UWBO_OK;
    }
    const size_t half = window / 2;
    for (size_t r = 0; r < m; ++r) {
        const double* x = in + r * n;
        double* y = out + r * n;
        for (size_t c = 0; c < n; ++c) {
            size_t h = half;
            if (c < h) h = c;
            if (n - 1 - c < h) h = n - 1 - c;
            double sum = 0.0;
            for (size_t k = c - h; k <= c + h; ++k) sum += x[k];
            y[c] = sum / (double)(2 * h + 1);
        }
    }
    return UWBO_OK;
}

/* pipeline.cpp:124-137 */
int uwbo_subtract_slow_time_mean(const double* in, size_t m, size_t n, double* out) {
    for (size_t r = 0; r < m; ++r) {
        double sum = 0.0;
        for (size_t c = 0; c < n; ++c) sum += in[r * n + c];
        const double mean = sum / (double)n;
        for (size_t c = 0; c < n; ++c) out[r * n + c] = in[r * n + c] - mean;
    }
    return UWBO_OK;
}

/* pipeline.cpp:139-155 */
int uwbo_normalize_slow(const double* in, size_t m, size_t n, double epsilon, double* out) {
    if (!(epsilon > 0.0)) return UWBO_PARAMETER;
    for (size_t r = 0; r < m; ++r) {
        double peak = 0.0;
        for (size_t c = 0; c < n; ++c) {
            const double a = fabs(in[r * n + c]);
            peak = peak < a ? a : peak; /* std::max(peak, |x|) */
        }
        const double scale = peak < epsilon ? epsilon : peak; /* std::max(peak, eps) */
        for (size_t c = 0; c < n; ++c) out[r * n + c] = in[r * n + c] / scale;
    }
    return UWBO_OK;
}

/* pipeline.cpp:157-190 with the FFTW r2c call restated by fft_provider.c */
int uwbo_slow_time_spectrum(const double* in, size_t m, size_t n, size_t fft_length, double* power) {
    if (fft_length < n) return UWBO_PARAMETER;
    const size_t L = fft_length, bins = L / 2 + 1;
    double* wr = (double*)malloc(sizeof(double) * L);
    double* wi = (double*)malloc(sizeof(double) * L);
    double* x = (double*)malloc(sizeof(double) * L);
    double* re = (double*)malloc(sizeof(double) * L);
    double* im = (double*)malloc(sizeof(double) * L);
    double* ore = (double*)malloc(sizeof(double) * bins);
    double* oim = (double*)malloc(sizeof(double) * bins);
    uwb_fft_twiddles(L, wr, wi);
    for (size_t r = 0; r < m; ++r) {
        for (size_t j = 0; j < L; ++j) x[j] = j < n ? in[r * n + j] : 0.0;
        uwb_rfft(x, L, wr, wi, re, im, ore, oim);
        for (size_t k = 0; k < bins; ++k) power[r * bins + k] = ore[k] * ore[k] + oim[k] * oim[k];
    }
    free(wr); free(wi); free(x); free(re); free(im); free(ore); free(oim);
    return UWBO_OK;
}

/* pipeline.cpp:192-213 with freq_axis[k] = k * prf / L (pipeline.cpp:169-172) */
int uwbo_band_range(size_t fft_length, double prf, double low, double high, size_t* first,
                    size_t* kept) {
    const size_t bins = fft_length / 2 + 1;
    size_t f = bins, l = 0;
    for (size_t k = 0; k < bins; ++k) {
        const double freq = (double)k * prf / (double)fft_length;
        if (freq >= low && freq <= high) {
            if (f == bins) f = k;
            l = k;
        }
    }
    if (f == bins) return UWBO_CONFIGURATION;
    *first = f;
    *kept = l - f + 1;
    return UWBO_OK;
}
