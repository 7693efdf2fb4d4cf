/*
 * TEST INFRASTRUCTURE ONLY (oracle/). CPU restatement, in plain C, of the
 * reference algorithms on the north-star path.
 * Each function cites the reference file:line it restates. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker. The product (paper_2012_11077_b200) never links it.
 *
 * Pinning: tests/test_oracle.py checks this restatement bit for bit against
 * the reference itself compiled from /root/reference (oracle/_ref/libuwbref.so)
 * and against the reference tests' known-answer values and the golden
 * fixtures in tests/golden/.
 *
 * Generalisation beyond the reference API (needed for BASELINE config 5):
 * per-axis guard/background radii (gr, gc, br, bc). With gr == gc and
 * br == bc every output is bit-identical to uwbvital::cfar2d_{naive,integral}.
 */
#ifndef UWB_ORACLE_H
#define UWB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    UWBO_OK = 0,
    UWBO_DIMENSION = 1,
    UWBO_INPUT = 2,
    UWBO_PARAMETER = 3,
    UWBO_BOUNDS = 4,
    UWBO_CONFIGURATION = 5,
};

typedef struct {
    int guard_rows;      /* g_r */
    int guard_cols;      /* g_c */
    int background_rows; /* b_r */
    int background_cols; /* b_c */
    double pfa;
} uwbo_params;

typedef struct {
    uint64_t row, col;
    double value, threshold;
} uwbo_detection;

/* sat.cpp:10-37 */
int uwbo_build_sat(const double* src, size_t rows, size_t cols, double* table, int64_t* bad_row,
                   int64_t* bad_col);
/* cfar.cpp:34-43 (no validation; callers validate) */
double uwbo_alpha(size_t n_train, double pfa);
/* cfar.cpp:28-32 generalised per axis */
size_t uwbo_interior_train_count(const uwbo_params* p);

/*
 * cfar.cpp:109-175 + 200-227. backend 0 = naive (explicit ring loops),
 * 1 = integral image. Cells of rows [row_begin, row_end) are evaluated; with
 * slab_local != 0 the integral backend builds its table only over rows
 * [row_begin - (g_r+b_r), row_end + (g_r+b_r)) clipped to the map (the row-slab
 * decomposition of SURVEY 8e); windows are always clamped to the global map.
 * mask (u8) and thr are full rows x cols arrays; only the evaluated rows are
 * written. Detections of the evaluated rows are written sorted
 * (value desc, row asc, col asc) up to det_cap; *n_det gets the total.
 * Returns a UWBO_* code; *bad_row/*bad_col name the offending cell for INPUT.
 */
int uwbo_cfar(const double* map, size_t rows, size_t cols, const uwbo_params* p, int backend,
              size_t row_begin, size_t row_end, int slab_local, uint8_t* mask, double* thr,
              uwbo_detection* dets, size_t det_cap, size_t* n_det, int64_t* bad_row,
              int64_t* bad_col);

/* pipeline.cpp:58-155; all return UWBO_* codes */
int uwbo_remove_dc(const double* in, size_t m, size_t n, double* out);
int uwbo_detrend_linear(const double* in, size_t m, size_t n, double* out);
int uwbo_mean_filter_slow(const double* in, size_t m, size_t n, size_t window, double* out);
int uwbo_subtract_slow_time_mean(const double* in, size_t m, size_t n, double* out);
int uwbo_normalize_slow(const double* in, size_t m, size_t n, double epsilon, double* out);
/* pipeline.cpp:157-190: power is m x (L/2+1) */
int uwbo_slow_time_spectrum(const double* in, size_t m, size_t n, size_t fft_length, double* power);
/* pipeline.cpp:192-223: returns first bin via *first and count via *kept */
int uwbo_band_range(size_t fft_length, double prf, double low, double high, size_t* first,
                    size_t* kept);

#ifdef __cplusplus
}
#endif

#endif
