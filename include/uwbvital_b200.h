/*
 * uwbvital_b200.h — the C ABI of the B200 (sm_100a) implementation of the
 * uwbvital north-star path: front-end preprocessing -> slow-time FFT /
 * band select -> summed-area table -> 2-D CA-CFAR.
 *
 * This is the drop-in boundary. The reference library exposes its path only
 * as C++ value-semantic functions (proj/include/uwbvital/{sat,cfar,pipeline}.hpp);
 * every host-level entry point below replaces exactly one of them and keeps its
 * argument meaning, its check order and its exception class (as a status code +
 * the reference's message text, fetched with uwb_last_error()). The C++ drop-in
 * (include/uwbvital/*.hpp, libuwbvital.so) and the Python mirror
 * (paper_2012_11077_b200) are thin layers over this header.
 *
 * Two families:
 *   uwb_*      host pointers in/out, synchronous, one call = one reference call;
 *   uwb_dev_*  device pointers, asynchronous on a caller stream, batched over
 *              maps; the throughput path used by bench.py and by multi-GPU runs.
 *
 * Numerics: every kernel computes in IEEE fp64 in the reference's operation
 * order (no FMA contraction), so the summed-area table, thresholds, masks and
 * detection lists are bit-identical to the reference CPU code on the same
 * inputs (UWB_SAT_GLOBAL). UWB_SAT_SLAB re-bases the table per row slab (SURVEY
 * 8e) and is bit-identical to the oracle run with the same slab decomposition.
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns UWB_CUDA_ERROR.
 */
#ifndef UWBVITAL_B200_H
#define UWBVITAL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UWB_B200_ABI_VERSION 2

/* Status codes; 1..5 correspond one-to-one to the reference exception classes
 * of proj/include/uwbvital/errors.hpp:13-41. */
typedef enum uwb_status {
    UWB_OK = 0,
    UWB_DIMENSION_ERROR = 1,     /* DimensionError */
    UWB_INPUT_ERROR = 2,         /* InputError */
    UWB_PARAMETER_ERROR = 3,     /* ParameterError */
    UWB_BOUNDS_ERROR = 4,        /* BoundsError */
    UWB_CONFIGURATION_ERROR = 5, /* ConfigurationError */
    UWB_CUDA_ERROR = 6,          /* no device / launch failure */
    UWB_CAPACITY_ERROR = 7,      /* detection buffer too small (count still reported) */
    UWB_INVALID_ARGUMENT = 8,    /* null pointer / bad layout */
    UWB_FORMAT_ERROR = 9         /* FormatError (frame files) */
} uwb_status;

typedef enum uwb_dtype { UWB_F32 = 0, UWB_F64 = 1 } uwb_dtype;

/* CFAR backends of cfar.hpp:77-84. */
typedef enum uwb_backend { UWB_NAIVE = 0, UWB_INTEGRAL = 1 } uwb_backend;

/* Table scope for the integral backend. */
typedef enum uwb_sat_mode {
    UWB_SAT_GLOBAL = 0, /* one (M+1)x(N+1) table per map: reference-exact */
    UWB_SAT_SLAB = 1,   /* row slabs, each with its own table over slab + halo */
    UWB_SAT_TILE = 2    /* row slabs (slab_rows, 0 = 1024) x column bands of 1024 owned
                           columns (UWB_TILE_COLS), each tile with its own table over the
                           tile + a 32-aligned halo >= g + b on each side: single large
                           maps run as a batch of short strip chains. Equal to GLOBAL
                           modulo the tie band; bit-identical to the reference run on
                           each tile's buffer (cols % 32 != 0: row slabs only) */
} uwb_sat_mode;

/* CfarParams (cfar.hpp:19-32) generalised to per-axis radii; the reference's
 * square window is guard_rows == guard_cols, background_rows == background_cols. */
typedef struct uwb_cfar_params {
    int32_t guard_rows;
    int32_t guard_cols;
    int32_t background_rows;
    int32_t background_cols;
    double pfa;
} uwb_cfar_params;

/* Detection (cfar.hpp:57-64); same field order and sizes as the reference on LP64. */
typedef struct uwb_detection {
    uint64_t row;
    uint64_t col;
    double value;
    double threshold;
} uwb_detection;

/* PipelineConfig (pipeline.hpp:18-30) with the CFAR radii per axis. */
typedef struct uwb_pipeline_config {
    uint64_t mean_filter_window;   /* odd */
    uint64_t fft_length;           /* 0 = next power of two >= traces */
    double band_low_hz;
    double band_high_hz;
    uwb_cfar_params cfar;
    int32_t backend;               /* uwb_backend */
    int32_t mean_filter_mode;      /* 0 Smoothing, 1 SubtractMean */
    double normalization_epsilon;
} uwb_pipeline_config;

/* ------------------------------------------------------------ errors --- */

/* Message of the last failing call on this host thread, in the reference's
 * wording (e.g. "build_sat: non-finite entry at (3, 4)"); "" after success. */
const char* uwb_last_error(void);
/* Offending cell of the last UWB_INPUT_ERROR (-1, -1 otherwise). */
void uwb_last_error_cell(int64_t* row, int64_t* col);
/* 1 if a CUDA device is usable by this library. */
int uwb_device_available(void);

/* ------------------------------------------- scalar reference helpers --- */

/* cfar.hpp:49 alpha_factor(n_train, pfa) = n (pfa^(-1/n) - 1); host libm. */
uwb_status uwb_alpha_factor(uint64_t n_train, double pfa, double* out);
/* CfarParams::validate (cfar.cpp:14-26), per axis. */
uwb_status uwb_cfar_params_validate(const uwb_cfar_params* params);
/* CfarParams::interior_train_count (cfar.cpp:28-32), per axis. */
uint64_t uwb_interior_train_count(const uwb_cfar_params* params);
/* cfar.hpp:54-55 training_window: out = {outer r0,r1,c0,c1, guard r0,r1,c0,c1, n_train}. */
uwb_status uwb_training_window(const uwb_cfar_params* params, uint64_t row, uint64_t col,
                               uint64_t rows, uint64_t cols, uint64_t out[9]);
/* alpha table alpha[n] for n = 0..interior_train_count (alpha[0] = 0), the
 * memoised AlphaTable of cfar.cpp:65-79 evaluated eagerly on the host. */
uwb_status uwb_alpha_table(const uwb_cfar_params* params, double* out, uint64_t len);

/* ----------------------------------------------- host-level drop-ins --- */

/* sat.hpp:52 build_sat: table is (rows+1) x (cols+1) row-major, zero row/col 0. */
uwb_status uwb_build_sat(const double* src, uint64_t rows, uint64_t cols, double* table);

/* cfar.hpp:77-84 cfar2d_naive / cfar2d_integral. mask: rows*cols bytes (0/1),
 * thresholds: rows*cols doubles (may be NULL), dets: capacity entries, sorted by
 * value desc, row asc, col asc; *n_det = total count (UWB_CAPACITY_ERROR if it
 * exceeds det_capacity; the buffer then holds the first det_capacity). */
uwb_status uwb_cfar2d(uwb_backend backend, const double* power_map, uint64_t rows, uint64_t cols,
                      const uwb_cfar_params* params, uint8_t* mask, double* thresholds,
                      uwb_detection* dets, uint64_t det_capacity, uint64_t* n_det);

/* pipeline.hpp:42-56 stages on an m x n frame (rows = fast time). */
uwb_status uwb_remove_dc(const double* in, uint64_t m, uint64_t n, double* out);
uwb_status uwb_detrend_linear(const double* in, uint64_t m, uint64_t n, double* out);
uwb_status uwb_mean_filter_slow(const double* in, uint64_t m, uint64_t n, uint64_t window,
                                double* out);
uwb_status uwb_subtract_slow_time_mean(const double* in, uint64_t m, uint64_t n, double* out);
uwb_status uwb_normalize_slow(const double* in, uint64_t m, uint64_t n, double epsilon,
                              double* out);
/* pipeline.hpp:62: power m x (fft_length/2+1); freq_axis fft_length/2+1; range_axis m. */
uwb_status uwb_slow_time_spectrum(const double* in, uint64_t m, uint64_t n, double fast_rate,
                                  double prf, uint64_t fft_length, double* power,
                                  double* freq_axis, double* range_axis);
/* pipeline.hpp:67-68: keeps bins with low <= f <= high; writes *first, *kept and
 * (if non-NULL) the selected m x kept power block and kept frequencies. */
uwb_status uwb_band_select(const double* power, uint64_t m, uint64_t bins, const double* freq_axis,
                           double band_low_hz, double band_high_hz, uint64_t* first,
                           uint64_t* kept, double* out_power, double* out_freq);
/* pipeline.hpp:79-80 detect. band_power: m * band_capacity doubles (row-major m x kept);
 * band_freq: band_capacity; range_axis: m; mask/thresholds: m * band_capacity.
 * *kept receives the band width. Stage errors carry the "<stage>: " prefix. */
uwb_status uwb_detect(const double* frame, uint64_t m, uint64_t n, double fast_rate, double prf,
                      const uwb_pipeline_config* config, uint64_t band_capacity,
                      double* band_power, double* band_freq, double* range_axis, uint64_t* kept,
                      uint8_t* mask, double* thresholds, uwb_detection* dets,
                      uint64_t det_capacity, uint64_t* n_det);

/* ------------------------------------------ device-level, batched path --- */

/* A batch of equally sized maps in device memory: map i, row r, col c at
 * element (maps + i*map_stride + r*ld + c). */
typedef struct uwb_map_batch {
    const void* maps;
    int32_t dtype;       /* uwb_dtype */
    int32_t reserved;
    uint64_t n_maps;
    uint64_t rows;
    uint64_t cols;
    uint64_t ld;         /* row pitch in elements (>= cols) */
    uint64_t map_stride; /* elements between maps (>= rows*ld) */
} uwb_map_batch;

/* Outputs of a batched CFAR call (device pointers; optional ones may be NULL). */
typedef struct uwb_cfar_outputs {
    uint32_t* mask_bits;       /* per map: rows * words_per_row words, bit c%32 of word c/32 */
    uint64_t words_per_row;    /* >= ceil(cols/32) */
    uint64_t mask_map_stride;  /* words between maps */
    uint8_t* mask_u8;          /* optional: per map rows*cols bytes, map stride rows*cols */
    double* thresholds;        /* optional: per map rows*cols doubles */
    uwb_detection* dets;       /* per map det_capacity entries, sorted as the reference */
    uint64_t det_capacity;
    uint64_t* det_counts;      /* per map total count (may exceed capacity) */
    uint64_t* first_bad;       /* per map 2 entries: first non-finite, first negative
                                  cell as row-major index, UINT64_MAX if none */
    /* Tie band of the north star (optional, certified path): cells whose CUT lies
     * within 1e-6 relative of T, |cut - T| <= 1e-6 T. tie_counts: per map count
     * (UINT64_MAX for a map the certified path handed to the exact path);
     * ties: per map tie_capacity records {row, col, cut, T} in no order. */
    uint64_t* tie_counts;
    uwb_detection* ties;
    uint64_t tie_capacity;
    /* optional, per map: 0 = decided by the certified path, bit 0 = candidate
     * list overflow, bit 1 = a value outside the certified range (both ran the
     * exact path instead; same results), UINT32_MAX = the call used the exact
     * path for every map. */
    uint32_t* cert_status;
} uwb_cfar_outputs;

/* Device workspace bytes needed by uwb_dev_cfar2d for this batch and mode.
 * slab_rows: rows owned per slab for UWB_SAT_SLAB (ignored for GLOBAL). */
uint64_t uwb_dev_cfar2d_workspace(const uwb_map_batch* batch, const uwb_cfar_params* params,
                                  int32_t sat_mode, uint64_t slab_rows, uint64_t det_capacity);

/* Integral-image CA-CFAR over every map of the batch (cfar.cpp:218-227 per map),
 * asynchronously on `stream` (a cudaStream_t; NULL = legacy default stream).
 * Parameters are validated on the host; input errors are reported per map in
 * outputs->first_bad (the call itself does not synchronise). alpha: device
 * array from uwb_alpha_table, length interior_train_count+1.
 * flags bit 0: skip the detection sort (list left in unspecified order).
 * flags bit 2: reuse the summed-area tables already in `workspace` from the
 *   previous call on the same maps with the same table geometry (GLOBAL mode, or
 *   SLAB mode with the same slab_rows and g_r + b_r), made without bit 4: one
 *   table, several CFAR parameter sets (the integral image's point). Non-finite
 *   inputs are reported only by the call that built the tables.
 * flags bit 4: fused SAT + CFAR for whole-map batches: one kernel whose table
 *   never leaves shared memory (same results, about a third of the HBM traffic;
 *   on an otherwise idle B200 the two-kernel default is measured slightly
 *   faster). No table is left in `workspace`.
 * flags bit 3: the naive backend instead (cfar.cpp:200-216: explicit ring sums,
 *   no table; GLOBAL mode only) - the baseline of the paper's Table I.
 * flags bit 6: force the exact two-kernel path (full table + cfar_ws_kernel).
 *   By default a call that wants masks and detection lists (no thresholds, no
 *   mask_u8, no bits 2/4) and whose window is one of the instantiated shapes
 *   (g+b, g) per axis in {(10,2), (5,1), (36,4), (19,3)} runs the certified-
 *   decision path (cfar_cert.cu): a quantised window-sum pass certifies almost
 *   every cell below T against an a-priori bound of the reference's table
 *   rounding, the SAT stores only the taps of the remaining candidates, and
 *   those are decided exactly. Results are identical to the exact path; a call
 *   that should leave its tables for a later bit-2 call must set bit 6.
 * flags bit 7 (test hook): the certified path's SAT writes whole tables.
 * flags bit 8 (test hook): the exact ring CFAR keeps 256-row chunks for small
 *   batches. Bits 7 and 8 change the schedule only, never the results.
 * flags bit 9: take the certified path also for a small batch (every table's
 *   strips resident at once, each table one thread-block cluster), which by
 *   default runs the exact path (latency-bound batches).
 * flags bit 10 (test hook): small batches build their tables with one CTA per
 *   table instead of one thread-block cluster per table (same results). */
uwb_status uwb_dev_cfar2d(const uwb_map_batch* batch, const uwb_cfar_params* params,
                          const double* alpha_dev, int32_t sat_mode, uint64_t slab_rows,
                          const uwb_cfar_outputs* out, void* workspace, uint64_t workspace_bytes,
                          uint32_t flags, void* stream);

/* Row window of larger maps (one rank's share of a map sharded by rows,
 * SURVEY 8e / BASELINE config 4): the batch buffer holds global rows
 * [buf_row0, buf_row0 + batch->rows) of maps that have global_rows rows, and
 * the call owns rows [row_begin, row_end). The buffer must hold the owned rows
 * plus g_r + b_r halo rows on each side (clipped to the map). Tables are
 * slab-local (UWB_SAT_SLAB semantics, slab_rows 0 = one slab for the window),
 * windows clamp with the global row count, detections carry global rows, and
 * mask rows / per-cell outputs are indexed by row - row_begin.
 * col_bands > 0 also cuts the columns into bands of col_bands owned columns
 * (rounded up to 128) with their own tables (UWB_SAT_TILE semantics); 0 = none. */
typedef struct uwb_row_window {
    uint64_t global_rows;
    uint64_t buf_row0;
    uint64_t row_begin;
    uint64_t row_end;
    uint64_t col_bands;
} uwb_row_window;

uint64_t uwb_dev_cfar2d_window_workspace(const uwb_map_batch* batch, const uwb_row_window* win,
                                         const uwb_cfar_params* params, uint64_t slab_rows,
                                         uint64_t det_capacity);
uwb_status uwb_dev_cfar2d_window(const uwb_map_batch* batch, const uwb_row_window* win,
                                 const uwb_cfar_params* params, const double* alpha_dev, uint64_t slab_rows,
                                 const uwb_cfar_outputs* out, void* workspace, uint64_t workspace_bytes,
                                 uint32_t flags, void* stream);

/* The global (M+1)x(N+1) tables of a batch in the device layout used by the
 * CFAR kernels: map i's padded element (i_r, j) at sat[i*sat_map_stride +
 * i_r*sat_ld + 31 + j] (the 31-element shift puts every 32-column group of a
 * row on two whole 128-byte lines). sat must be 256-byte aligned and sat_ld a
 * multiple of 32 with sat_ld >= cols + 32. Elements of a row past padded column
 * `cols` (the pitch padding) are unspecified. */
uwb_status uwb_dev_build_sat(const uwb_map_batch* batch, double* sat, uint64_t sat_ld,
                             uint64_t sat_map_stride, uint64_t* first_nonfinite,
                             void* workspace, uint64_t workspace_bytes, void* stream);
uint64_t uwb_dev_build_sat_workspace(const uwb_map_batch* batch);

/* Host-buffer batched CFAR for the end-to-end path: maps in (pinned) host
 * memory are streamed through the device in chunks with copy/compute overlap;
 * mask bits, detection lists and counts come back to host buffers. A map with
 * a non-finite or negative cell fails the call with UWB_INPUT_ERROR and the
 * message cfar2d_integral raises on that map (the first such map in batch
 * order; sat.cpp:28-32 before cfar.cpp:85-92). */
uwb_status uwb_host_cfar2d_batch(const uwb_map_batch* host_batch, const uwb_cfar_params* params,
                                 int32_t sat_mode, uint64_t slab_rows, uint32_t* mask_bits,
                                 uwb_detection* dets, uint64_t det_capacity,
                                 uint64_t* det_counts, uint64_t maps_per_chunk);

/* Batched detect() on the device (pipeline.cpp:246-275 per record; SURVEY 8f
 * rank 1): `records` holds n_records frames of m fast-time rows x n slow-time
 * columns (dtype f32/f64, dense). The front end writes each record's band power
 * (m x kept fp64, kept = *kept_out) straight into `band` (n_records maps, the
 * CFAR input), then the CFAR of the configuration runs over all band maps into
 * `out` (one map per record). Configuration and stage errors are returned with
 * the reference's messages before any work; per-record input errors go to
 * out->first_bad (entry 0: first non-finite frame sample, row-major). Query the
 * band width and workspace first (uwb_dev_detect_batch_workspace returns 0 for
 * a configuration error). `flags` as uwb_dev_cfar2d for the CFAR (bits 2 and 8
 * ignored there); bit 8 (test hook) runs the per-stage front-end kernels
 * instead of the fused two-kernel front end (same results). */
uint64_t uwb_dev_detect_batch_workspace(uint64_t n_records, uint64_t m, uint64_t n, double prf,
                                        const uwb_pipeline_config* cfg, uint64_t det_capacity);
uwb_status uwb_dev_detect_batch(const void* records, int32_t dtype, uint64_t n_records, uint64_t m, uint64_t n,
                                double fast_rate, double prf, const uwb_pipeline_config* cfg, double* band,
                                uint64_t* kept_out, const uwb_cfar_outputs* out, void* workspace,
                                uint64_t workspace_bytes, uint32_t flags, void* stream);

/* ---- RFRM frame files (frame_io.hpp:10-23) ----
 * uwb_rfrm_parse validates a whole file image exactly as read_frame does
 * (frame_io.cpp:69-122: magic, version, header, 2x2 minimum, payload length,
 * trailing bytes, RadarFrame rates; UWB_FORMAT_ERROR with the reference's
 * message) and locates its payload. uwb_dev_rfrm_to_frames transposes n_rec
 * payloads (each n_traces x m_samples f32, trace-major, packed back to back on
 * the device) into range-major frames [n_rec][m][n] of out_dtype, and writes
 * each record's first non-finite sample (row-major index, UINT64_MAX if none)
 * to first_nonfinite[i] ("frame file: RadarFrame: non-finite sample"). */
typedef struct uwb_rfrm_info {
    uint32_t m_samples;
    uint32_t n_traces;
    double fast_rate;
    double prf;
    uint64_t payload_offset; /* bytes from the file start */
    uint64_t payload_bytes;  /* m_samples * n_traces * 4 */
} uwb_rfrm_info;

uwb_status uwb_rfrm_parse(const void* file_bytes, uint64_t len, uwb_rfrm_info* info);
uwb_status uwb_dev_rfrm_to_frames(const float* payload, uint64_t n_rec, uint64_t m_samples, uint64_t n_traces,
                                  int32_t out_dtype, void* frames, uint64_t* first_nonfinite, void* stream);

/* Instrumentation. uwb_kernel_launches: number of kernels this library has
 * launched in the process. With flags bit 1 set, uwb_dev_cfar2d records CUDA
 * events around its phases (SAT, CFAR, sort) into a 1024-slot ring without
 * synchronising; uwb_dev_phase_ms synchronises on them, writes up to max_calls
 * triples {sat_ms, cfar_ms, sort_ms} and clears the ring. Returns the count. */
uint64_t uwb_kernel_launches(void);
int32_t uwb_dev_phase_ms(float* out, int32_t max_calls);
/* Same ring, four phases per call {certify (+ tap marking), SAT, CFAR (certified
 * resolve or the exact kernel), sort}; the exact path's certify phase is ~0. */
int32_t uwb_dev_phase_ms4(float* out, int32_t max_calls);

/* Pinned host allocation helpers (cudaHostAlloc / cudaFreeHost). */
void* uwb_host_alloc(uint64_t bytes);
void uwb_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* UWBVITAL_B200_H */
