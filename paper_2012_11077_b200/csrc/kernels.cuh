// Launch descriptors shared between the kernels and the host-side C ABI.
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "uwbvital_b200.h"

namespace uwb {

// Kernels launched by this library (uwb_kernel_launches()).
extern std::atomic<uint64_t> g_kernel_launches;

// Device table layout ("shifted pitched"): padded element (i, j) of the
// (M+1) x (N+1) summed-area table lives at table[i * ld + kTabShift + j], with
// ld a multiple of 32 doubles. S(r, c) = padded (r+1, c+1) then sits at index
// (r+1)*ld + 32 + c, so the 32 values a warp writes for columns 32k..32k+31
// fill two whole, 256-byte aligned L2 lines (no partial-line write-back).
constexpr int kTabShift = 31;
constexpr int kTabAlign = 32;
__host__ __device__ constexpr int64_t table_ld_for(int64_t cols) {
    return (cols + kTabShift + 1 + kTabAlign - 1) / kTabAlign * kTabAlign;
}

// A batch is split into jobs: job = (map, slab). GLOBAL mode has one slab per
// map covering all rows; SLAB mode owns rows [s*slab_rows, (s+1)*slab_rows) and
// builds its table over the owned rows plus `halo` rows on each side (clipped).
//
// A call may also cover only a row window of larger maps (one rank's share of a
// map sharded by rows): the buffer then holds global rows
// [buf_row0, buf_row0 + buf_rows), the call owns rows [row_lo, row_hi), windows
// clamp with the global row count `rows`, and outputs are indexed by row - row_lo.
struct JobGeometry {
    int64_t rows;       // global map rows (clamp bounds)
    int64_t slab_rows;  // owned rows per slab (== owned rows in GLOBAL mode)
    int64_t n_slabs;
    int64_t halo;       // g_r + b_r in SLAB mode, 0 in GLOBAL mode
    int64_t row_lo;     // first owned row of the call
    int64_t row_hi;     // end of the owned rows
    int64_t buf_row0;   // global row of the input buffer's row 0
    int64_t buf_rows;   // rows present in the input buffer
    // Column bands (UWB_SAT_TILE): band k owns columns [k*band_cols, (k+1)*band_cols)
    // and its table covers band_width source columns from band_c0(k) (the owned
    // columns plus a 32-aligned halo >= g_c + b_c on each side, moved inward at
    // the map edges, so every band table has the same width). Band tables are
    // separate pitched tables (ld = band_seg), band k of CFAR job j at table
    // index j * n_bands + k. n_bands == 1: no bands (band_width = map_cols).
    int64_t map_cols;   // global map columns (clamp bounds)
    int64_t n_bands;
    int64_t band_cols;
    int64_t band_width;
    int64_t band_seg;

    __host__ __device__ int64_t owned_begin(int64_t s) const { return row_lo + s * slab_rows; }
    __host__ __device__ int64_t owned_end(int64_t s) const {
        const int64_t e = row_lo + (s + 1) * slab_rows;
        return e < row_hi ? e : row_hi;
    }
    __host__ __device__ int64_t out_rows() const { return row_hi - row_lo; }
    __host__ __device__ int64_t table_begin(int64_t s) const {
        const int64_t b = owned_begin(s) - halo;
        return b > 0 ? b : 0;
    }
    __host__ __device__ int64_t table_end(int64_t s) const {
        const int64_t e = owned_end(s) + halo;
        return e < rows ? e : rows;
    }
    __host__ __device__ int64_t band_c0(int64_t k) const {
        if (n_bands <= 1) return 0;
        int64_t c = k * band_cols - (band_width - band_cols) / 2;
        c = c > 0 ? c : 0;
        return c < map_cols - band_width ? c : map_cols - band_width;
    }
    __host__ __device__ int64_t band_of(int64_t c) const { return n_bands > 1 ? c / band_cols : 0; }
    // rows of the largest table (source rows, excluding the zero row)
    __host__ __device__ int64_t max_table_rows() const {
        const int64_t r = slab_rows + 2 * halo;
        return r < rows ? r : rows;
    }
};

struct SatLaunch {
    const void* maps;
    int64_t ld;          // source row pitch (elements)
    int64_t map_stride;  // elements between maps
    int64_t cols;
    JobGeometry geo;
    int64_t n_jobs;      // n_maps * n_slabs * n_bands
    double* table;       // padded tables, shifted layout
    int64_t table_ld;
    int64_t table_stride; // doubles between job tables
    int64_t strips;
    double* gedge;       // strips > 1: (n_jobs * strips) edge columns
    int64_t edge_stride;
    unsigned* gprog;     // (n_jobs * strips) row counters, zeroed before launch
    unsigned* tile_counter;
    unsigned long long* first_bad; // per map 2 slots; slot 0 = first non-finite
    bool vec_ok;         // 16-byte vector loads legal
    int elem_bytes;
    unsigned flags;      // bit 1: low-latency strip chain (set by the launcher)
    int cpl;             // columns per lane (strips of 32 * cpl columns): 1, 2 or 4
    // Sparse mode (certified CFAR, cfar_cert.cu): when `need` is set, only the
    // 32-byte segments of S(r, .) marked in need[(job * strips + strip) *
    // need_rows + r] (bit = lane) are stored; maps with map_full[map] != 0
    // store every segment. Padded row / column 0 are not stored.
    const unsigned* need;
    int64_t need_rows;
    const unsigned* map_full;
    int64_t jobs_per_map; // SAT jobs per map (n_slabs * n_bands)
    int l2_ahead;         // sparse mode: L2 prefetch distance in rows (set by the launcher)
};

struct SatJobView {
    const void* src;
    int64_t rows;
    int64_t row0;        // map row of table source row 0
    int64_t col0;        // map column of table source column 0 (column bands)
    double* table;
    unsigned long long* nonfinite;
};

__host__ __device__ inline SatJobView sat_job(const SatLaunch& L, int64_t job) {
    // SAT jobs are (map, slab, band); the CFAR's jobs are (map, slab)
    const int64_t k = job % L.geo.n_bands;
    const int64_t ms = job / L.geo.n_bands;
    const int64_t m = ms / L.geo.n_slabs;
    const int64_t s = ms % L.geo.n_slabs;
    const int64_t b = L.geo.table_begin(s);
    const int64_t c0 = L.geo.band_c0(k);
    SatJobView v;
    v.src = static_cast<const char*>(L.maps) + (m * L.map_stride + (b - L.geo.buf_row0) * L.ld + c0) * L.elem_bytes;
    v.rows = L.geo.table_end(s) - b;
    v.row0 = b;
    v.col0 = c0;
    v.table = L.table + job * L.table_stride;
    v.nonfinite = L.first_bad ? L.first_bad + 2 * m : nullptr;
    return v;
}

struct CfarLaunch {
    const void* maps;
    int64_t ld;
    int64_t map_stride;
    int64_t cols;
    JobGeometry geo;
    int64_t n_jobs;
    const double* table;
    int64_t table_ld;
    int64_t table_stride;
    int gr, gc, hr, hc;  // guard radii and outer half-widths (g + b) per axis
    const double* alpha; // alpha[n], n = 0..n_int
    // outputs
    uint32_t* mask_bits;
    int64_t words_per_row;
    int64_t mask_map_stride;
    uint8_t* mask_u8;
    double* thresholds;
    uwb_detection* dets;
    int64_t det_cap;
    unsigned long long* det_counts;
    unsigned long long* first_bad;
    int64_t row_chunks;  // row chunks per job
    int64_t ring_rows;   // CFAR ring kernel: output rows per CTA (row chunk height)
    unsigned sleep_ns;   // barrier-wait suspend hint of the CFAR ring kernel (ns)
    unsigned debug;      // bit 0: consumers skip the cell arithmetic (data-movement probe; tuning build only)
    bool fixed_rows;     // CFAR ring: keep 256-row chunks for small batches (test hook, same results)
    int ring_ahead;      // CFAR ring: table groups of look-ahead beyond the window
    int pf_groups;       // CFAR ring: L2 prefetch distance of both streams (groups)
    int64_t col_tiles;
    // launch_cfar_integral_filtered: the flagged maps, compacted on the device
    const unsigned* flagged_maps;
    const unsigned* flagged_count;
};

// Certified-decision CFAR (cfar_cert.cu): one launch description shared by the
// certify, mark and resolve kernels.
struct CertLaunch {
    const void* maps;
    int elem_bytes;
    int64_t ld, map_stride, cols;
    JobGeometry geo;     // the CFAR call's geometry (slabs / bands of the tables)
    int64_t n_maps;
    int gr, gc, hr, hc;
    const double* alpha;
    int n_int;           // interior training count
    // quantisation q = round(x * 2^s) and the a-priori bound of the reference's rounding
    int s_bits;
    double scale, inv_scale_d, xlim, s_bound;
    float inv_scale, magic;
    uint32_t bits_magic, xlim_bits, ring_off;
    const float4* ke;    // per n: {K_n, K_n 2^-(s+1), E_n}
    // candidates
    int2* cand;          // per map cand_cap (row, col), global rows
    unsigned* cand_count;
    int64_t cand_cap;
    unsigned* status;    // per map: bit 0 list overflow, bit 1 value outside the certified range
    unsigned* flagged;   // the maps with status != 0, compacted by cert_resolve_kernel
    unsigned* flagged_count;
    unsigned long long* first_bad;
    int64_t col_ctas, row_chunk, row_chunks;
    int l2_ahead_t;      // L2 prefetch distance of the certify pass (tile-rows; set by the launcher)
    // sparse-table taps
    unsigned* need;
    int64_t need_rows, strips;
    int cpl;
    const double* table;
    int64_t table_ld, table_stride;
    // outputs
    uint32_t* mask_bits;
    int64_t words_per_row, mask_map_stride;
    uwb_detection* dets;
    int64_t det_cap;
    unsigned long long* det_counts;
    unsigned long long* tie_counts;
    uwb_detection* ties;
    int64_t tie_cap;
};

cudaError_t launch_sat(const SatLaunch& L, int dtype, cudaStream_t stream);
int64_t sat_strips(int64_t cols, int cpl);       // strips of 32 * cpl columns
int sat_cpl_for(int64_t n_jobs, int64_t cols);   // columns per lane for a batch
// small batches whose tables each fit one CTA (sat_cta_kernel: strips hand over in shared memory)
bool sat_cta_eligible(int64_t n_jobs, int64_t cols, int dtype);
// small batches whose tables each run as one thread-block cluster (sat_cluster.cu: strips hand
// over through distributed shared memory); _fits: by shape, _eligible: shape and alignment
bool sat_cluster_fits(int64_t n_jobs, int64_t cols, int64_t max_rows, int dtype, bool allow_chain = false);
bool sat_cluster_eligible(const SatLaunch& L, int dtype);
cudaError_t launch_sat_cluster(const SatLaunch& L, int dtype, cudaStream_t stream);

cudaError_t launch_cfar_integral(const CfarLaunch& L, int dtype, cudaStream_t stream);
// the same over the flagged maps L.flagged_maps[0 .. *L.flagged_count) only (certified path's exact fallback)
cudaError_t launch_cfar_integral_filtered(const CfarLaunch& L, int dtype, cudaStream_t stream);
// SAT + CFAR in one kernel, table kept on chip (cfar_fused.cu). Whole-map
// batches only; cudaErrorNotSupported when the geometry does not qualify.
cudaError_t launch_cfar_fused(const SatLaunch& S, const CfarLaunch& C, int dtype, cudaStream_t stream);
cudaError_t launch_cfar_naive(const CfarLaunch& L, int dtype, cudaStream_t stream);
// certified-decision CFAR (cfar_cert.cu)
bool cert_supported(int hr, int gr, int hc, int gc);
void cert_prepare(CertLaunch& L, int range_log2);
cudaError_t launch_cert_table(const CertLaunch& L, float4* ke, int n_max, cudaStream_t stream);
cudaError_t launch_cert(const CertLaunch& L, int dtype, cudaStream_t stream);
cudaError_t launch_cert_mark(const CertLaunch& L, cudaStream_t stream);
cudaError_t launch_cert_resolve(const CertLaunch& L, int dtype, cudaStream_t stream);
// Sort each map's detection list: value desc, row asc, col asc (cfar.cpp:170-173).
cudaError_t launch_sort_detections(uwb_detection* dets, int64_t cap,
                                   const unsigned long long* counts, int64_t n_maps,
                                   uwb_detection* scratch, cudaStream_t stream);

// Front-end (pipeline.cpp:58-223)
struct FrontendLaunch {
    const void* frame;   // m x n, row pitch n
    int dtype;
    int64_t m, n;
    double* work;        // m x n doubles (detrended frame)
    unsigned long long* first_nonfinite;
    uint64_t window;     // mean filter window (odd); 1 = identity
    int mode;            // 0 smoothing, 1 subtract mean
    double epsilon;
    int64_t L;           // fft length
    const double* wr;    // twiddles, L entries
    const double* wi;
    int64_t first_bin, kept;
    double* band;        // m x kept
    double* full_power;  // optional m x (L/2+1) (slow_time_spectrum)
    int stage_mask;      // which stages to run (see frontend.cu)
    int64_t n_rec;       // records in the batch (0 = 1); record i's frame, work,
                         // band and spectrum follow record i-1's densely, and its
                         // non-finite report goes to first_nonfinite[i]
};
cudaError_t launch_frontend_columns(const FrontendLaunch& F, cudaStream_t stream);
// RFRM payloads (trace-major f32) -> range-major frames (ingest.cu)
cudaError_t launch_rfrm_transpose(const float* payload, int64_t n_rec, int64_t m, int64_t n, int out_dtype,
                                  void* frames, unsigned long long* first_bad, cudaStream_t stream);
cudaError_t launch_frontend_rows(const FrontendLaunch& F, cudaStream_t stream);
// stats + fft1024 kernels for the whole front end (detect paths); cudaErrorNotSupported
// when the configuration needs launch_frontend_columns + launch_frontend_rows
cudaError_t launch_frontend_fused(const FrontendLaunch& F, cudaStream_t stream);

} // namespace uwb
