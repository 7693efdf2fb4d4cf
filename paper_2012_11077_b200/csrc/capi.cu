// Host side of the C ABI (include/uwbvital_b200.h).
//
// Every host-level entry point restates the reference function's validation
// order and message text (proj/src/{sat,cfar,pipeline}.cpp) and runs the
// arithmetic on the GPU; there is no host compute fallback. Scalar helpers
// that the reference evaluates on the host with libm (alpha_factor, the FFT
// twiddles the oracle's FFTW provider uses, the window clamps) stay on the host
// so their bits match.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "kernels.cuh"

namespace uwb {

size_t frontend_rows_smem(int64_t n, int64_t L);

namespace {

struct ErrorState {
    std::string message;
    int64_t row = -1;
    int64_t col = -1;
};
thread_local ErrorState g_err;

std::string fmt_double(double v) { // std::to_string(double) == "%f"
    char buf[64];
    std::snprintf(buf, sizeof buf, "%f", v);
    return buf;
}
std::string S(uint64_t v) { return std::to_string(v); }
std::string S(int64_t v) { return std::to_string(v); }
std::string S(int v) { return std::to_string(v); }

uwb_status ok() {
    g_err.message.clear();
    g_err.row = g_err.col = -1;
    return UWB_OK;
}

uwb_status fail(uwb_status s, const std::string& msg, int64_t row = -1, int64_t col = -1) {
    g_err.message = msg;
    g_err.row = row;
    g_err.col = col;
    return s;
}

// Per host thread non-blocking stream for the synchronous host-level calls.
cudaStream_t host_stream() {
    thread_local cudaStream_t s = nullptr;
    if (!s) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    return s;
}

// Stream-ordered device buffer.
struct DevBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
    cudaError_t alloc(size_t bytes, cudaStream_t stream) {
        s = stream;
        return cudaMallocAsync(&p, bytes ? bytes : 16, stream);
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

bool device_ok() {
    int n = 0;
    return cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
}

uwb_status need_device() {
    if (!device_ok()) return fail(UWB_CUDA_ERROR, "uwbvital_b200: no CUDA device available (no CPU fallback)");
    // stream-ordered scratch is returned to the device's default pool, not to the
    // driver, so repeated calls do not re-map their workspaces
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
    return UWB_OK;
}

int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// --- scalar reference logic (cfar.cpp) ---------------------------------------

uwb_status validate_params(const uwb_cfar_params& p) {
    // cfar.cpp:14-26 (per axis: rows first, then cols)
    if (p.guard_rows < 0) return fail(UWB_PARAMETER_ERROR, "CfarParams: guard_radius must be >= 0, got " + S(p.guard_rows));
    if (p.guard_cols < 0) return fail(UWB_PARAMETER_ERROR, "CfarParams: guard_radius must be >= 0, got " + S(p.guard_cols));
    if (p.background_rows < 1) return fail(UWB_PARAMETER_ERROR, "CfarParams: background_radius must be >= 1, got " + S(p.background_rows));
    if (p.background_cols < 1) return fail(UWB_PARAMETER_ERROR, "CfarParams: background_radius must be >= 1, got " + S(p.background_cols));
    if (!(p.pfa > 0.0) || !(p.pfa < 1.0)) return fail(UWB_PARAMETER_ERROR, "CfarParams: pfa must lie in (0,1), got " + fmt_double(p.pfa));
    return ok();
}

uint64_t interior_count(const uwb_cfar_params& p) {
    const uint64_t orr = 2 * static_cast<uint64_t>(p.guard_rows + p.background_rows) + 1;
    const uint64_t oc = 2 * static_cast<uint64_t>(p.guard_cols + p.background_cols) + 1;
    const uint64_t gr = 2 * static_cast<uint64_t>(p.guard_rows) + 1;
    const uint64_t gc = 2 * static_cast<uint64_t>(p.guard_cols) + 1;
    return orr * oc - gr * gc;
}

double alpha_value(uint64_t n_train, double pfa) { // cfar.cpp:41-42
    const double n = static_cast<double>(n_train);
    return n * (std::pow(pfa, -1.0 / n) - 1.0);
}

std::vector<double> alpha_table_host(const uwb_cfar_params& p) {
    const uint64_t n_int = interior_count(p);
    std::vector<double> a(n_int + 1, 0.0);
    for (uint64_t n = 1; n <= n_int; ++n) a[n] = alpha_value(n, p.pfa);
    return a;
}

bool degenerate(const uwb_cfar_params& p, uint64_t rows, uint64_t cols) { // cfar.cpp:99-107
    return rows <= 2 * static_cast<uint64_t>(p.guard_rows) + 1 &&
           cols <= 2 * static_cast<uint64_t>(p.guard_cols) + 1;
}

std::string degenerate_msg(const uwb_cfar_params& p, uint64_t rows, uint64_t cols) {
    const uint64_t sr = 2 * static_cast<uint64_t>(p.guard_rows) + 1;
    const uint64_t sc = 2 * static_cast<uint64_t>(p.guard_cols) + 1;
    return "cfar2d: " + S(rows) + "x" + S(cols) + " map fits inside the " + S(sr) + "x" + S(sc) +
           " guard window; no training cells remain";
}

// --- batch plumbing -----------------------------------------------------------

struct Plan {
    JobGeometry geo;
    int64_t n_maps, cols, n_jobs, table_ld, table_stride, strips, max_rows, edge_stride;
    int64_t sat_jobs, sat_cols; // SAT jobs (map, slab, band) and table source columns per job
    int cpl;
    size_t off_tables, off_edge, off_prog, off_counter, off_scratch;
    // certified-decision CFAR (cfar_cert.cu): candidate lists, status, tap bitmap, K/E table
    int64_t cand_cap, need_rows, n_int;
    size_t off_cand, off_cand_count, off_status, off_need, off_ke, off_flagged, total;
};

// win == nullptr: the batch holds whole maps. Otherwise the batch buffer holds
// rows [win->buf_row0, +b.rows) of maps with win->global_rows rows and the call
// owns rows [win->row_begin, win->row_end) (always slab-local tables with halo).
Plan make_plan(const uwb_map_batch& b, const uwb_cfar_params* p, int sat_mode, uint64_t slab_rows,
               int64_t det_cap, const uwb_row_window* win = nullptr) {
    Plan P{};
    P.n_maps = static_cast<int64_t>(b.n_maps);
    P.cols = static_cast<int64_t>(b.cols);
    P.geo.rows = static_cast<int64_t>(win ? win->global_rows : b.rows);
    P.geo.row_lo = static_cast<int64_t>(win ? win->row_begin : 0);
    P.geo.row_hi = static_cast<int64_t>(win ? win->row_end : b.rows);
    P.geo.buf_row0 = static_cast<int64_t>(win ? win->buf_row0 : 0);
    P.geo.buf_rows = static_cast<int64_t>(b.rows);
    const int64_t owned = P.geo.row_hi - P.geo.row_lo;
    if (sat_mode == UWB_SAT_TILE && !win && slab_rows == 0) slab_rows = 1024;
    if (win || ((sat_mode == UWB_SAT_SLAB || sat_mode == UWB_SAT_TILE) && slab_rows > 0 &&
                static_cast<int64_t>(slab_rows) < owned)) {
        P.geo.slab_rows = slab_rows > 0 && static_cast<int64_t>(slab_rows) < owned ? static_cast<int64_t>(slab_rows)
                                                                                  : (owned > 0 ? owned : 1);
        P.geo.halo = p ? p->guard_rows + p->background_rows : 0;
    } else {
        P.geo.slab_rows = owned > 0 ? owned : 1;
        P.geo.halo = 0;
    }
    P.geo.n_slabs = owned > 0 ? (owned + P.geo.slab_rows - 1) / P.geo.slab_rows : 0;
    P.n_jobs = P.n_maps * P.geo.n_slabs;
    P.max_rows = P.geo.max_table_rows();
    // column bands (UWB_SAT_TILE): band tables of band_cols owned columns plus a
    // 32-aligned halo >= g_c + b_c per side; only when the bands are narrower
    // than the map and the map width keeps every band start 32-aligned
    P.geo.map_cols = P.cols;
    P.geo.n_bands = 1;
    P.geo.band_cols = P.cols;
    P.geo.band_width = P.cols;
    P.sat_cols = P.cols;
    if (((sat_mode == UWB_SAT_TILE && !win) || (win && win->col_bands)) && p && P.cols % 32 == 0) {
        int64_t bc = win ? static_cast<int64_t>(win->col_bands) : 1024;
        if (const char* e = UWB_KNOB("UWB_TILE_COLS"); e && !win) bc = atoll(e);
        bc = round_up(bc < 128 ? 128 : bc, 128);
        const int64_t hp = round_up(p->guard_cols + p->background_cols, 32);
        if (bc + 2 * hp < P.cols) {
            P.geo.n_bands = (P.cols + bc - 1) / bc;
            P.geo.band_cols = bc;
            P.geo.band_width = bc + 2 * hp;
            P.sat_cols = P.geo.band_width;
        }
    }
    P.geo.band_seg = table_ld_for(P.sat_cols);
    P.table_ld = P.geo.band_seg;
    P.table_stride = (P.max_rows + 1) * P.table_ld;
    P.sat_jobs = P.n_jobs * P.geo.n_bands;
    P.cpl = sat_cpl_for(P.sat_jobs, P.sat_cols);
    P.strips = sat_strips(P.sat_cols, P.cpl);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += round_up(static_cast<int64_t>(bytes), 256);
        return o;
    };
    P.off_tables = take(sizeof(double) * static_cast<size_t>(P.sat_jobs) * P.table_stride);
    P.edge_stride = round_up(P.max_rows, 32);
    // S(r, strip's last column) handed from each strip to the next, contiguous per strip
    P.off_edge = take(P.strips > 1 ? sizeof(double) * static_cast<size_t>(P.sat_jobs) * P.strips * P.edge_stride : 0);
    P.off_prog = take(sizeof(unsigned) * P.sat_jobs * P.strips);
    P.off_counter = take(sizeof(unsigned) * 4);
    P.off_scratch = take(det_cap > 2048 ? sizeof(uwb_detection) * P.n_maps * det_cap : 0);
    if (p) {
        // candidates: detections (about Pfa of the cells) plus the cells within
        // the certification margin of T; 1/256 of the owned cells is >> both
        const int64_t cells = owned * P.cols;
        P.cand_cap = std::max<int64_t>(1024, (cells / 256 + 255) / 256 * 256);
        P.need_rows = round_up(P.max_rows, 32);
        P.n_int = static_cast<int64_t>(interior_count(*p));
        P.off_cand = take(sizeof(int2) * P.n_maps * P.cand_cap);
        P.off_cand_count = take(sizeof(unsigned) * P.n_maps);
        P.off_status = take(sizeof(unsigned) * P.n_maps);
        P.off_need = take(sizeof(unsigned) * P.sat_jobs * P.strips * P.need_rows);
        P.off_ke = take(sizeof(float4) * (P.n_int + 1));
        P.off_flagged = take(sizeof(unsigned) * (P.n_maps + 1)); // [0] count, [1..] maps
    }
    P.total = off;
    return P;
}

SatLaunch sat_launch(const Plan& P, const uwb_map_batch& b, char* ws, unsigned long long* first_bad) {
    SatLaunch L{};
    L.maps = b.maps;
    L.ld = static_cast<int64_t>(b.ld);
    L.map_stride = static_cast<int64_t>(b.map_stride);
    L.cols = P.sat_cols;
    L.geo = P.geo;
    L.n_jobs = P.sat_jobs;
    L.table = reinterpret_cast<double*>(ws + P.off_tables);
    L.table_ld = P.table_ld;
    L.table_stride = P.table_stride;
    L.strips = P.strips;
    L.cpl = P.cpl;
    L.gedge = reinterpret_cast<double*>(ws + P.off_edge);
    L.edge_stride = P.edge_stride;
    L.gprog = reinterpret_cast<unsigned*>(ws + P.off_prog);
    L.tile_counter = reinterpret_cast<unsigned*>(ws + P.off_counter);
    L.first_bad = first_bad;
    L.elem_bytes = b.dtype == UWB_F32 ? 4 : 8;
    const uintptr_t a = reinterpret_cast<uintptr_t>(b.maps);
    L.vec_ok = (a % 16 == 0) && ((b.ld * L.elem_bytes) % 16 == 0) &&
               ((b.map_stride * L.elem_bytes) % 16 == 0);
    return L;
}

cudaError_t run_sat(const Plan& P, const SatLaunch& L, int dtype, cudaStream_t s) {
    // the cluster kernel (small batches) needs no counters
    if (!(L.flags & 256u) && sat_cluster_eligible(L, dtype)) return launch_sat(L, dtype, s);
    cudaError_t e = cudaMemsetAsync(L.gprog, 0, sizeof(unsigned) * P.sat_jobs * P.strips, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(L.tile_counter, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    return launch_sat(L, dtype, s);
}

CfarLaunch cfar_launch(const Plan& P, const uwb_map_batch& b, const uwb_cfar_params& p,
                       const double* alpha, char* ws, const uwb_cfar_outputs& o) {
    CfarLaunch L{};
    L.maps = b.maps;
    L.ld = static_cast<int64_t>(b.ld);
    L.map_stride = static_cast<int64_t>(b.map_stride);
    L.cols = P.cols;
    L.geo = P.geo;
    L.n_jobs = P.n_jobs;
    L.table = ws ? reinterpret_cast<const double*>(ws + P.off_tables) : nullptr;
    L.table_ld = P.table_ld;
    L.table_stride = P.table_stride;
    L.gr = p.guard_rows;
    L.gc = p.guard_cols;
    L.hr = p.guard_rows + p.background_rows;
    L.hc = p.guard_cols + p.background_cols;
    L.alpha = alpha;
    L.mask_bits = o.mask_bits;
    L.words_per_row = static_cast<int64_t>(o.words_per_row);
    L.mask_map_stride = static_cast<int64_t>(o.mask_map_stride);
    L.mask_u8 = o.mask_u8;
    L.thresholds = o.thresholds;
    L.dets = o.dets;
    L.det_cap = static_cast<int64_t>(o.det_capacity);
    L.det_counts = reinterpret_cast<unsigned long long*>(o.det_counts);
    L.first_bad = reinterpret_cast<unsigned long long*>(o.first_bad);
    return L;
}

uwb_status check_batch(const uwb_map_batch* b) {
    if (!b || (!b->maps && b->n_maps && b->rows && b->cols)) return fail(UWB_INVALID_ARGUMENT, "uwb: null batch");
    if (b->dtype != UWB_F32 && b->dtype != UWB_F64) return fail(UWB_INVALID_ARGUMENT, "uwb: bad dtype");
    if (b->ld < b->cols || (b->n_maps > 1 && b->map_stride < b->rows * b->ld))
        return fail(UWB_INVALID_ARGUMENT, "uwb: bad batch layout");
    return UWB_OK;
}


// Phase-event ring (flags bit 1 of uwb_dev_cfar2d): 5 events per call around
// the phases {certify (+ tap marking), SAT, CFAR (certified resolve or the exact
// ring kernel), sort}; the exact path's certify phase is empty.
struct PhaseRing {
    static constexpr int kSlots = 1024;
    static constexpr int kEv = 5;
    std::mutex mu;
    std::vector<cudaEvent_t> ev;
    int used = 0;
    cudaEvent_t* slot() {
        std::lock_guard<std::mutex> lk(mu);
        if (ev.empty()) {
            ev.resize(static_cast<size_t>(kSlots) * kEv);
            for (auto& e : ev) cudaEventCreate(&e);
        }
        if (used >= kSlots) return nullptr;
        return &ev[static_cast<size_t>(used++) * kEv];
    }
};
PhaseRing g_phase;

CertLaunch cert_launch(const Plan& P, const uwb_map_batch& b, const uwb_cfar_params& p, const double* alpha,
                       char* ws, const uwb_cfar_outputs& o) {
    CertLaunch L{};
    L.maps = b.maps;
    L.elem_bytes = b.dtype == UWB_F32 ? 4 : 8;
    L.ld = static_cast<int64_t>(b.ld);
    L.map_stride = static_cast<int64_t>(b.map_stride);
    L.cols = P.cols;
    L.geo = P.geo;
    L.n_maps = P.n_maps;
    L.gr = p.guard_rows;
    L.gc = p.guard_cols;
    L.hr = p.guard_rows + p.background_rows;
    L.hc = p.guard_cols + p.background_cols;
    L.alpha = alpha;
    L.n_int = static_cast<int>(P.n_int);
    L.ke = reinterpret_cast<const float4*>(ws + P.off_ke);
    L.cand = reinterpret_cast<int2*>(ws + P.off_cand);
    L.cand_count = reinterpret_cast<unsigned*>(ws + P.off_cand_count);
    L.cand_cap = P.cand_cap;
    L.status = reinterpret_cast<unsigned*>(ws + P.off_status);
    L.flagged_count = reinterpret_cast<unsigned*>(ws + P.off_flagged);
    L.flagged = L.flagged_count + 1;
    L.first_bad = reinterpret_cast<unsigned long long*>(o.first_bad);
    L.need = reinterpret_cast<unsigned*>(ws + P.off_need);
    L.need_rows = P.need_rows;
    L.strips = P.strips;
    L.cpl = P.cpl;
    L.table = reinterpret_cast<const double*>(ws + P.off_tables);
    L.table_ld = P.table_ld;
    L.table_stride = P.table_stride;
    L.mask_bits = o.mask_bits;
    L.words_per_row = static_cast<int64_t>(o.words_per_row);
    L.mask_map_stride = static_cast<int64_t>(o.mask_map_stride);
    L.dets = o.dets;
    L.det_cap = static_cast<int64_t>(o.det_capacity);
    L.det_counts = reinterpret_cast<unsigned long long*>(o.det_counts);
    L.tie_counts = reinterpret_cast<unsigned long long*>(o.tie_counts);
    L.ties = o.ties;
    L.tie_cap = static_cast<int64_t>(o.tie_capacity);
    int range = 9; // certified values lie in [0, 2^range)
    if (const char* e = UWB_KNOB("UWB_CERT_RANGE_LOG2")) range = std::max(0, std::min(20, atoi(e)));
    cert_prepare(L, range);
    return L;
}

// The certified path applies to mask + list outputs of the integral backend
// with a window instantiated in cfar_cert.cu (the exact two-kernel path
// otherwise; flags bit 6 forces it).
bool cert_applies(const Plan& P, const uwb_map_batch& b, const uwb_cfar_params& p, const uwb_cfar_outputs& o,
                  int backend, uint32_t flags) {
    if (backend != UWB_INTEGRAL || (flags & (4u | 16u | 64u)) || o.thresholds || o.mask_u8 || !o.mask_bits)
        return false;
    // the certify kernel reads aligned column pairs (2x2 tiles)
    const uint64_t esz = b.dtype == UWB_F32 ? 4 : 8;
    if (b.cols % 2 || b.ld % 2 || (b.n_maps > 1 && b.map_stride % 2) ||
        reinterpret_cast<uintptr_t>(b.maps) % (2 * esz))
        return false;
    if (P.cand_cap == 0 || P.geo.rows >= (int64_t(1) << 30) || P.cols >= (int64_t(1) << 30)) return false;
    // small batches are latency-bound: the one-CTA-per-table exact SAT and the
    // ring CFAR take fewer dependent steps than certify + sparse SAT + resolve
    if (!(flags & 512u) && (sat_cta_eligible(P.sat_jobs, P.sat_cols, b.dtype) ||
                            sat_cluster_fits(P.sat_jobs, P.sat_cols, P.geo.max_table_rows(), b.dtype)))
        return false;
    return cert_supported(p.guard_rows + p.background_rows, p.guard_rows, p.guard_cols + p.background_cols,
                          p.guard_cols);
}

// NVTX range over the launches of one stage (host side; visible in nsys / ncu
// NVTX filters; no cost without an attached tool).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Device-resident CFAR of a batch (no validation beyond layout; see uwb_dev_cfar2d).
uwb_status dev_cfar(const uwb_map_batch& b, const uwb_cfar_params& p, const double* alpha,
                    int backend, int sat_mode, uint64_t slab_rows, const uwb_cfar_outputs& o,
                    void* workspace, uint64_t ws_bytes, uint32_t flags, cudaStream_t s,
                    const uwb_row_window* win = nullptr) {
    const Plan P = make_plan(b, &p, backend == UWB_INTEGRAL ? sat_mode : UWB_SAT_GLOBAL, slab_rows,
                             static_cast<int64_t>(o.det_capacity), win);
    if (P.n_jobs > 65535) return fail(UWB_INVALID_ARGUMENT, "uwb: more than 65535 (map, slab) jobs per call");
    if (backend == UWB_INTEGRAL && ws_bytes < P.total) return fail(UWB_INVALID_ARGUMENT, "uwb: workspace too small");
    char* ws = static_cast<char*>(workspace);
    cudaEvent_t* ev = (flags & 2u) ? g_phase.slot() : nullptr;
    UWB_CUDA_TRY(cudaMemsetAsync(o.det_counts, 0, sizeof(uint64_t) * b.n_maps, s));
    if (o.first_bad) UWB_CUDA_TRY(cudaMemsetAsync(o.first_bad, 0xff, sizeof(uint64_t) * 2 * b.n_maps, s));
    if (o.tie_counts) UWB_CUDA_TRY(cudaMemsetAsync(o.tie_counts, 0, sizeof(uint64_t) * b.n_maps, s));
    if (ev) UWB_CUDA_TRY(cudaEventRecord(ev[0], s));
    const bool cert = cert_applies(P, b, p, o, backend, flags);
    if (o.cert_status) {
        if (cert) UWB_CUDA_TRY(cudaMemsetAsync(o.cert_status, 0, sizeof(uint32_t) * b.n_maps, s));
        else UWB_CUDA_TRY(cudaMemsetAsync(o.cert_status, 0xff, sizeof(uint32_t) * b.n_maps, s));
    }
    if (cert) {
        // certify -> mark taps -> sparse SAT -> resolve (+ exact path for flagged maps)
        const CertLaunch CL = cert_launch(P, b, p, alpha, ws, o);
        UWB_CUDA_TRY(cudaMemsetAsync(CL.cand_count, 0, sizeof(unsigned) * P.n_maps, s));
        UWB_CUDA_TRY(cudaMemsetAsync(CL.status, 0, sizeof(unsigned) * P.n_maps, s));
        UWB_CUDA_TRY(cudaMemsetAsync(CL.flagged_count, 0, sizeof(unsigned), s));
        UWB_CUDA_TRY(cudaMemsetAsync(CL.need, 0, sizeof(unsigned) * P.sat_jobs * P.strips * P.need_rows, s));
        UWB_CUDA_TRY(cudaMemset2DAsync(o.mask_bits, sizeof(uint32_t) * o.mask_map_stride, 0,
                                       sizeof(uint32_t) * o.words_per_row * P.geo.out_rows(), b.n_maps, s));
        UWB_CUDA_TRY(launch_cert_table(CL, const_cast<float4*>(CL.ke), static_cast<int>(P.n_int), s));
        SatLaunch SL = sat_launch(P, b, ws, reinterpret_cast<unsigned long long*>(o.first_bad));
        SL.need = (flags & 128u) ? nullptr : CL.need; // bit 7 (test hook): full tables, same results
        SL.need_rows = P.need_rows;
        SL.map_full = CL.status;
        SL.jobs_per_map = P.geo.n_slabs * P.geo.n_bands;
        {
            NvtxRange r("uwb.certify");
            UWB_CUDA_TRY(launch_cert(CL, b.dtype, s));
            UWB_CUDA_TRY(launch_cert_mark(CL, s));
        }
        if (ev) UWB_CUDA_TRY(cudaEventRecord(ev[1], s));
        {
            NvtxRange r("uwb.sat.sparse");
            UWB_CUDA_TRY(run_sat(P, SL, b.dtype, s));
        }
        if (ev) UWB_CUDA_TRY(cudaEventRecord(ev[2], s));
        NvtxRange r("uwb.resolve");
        UWB_CUDA_TRY(launch_cert_resolve(CL, b.dtype, s));
        // maps the certificate could not cover (values outside its range, or
        // more candidates than the list holds) have full tables: exact kernel
        CfarLaunch FL = cfar_launch(P, b, p, alpha, ws, o);
        FL.flagged_maps = CL.flagged;
        FL.flagged_count = CL.flagged_count;
        UWB_CUDA_TRY(launch_cfar_integral_filtered(FL, b.dtype, s));
        if (o.cert_status)
            UWB_CUDA_TRY(cudaMemcpyAsync(o.cert_status, CL.status, sizeof(uint32_t) * b.n_maps,
                                         cudaMemcpyDeviceToDevice, s));
    } else if (backend == UWB_INTEGRAL) {
        if (ev) UWB_CUDA_TRY(cudaEventRecord(ev[1], s));
        bool fused = false;
        if ((flags & 16u) && !(flags & 4u)) {
            // bit 4: SAT and CFAR as one kernel with the table on chip (no table
            // is left in the workspace; falls through to the two kernels when
            // the geometry does not qualify)
            const SatLaunch SL = sat_launch(P, b, ws, reinterpret_cast<unsigned long long*>(o.first_bad));
            UWB_CUDA_TRY(cudaMemsetAsync(SL.gprog, 0, sizeof(unsigned) * P.sat_jobs * P.strips, s));
            UWB_CUDA_TRY(cudaMemsetAsync(SL.tile_counter, 0, sizeof(unsigned), s));
            if (ev) UWB_CUDA_TRY(cudaEventRecord(ev[2], s));
            const cudaError_t e = launch_cfar_fused(SL, cfar_launch(P, b, p, alpha, ws, o), b.dtype, s);
            if (e == cudaSuccess) {
                fused = true;
            } else if (e != cudaErrorNotSupported) {
                return set_cuda_error(e, "launch_cfar_fused");
            } else {
                cudaGetLastError();
            }
        }
        if (!fused) {
            if (!(flags & 4u)) { // bit 2: the workspace already holds this batch's tables
                NvtxRange r("uwb.sat");
                SatLaunch SL = sat_launch(P, b, ws, reinterpret_cast<unsigned long long*>(o.first_bad));
                if (flags & 1024u) SL.flags |= 256u; // bit 10 (test hook): no cluster kernel, same results
                UWB_CUDA_TRY(run_sat(P, SL, b.dtype, s));
            }
            NvtxRange r("uwb.cfar");
            if (ev) UWB_CUDA_TRY(cudaEventRecord(ev[2], s));
            CfarLaunch FL = cfar_launch(P, b, p, alpha, ws, o);
            FL.fixed_rows = (flags & 256u) != 0; // bit 8 (test hook): 256-row ring chunks, same results
            UWB_CUDA_TRY(launch_cfar_integral(FL, b.dtype, s));
        }
    } else {
        if (ev) UWB_CUDA_TRY(cudaEventRecord(ev[1], s));
        if (ev) UWB_CUDA_TRY(cudaEventRecord(ev[2], s));
        UWB_CUDA_TRY(launch_cfar_naive(cfar_launch(P, b, p, alpha, nullptr, o), b.dtype, s));
    }
    if (ev) UWB_CUDA_TRY(cudaEventRecord(ev[3], s));
    struct Tail {
        cudaEvent_t* ev;
        cudaStream_t s;
        ~Tail() {
            if (ev) cudaEventRecord(ev[4], s);
        }
    } tail{ev, s};
    if (!(flags & 1u)) {
        uwb_detection* scratch = (o.det_capacity > 2048 && ws && ws_bytes >= P.total)
                                     ? reinterpret_cast<uwb_detection*>(ws + P.off_scratch)
                                     : nullptr;
        NvtxRange r("uwb.sort");
        UWB_CUDA_TRY(launch_sort_detections(o.dets, static_cast<int64_t>(o.det_capacity),
                                            reinterpret_cast<const unsigned long long*>(o.det_counts),
                                            static_cast<int64_t>(b.n_maps), scratch, s));
    }
    return UWB_OK;
}

void twiddles(int64_t L, std::vector<double>& wr, std::vector<double>& wi) {
    // identical expression to oracle/fftw_shim/fft_provider.c:uwb_fft_twiddles
    wr.resize(static_cast<size_t>(L));
    wi.resize(static_cast<size_t>(L));
    for (int64_t k = 0; k < L; ++k) {
        const double angle = (2.0 * M_PI * static_cast<double>(k)) / static_cast<double>(L);
        wr[static_cast<size_t>(k)] = std::cos(angle);
        wi[static_cast<size_t>(k)] = -std::sin(angle);
    }
}

uint64_t next_pow2(uint64_t n) {
    uint64_t p = 1;
    while (p < n) p <<= 1;
    return p;
}

} // namespace

uwb_status set_error(uwb_status s, const char* msg, int64_t row, int64_t col) {
    return fail(s, msg, row, col);
}

uwb_status set_cuda_error(cudaError_t e, const char* what) {
    return fail(UWB_CUDA_ERROR, std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what);
}

// PipelineConfig::validate / effective_fft_length and the stage checks of
// detect (pipeline.cpp:40-56, 100-105, 157-223), evaluated on the host. The
// configuration error is reported after the frame's finiteness check and the
// stage error after it, as in the reference.
struct DetectPlan {
    uint64_t L = 0, first = 0, kept = 0;
    uwb_status cfg_status = UWB_OK, stage_status = UWB_OK;
    std::string cfg_msg, stage_msg;
    bool ok() const { return cfg_status == UWB_OK && stage_status == UWB_OK; }
};

DetectPlan detect_plan(uint64_t m, uint64_t n, double prf, const uwb_pipeline_config& c) {
    (void)m;
    DetectPlan D;
    const uint64_t L = c.fft_length == 0 ? next_pow2(n) : c.fft_length;
    D.L = L;
    std::string& cfg_msg = D.cfg_msg;
    uwb_status& cfg_status = D.cfg_status;
    std::string& stage_msg = D.stage_msg;
    uwb_status& stage_status = D.stage_status;

    // configuration checks that do not need data; reported after the
    // finiteness check below to keep the reference's order

    if (c.mean_filter_window == 0 || c.mean_filter_window % 2 == 0) {
        cfg_status = UWB_PARAMETER_ERROR;
        cfg_msg = "PipelineConfig: mean_filter_window must be odd and positive, got " + S(c.mean_filter_window);
    } else if (!(c.band_low_hz > 0.0) || !(c.band_low_hz < c.band_high_hz)) {
        cfg_status = UWB_PARAMETER_ERROR;
        cfg_msg = "PipelineConfig: need 0 < band_low_hz < band_high_hz";
    } else if (!(c.normalization_epsilon > 0.0)) {
        cfg_status = UWB_PARAMETER_ERROR;
        cfg_msg = "PipelineConfig: normalization_epsilon must be positive";
    } else if (validate_params(c.cfar) != UWB_OK) {
        cfg_status = UWB_PARAMETER_ERROR;
        cfg_msg = g_err.message;
    } else if (!(c.band_high_hz < prf / 2.0)) {
        cfg_status = UWB_PARAMETER_ERROR;
        cfg_msg = "detect: band_high_hz must be below prf/2 = " + fmt_double(prf / 2.0) + " Hz";
    }
    const bool smooth = c.mean_filter_mode == 0;

    if (cfg_status == UWB_OK) {
        if (smooth && (c.mean_filter_window > n)) {
            stage_status = UWB_PARAMETER_ERROR;
            stage_msg = "mean_filter_slow: mean_filter_slow: window must be odd and in [1, " + S(n) + "], got " +
                        S(c.mean_filter_window);
        } else if (L < n) {
            stage_status = UWB_PARAMETER_ERROR;
            stage_msg = "slow_time_spectrum: slow_time_spectrum: fft_length " + S(L) + " < trace count " + S(n);
        }
    }

    if (cfg_status == UWB_OK && stage_status == UWB_OK) {
        const uint64_t bins = L / 2 + 1;
        uint64_t f = bins, l = 0;
        for (uint64_t k = 0; k < bins; ++k) {
            const double fr = static_cast<double>(k) * prf / static_cast<double>(L);
            if (fr >= c.band_low_hz && fr <= c.band_high_hz) {
                if (f == bins) f = k;
                l = k;
            }
        }
        if (f == bins) {
            const double res = bins > 1 ? (1.0 * prf / static_cast<double>(L)) - (0.0 * prf / static_cast<double>(L))
                                        : 0.0 * prf / static_cast<double>(L);
            stage_status = UWB_CONFIGURATION_ERROR;
            stage_msg = "band_select: band_select: no FFT bin falls in [" + fmt_double(c.band_low_hz) + ", " +
                        fmt_double(c.band_high_hz) + "] Hz at bin resolution " + fmt_double(res) + " Hz";
        } else {
            D.first = f;
            D.kept = l - f + 1;
        }
    }
    return D;
}

} // namespace uwb

using namespace uwb;

// ======================================================================== API

extern "C" {

const char* uwb_last_error(void) { return g_err.message.c_str(); }

void uwb_last_error_cell(int64_t* row, int64_t* col) {
    if (row) *row = g_err.row;
    if (col) *col = g_err.col;
}

int uwb_device_available(void) { return device_ok() ? 1 : 0; }

uwb_status uwb_alpha_factor(uint64_t n_train, double pfa, double* out) {
    if (n_train == 0) return fail(UWB_PARAMETER_ERROR, "alpha_factor: n_train must be >= 1");
    if (!(pfa > 0.0) || !(pfa < 1.0))
        return fail(UWB_PARAMETER_ERROR, "alpha_factor: pfa must lie in (0,1), got " + fmt_double(pfa));
    *out = alpha_value(n_train, pfa);
    return ok();
}

uwb_status uwb_cfar_params_validate(const uwb_cfar_params* p) {
    if (!p) return fail(UWB_INVALID_ARGUMENT, "uwb: null params");
    return validate_params(*p);
}

uint64_t uwb_interior_train_count(const uwb_cfar_params* p) { return p ? interior_count(*p) : 0; }

uwb_status uwb_training_window(const uwb_cfar_params* p, uint64_t row, uint64_t col, uint64_t rows,
                               uint64_t cols, uint64_t out[9]) {
    // cfar.cpp:179-198
    if (uwb_status s = validate_params(*p)) return s;
    if (row >= rows || col >= cols)
        return fail(UWB_BOUNDS_ERROR, "training_window: cell (" + S(row) + ", " + S(col) + ") outside " +
                                          S(rows) + "x" + S(cols) + " map");
    auto lo = [](uint64_t c, int r) -> uint64_t {
        const long long v = static_cast<long long>(c) - r;
        return v < 0 ? 0 : static_cast<uint64_t>(v);
    };
    auto hi = [](uint64_t c, int r, uint64_t d) -> uint64_t {
        const uint64_t v = c + static_cast<uint64_t>(r);
        return v >= d ? d - 1 : v;
    };
    const int hr = p->guard_rows + p->background_rows, hc = p->guard_cols + p->background_cols;
    out[0] = lo(row, hr); out[1] = hi(row, hr, rows); out[2] = lo(col, hc); out[3] = hi(col, hc, cols);
    out[4] = lo(row, p->guard_rows); out[5] = hi(row, p->guard_rows, rows);
    out[6] = lo(col, p->guard_cols); out[7] = hi(col, p->guard_cols, cols);
    out[8] = (out[1] - out[0] + 1) * (out[3] - out[2] + 1) - (out[5] - out[4] + 1) * (out[7] - out[6] + 1);
    if (out[8] == 0)
        return fail(UWB_CONFIGURATION_ERROR, "training_window: " + S(rows) + "x" + S(cols) +
                                                 " map leaves no training cells at (" + S(row) + ", " +
                                                 S(col) + ")");
    return ok();
}

uwb_status uwb_alpha_table(const uwb_cfar_params* p, double* out, uint64_t len) {
    if (uwb_status s = validate_params(*p)) return s;
    const std::vector<double> a = alpha_table_host(*p);
    if (len < a.size()) return fail(UWB_INVALID_ARGUMENT, "uwb_alpha_table: buffer shorter than interior_train_count+1");
    std::memcpy(out, a.data(), sizeof(double) * a.size());
    return ok();
}

// ------------------------------------------------------------ build_sat ---

uwb_status uwb_build_sat(const double* src, uint64_t rows, uint64_t cols, double* table) {
    if (rows == 0 || cols == 0)
        return fail(UWB_DIMENSION_ERROR, "build_sat: source matrix must be at least 1x1, got " + S(rows) + "x" + S(cols));
    if (uwb_status s = need_device()) return s;
    cudaStream_t s = host_stream();
    uwb_map_batch b{};
    b.dtype = UWB_F64;
    b.n_maps = 1;
    b.rows = rows;
    b.cols = cols;
    b.ld = cols;
    b.map_stride = rows * cols;
    DevBuf d_src, d_ws, d_bad;
    UWB_CUDA_TRY(d_src.alloc(sizeof(double) * rows * cols, s));
    UWB_CUDA_TRY(cudaMemcpyAsync(d_src.p, src, sizeof(double) * rows * cols, cudaMemcpyHostToDevice, s));
    b.maps = d_src.p;
    const uint64_t wsb = uwb_dev_build_sat_workspace(&b);
    UWB_CUDA_TRY(d_ws.alloc(wsb, s));
    UWB_CUDA_TRY(d_bad.alloc(sizeof(uint64_t) * 2, s));
    const Plan P = make_plan(b, nullptr, UWB_SAT_GLOBAL, 0, 0);
    double* d_table = reinterpret_cast<double*>(static_cast<char*>(d_ws.p) + P.off_tables);
    if (uwb_status st = uwb_dev_build_sat(&b, d_table, P.table_ld, P.table_stride, d_bad.as<uint64_t>(),
                                          d_ws.p, wsb, s))
        return st;
    uint64_t bad[2];
    UWB_CUDA_TRY(cudaMemcpyAsync(bad, d_bad.p, sizeof(bad), cudaMemcpyDeviceToHost, s));
    UWB_CUDA_TRY(cudaMemcpy2DAsync(table, sizeof(double) * (cols + 1), d_table + kTabShift,
                                   sizeof(double) * P.table_ld, sizeof(double) * (cols + 1), rows + 1,
                                   cudaMemcpyDeviceToHost, s));
    UWB_CUDA_TRY(cudaStreamSynchronize(s));
    if (bad[0] != ~0ull) {
        const int64_t r = static_cast<int64_t>(bad[0] / cols), c = static_cast<int64_t>(bad[0] % cols);
        return fail(UWB_INPUT_ERROR, "build_sat: non-finite entry at (" + S(r) + ", " + S(c) + ")", r, c);
    }
    return ok();
}

uint64_t uwb_dev_build_sat_workspace(const uwb_map_batch* b) {
    return make_plan(*b, nullptr, UWB_SAT_GLOBAL, 0, 0).total;
}

uwb_status uwb_dev_build_sat(const uwb_map_batch* b, double* sat, uint64_t sat_ld, uint64_t sat_map_stride,
                             uint64_t* first_nonfinite, void* workspace, uint64_t ws_bytes, void* stream) {
    if (uwb_status s = check_batch(b)) return s;
    if (uwb_status s = need_device()) return s;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Plan P = make_plan(*b, nullptr, UWB_SAT_GLOBAL, 0, 0);
    if (ws_bytes < P.total) return fail(UWB_INVALID_ARGUMENT, "uwb: workspace too small");
    if (sat_ld < static_cast<uint64_t>(table_ld_for(P.cols)) || sat_ld % kTabAlign ||
        reinterpret_cast<uintptr_t>(sat) % 256)
        return fail(UWB_INVALID_ARGUMENT,
                    "uwb_dev_build_sat: table must be 256-byte aligned with ld a multiple of 32 and >= cols+32");
    char* ws = static_cast<char*>(workspace);
    // first_nonfinite uses the 2-slot-per-map layout internally
    DevBuf bad;
    UWB_CUDA_TRY(bad.alloc(sizeof(uint64_t) * 2 * b->n_maps, s));
    UWB_CUDA_TRY(cudaMemsetAsync(bad.p, 0xff, sizeof(uint64_t) * 2 * b->n_maps, s));
    SatLaunch L = sat_launch(P, *b, ws, bad.as<unsigned long long>());
    L.table = sat;
    L.table_ld = static_cast<int64_t>(sat_ld);
    L.table_stride = static_cast<int64_t>(sat_map_stride);
    UWB_CUDA_TRY(run_sat(P, L, b->dtype, s));
    if (first_nonfinite)
        UWB_CUDA_TRY(cudaMemcpy2DAsync(first_nonfinite, sizeof(uint64_t), bad.p, 2 * sizeof(uint64_t),
                                       sizeof(uint64_t), b->n_maps, cudaMemcpyDeviceToDevice, s));
    return ok();
}

// ---------------------------------------------------------------- CFAR ---

uint64_t uwb_dev_cfar2d_workspace(const uwb_map_batch* b, const uwb_cfar_params* p, int32_t sat_mode,
                                  uint64_t slab_rows, uint64_t det_capacity) {
    return make_plan(*b, p, sat_mode, slab_rows, static_cast<int64_t>(det_capacity)).total;
}

uwb_status uwb_dev_cfar2d(const uwb_map_batch* b, const uwb_cfar_params* p, const double* alpha_dev,
                          int32_t sat_mode, uint64_t slab_rows, const uwb_cfar_outputs* out,
                          void* workspace, uint64_t ws_bytes, uint32_t flags, void* stream) {
    if (uwb_status s = check_batch(b)) return s;
    if (uwb_status s = validate_params(*p)) return s;
    if (b->rows == 0 || b->cols == 0) return fail(UWB_DIMENSION_ERROR, "cfar2d: power map must be at least 1x1");
    if (degenerate(*p, b->rows, b->cols)) return fail(UWB_CONFIGURATION_ERROR, degenerate_msg(*p, b->rows, b->cols));
    if (uwb_status s = need_device()) return s;
    const Plan P = make_plan(*b, p, sat_mode, slab_rows, static_cast<int64_t>(out->det_capacity));
    if (ws_bytes < P.total) return fail(UWB_INVALID_ARGUMENT, "uwb: workspace too small (need " + S(static_cast<uint64_t>(P.total)) + ")");
    // flags bit 3: the naive backend (cfar2d_naive, cfar.cpp:200-216; no table)
    const int backend = (flags & 8u) ? UWB_NAIVE : UWB_INTEGRAL;
    if (uwb_status s = dev_cfar(*b, *p, alpha_dev, backend, sat_mode, slab_rows, *out, workspace, ws_bytes, flags,
                                static_cast<cudaStream_t>(stream)))
        return s;
    return ok();
}

static uwb_status check_window(const uwb_map_batch* b, const uwb_row_window* w, const uwb_cfar_params* p) {
    if (!w) return fail(UWB_INVALID_ARGUMENT, "uwb: null row window");
    if (w->row_begin >= w->row_end || w->row_end > w->global_rows)
        return fail(UWB_BOUNDS_ERROR, "uwb: row window [" + S(w->row_begin) + ", " + S(w->row_end) +
                                          ") outside a map of " + S(w->global_rows) + " rows");
    const uint64_t halo = static_cast<uint64_t>(p->guard_rows + p->background_rows);
    const uint64_t need0 = w->row_begin > halo ? w->row_begin - halo : 0;
    const uint64_t need1 = std::min(w->global_rows, w->row_end + halo);
    if (w->buf_row0 > need0 || w->buf_row0 + b->rows < need1)
        return fail(UWB_BOUNDS_ERROR, "uwb: the buffer holds rows [" + S(w->buf_row0) + ", " +
                                          S(w->buf_row0 + b->rows) + "), the window needs [" + S(need0) + ", " +
                                          S(need1) + ")");
    return UWB_OK;
}

uint64_t uwb_dev_cfar2d_window_workspace(const uwb_map_batch* b, const uwb_row_window* win,
                                         const uwb_cfar_params* p, uint64_t slab_rows, uint64_t det_capacity) {
    return make_plan(*b, p, UWB_SAT_SLAB, slab_rows, static_cast<int64_t>(det_capacity), win).total;
}

uwb_status uwb_dev_cfar2d_window(const uwb_map_batch* b, const uwb_row_window* win, const uwb_cfar_params* p,
                                 const double* alpha_dev, uint64_t slab_rows, const uwb_cfar_outputs* out,
                                 void* workspace, uint64_t ws_bytes, uint32_t flags, void* stream) {
    if (uwb_status s = check_batch(b)) return s;
    if (uwb_status s = validate_params(*p)) return s;
    if (b->rows == 0 || b->cols == 0) return fail(UWB_DIMENSION_ERROR, "cfar2d: power map must be at least 1x1");
    if (uwb_status s = check_window(b, win, p)) return s;
    if (degenerate(*p, win->global_rows, b->cols))
        return fail(UWB_CONFIGURATION_ERROR, degenerate_msg(*p, win->global_rows, b->cols));
    if (uwb_status s = need_device()) return s;
    const Plan P = make_plan(*b, p, UWB_SAT_SLAB, slab_rows, static_cast<int64_t>(out->det_capacity), win);
    if (ws_bytes < P.total) return fail(UWB_INVALID_ARGUMENT, "uwb: workspace too small (need " + S(static_cast<uint64_t>(P.total)) + ")");
    if (uwb_status s = dev_cfar(*b, *p, alpha_dev, UWB_INTEGRAL, UWB_SAT_SLAB, slab_rows, *out, workspace, ws_bytes,
                                flags, static_cast<cudaStream_t>(stream), win))
        return s;
    return ok();
}

uwb_status uwb_cfar2d(uwb_backend backend, const double* map, uint64_t rows, uint64_t cols,
                      const uwb_cfar_params* p, uint8_t* mask, double* thresholds, uwb_detection* dets,
                      uint64_t det_capacity, uint64_t* n_det) {
    *n_det = 0;
    const uint64_t cells = rows * cols;
    if (backend == UWB_INTEGRAL && cells == 0) // sat.cpp:13-16 runs first
        return fail(UWB_DIMENSION_ERROR, "build_sat: source matrix must be at least 1x1, got " + S(rows) + "x" + S(cols));
    if (backend == UWB_NAIVE) {
        if (uwb_status s = validate_params(*p)) return s;
        if (cells == 0) return fail(UWB_DIMENSION_ERROR, "cfar2d: power map must be at least 1x1");
    }
    if (uwb_status s = need_device()) return s;
    cudaStream_t s = host_stream();

    uwb_map_batch b{};
    b.dtype = UWB_F64;
    b.n_maps = 1;
    b.rows = rows;
    b.cols = cols;
    b.ld = cols;
    b.map_stride = cells;
    // parameters may be invalid at this point for the integral backend (the
    // reference validates them after building the table); keep the kernels safe
    uwb_cfar_params q = *p;
    const bool params_ok = validate_params(q) == UWB_OK;
    if (!params_ok) q = uwb_cfar_params{0, 0, 1, 1, 0.5};
    const std::vector<double> alpha = alpha_table_host(q);
    // first pass with a bounded list; rerun with the exact count on overflow
    uint64_t cap = std::max<uint64_t>(std::min<uint64_t>(cells, 1u << 16), 1);
retry:
    DevBuf d_map, d_alpha, d_mask, d_thr, d_dets, d_cnt, d_bad, d_bits, d_ws;
    UWB_CUDA_TRY(d_map.alloc(sizeof(double) * cells, s));
    UWB_CUDA_TRY(cudaMemcpyAsync(d_map.p, map, sizeof(double) * cells, cudaMemcpyHostToDevice, s));
    b.maps = d_map.p;
    UWB_CUDA_TRY(d_alpha.alloc(sizeof(double) * alpha.size(), s));
    UWB_CUDA_TRY(cudaMemcpyAsync(d_alpha.p, alpha.data(), sizeof(double) * alpha.size(), cudaMemcpyHostToDevice, s));
    UWB_CUDA_TRY(d_mask.alloc(cells, s));
    UWB_CUDA_TRY(d_thr.alloc(sizeof(double) * cells, s));
    UWB_CUDA_TRY(d_dets.alloc(sizeof(uwb_detection) * cap, s));
    UWB_CUDA_TRY(d_cnt.alloc(sizeof(uint64_t), s));
    UWB_CUDA_TRY(d_bad.alloc(sizeof(uint64_t) * 2, s));
    const uint64_t words = (cols + 31) / 32;
    UWB_CUDA_TRY(d_bits.alloc(sizeof(uint32_t) * words * rows, s));

    uwb_cfar_outputs o{};
    o.mask_bits = d_bits.as<uint32_t>();
    o.words_per_row = words;
    o.mask_map_stride = words * rows;
    o.mask_u8 = d_mask.as<uint8_t>();
    o.thresholds = d_thr.as<double>();
    o.dets = d_dets.as<uwb_detection>();
    o.det_capacity = cap;
    o.det_counts = d_cnt.as<uint64_t>();
    o.first_bad = d_bad.as<uint64_t>();

    const Plan P = make_plan(b, &q, UWB_SAT_GLOBAL, 0, static_cast<int64_t>(cap));
    UWB_CUDA_TRY(d_ws.alloc(P.total, s));
    if (uwb_status st = dev_cfar(b, q, d_alpha.as<double>(), backend, UWB_SAT_GLOBAL, 0, o, d_ws.p, P.total, 0, s))
        return st;
    uint64_t bad[2], cnt = 0;
    UWB_CUDA_TRY(cudaMemcpyAsync(bad, d_bad.p, sizeof(bad), cudaMemcpyDeviceToHost, s));
    UWB_CUDA_TRY(cudaMemcpyAsync(&cnt, d_cnt.p, sizeof(cnt), cudaMemcpyDeviceToHost, s));
    UWB_CUDA_TRY(cudaStreamSynchronize(s));

    auto cell_rc = [&](uint64_t idx, int64_t& r, int64_t& c) {
        r = static_cast<int64_t>(idx / cols);
        c = static_cast<int64_t>(idx % cols);
    };
    if (backend == UWB_INTEGRAL) {
        if (bad[0] != ~0ull) { // sat.cpp:28-32
            int64_t r, c;
            cell_rc(bad[0], r, c);
            return fail(UWB_INPUT_ERROR, "build_sat: non-finite entry at (" + S(r) + ", " + S(c) + ")", r, c);
        }
        if (!params_ok) return validate_params(*p);
    }
    if (bad[1] != ~0ull) { // cfar.cpp:85-92
        int64_t r, c;
        cell_rc(bad[1], r, c);
        return fail(UWB_INPUT_ERROR, "cfar2d: cell (" + S(r) + ", " + S(c) + ") is not a finite non-negative power", r, c);
    }
    if (degenerate(*p, rows, cols)) return fail(UWB_CONFIGURATION_ERROR, degenerate_msg(*p, rows, cols));
    if (cnt > cap) {
        cap = cnt;
        goto retry;
    }

    *n_det = cnt;
    const uint64_t n_copy = std::min(cnt, det_capacity);
    if (mask) UWB_CUDA_TRY(cudaMemcpyAsync(mask, d_mask.p, cells, cudaMemcpyDeviceToHost, s));
    if (thresholds) UWB_CUDA_TRY(cudaMemcpyAsync(thresholds, d_thr.p, sizeof(double) * cells, cudaMemcpyDeviceToHost, s));
    if (dets && n_copy)
        UWB_CUDA_TRY(cudaMemcpyAsync(dets, d_dets.p, sizeof(uwb_detection) * n_copy, cudaMemcpyDeviceToHost, s));
    UWB_CUDA_TRY(cudaStreamSynchronize(s));
    if (cnt > det_capacity) return fail(UWB_CAPACITY_ERROR, "uwb_cfar2d: detection buffer too small");
    return ok();
}

// ----------------------------------------------------------- front-end ---

namespace {

// Runs the requested front-end stages on the device. in_host: m x n doubles.
// Outputs (host, optional): frame_out m x n, band m x kept, full m x bins.
uwb_status run_frontend(const double* in_host, uint64_t m, uint64_t n, int stages, uint64_t window,
                        int mode, double eps, uint64_t L, uint64_t first, uint64_t kept, double* frame_out,
                        double* band_out, double* full_out, bool check_finite, uint64_t* first_nonfinite) {
    if (uwb_status s = need_device()) return s;
    cudaStream_t s = host_stream();
    if (L > 8192 && (stages & 16)) return fail(UWB_INVALID_ARGUMENT, "uwb: fft_length > 8192 not supported on the device path");
    DevBuf d_in, d_work, d_band, d_full, d_wr, d_wi, d_bad;
    UWB_CUDA_TRY(d_in.alloc(sizeof(double) * m * n, s));
    UWB_CUDA_TRY(cudaMemcpyAsync(d_in.p, in_host, sizeof(double) * m * n, cudaMemcpyHostToDevice, s));
    UWB_CUDA_TRY(d_work.alloc(sizeof(double) * m * n, s));
    UWB_CUDA_TRY(d_bad.alloc(sizeof(uint64_t), s));
    UWB_CUDA_TRY(cudaMemsetAsync(d_bad.p, 0xff, sizeof(uint64_t), s));
    FrontendLaunch F{};
    F.frame = d_in.p;
    F.dtype = UWB_F64;
    F.m = static_cast<int64_t>(m);
    F.n = static_cast<int64_t>(n);
    F.work = d_work.as<double>();
    F.first_nonfinite = check_finite ? d_bad.as<unsigned long long>() : nullptr;
    F.window = window;
    F.mode = mode;
    F.epsilon = eps;
    F.L = static_cast<int64_t>(L);
    F.first_bin = static_cast<int64_t>(first);
    F.kept = static_cast<int64_t>(kept);
    std::vector<double> wr, wi;
    if (stages & 16) {
        twiddles(F.L, wr, wi);
        UWB_CUDA_TRY(d_wr.alloc(sizeof(double) * L, s));
        UWB_CUDA_TRY(d_wi.alloc(sizeof(double) * L, s));
        UWB_CUDA_TRY(cudaMemcpyAsync(d_wr.p, wr.data(), sizeof(double) * L, cudaMemcpyHostToDevice, s));
        UWB_CUDA_TRY(cudaMemcpyAsync(d_wi.p, wi.data(), sizeof(double) * L, cudaMemcpyHostToDevice, s));
        F.wr = d_wr.as<double>();
        F.wi = d_wi.as<double>();
        if (band_out) {
            UWB_CUDA_TRY(d_band.alloc(sizeof(double) * m * kept, s));
            F.band = d_band.as<double>();
        }
        if (full_out) {
            UWB_CUDA_TRY(d_full.alloc(sizeof(double) * m * (L / 2 + 1), s));
            F.full_power = d_full.as<double>();
        }
    }
    // columns stage (always runs: it also moves the input into the work buffer)
    F.stage_mask = stages & 3;
    UWB_CUDA_TRY(launch_frontend_columns(F, s));
    if (stages & (4 | 8 | 16)) {
        F.stage_mask = stages & (4 | 8 | 16);
        UWB_CUDA_TRY(launch_frontend_rows(F, s));
    }
    uint64_t bad = ~0ull;
    UWB_CUDA_TRY(cudaMemcpyAsync(&bad, d_bad.p, sizeof(bad), cudaMemcpyDeviceToHost, s));
    if (frame_out) UWB_CUDA_TRY(cudaMemcpyAsync(frame_out, d_work.p, sizeof(double) * m * n, cudaMemcpyDeviceToHost, s));
    if (band_out && (stages & 16))
        UWB_CUDA_TRY(cudaMemcpyAsync(band_out, d_band.p, sizeof(double) * m * kept, cudaMemcpyDeviceToHost, s));
    if (full_out && (stages & 16))
        UWB_CUDA_TRY(cudaMemcpyAsync(full_out, d_full.p, sizeof(double) * m * (L / 2 + 1), cudaMemcpyDeviceToHost, s));
    UWB_CUDA_TRY(cudaStreamSynchronize(s));
    if (first_nonfinite) *first_nonfinite = bad;
    return UWB_OK;
}

} // namespace

uwb_status uwb_remove_dc(const double* in, uint64_t m, uint64_t n, double* out) {
    if (m == 0 || n == 0) return ok();
    if (uwb_status s = run_frontend(in, m, n, 1, 1, 0, 1.0, 0, 0, 0, out, nullptr, nullptr, false, nullptr)) return s;
    return ok();
}

uwb_status uwb_detrend_linear(const double* in, uint64_t m, uint64_t n, double* out) {
    if (m == 0 || n == 0) return ok();
    if (uwb_status s = run_frontend(in, m, n, 2, 1, 0, 1.0, 0, 0, 0, out, nullptr, nullptr, false, nullptr)) return s;
    return ok();
}

uwb_status uwb_mean_filter_slow(const double* in, uint64_t m, uint64_t n, uint64_t window, double* out) {
    // pipeline.cpp:101-106
    if (window == 0 || window % 2 == 0 || window > n)
        return fail(UWB_PARAMETER_ERROR, "mean_filter_slow: window must be odd and in [1, " + S(n) + "], got " + S(window));
    if (m == 0) return ok();
    if (uwb_status s = run_frontend(in, m, n, 4, window, 0, 1.0, 0, 0, 0, out, nullptr, nullptr, false, nullptr)) return s;
    return ok();
}

uwb_status uwb_subtract_slow_time_mean(const double* in, uint64_t m, uint64_t n, double* out) {
    if (m == 0 || n == 0) return ok();
    if (uwb_status s = run_frontend(in, m, n, 4, 1, 1, 1.0, 0, 0, 0, out, nullptr, nullptr, false, nullptr)) return s;
    return ok();
}

uwb_status uwb_normalize_slow(const double* in, uint64_t m, uint64_t n, double epsilon, double* out) {
    if (!(epsilon > 0.0)) return fail(UWB_PARAMETER_ERROR, "normalize_slow: epsilon must be positive");
    if (m == 0 || n == 0) return ok();
    if (uwb_status s = run_frontend(in, m, n, 8, 1, 0, epsilon, 0, 0, 0, out, nullptr, nullptr, false, nullptr)) return s;
    return ok();
}

uwb_status uwb_slow_time_spectrum(const double* in, uint64_t m, uint64_t n, double fast_rate, double prf,
                                  uint64_t fft_length, double* power, double* freq_axis, double* range_axis) {
    if (fft_length < n)
        return fail(UWB_PARAMETER_ERROR, "slow_time_spectrum: fft_length " + S(fft_length) + " < trace count " + S(n));
    const uint64_t bins = fft_length / 2 + 1;
    // pipeline.cpp:169-175 axes (host scalar arithmetic, as the reference)
    if (freq_axis)
        for (uint64_t k = 0; k < bins; ++k)
            freq_axis[k] = static_cast<double>(k) * prf / static_cast<double>(fft_length);
    if (range_axis)
        for (uint64_t r = 0; r < m; ++r)
            range_axis[r] = static_cast<double>(r) * 299792458.0 / (2.0 * fast_rate);
    if (m == 0) return ok();
    if (uwb_status s = run_frontend(in, m, n, 16, 1, 0, 1.0, fft_length, 0, 0, nullptr, nullptr, power, false, nullptr))
        return s;
    return ok();
}

uwb_status uwb_band_select(const double* power, uint64_t m, uint64_t bins, const double* freq_axis,
                           double low, double high, uint64_t* first_out, uint64_t* kept_out,
                           double* out_power, double* out_freq) {
    // pipeline.cpp:192-223
    uint64_t first = bins, last = 0;
    for (uint64_t k = 0; k < bins; ++k) {
        const double f = freq_axis[k];
        if (f >= low && f <= high) {
            if (first == bins) first = k;
            last = k;
        }
    }
    if (first == bins) {
        const double res = bins > 1 ? freq_axis[1] - freq_axis[0] : freq_axis[0];
        return fail(UWB_CONFIGURATION_ERROR, "band_select: no FFT bin falls in [" + fmt_double(low) + ", " +
                                                 fmt_double(high) + "] Hz at bin resolution " + fmt_double(res) + " Hz");
    }
    const uint64_t kept = last - first + 1;
    *first_out = first;
    *kept_out = kept;
    if (out_freq) std::memcpy(out_freq, freq_axis + first, sizeof(double) * kept);
    if (out_power && m) {
        if (uwb_status s = need_device()) return s;
        UWB_CUDA_TRY(cudaMemcpy2D(out_power, sizeof(double) * kept, power + first, sizeof(double) * bins,
                                  sizeof(double) * kept, m, cudaMemcpyHostToHost));
    }
    return ok();
}

uwb_status uwb_detect(const double* frame, uint64_t m, uint64_t n, double fast_rate, double prf,
                      const uwb_pipeline_config* cfg, uint64_t band_capacity, double* band_power,
                      double* band_freq, double* range_axis, uint64_t* kept_out, uint8_t* mask,
                      double* thresholds, uwb_detection* dets, uint64_t det_capacity, uint64_t* n_det) {
    *n_det = 0;
    *kept_out = 0;
    // RadarFrame::validate (pipeline.cpp:27-38)
    if (m < 2 || n < 2)
        return fail(UWB_DIMENSION_ERROR, "RadarFrame: need at least 2x2 samples, got " + S(m) + "x" + S(n));
    if (!(fast_rate > 0.0) || !(prf > 0.0))
        return fail(UWB_PARAMETER_ERROR, "RadarFrame: fast_rate and prf must be positive");
    if (uwb_status s = need_device()) return s;
    cudaStream_t s = host_stream();

    const uwb_pipeline_config& c = *cfg;
    const DetectPlan D = detect_plan(m, n, prf, c);
    const uint64_t L = D.L, first = D.first, kept = D.kept;
    const uwb_status cfg_status = D.cfg_status, stage_status = D.stage_status;
    const std::string& cfg_msg = D.cfg_msg;
    const std::string& stage_msg = D.stage_msg;
    const bool smooth = c.mean_filter_mode == 0;
    const bool run_all = cfg_status == UWB_OK && stage_status == UWB_OK;
    if (run_all && L > 8192) return fail(UWB_INVALID_ARGUMENT, "uwb: fft_length > 8192 not supported on the device path");
    if (run_all && kept > band_capacity) return fail(UWB_INVALID_ARGUMENT, "uwb_detect: band_capacity too small");

    // ---- device pipeline
    DevBuf d_in, d_work, d_band, d_wr, d_wi, d_bad;
    UWB_CUDA_TRY(d_in.alloc(sizeof(double) * m * n, s));
    UWB_CUDA_TRY(cudaMemcpyAsync(d_in.p, frame, sizeof(double) * m * n, cudaMemcpyHostToDevice, s));
    UWB_CUDA_TRY(d_work.alloc(sizeof(double) * m * n, s));
    UWB_CUDA_TRY(d_bad.alloc(sizeof(uint64_t), s));
    UWB_CUDA_TRY(cudaMemsetAsync(d_bad.p, 0xff, sizeof(uint64_t), s));
    FrontendLaunch F{};
    F.frame = d_in.p;
    F.dtype = UWB_F64;
    F.m = static_cast<int64_t>(m);
    F.n = static_cast<int64_t>(n);
    F.work = d_work.as<double>();
    F.first_nonfinite = d_bad.as<unsigned long long>();
    F.window = c.mean_filter_window;
    F.mode = smooth ? 0 : 1;
    F.epsilon = c.normalization_epsilon;
    F.L = static_cast<int64_t>(L);
    F.first_bin = static_cast<int64_t>(first);
    F.kept = static_cast<int64_t>(kept);
    std::vector<double> wr, wi;
    cudaError_t fused = cudaErrorNotSupported;
    if (run_all) {
        twiddles(F.L, wr, wi);
        UWB_CUDA_TRY(d_wr.alloc(sizeof(double) * L, s));
        UWB_CUDA_TRY(d_wi.alloc(sizeof(double) * L, s));
        UWB_CUDA_TRY(cudaMemcpyAsync(d_wr.p, wr.data(), sizeof(double) * L, cudaMemcpyHostToDevice, s));
        UWB_CUDA_TRY(cudaMemcpyAsync(d_wi.p, wi.data(), sizeof(double) * L, cudaMemcpyHostToDevice, s));
        UWB_CUDA_TRY(d_band.alloc(sizeof(double) * m * kept, s));
        F.wr = d_wr.as<double>();
        F.wi = d_wi.as<double>();
        F.band = d_band.as<double>();
        fused = launch_frontend_fused(F, s); // whole front end in two kernels when it applies
        if (fused != cudaErrorNotSupported) UWB_CUDA_TRY(fused);
    }
    if (fused == cudaErrorNotSupported) {
        // the columns stage also runs on its own: it reports non-finite samples
        F.stage_mask = 3;
        UWB_CUDA_TRY(launch_frontend_columns(F, s));
        if (run_all) {
            F.stage_mask = 4 | 8 | 16;
            UWB_CUDA_TRY(launch_frontend_rows(F, s));
        }
    }
    uint64_t bad = ~0ull;
    UWB_CUDA_TRY(cudaMemcpyAsync(&bad, d_bad.p, sizeof(bad), cudaMemcpyDeviceToHost, s));
    UWB_CUDA_TRY(cudaStreamSynchronize(s));
    if (bad != ~0ull) return fail(UWB_INPUT_ERROR, "RadarFrame: non-finite sample");
    if (cfg_status) return fail(cfg_status, cfg_msg);
    if (stage_status) return fail(stage_status, stage_msg);

    // ---- CFAR stage on the band map ("cfar2d: " prefix, pipeline.cpp:269-273)
    if (band_freq)
        for (uint64_t k = 0; k < kept; ++k)
            band_freq[k] = static_cast<double>(first + k) * prf / static_cast<double>(L);
    if (range_axis)
        for (uint64_t r = 0; r < m; ++r) range_axis[r] = static_cast<double>(r) * 299792458.0 / (2.0 * fast_rate);
    if (band_power)
        UWB_CUDA_TRY(cudaMemcpyAsync(band_power, d_band.p, sizeof(double) * m * kept, cudaMemcpyDeviceToHost, s));
    *kept_out = kept;
    if (degenerate(c.cfar, m, kept))
        return fail(UWB_CONFIGURATION_ERROR, "cfar2d: " + degenerate_msg(c.cfar, m, kept));

    const uint64_t cells = m * kept;
    const std::vector<double> alpha = alpha_table_host(c.cfar);
    DevBuf d_alpha, d_mask, d_thr, d_dets, d_cnt, d_fb, d_bits, d_ws;
    UWB_CUDA_TRY(d_alpha.alloc(sizeof(double) * alpha.size(), s));
    UWB_CUDA_TRY(cudaMemcpyAsync(d_alpha.p, alpha.data(), sizeof(double) * alpha.size(), cudaMemcpyHostToDevice, s));
    UWB_CUDA_TRY(d_mask.alloc(cells, s));
    UWB_CUDA_TRY(d_thr.alloc(sizeof(double) * cells, s));
    UWB_CUDA_TRY(d_dets.alloc(sizeof(uwb_detection) * cells, s));
    UWB_CUDA_TRY(d_cnt.alloc(sizeof(uint64_t), s));
    UWB_CUDA_TRY(d_fb.alloc(sizeof(uint64_t) * 2, s));
    const uint64_t words = (kept + 31) / 32;
    UWB_CUDA_TRY(d_bits.alloc(sizeof(uint32_t) * words * m, s));
    uwb_map_batch b{};
    b.maps = d_band.p;
    b.dtype = UWB_F64;
    b.n_maps = 1;
    b.rows = m;
    b.cols = kept;
    b.ld = kept;
    b.map_stride = cells;
    uwb_cfar_outputs o{};
    o.mask_bits = d_bits.as<uint32_t>();
    o.words_per_row = words;
    o.mask_map_stride = words * m;
    o.mask_u8 = d_mask.as<uint8_t>();
    o.thresholds = d_thr.as<double>();
    o.dets = d_dets.as<uwb_detection>();
    o.det_capacity = cells;
    o.det_counts = d_cnt.as<uint64_t>();
    o.first_bad = d_fb.as<uint64_t>();
    const Plan P = make_plan(b, &c.cfar, UWB_SAT_GLOBAL, 0, static_cast<int64_t>(cells));
    UWB_CUDA_TRY(d_ws.alloc(P.total, s));
    const int backend = c.backend == UWB_NAIVE ? UWB_NAIVE : UWB_INTEGRAL;
    if (uwb_status st = dev_cfar(b, c.cfar, d_alpha.as<double>(), backend, UWB_SAT_GLOBAL, 0, o, d_ws.p, P.total, 0, s))
        return st;
    uint64_t cnt = 0, fb[2];
    UWB_CUDA_TRY(cudaMemcpyAsync(&cnt, d_cnt.p, sizeof(cnt), cudaMemcpyDeviceToHost, s));
    UWB_CUDA_TRY(cudaMemcpyAsync(fb, d_fb.p, sizeof(fb), cudaMemcpyDeviceToHost, s));
    UWB_CUDA_TRY(cudaStreamSynchronize(s));
    if (backend == UWB_INTEGRAL && fb[0] != ~0ull) {
        const int64_t r = static_cast<int64_t>(fb[0] / kept), cc = static_cast<int64_t>(fb[0] % kept);
        return fail(UWB_INPUT_ERROR, "cfar2d: build_sat: non-finite entry at (" + S(r) + ", " + S(cc) + ")", r, cc);
    }
    if (fb[1] != ~0ull) {
        const int64_t r = static_cast<int64_t>(fb[1] / kept), cc = static_cast<int64_t>(fb[1] % kept);
        return fail(UWB_INPUT_ERROR, "cfar2d: cfar2d: cell (" + S(r) + ", " + S(cc) + ") is not a finite non-negative power", r, cc);
    }
    *n_det = cnt;
    if (mask) UWB_CUDA_TRY(cudaMemcpyAsync(mask, d_mask.p, cells, cudaMemcpyDeviceToHost, s));
    if (thresholds) UWB_CUDA_TRY(cudaMemcpyAsync(thresholds, d_thr.p, sizeof(double) * cells, cudaMemcpyDeviceToHost, s));
    const uint64_t n_copy = std::min(cnt, det_capacity);
    if (dets && n_copy)
        UWB_CUDA_TRY(cudaMemcpyAsync(dets, d_dets.p, sizeof(uwb_detection) * n_copy, cudaMemcpyDeviceToHost, s));
    UWB_CUDA_TRY(cudaStreamSynchronize(s));
    if (cnt > det_capacity) return fail(UWB_CAPACITY_ERROR, "uwb_detect: detection buffer too small");
    return ok();
}

// ------------------------------------------------- host-buffer batch (e2e) ---

uwb_status uwb_host_cfar2d_batch(const uwb_map_batch* hb, const uwb_cfar_params* p, int32_t sat_mode,
                                 uint64_t slab_rows, uint32_t* mask_bits, uwb_detection* dets,
                                 uint64_t det_capacity, uint64_t* det_counts, uint64_t maps_per_chunk) {
    if (uwb_status s = check_batch(hb)) return s;
    if (uwb_status s = validate_params(*p)) return s;
    if (hb->rows == 0 || hb->cols == 0) return fail(UWB_DIMENSION_ERROR, "cfar2d: power map must be at least 1x1");
    if (degenerate(*p, hb->rows, hb->cols)) return fail(UWB_CONFIGURATION_ERROR, degenerate_msg(*p, hb->rows, hb->cols));
    if (uwb_status s = need_device()) return s;
    if (hb->ld != hb->cols || hb->map_stride != hb->rows * hb->cols)
        return fail(UWB_INVALID_ARGUMENT, "uwb_host_cfar2d_batch: host maps must be dense");
    const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(maps_per_chunk ? maps_per_chunk : 64, hb->n_maps));
    const size_t esz = hb->dtype == UWB_F32 ? 4 : 8;
    const uint64_t cells = hb->rows * hb->cols;
    const uint64_t words = (hb->cols + 31) / 32;
    const uint64_t mask_words = words * hb->rows;

    // Three engines, three streams: the copy-in stream streams chunks back to
    // back (the PCIe H2D link is the bound of this call), the compute stream runs
    // SAT+CFAR+sort per chunk in one workspace, the copy-out stream drains
    // results. kSlots input/output slots rotate; events order reuse.
    constexpr int kSlots = 3;
    struct Streams {
        cudaStream_t in = nullptr, comp = nullptr, out = nullptr;
        cudaEvent_t loaded[kSlots] = {}, done[kSlots] = {}, drained[kSlots] = {};
        ~Streams() {
            for (cudaStream_t x : {in, comp, out})
                if (x) cudaStreamSynchronize(x);
            for (int i = 0; i < kSlots; ++i)
                for (cudaEvent_t e : {loaded[i], done[i], drained[i]})
                    if (e) cudaEventDestroy(e);
            for (cudaStream_t x : {in, comp, out})
                if (x) cudaStreamDestroy(x);
        }
    } S;
    UWB_CUDA_TRY(cudaStreamCreateWithFlags(&S.in, cudaStreamNonBlocking));
    UWB_CUDA_TRY(cudaStreamCreateWithFlags(&S.comp, cudaStreamNonBlocking));
    UWB_CUDA_TRY(cudaStreamCreateWithFlags(&S.out, cudaStreamNonBlocking));
    for (int i = 0; i < kSlots; ++i) {
        UWB_CUDA_TRY(cudaEventCreateWithFlags(&S.loaded[i], cudaEventDisableTiming));
        UWB_CUDA_TRY(cudaEventCreateWithFlags(&S.done[i], cudaEventDisableTiming));
        UWB_CUDA_TRY(cudaEventCreateWithFlags(&S.drained[i], cudaEventDisableTiming));
    }
    struct Slot {
        DevBuf in, bits, dets, cnt, bad;
    } slots[kSlots];
    uwb_map_batch cb = *hb;
    cb.n_maps = chunk;
    const Plan P = make_plan(cb, p, sat_mode, slab_rows, static_cast<int64_t>(det_capacity));
    const std::vector<double> alpha = alpha_table_host(*p);
    DevBuf d_alpha, ws;
    struct Drain { // on every exit: copies finish before the buffers are freed on the compute stream
        const Streams& s;
        ~Drain() {
            cudaStreamSynchronize(s.in);
            cudaStreamSynchronize(s.out);
        }
    } drain{S};
    UWB_CUDA_TRY(d_alpha.alloc(sizeof(double) * alpha.size(), S.comp));
    UWB_CUDA_TRY(cudaMemcpyAsync(d_alpha.p, alpha.data(), sizeof(double) * alpha.size(), cudaMemcpyHostToDevice, S.comp));
    UWB_CUDA_TRY(ws.alloc(P.total, S.comp));
    for (auto& sl : slots) {
        UWB_CUDA_TRY(sl.in.alloc(esz * cells * chunk, S.comp));
        UWB_CUDA_TRY(sl.bits.alloc(sizeof(uint32_t) * mask_words * chunk, S.comp));
        UWB_CUDA_TRY(sl.dets.alloc(sizeof(uwb_detection) * std::max<uint64_t>(det_capacity, 1) * chunk, S.comp));
        UWB_CUDA_TRY(sl.cnt.alloc(sizeof(uint64_t) * chunk, S.comp));
        UWB_CUDA_TRY(sl.bad.alloc(sizeof(uint64_t) * 2 * chunk, S.comp));
    }
    // per-map first bad cells {non-finite, negative} (row-major index), read back
    // with the counts and reported as the reference's InputError below
    struct PinnedBad {
        uint64_t* p = nullptr;
        ~PinnedBad() {
            if (p) cudaFreeHost(p);
        }
    } bad;
    UWB_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&bad.p), sizeof(uint64_t) * 2 * hb->n_maps));
    UWB_CUDA_TRY(cudaStreamSynchronize(S.comp)); // allocations visible to the other streams
    uwb_status result = UWB_OK;
    for (uint64_t m0 = 0, k = 0; m0 < hb->n_maps; m0 += chunk, ++k) {
        const int i = static_cast<int>(k % kSlots);
        const uint64_t nm = std::min(chunk, hb->n_maps - m0);
        Slot& sl = slots[i];
        const char* src = static_cast<const char*>(hb->maps) + esz * cells * m0;
        if (k >= kSlots) UWB_CUDA_TRY(cudaStreamWaitEvent(S.in, S.done[i], 0)); // input slot consumed
        UWB_CUDA_TRY(cudaMemcpyAsync(sl.in.p, src, esz * cells * nm, cudaMemcpyHostToDevice, S.in));
        UWB_CUDA_TRY(cudaEventRecord(S.loaded[i], S.in));
        UWB_CUDA_TRY(cudaStreamWaitEvent(S.comp, S.loaded[i], 0));
        if (k >= kSlots) UWB_CUDA_TRY(cudaStreamWaitEvent(S.comp, S.drained[i], 0)); // output slot drained
        uwb_map_batch db = cb;
        db.maps = sl.in.p;
        db.n_maps = nm;
        uwb_cfar_outputs o{};
        o.mask_bits = sl.bits.as<uint32_t>();
        o.words_per_row = words;
        o.mask_map_stride = mask_words;
        o.dets = sl.dets.as<uwb_detection>();
        o.det_capacity = det_capacity;
        o.det_counts = sl.cnt.as<uint64_t>();
        o.first_bad = sl.bad.as<uint64_t>();
        if (uwb_status s2 = dev_cfar(db, *p, d_alpha.as<double>(), UWB_INTEGRAL, sat_mode, slab_rows, o, ws.p,
                                     P.total, 0, S.comp))
            return s2;
        UWB_CUDA_TRY(cudaEventRecord(S.done[i], S.comp));
        UWB_CUDA_TRY(cudaStreamWaitEvent(S.out, S.done[i], 0));
        if (mask_bits)
            UWB_CUDA_TRY(cudaMemcpyAsync(mask_bits + mask_words * m0, sl.bits.p, sizeof(uint32_t) * mask_words * nm,
                                         cudaMemcpyDeviceToHost, S.out));
        if (dets && det_capacity)
            UWB_CUDA_TRY(cudaMemcpyAsync(dets + det_capacity * m0, sl.dets.p, sizeof(uwb_detection) * det_capacity * nm,
                                         cudaMemcpyDeviceToHost, S.out));
        UWB_CUDA_TRY(cudaMemcpyAsync(det_counts + m0, sl.cnt.p, sizeof(uint64_t) * nm, cudaMemcpyDeviceToHost, S.out));
        UWB_CUDA_TRY(cudaMemcpyAsync(bad.p + 2 * m0, sl.bad.p, sizeof(uint64_t) * 2 * nm, cudaMemcpyDeviceToHost, S.out));
        UWB_CUDA_TRY(cudaEventRecord(S.drained[i], S.out));
    }
    UWB_CUDA_TRY(cudaStreamSynchronize(S.out));
    UWB_CUDA_TRY(cudaStreamSynchronize(S.comp));
    // the first map with a bad cell raises what cfar2d_integral raises on it:
    // build_sat's non-finite check first (sat.cpp:28-32), then run_cfar's
    // power-map check (cfar.cpp:85-92); its outputs are not meaningful
    for (uint64_t i = 0; i < hb->n_maps; ++i) {
        const uint64_t nf = bad.p[2 * i], neg = bad.p[2 * i + 1];
        if (nf == ~0ull && neg == ~0ull) continue;
        const uint64_t idx = nf != ~0ull ? nf : neg;
        const int64_t r = static_cast<int64_t>(idx / hb->cols), c = static_cast<int64_t>(idx % hb->cols);
        const std::string at = "(" + std::to_string(r) + ", " + std::to_string(c) + ")";
        if (nf != ~0ull) return fail(UWB_INPUT_ERROR, "build_sat: non-finite entry at " + at, r, c);
        return fail(UWB_INPUT_ERROR, "cfar2d: cell " + at + " is not a finite non-negative power", r, c);
    }
    for (uint64_t i = 0; i < hb->n_maps; ++i)
        if (det_counts[i] > det_capacity) result = fail(UWB_CAPACITY_ERROR, "uwb_host_cfar2d_batch: detection buffer too small");
    return result ? result : ok();
}

// ---- batched device detect() ------------------------------

static uint64_t detect_ws_layout(uint64_t n_rec, uint64_t m, uint64_t n, uint64_t L, const Plan& P,
                                 size_t* off_work, size_t* off_tw, size_t* off_bad, size_t* off_cfar) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += static_cast<size_t>(round_up(static_cast<int64_t>(bytes), 256));
        return o;
    };
    *off_work = take(sizeof(double) * n_rec * m * n);
    *off_tw = take(sizeof(double) * 2 * L);
    *off_bad = take(sizeof(uint64_t) * n_rec);
    *off_cfar = take(P.total);
    return off;
}

uint64_t uwb_dev_detect_batch_workspace(uint64_t n_records, uint64_t m, uint64_t n, double prf,
                                        const uwb_pipeline_config* cfg, uint64_t det_capacity) {
    const DetectPlan D = detect_plan(m, n, prf, *cfg);
    if (!D.ok()) return 0;
    uwb_map_batch b{};
    b.dtype = UWB_F64;
    b.n_maps = n_records;
    b.rows = m;
    b.cols = D.kept;
    b.ld = D.kept;
    b.map_stride = m * D.kept;
    const Plan P = make_plan(b, &cfg->cfar, UWB_SAT_GLOBAL, 0, static_cast<int64_t>(det_capacity));
    size_t a, t, bd, cf;
    return detect_ws_layout(n_records, m, n, D.L, P, &a, &t, &bd, &cf);
}

uwb_status uwb_dev_detect_batch(const void* records, int32_t dtype, uint64_t n_records, uint64_t m, uint64_t n,
                                double fast_rate, double prf, const uwb_pipeline_config* cfg, double* band,
                                uint64_t* kept_out, const uwb_cfar_outputs* out, void* workspace,
                                uint64_t ws_bytes, uint32_t flags, void* stream) {
    if (kept_out) *kept_out = 0;
    if (!cfg || !out || (!records && n_records)) return fail(UWB_INVALID_ARGUMENT, "uwb: null argument");
    if (dtype != UWB_F32 && dtype != UWB_F64) return fail(UWB_INVALID_ARGUMENT, "uwb: bad dtype");
    if (m < 2 || n < 2)
        return fail(UWB_DIMENSION_ERROR, "RadarFrame: need at least 2x2 samples, got " + S(m) + "x" + S(n));
    if (!(fast_rate > 0.0) || !(prf > 0.0))
        return fail(UWB_PARAMETER_ERROR, "RadarFrame: fast_rate and prf must be positive");
    const DetectPlan D = detect_plan(m, n, prf, *cfg);
    if (D.cfg_status) return fail(D.cfg_status, D.cfg_msg);
    if (D.stage_status) return fail(D.stage_status, D.stage_msg);
    if (D.L > 8192) return fail(UWB_INVALID_ARGUMENT, "uwb: fft_length > 8192 not supported on the device path");
    if (degenerate(cfg->cfar, m, D.kept))
        return fail(UWB_CONFIGURATION_ERROR, "cfar2d: " + degenerate_msg(cfg->cfar, m, D.kept));
    if (uwb_status st = need_device()) return st;
    if (kept_out) *kept_out = D.kept;
    if (n_records == 0) return ok();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uwb_map_batch b{};
    b.maps = band;
    b.dtype = UWB_F64;
    b.n_maps = n_records;
    b.rows = m;
    b.cols = D.kept;
    b.ld = D.kept;
    b.map_stride = m * D.kept;
    const Plan P = make_plan(b, &cfg->cfar, UWB_SAT_GLOBAL, 0, static_cast<int64_t>(out->det_capacity));
    size_t off_work, off_tw, off_bad, off_cfar;
    const uint64_t need = detect_ws_layout(n_records, m, n, D.L, P, &off_work, &off_tw, &off_bad, &off_cfar);
    if (ws_bytes < need) return fail(UWB_INVALID_ARGUMENT, "uwb: workspace too small (need " + S(need) + ")");
    char* ws = static_cast<char*>(workspace);
    // twiddles (host, identical to the oracle's FFT provider) and the alpha table
    std::vector<double> wr, wi;
    twiddles(static_cast<int64_t>(D.L), wr, wi);
    std::vector<double> tw(wr);
    tw.insert(tw.end(), wi.begin(), wi.end());
    const std::vector<double> alpha = alpha_table_host(cfg->cfar);
    DevBuf d_alpha;
    UWB_CUDA_TRY(d_alpha.alloc(sizeof(double) * alpha.size(), s));
    UWB_CUDA_TRY(cudaMemcpyAsync(d_alpha.p, alpha.data(), sizeof(double) * alpha.size(), cudaMemcpyHostToDevice, s));
    UWB_CUDA_TRY(cudaMemcpyAsync(ws + off_tw, tw.data(), sizeof(double) * tw.size(), cudaMemcpyHostToDevice, s));
    UWB_CUDA_TRY(cudaMemsetAsync(ws + off_bad, 0xff, sizeof(uint64_t) * n_records, s));
    // front end (pipeline.cpp:246-268): columns, then rows straight into the band maps
    FrontendLaunch F{};
    F.frame = records;
    F.dtype = dtype;
    F.m = static_cast<int64_t>(m);
    F.n = static_cast<int64_t>(n);
    F.n_rec = static_cast<int64_t>(n_records);
    F.work = reinterpret_cast<double*>(ws + off_work);
    F.first_nonfinite = reinterpret_cast<unsigned long long*>(ws + off_bad);
    F.window = cfg->mean_filter_window;
    F.mode = cfg->mean_filter_mode == 0 ? 0 : 1;
    F.epsilon = cfg->normalization_epsilon;
    F.L = static_cast<int64_t>(D.L);
    F.wr = reinterpret_cast<const double*>(ws + off_tw);
    F.wi = F.wr + D.L;
    F.first_bin = static_cast<int64_t>(D.first);
    F.kept = static_cast<int64_t>(D.kept);
    F.band = band;
    // flags bit 8 (test hook): the general front-end kernels (same results)
    NvtxRange fe("uwb.detect_batch");
    const cudaError_t fused = (flags & 256u) ? cudaErrorNotSupported : launch_frontend_fused(F, s);
    if (fused == cudaErrorNotSupported) {
        F.stage_mask = 3;
        UWB_CUDA_TRY(launch_frontend_columns(F, s));
        F.stage_mask = 4 | 8 | 16;
        UWB_CUDA_TRY(launch_frontend_rows(F, s));
    } else {
        UWB_CUDA_TRY(fused);
    }
    // CFAR over the band maps (pipeline.cpp:269-273)
    const int backend = cfg->backend == UWB_NAIVE ? UWB_NAIVE : UWB_INTEGRAL;
    if (uwb_status st = dev_cfar(b, cfg->cfar, d_alpha.as<double>(), backend, UWB_SAT_GLOBAL, 0, *out,
                                 ws + off_cfar, P.total, flags & ~(4u | 256u), s))
        return st;
    // a record's first non-finite sample (row-major over its m x n frame) is its
    // entry 0 of first_bad (RadarFrame::validate, pipeline.cpp:27-38)
    if (out->first_bad)
        UWB_CUDA_TRY(cudaMemcpy2DAsync(out->first_bad, 2 * sizeof(uint64_t), ws + off_bad, sizeof(uint64_t),
                                       sizeof(uint64_t), n_records, cudaMemcpyDeviceToDevice, s));
    return ok();
}

// ---- RFRM frame files (frame_io.cpp:69-122) ---------------------------------

uwb_status uwb_rfrm_parse(const void* file_bytes, uint64_t len, uwb_rfrm_info* info) {
    if (!info || (!file_bytes && len)) return fail(UWB_INVALID_ARGUMENT, "uwb: null argument");
    const unsigned char* b = static_cast<const unsigned char*>(file_bytes);
    if (len < 4 || std::memcmp(b, "RFRM", 4) != 0) return fail(UWB_FORMAT_ERROR, "frame file: bad magic, expected \"RFRM\"");
    uint64_t pos = 4;
    auto get = [&](int bytes, uint64_t& v) { // little-endian field; false when the header is cut short
        if (pos + static_cast<uint64_t>(bytes) > len) return false;
        v = 0;
        for (int i = 0; i < bytes; ++i) v |= static_cast<uint64_t>(b[pos + i]) << (8 * i);
        pos += static_cast<uint64_t>(bytes);
        return true;
    };
    uint64_t version = 0, m = 0, n = 0, fr = 0, pr = 0;
    if (!get(2, version)) return fail(UWB_FORMAT_ERROR, "frame file: truncated header");
    if (version != 1) return fail(UWB_FORMAT_ERROR, "frame file: unsupported version " + S(version));
    if (!get(4, m) || !get(4, n) || !get(8, fr) || !get(8, pr))
        return fail(UWB_FORMAT_ERROR, "frame file: truncated header");
    if (m < 2 || n < 2)
        return fail(UWB_FORMAT_ERROR, "frame file: header declares " + S(m) + "x" + S(n) + " frame, need at least 2x2");
    double fast_rate, prf;
    std::memcpy(&fast_rate, &fr, 8);
    std::memcpy(&prf, &pr, 8);
    const uint64_t payload = m * n * 4;
    if (len - pos < payload)
        return fail(UWB_FORMAT_ERROR, "frame file: truncated payload, expected " + S(payload) + " bytes");
    if (len - pos > payload) return fail(UWB_FORMAT_ERROR, "frame file: trailing bytes after payload");
    // RadarFrame::validate (pipeline.cpp:27-38); finiteness is checked on the device
    if (!(fast_rate > 0.0) || !(prf > 0.0))
        return fail(UWB_FORMAT_ERROR, "frame file: RadarFrame: fast_rate and prf must be positive");
    info->m_samples = static_cast<uint32_t>(m);
    info->n_traces = static_cast<uint32_t>(n);
    info->fast_rate = fast_rate;
    info->prf = prf;
    info->payload_offset = pos;
    info->payload_bytes = payload;
    return ok();
}

uwb_status uwb_dev_rfrm_to_frames(const float* payload, uint64_t n_rec, uint64_t m, uint64_t n, int32_t out_dtype,
                                  void* frames, uint64_t* first_nonfinite, void* stream) {
    if ((!payload || !frames) && n_rec) return fail(UWB_INVALID_ARGUMENT, "uwb: null argument");
    if (out_dtype != UWB_F32 && out_dtype != UWB_F64) return fail(UWB_INVALID_ARGUMENT, "uwb: bad dtype");
    if (uwb_status st = need_device()) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (first_nonfinite && n_rec) UWB_CUDA_TRY(cudaMemsetAsync(first_nonfinite, 0xff, sizeof(uint64_t) * n_rec, s));
    UWB_CUDA_TRY(launch_rfrm_transpose(payload, static_cast<int64_t>(n_rec), static_cast<int64_t>(m),
                                       static_cast<int64_t>(n), out_dtype, frames,
                                       reinterpret_cast<unsigned long long*>(first_nonfinite), s));
    return ok();
}

uint64_t uwb_kernel_launches(void) { return g_kernel_launches.load(); }

int32_t uwb_dev_phase_ms4(float* out, int32_t max_calls) {
    std::lock_guard<std::mutex> lk(g_phase.mu);
    const int n = std::min<int>(g_phase.used, max_calls);
    for (int i = 0; i < n; ++i) {
        cudaEvent_t* e = &g_phase.ev[static_cast<size_t>(i) * PhaseRing::kEv];
        cudaEventSynchronize(e[4]);
        for (int k = 0; k < 4; ++k) cudaEventElapsedTime(&out[4 * i + k], e[k], e[k + 1]);
    }
    g_phase.used = 0;
    return n;
}

int32_t uwb_dev_phase_ms(float* out, int32_t max_calls) {
    std::vector<float> q(static_cast<size_t>(std::max(0, max_calls)) * 4);
    const int n = uwb_dev_phase_ms4(q.data(), max_calls);
    for (int i = 0; i < n; ++i) { // {sat, cfar (certify + resolve), sort}
        out[3 * i + 0] = q[4 * i + 1];
        out[3 * i + 1] = q[4 * i + 0] + q[4 * i + 2];
        out[3 * i + 2] = q[4 * i + 3];
    }
    return n;
}

void* uwb_host_alloc(uint64_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
    return p;
}

void uwb_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

} // extern "C"
