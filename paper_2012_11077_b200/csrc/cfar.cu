// Kernel (d) fallbacks, the naive backend and the detection sort.
//
// launch_cfar_integral() uses the shared-memory ring kernel of cfar_ring.cu and
// falls back to cfar_integral_kernel below (taps read straight from the
// global table through L1) when the rings do not fit in shared memory.
//
// Per cell (cfar.cpp:115-127): clamped outer and guard rectangles, their n_train,
// the two four-tap region sums in the association of sat.hpp:32-33,
//     RS = (t[r0][c0] + t[r1+1][c1+1]) - (t[r0][c1+1] + t[r1+1][c0]),
// sum = RS(outer) - RS(guard), mean = sum / n (IEEE division), T = alpha[n] * mean
// with alpha tabulated on the host by the same libm pow, and mask = cut > T
// (ties are H0). Same operations in the same order => bit-identical thresholds.
// Detections are compacted with one warp-aggregated atomicAdd per warp-row into
// the map's list, which is then sorted (value desc, row asc, col asc,
// cfar.cpp:170-173); the final order is independent of the atomic order.
#include <cfloat>

#include "cfar_common.cuh"

namespace uwb {

cudaError_t launch_cfar_ring(const CfarLaunch& L, int dtype, cudaStream_t stream);

namespace {

constexpr int kCfarThreads = 128;
constexpr int kCfarRowChunk = 32;

template <typename T>
__device__ __forceinline__ double load_cell(const T* p) {
    return static_cast<double>(__ldg(p));
}

__device__ __forceinline__ double tap(const double* t, int64_t ld, int64_t i, int64_t j) {
    return __ldg(t + i * ld + kTabShift + j);
}

template <typename T>
__device__ __forceinline__ void cfar_integral_tile(const CfarLaunch& L, const int64_t job) {
    const int64_t map = job / L.geo.n_slabs;
    const int64_t slab = job % L.geo.n_slabs;
    const int col_tile = static_cast<int>(blockIdx.x % L.col_tiles);
    const int chunk = static_cast<int>(blockIdx.x / L.col_tiles);
    const int c = col_tile * kCfarThreads + static_cast<int>(threadIdx.x);
    const int cols = static_cast<int>(L.cols), rows = static_cast<int>(L.geo.rows);
    const bool col_ok = c < cols;
    const int ra = static_cast<int>(L.geo.owned_begin(slab)) + chunk * kCfarRowChunk;
    const int rb = min(ra + kCfarRowChunk, static_cast<int>(L.geo.owned_end(slab)));
    if (ra >= rb) return;
    const int trow0 = static_cast<int>(L.geo.table_begin(slab));
    const int64_t band = col_ok ? L.geo.band_of(c) : 0; // band tables: local columns
    const double* tab = L.table + (job * L.geo.n_bands + band) * L.table_stride - L.geo.band_c0(band);
    const int64_t ld = L.table_ld;
    const T* cut_base = static_cast<const T*>(L.maps) + map * L.map_stride;

    const int oc0 = clamp_lo32(c, L.hc), oc1 = clamp_hi32(c, L.hc, cols);
    const int gc0 = clamp_lo32(c, L.gc), gc1 = clamp_hi32(c, L.gc, cols);
    const int ow = oc1 - oc0 + 1, gw = gc1 - gc0 + 1;

    for (int r = ra; r < rb; ++r) {
        bool hit = false;
        double v = 0.0, thr = 0.0;
        if (col_ok) {
            const int or0 = clamp_lo32(r, L.hr), or1 = clamp_hi32(r, L.hr, rows);
            const int gr0 = clamp_lo32(r, L.gr), gr1 = clamp_hi32(r, L.gr, rows);
            const int n = (or1 - or0 + 1) * ow - (gr1 - gr0 + 1) * gw;
            const int ti0 = or0 - trow0, ti1 = or1 + 1 - trow0;
            const int gi0 = gr0 - trow0, gi1 = gr1 + 1 - trow0;
            const double rs_o = dsub(dadd(tap(tab, ld, ti0, oc0), tap(tab, ld, ti1, oc1 + 1)),
                                     dadd(tap(tab, ld, ti0, oc1 + 1), tap(tab, ld, ti1, oc0)));
            const double rs_g = dsub(dadd(tap(tab, ld, gi0, gc0), tap(tab, ld, gi1, gc1 + 1)),
                                     dadd(tap(tab, ld, gi0, gc1 + 1), tap(tab, ld, gi1, gc0)));
            const double sum = dsub(rs_o, rs_g);
            const double mean = ddiv(sum, static_cast<double>(n));
            thr = dmul(__ldg(L.alpha + n), mean);
            v = load_cell(cut_base + (r - L.geo.buf_row0) * L.ld + c);
            hit = v > thr; // cfar.cpp:125, ties -> H0
            if (v < 0.0)
                report_min(L.first_bad + 2 * map + 1, static_cast<unsigned long long>(static_cast<int64_t>(r) * cols + c));
        }
        emit_cells(L, map, r, c, col_ok, hit, v, thr);
    }
}

template <typename T>
__global__ void __launch_bounds__(kCfarThreads)
cfar_integral_kernel(CfarLaunch L) {
    if (!L.flagged_count) {
        cfar_integral_tile<T>(L, blockIdx.y);
        return;
    }
    // certified path's exact fallback: a short grid strides over the jobs of
    // the maps the certificate flagged (compacted by cert_resolve_kernel;
    // usually none)
    const int64_t n = static_cast<int64_t>(*L.flagged_count) * L.geo.n_slabs;
    for (int64_t i = blockIdx.y; i < n; i += gridDim.y)
        cfar_integral_tile<T>(L, static_cast<int64_t>(L.flagged_maps[i / L.geo.n_slabs]) * L.geo.n_slabs +
                                     i % L.geo.n_slabs);
}

// cfar.cpp:200-216: explicit ring loop, row-major accumulation order.
template <typename T>
__global__ void __launch_bounds__(kCfarThreads)
cfar_naive_kernel(CfarLaunch L) {
    const int64_t map = blockIdx.y;
    const int col_tile = static_cast<int>(blockIdx.x % L.col_tiles);
    const int chunk = static_cast<int>(blockIdx.x / L.col_tiles);
    const int c = col_tile * kCfarThreads + static_cast<int>(threadIdx.x);
    const int cols = static_cast<int>(L.cols), rows = static_cast<int>(L.geo.rows);
    const bool col_ok = c < cols;
    const int ra = chunk * kCfarRowChunk;
    const int rb = min(ra + kCfarRowChunk, rows);
    if (ra >= rb) return;
    const T* m = static_cast<const T*>(L.maps) + map * L.map_stride;
    const int oc0 = clamp_lo32(c, L.hc), oc1 = clamp_hi32(c, L.hc, cols);
    const int gc0 = clamp_lo32(c, L.gc), gc1 = clamp_hi32(c, L.gc, cols);
    const int ow = oc1 - oc0 + 1, gw = gc1 - gc0 + 1;
    for (int r = ra; r < rb; ++r) {
        bool hit = false;
        double v = 0.0, thr = 0.0;
        if (col_ok) {
            const int or0 = clamp_lo32(r, L.hr), or1 = clamp_hi32(r, L.hr, rows);
            const int gr0 = clamp_lo32(r, L.gr), gr1 = clamp_hi32(r, L.gr, rows);
            const int n = (or1 - or0 + 1) * ow - (gr1 - gr0 + 1) * gw;
            double sum = 0.0;
            for (int rr = or0; rr <= or1; ++rr) {
                const bool guard_row = rr >= gr0 && rr <= gr1;
                const T* row = m + static_cast<int64_t>(rr) * L.ld;
                for (int cc = oc0; cc <= oc1; ++cc) {
                    if (guard_row && cc >= gc0 && cc <= gc1) continue;
                    sum = dadd(sum, load_cell(row + cc));
                }
            }
            const double mean = ddiv(sum, static_cast<double>(n));
            thr = dmul(__ldg(L.alpha + n), mean);
            v = load_cell(m + static_cast<int64_t>(r) * L.ld + c);
            hit = v > thr;
            if (!isfinite(v) || v < 0.0)
                report_min(L.first_bad + 2 * map + 1, static_cast<unsigned long long>(static_cast<int64_t>(r) * cols + c));
        }
        emit_cells(L, map, r, c, col_ok, hit, v, thr);
    }
}

// ---------------------------------------------------------------- sorting ---

__device__ __forceinline__ bool before(const uwb_detection& a, const uwb_detection& b) {
    // std::tie(b.value, a.row, a.col) < std::tie(a.value, b.row, b.col)
    if (b.value < a.value) return true;
    if (a.value < b.value) return false;
    if (a.row != b.row) return a.row < b.row;
    return a.col < b.col;
}

constexpr int kSortThreads = 1024;
constexpr int kSortRun = 2048; // entries sorted in shared memory at once

__device__ uwb_detection sentinel() {
    uwb_detection s;
    s.row = ~0ull;
    s.col = ~0ull;
    s.value = -DBL_MAX;
    s.threshold = 0.0;
    return s;
}

// Bitonic sort of up to kSortRun entries in shared memory.
__device__ void smem_bitonic(uwb_detection* s, int n_pow2) {
    for (int k = 2; k <= n_pow2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const bool asc = (i & k) == 0;
                    uwb_detection a = s[i], b = s[p];
                    const bool swap = asc ? before(b, a) : before(a, b);
                    if (swap) {
                        s[i] = b;
                        s[p] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__device__ int merge_path(const uwb_detection* a, int na, const uwb_detection* b, int nb, int diag) {
    int lo = max(0, diag - nb), hi = min(diag, na);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (!before(b[diag - 1 - mid], a[mid])) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Phase 1 of the detection sort: CTA (map, y) sorts run y of the map's list
// (kSortRun entries) in shared memory, so the runs of one long list sort in parallel.
__global__ void __launch_bounds__(kSortThreads)
sort_runs_kernel(uwb_detection* dets, int64_t cap, const unsigned long long* counts) {
    extern __shared__ uwb_detection smem_det[];
    const int64_t map = blockIdx.x;
    const int64_t count = imin(static_cast<int64_t>(counts[map]), cap);
    const int64_t base = static_cast<int64_t>(blockIdx.y) * kSortRun;
    if (count <= 1 || base >= count) return;
    uwb_detection* src = dets + map * cap;
    const int n = static_cast<int>(imin(kSortRun, count - base));
    int p2 = 1;
    while (p2 < n) p2 <<= 1;
    for (int i = threadIdx.x; i < p2; i += blockDim.x) smem_det[i] = i < n ? src[base + i] : sentinel();
    __syncthreads();
    smem_bitonic(smem_det, p2);
    for (int i = threadIdx.x; i < n; i += blockDim.x) src[base + i] = smem_det[i];
}

// Phase 2: merge passes (merge path) over the sorted runs, one CTA per map
// (runs_sorted = false: the CTA also sorts the runs itself, one after another).
__global__ void __launch_bounds__(kSortThreads)
sort_detections_kernel(uwb_detection* dets, int64_t cap, const unsigned long long* counts,
                       uwb_detection* scratch, bool runs_sorted) {
    extern __shared__ uwb_detection smem_det[];
    const int64_t map = blockIdx.x;
    const int64_t count = imin(static_cast<int64_t>(counts[map]), cap);
    if (count <= 1 || (runs_sorted && count <= kSortRun)) return;
    uwb_detection* src = dets + map * cap;
    uwb_detection* alt = scratch ? scratch + map * cap : nullptr;

    // 1. sort runs of kSortRun in shared memory
    for (int64_t base = 0; !runs_sorted && base < count; base += kSortRun) {
        const int n = static_cast<int>(imin(kSortRun, count - base));
        int p2 = 1;
        while (p2 < n) p2 <<= 1;
        for (int i = threadIdx.x; i < p2; i += blockDim.x) smem_det[i] = i < n ? src[base + i] : sentinel();
        __syncthreads();
        smem_bitonic(smem_det, p2);
        for (int i = threadIdx.x; i < n; i += blockDim.x) src[base + i] = smem_det[i];
        __syncthreads();
    }
    if (count <= kSortRun || alt == nullptr) return;

    // 2. merge passes (merge path), ping-pong between src and alt
    constexpr int kItems = 8;
    uwb_detection* in = src;
    uwb_detection* out = alt;
    for (int64_t width = kSortRun; width < count; width *= 2) {
        for (int64_t k0 = static_cast<int64_t>(threadIdx.x) * kItems; k0 < count;
             k0 += static_cast<int64_t>(blockDim.x) * kItems) {
            const int64_t base = (k0 / (2 * width)) * (2 * width);
            const int64_t a0 = base, a1 = imin(base + width, count);
            const int64_t b0 = a1, b1 = imin(base + 2 * width, count);
            const int na = static_cast<int>(a1 - a0), nb = static_cast<int>(b1 - b0);
            const int diag = static_cast<int>(k0 - base);
            int i = merge_path(in + a0, na, in + b0, nb, diag);
            int j = diag - i;
            const int64_t kend = imin(k0 + kItems, b1);
            for (int64_t k = k0; k < kend; ++k) {
                const bool take_a = i < na && (j >= nb || !before(in[b0 + j], in[a0 + i]));
                out[k] = take_a ? in[a0 + i++] : in[b0 + j++];
            }
        }
        __syncthreads();
        uwb_detection* t = in;
        in = out;
        out = t;
    }
    if (in != src)
        for (int64_t i = threadIdx.x; i < count; i += blockDim.x) src[i] = in[i];
}

// Phase 2 for few long lists: one merge pass over every list, CTA (x, map)
// producing output entries [x * kMergeTile, +kMergeTile) of the map's merged
// pairs of width-`width` runs (kMergeTile divides 2 * width). The CTA finds its
// input ranges by two merge-path searches, stages them in shared memory and
// merges kItems per thread there. A list needs P = ceil(log2(count / kSortRun))
// passes; pass q >= P does nothing, except that an odd P ends in the scratch
// buffer and pass P (reading it, width >= count) copies the list back.
constexpr int kMergeTile = 2048;
constexpr int kMergeThreads = 256;
__global__ void __launch_bounds__(kMergeThreads)
merge_pass_kernel(const uwb_detection* in_all, uwb_detection* out_all, int64_t cap,
                  const unsigned long long* counts, int64_t width, int q) {
    extern __shared__ uwb_detection smem_det[];
    __shared__ int split[2];
    const int64_t map = blockIdx.y;
    const int64_t count = imin(static_cast<int64_t>(counts[map]), cap);
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kMergeTile;
    if (count <= kSortRun || t0 >= count) return; // short lists stay sorted in place
    int passes = 0;
    for (int64_t w = kSortRun; w < count; w *= 2) ++passes;
    if (q > passes || (q == passes && passes % 2 == 0)) return;
    const uwb_detection* in = in_all + map * cap;
    uwb_detection* out = out_all + map * cap;
    const int64_t base = (t0 / (2 * width)) * (2 * width);
    const int64_t a0 = base, a1 = imin(base + width, count);
    const int64_t b0 = a1, b1 = imin(base + 2 * width, count);
    const int na = static_cast<int>(a1 - a0), nb = static_cast<int>(b1 - b0);
    const int d0 = static_cast<int>(t0 - base);
    const int d1 = min(d0 + kMergeTile, na + nb);
    if (threadIdx.x == 0) split[0] = merge_path(in + a0, na, in + b0, nb, d0);
    if (threadIdx.x == 32) split[1] = merge_path(in + a0, na, in + b0, nb, d1);
    __syncthreads();
    const int i0 = split[0], j0 = d0 - split[0];
    const int la = split[1] - i0, lb = (d1 - split[1]) - j0;
    for (int k = threadIdx.x; k < la + lb; k += blockDim.x)
        smem_det[k] = k < la ? in[a0 + i0 + k] : in[b0 + j0 + (k - la)];
    __syncthreads();
    constexpr int kItems = kMergeTile / kMergeThreads;
    const int k0 = static_cast<int>(threadIdx.x) * kItems;
    if (k0 >= la + lb) return;
    const uwb_detection* sa = smem_det;
    const uwb_detection* sb = smem_det + la;
    int i = merge_path(sa, la, sb, lb, k0);
    int j = k0 - i;
    const int kend = min(k0 + kItems, la + lb);
    for (int k = k0; k < kend; ++k) {
        const bool take_a = i < la && (j >= lb || !before(sb[j], sa[i]));
        out[t0 + k] = take_a ? sa[i++] : sb[j++];
    }
}

CfarLaunch grid_shape(const CfarLaunch& L0, dim3& grid) {
    CfarLaunch L = L0;
    L.col_tiles = (L.cols + kCfarThreads - 1) / kCfarThreads;
    L.row_chunks = (L.geo.slab_rows + kCfarRowChunk - 1) / kCfarRowChunk;
    grid = dim3(static_cast<unsigned>(L.col_tiles * L.row_chunks), static_cast<unsigned>(L.n_jobs), 1);
    return L;
}

} // namespace

cudaError_t launch_cfar_integral(const CfarLaunch& L0, int dtype, cudaStream_t stream) {
    if (L0.n_jobs == 0 || L0.cols == 0 || L0.geo.rows == 0) return cudaSuccess;
    const cudaError_t e = launch_cfar_ring(L0, dtype, stream);
    if (e != cudaErrorNotSupported) return e;
    dim3 grid;
    const CfarLaunch L = grid_shape(L0, grid);
    ++g_kernel_launches;
    if (dtype == UWB_F32) cfar_integral_kernel<float><<<grid, kCfarThreads, 0, stream>>>(L);
    else cfar_integral_kernel<double><<<grid, kCfarThreads, 0, stream>>>(L);
    return cudaGetLastError();
}

// The certified path's exact fallback over the flagged maps (L.flagged_maps,
// *L.flagged_count, written on the device): a grid of at most kFilteredJobs job
// rows striding over them, so a batch with nothing flagged costs one small
// launch (the ring kernel's full grid of early-exiting CTAs took ~0.13 ms for
// 4096 maps).
cudaError_t launch_cfar_integral_filtered(const CfarLaunch& L0, int dtype, cudaStream_t stream) {
    if (L0.n_jobs == 0 || L0.cols == 0 || L0.geo.rows == 0) return cudaSuccess;
    constexpr int64_t kFilteredJobs = 8;
    dim3 grid;
    const CfarLaunch L = grid_shape(L0, grid);
    grid.y = static_cast<unsigned>(L.n_jobs < kFilteredJobs ? L.n_jobs : kFilteredJobs);
    ++g_kernel_launches;
    if (dtype == UWB_F32) cfar_integral_kernel<float><<<grid, kCfarThreads, 0, stream>>>(L);
    else cfar_integral_kernel<double><<<grid, kCfarThreads, 0, stream>>>(L);
    return cudaGetLastError();
}

cudaError_t launch_cfar_naive(const CfarLaunch& L0, int dtype, cudaStream_t stream) {
    if (L0.n_jobs == 0 || L0.cols == 0 || L0.geo.rows == 0) return cudaSuccess;
    dim3 grid;
    const CfarLaunch L = grid_shape(L0, grid);
    ++g_kernel_launches;
    if (dtype == UWB_F32) cfar_naive_kernel<float><<<grid, kCfarThreads, 0, stream>>>(L);
    else cfar_naive_kernel<double><<<grid, kCfarThreads, 0, stream>>>(L);
    return cudaGetLastError();
}

cudaError_t launch_sort_detections(uwb_detection* dets, int64_t cap, const unsigned long long* counts,
                                   int64_t n_maps, uwb_detection* scratch, cudaStream_t stream) {
    if (n_maps == 0 || cap <= 1) return cudaSuccess;
    const size_t smem = sizeof(uwb_detection) * kSortRun;
    cudaError_t e = cudaFuncSetAttribute(sort_detections_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int64_t runs = (cap + kSortRun - 1) / kSortRun;
    if (runs > 1 && runs <= 8 && n_maps <= 16 && scratch) {
        // a few lists of modest capacity (single-map calls): one launch, one CTA per
        // list sorting its runs and merging them; a short list (the usual case) is one
        // bitonic sort, and the call saves the 2-4 launches of the multi-CTA passes
        ++g_kernel_launches;
        sort_detections_kernel<<<static_cast<unsigned>(n_maps), kSortThreads, smem, stream>>>(dets, cap, counts, scratch,
                                                                                            false);
        return cudaGetLastError();
    }
    if (runs > 1 && runs <= 65535) {
        // long lists: the runs of every list sort in parallel CTAs
        e = cudaFuncSetAttribute(sort_runs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        ++g_kernel_launches;
        sort_runs_kernel<<<dim3(static_cast<unsigned>(n_maps), static_cast<unsigned>(runs)), kSortThreads, smem,
                           stream>>>(dets, cap, counts);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (!scratch) return cudaSuccess;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (n_maps < sms && !UWB_KNOB("UWB_SORT_ONE_CTA")) {
            // few long lists (single large maps): every merge pass spreads each
            // list over many CTAs; an even number of passes ends in `dets`
            const int64_t tiles = (cap + kMergeTile - 1) / kMergeTile;
            if (tiles > 65535) return cudaErrorNotSupported;
            const size_t msmem = sizeof(uwb_detection) * kMergeTile;
            e = cudaFuncSetAttribute(merge_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(msmem));
            if (e != cudaSuccess) return e;
            int passes = 0;
            for (int64_t w = kSortRun; w < cap; w *= 2) ++passes;
            passes += passes & 1;
            int64_t w = kSortRun;
            for (int q = 0; q < passes; ++q, w *= 2) {
                ++g_kernel_launches;
                merge_pass_kernel<<<dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(n_maps)), kMergeThreads,
                                    msmem, stream>>>(q % 2 ? scratch : dets, q % 2 ? dets : scratch, cap, counts, w, q);
                if ((e = cudaGetLastError()) != cudaSuccess) return e;
            }
            return cudaSuccess;
        }
        ++g_kernel_launches;
        sort_detections_kernel<<<static_cast<unsigned>(n_maps), kSortThreads, smem, stream>>>(dets, cap, counts, scratch,
                                                                                            true);
        return cudaGetLastError();
    }
    // one run per list: shared memory for the capacity's power of two only, so
    // short lists (cfg 3: 512 entries) sort with many CTAs per SM
    int64_t p2 = 1;
    while (p2 < cap) p2 <<= 1;
    const size_t smem1 = sizeof(uwb_detection) * static_cast<size_t>(p2);
    const int threads = static_cast<int>(imin(kSortThreads, imax(64, p2 / 2)));
    ++g_kernel_launches;
    sort_detections_kernel<<<static_cast<unsigned>(n_maps), threads, smem1, stream>>>(dets, cap, counts, scratch,
                                                                                    false);
    return cudaGetLastError();
}

} // namespace uwb
