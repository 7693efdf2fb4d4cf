// Kernel (d): CA-CFAR threshold + mask + detection compaction, replacing
// run_cfar / cfar_rows / cfar2d_integral (/root/reference/proj/src/cfar.cpp:109-175,
// 218-227) and, for the naive backend, cfar2d_naive (cfar.cpp:200-216).
//
// Per cell (cfar.cpp:115-127): clamped outer and guard rectangles, their n_train,
// the two four-tap region sums in the association of sat.hpp:32-33,
//     RS = (t[r0][c0] + t[r1+1][c1+1]) - (t[r0][c1+1] + t[r1+1][c0]),
// sum = RS(outer) - RS(guard), mean = sum / n (IEEE division), T = alpha[n] * mean
// with alpha tabulated on the host by the same libm pow, and mask = cut > T
// (ties are H0). Same operations in the same order => bit-identical thresholds.
//
// Layout: a CTA of 128 threads owns a 128-column x 32-row tile of one job; a
// warp covers 32 aligned columns, so the mask bits of a row segment come out of
// one __ballot_sync as one 32-bit word. Detections are compacted with one
// warp-aggregated atomicAdd per warp-row into the map's list; the list is then
// sorted (value desc, row asc, col asc, cfar.cpp:170-173), which makes the
// final order independent of the atomic order.
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace uwb {

namespace {

constexpr int kCfarThreads = 128;
constexpr int kCfarRowChunk = 32;

template <typename T>
__device__ __forceinline__ double load_cell(const T* p) {
    return static_cast<double>(__ldg(p));
}

__device__ __forceinline__ double tap(const double* t, int64_t ld, int64_t i, int64_t j) {
    return __ldg(t + i * ld + 1 + j);
}

struct Window {
    int64_t r0, r1, c0, c1;
};

__device__ __forceinline__ int64_t clamp_lo(int64_t c, int rad) {
    const int64_t v = c - rad;
    return v < 0 ? 0 : v;
}
__device__ __forceinline__ int64_t clamp_hi(int64_t c, int rad, int64_t dim) {
    const int64_t v = c + rad;
    return v >= dim ? dim - 1 : v;
}

// Emits the mask word, optional per-cell outputs and compacted detections for
// one row segment of 32 cells held by a warp.
__device__ __forceinline__ void emit(const CfarLaunch& L, int64_t map, int64_t r, int64_t c,
                                     bool valid, bool hit, double v, double thr) {
    const unsigned lane = threadIdx.x % kWarp;
    const unsigned bits = __ballot_sync(0xffffffffu, valid && hit);
    if (lane == 0 && L.mask_bits) {
        const int64_t word = c / 32;
        if (word < L.words_per_row)
            L.mask_bits[map * L.mask_map_stride + r * L.words_per_row + word] = bits;
    }
    if (valid) {
        const int64_t cell = r * L.cols + c;
        if (L.mask_u8) L.mask_u8[map * L.geo.rows * L.cols + cell] = hit ? 1 : 0;
        if (L.thresholds) L.thresholds[map * L.geo.rows * L.cols + cell] = thr;
    }
    if (bits) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(L.det_counts + map, static_cast<unsigned long long>(__popc(bits)));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (valid && hit) {
            const unsigned long long slot = base + __popc(bits & ((1u << lane) - 1u));
            if (slot < static_cast<unsigned long long>(L.det_cap)) {
                uwb_detection d;
                d.row = static_cast<uint64_t>(r);
                d.col = static_cast<uint64_t>(c);
                d.value = v;
                d.threshold = thr;
                L.dets[map * L.det_cap + slot] = d;
            }
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kCfarThreads)
cfar_integral_kernel(CfarLaunch L) {
    const int64_t job = blockIdx.y;
    const int64_t map = job / L.geo.n_slabs;
    const int64_t slab = job % L.geo.n_slabs;
    const int64_t col_tile = blockIdx.x % L.col_tiles;
    const int64_t chunk = blockIdx.x / L.col_tiles;
    const int64_t c = col_tile * kCfarThreads + threadIdx.x;
    const bool col_ok = c < L.cols;
    const int64_t rows = L.geo.rows;
    const int64_t ra = L.geo.owned_begin(slab) + chunk * kCfarRowChunk;
    const int64_t rb = imin(ra + kCfarRowChunk, L.geo.owned_end(slab));
    if (ra >= rb) return;
    const int64_t trow0 = L.geo.table_begin(slab);
    const double* tab = L.table + job * L.table_stride;
    const int64_t ld = L.table_ld;
    const T* cut_base = static_cast<const T*>(L.maps) + map * L.map_stride;

    // column extents do not depend on the row
    const int64_t oc0 = clamp_lo(c, L.hc), oc1 = clamp_hi(c, L.hc, L.cols);
    const int64_t gc0 = clamp_lo(c, L.gc), gc1 = clamp_hi(c, L.gc, L.cols);
    const int64_t ow = oc1 - oc0 + 1, gw = gc1 - gc0 + 1;

    for (int64_t r = ra; r < rb; ++r) {
        bool hit = false;
        double v = 0.0, thr = 0.0;
        if (col_ok) {
            const int64_t or0 = clamp_lo(r, L.hr), or1 = clamp_hi(r, L.hr, rows);
            const int64_t gr0 = clamp_lo(r, L.gr), gr1 = clamp_hi(r, L.gr, rows);
            const int64_t n = (or1 - or0 + 1) * ow - (gr1 - gr0 + 1) * gw;
            const int64_t ti0 = or0 - trow0, ti1 = or1 + 1 - trow0;
            const int64_t gi0 = gr0 - trow0, gi1 = gr1 + 1 - trow0;
            // sat.hpp:32-33, outer then guard
            const double rs_o = dsub(dadd(tap(tab, ld, ti0, oc0), tap(tab, ld, ti1, oc1 + 1)),
                                     dadd(tap(tab, ld, ti0, oc1 + 1), tap(tab, ld, ti1, oc0)));
            const double rs_g = dsub(dadd(tap(tab, ld, gi0, gc0), tap(tab, ld, gi1, gc1 + 1)),
                                     dadd(tap(tab, ld, gi0, gc1 + 1), tap(tab, ld, gi1, gc0)));
            const double sum = dsub(rs_o, rs_g);
            const double mean = ddiv(sum, static_cast<double>(n));
            thr = dmul(__ldg(L.alpha + n), mean);
            v = load_cell(cut_base + r * L.ld + c);
            hit = v > thr; // cfar.cpp:125, ties -> H0
            if (v < 0.0) report_min(L.first_bad + 2 * map + 1,
                                    static_cast<unsigned long long>(r * L.cols + c));
        }
        emit(L, map, r, c, col_ok, hit, v, thr);
    }
}

// cfar.cpp:200-216: explicit ring loop, row-major accumulation order.
template <typename T>
__global__ void __launch_bounds__(kCfarThreads)
cfar_naive_kernel(CfarLaunch L) {
    const int64_t map = blockIdx.y;
    const int64_t col_tile = blockIdx.x % L.col_tiles;
    const int64_t chunk = blockIdx.x / L.col_tiles;
    const int64_t c = col_tile * kCfarThreads + threadIdx.x;
    const bool col_ok = c < L.cols;
    const int64_t rows = L.geo.rows;
    const int64_t ra = chunk * kCfarRowChunk;
    const int64_t rb = imin(ra + kCfarRowChunk, rows);
    if (ra >= rb) return;
    const T* m = static_cast<const T*>(L.maps) + map * L.map_stride;
    const int64_t oc0 = clamp_lo(c, L.hc), oc1 = clamp_hi(c, L.hc, L.cols);
    const int64_t gc0 = clamp_lo(c, L.gc), gc1 = clamp_hi(c, L.gc, L.cols);
    const int64_t ow = oc1 - oc0 + 1, gw = gc1 - gc0 + 1;
    for (int64_t r = ra; r < rb; ++r) {
        bool hit = false;
        double v = 0.0, thr = 0.0;
        if (col_ok) {
            const int64_t or0 = clamp_lo(r, L.hr), or1 = clamp_hi(r, L.hr, rows);
            const int64_t gr0 = clamp_lo(r, L.gr), gr1 = clamp_hi(r, L.gr, rows);
            const int64_t n = (or1 - or0 + 1) * ow - (gr1 - gr0 + 1) * gw;
            double sum = 0.0;
            for (int64_t rr = or0; rr <= or1; ++rr) {
                const bool guard_row = rr >= gr0 && rr <= gr1;
                const T* row = m + rr * L.ld;
                for (int64_t cc = oc0; cc <= oc1; ++cc) {
                    if (guard_row && cc >= gc0 && cc <= gc1) continue;
                    sum = dadd(sum, load_cell(row + cc));
                }
            }
            const double mean = ddiv(sum, static_cast<double>(n));
            thr = dmul(__ldg(L.alpha + n), mean);
            v = load_cell(m + r * L.ld + c);
            hit = v > thr;
            if (!isfinite(v) || v < 0.0)
                report_min(L.first_bad + 2 * map + 1, static_cast<unsigned long long>(r * L.cols + c));
        }
        emit(L, map, r, c, col_ok, hit, v, thr);
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
                    if (swap) { s[i] = b; s[p] = a; }
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

__global__ void __launch_bounds__(kSortThreads)
sort_detections_kernel(uwb_detection* dets, int64_t cap, const unsigned long long* counts,
                       uwb_detection* scratch) {
    extern __shared__ uwb_detection smem[];
    const int64_t map = blockIdx.x;
    const int64_t count = imin(static_cast<int64_t>(counts[map]), cap);
    if (count <= 1) return;
    uwb_detection* src = dets + map * cap;
    uwb_detection* alt = scratch ? scratch + map * cap : nullptr;

    // 1. sort runs of kSortRun in shared memory
    for (int64_t base = 0; base < count; base += kSortRun) {
        const int n = static_cast<int>(imin(kSortRun, count - base));
        int p2 = 1;
        while (p2 < n) p2 <<= 1;
        for (int i = threadIdx.x; i < p2; i += blockDim.x) smem[i] = i < n ? src[base + i] : sentinel();
        __syncthreads();
        smem_bitonic(smem, p2);
        for (int i = threadIdx.x; i < n; i += blockDim.x) src[base + i] = smem[i];
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
            const int64_t a0 = base, a1 = min(base + width, count);
            const int64_t b0 = a1, b1 = min(base + 2 * width, count);
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
    dim3 grid;
    const CfarLaunch L = grid_shape(L0, grid);
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
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(sort_detections_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        attr_set = true;
    }
    ++g_kernel_launches;
    sort_detections_kernel<<<static_cast<unsigned>(n_maps), kSortThreads, smem, stream>>>(
        dets, cap, counts, scratch);
    return cudaGetLastError();
}

} // namespace uwb
