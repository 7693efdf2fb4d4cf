// Kernels (a1), (a2), (b): the front-end of detect()
// (/root/reference/proj/src/pipeline.cpp:58-223).
//
// (a1) frontend_columns_kernel — one thread per trace (column); adjacent threads
//      own adjacent columns, so every row access of the warp is one coalesced
//      segment. remove_dc (pipeline.cpp:58-69) then detrend_linear (:71-98), each
//      with its own serial sums over fast time in the reference's order, so the
//      output is bit-identical (DC removal is NOT folded into the affine fit:
//      the reference rounds after each stage).
// (a2)+(b) frontend_rows_kernel — one CTA per range row, everything in shared
//      memory: mean_filter_slow (:100-122) or subtract_slow_time_mean (:124-137),
//      normalize_slow (:139-155), zero padding, the r2c transform and |X|^2 for
//      the band-select bins only (:157-223), written straight into the band map.
//      The transform is the radix-2 decimation-in-time FFT restated by the
//      oracle's FFTW provider (oracle/fftw_shim/fft_provider.c) with the same
//      host-computed twiddles and the same operation order, or the direct DFT
//      for non-power-of-two lengths, so the band map reproduces the oracle bit for
//      bit and FFTW within the reference tests' 1e-9.
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace uwb {

namespace {

enum : int {
    kStageRemoveDc = 1,
    kStageDetrend = 2,
    kStageFilter = 4,
    kStageNormalize = 8,
    kStageSpectrum = 16,
};

template <typename T>
__global__ void __launch_bounds__(128) frontend_columns_kernel(FrontendLaunch F) {
    const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= F.n) return;
    const int64_t m = F.m, n = F.n;
    const int64_t rec = blockIdx.y;
    const T* x = static_cast<const T*>(F.frame) + rec * m * n;
    double* work = F.work + rec * m * n;
    unsigned long long* bad = F.first_nonfinite ? F.first_nonfinite + rec : nullptr;
    const double dm = static_cast<double>(m);

    double mean = 0.0;
    if (F.stage_mask & kStageRemoveDc) {
        double sum = 0.0;
        for (int64_t r = 0; r < m; ++r) sum = dadd(sum, static_cast<double>(x[r * n + c]));
        mean = ddiv(sum, dm);
    }
    if (bad) {
        for (int64_t r = 0; r < m; ++r)
            if (!isfinite(static_cast<double>(x[r * n + c])))
                report_min(bad, static_cast<unsigned long long>(r * n + c));
    }
    const bool dc = (F.stage_mask & kStageRemoveDc) != 0;
    if (!(F.stage_mask & kStageDetrend)) {
        for (int64_t r = 0; r < m; ++r) {
            const double v = static_cast<double>(x[r * n + c]);
            work[r * n + c] = dc ? dsub(v, mean) : v;
        }
        return;
    }
    // pipeline.cpp:78-81
    const double sum_r = ddiv(dmul(dm, dsub(dm, 1.0)), 2.0);
    const double sum_rr = ddiv(dmul(dmul(dsub(dm, 1.0), dm), dsub(dmul(2.0, dm), 1.0)), 6.0);
    const double det = dsub(dmul(dm, sum_rr), dmul(sum_r, sum_r));
    double sum_x = 0.0, sum_rx = 0.0;
    for (int64_t r = 0; r < m; ++r) {
        const double v0 = static_cast<double>(x[r * n + c]);
        const double v = dc ? dsub(v0, mean) : v0;
        sum_x = dadd(sum_x, v);
        sum_rx = dadd(sum_rx, dmul(static_cast<double>(r), v));
    }
    const double slope = ddiv(dsub(dmul(dm, sum_rx), dmul(sum_r, sum_x)), det);
    const double intercept = ddiv(dsub(sum_x, dmul(slope, sum_r)), dm);
    for (int64_t r = 0; r < m; ++r) {
        const double v0 = static_cast<double>(x[r * n + c]);
        const double v = dc ? dsub(v0, mean) : v0;
        work[r * n + c] = dsub(v, dadd(intercept, dmul(slope, static_cast<double>(r))));
    }
}

__device__ __forceinline__ unsigned bitrev(unsigned i, int bits) { return __brev(i) >> (32 - bits); }

__global__ void __launch_bounds__(256) frontend_rows_kernel(FrontendLaunch F) {
    extern __shared__ double sm[];
    const int64_t n = F.n, L = F.L;
    const int64_t r = static_cast<int64_t>(blockIdx.y) * F.m + blockIdx.x; // row across the batch
    double* row = sm;        // n
    double* re = sm + n;     // L
    double* im = re + L;     // L (also used as filter scratch)
    const double* in = F.work + r * n;

    for (int64_t c = threadIdx.x; c < n; c += blockDim.x) row[c] = in[c];
    __syncthreads();

    // ---- slow-time filter: result in im[0..n)
    if ((F.stage_mask & kStageFilter) && F.mode == 0 && F.window > 1) {
        const int64_t half = static_cast<int64_t>(F.window / 2);
        for (int64_t c = threadIdx.x; c < n; c += blockDim.x) {
            int64_t h = half;
            if (c < h) h = c;
            if (n - 1 - c < h) h = n - 1 - c;
            double sum = 0.0;
            for (int64_t k = c - h; k <= c + h; ++k) sum = dadd(sum, row[k]);
            im[c] = ddiv(sum, static_cast<double>(2 * h + 1));
        }
    } else if ((F.stage_mask & kStageFilter) && F.mode == 1) {
        __shared__ double mean_s;
        if (threadIdx.x == 0) {
            double sum = 0.0;
            for (int64_t c = 0; c < n; ++c) sum = dadd(sum, row[c]);
            mean_s = ddiv(sum, static_cast<double>(n));
        }
        __syncthreads();
        for (int64_t c = threadIdx.x; c < n; c += blockDim.x) im[c] = dsub(row[c], mean_s);
    } else {
        for (int64_t c = threadIdx.x; c < n; c += blockDim.x) im[c] = row[c];
    }
    __syncthreads();

    // ---- normalize_slow: divide by max(max|x|, eps)
    if (F.stage_mask & kStageNormalize) {
        __shared__ double warp_max[32];
        double peak = 0.0;
        for (int64_t c = threadIdx.x; c < n; c += blockDim.x) peak = fmax(peak, fabs(im[c]));
        for (int o = 16; o > 0; o >>= 1) peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
        if ((threadIdx.x & 31) == 0) warp_max[threadIdx.x >> 5] = peak;
        __syncthreads();
        if (threadIdx.x < 32) {
            double p = threadIdx.x < (blockDim.x >> 5) ? warp_max[threadIdx.x] : 0.0;
            for (int o = 16; o > 0; o >>= 1) p = fmax(p, __shfl_xor_sync(0xffffffffu, p, o));
            if (threadIdx.x == 0) warp_max[0] = p;
        }
        __syncthreads();
        const double pk = warp_max[0];
        const double scale = pk < F.epsilon ? F.epsilon : pk;
        for (int64_t c = threadIdx.x; c < n; c += blockDim.x) im[c] = ddiv(im[c], scale);
        __syncthreads();
    }

    if (!(F.stage_mask & kStageSpectrum)) {
        for (int64_t c = threadIdx.x; c < n; c += blockDim.x) F.work[r * n + c] = im[c];
        return;
    }

    // ---- r2c transform of the zero-padded row
    const bool pow2 = (L & (L - 1)) == 0;
    const int64_t bins = L / 2 + 1;
    if (pow2) {
        int bits = 0;
        while ((int64_t(1) << bits) < L) ++bits;
        // bit-reversal permutation (fft_provider.c swap loop): re[i] = x[rev(i)]
        for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
            const int64_t src = bits ? static_cast<int64_t>(bitrev(static_cast<unsigned>(i), bits)) : 0;
            re[i] = src < n ? im[src] : 0.0;
        }
        __syncthreads();
        for (int64_t i = threadIdx.x; i < L; i += blockDim.x) im[i] = 0.0;
        __syncthreads();
        // stage with half-length 2^lh: butterfly b pairs p = (b >> lh) * 2^(lh+1) + j and
        // p + 2^lh, j = b mod 2^lh, twiddle j * (L >> (lh + 1)) (powers of two: shifts)
        for (int lh = 0; lh < bits; ++lh) {
            const int half = 1 << lh;
            const int tw_shift = bits - lh - 1;
            for (int b = threadIdx.x; b < (1 << (bits - 1)); b += blockDim.x) {
                const int j = b & (half - 1);
                const int p = ((b >> lh) << (lh + 1)) + j;
                const int q = p + half;
                const double w_r = __ldg(F.wr + (j << tw_shift)), w_i = __ldg(F.wi + (j << tw_shift));
                const double br = re[q], bi = im[q];
                const double tr = dsub(dmul(w_r, br), dmul(w_i, bi));
                const double ti = dadd(dmul(w_r, bi), dmul(w_i, br));
                const double ur = re[p], ui = im[p];
                re[p] = dadd(ur, tr);
                im[p] = dadd(ui, ti);
                re[q] = dsub(ur, tr);
                im[q] = dsub(ui, ti);
            }
            __syncthreads();
        }
        for (int64_t k = threadIdx.x; k < bins; k += blockDim.x) {
            const double pw = dadd(dmul(re[k], re[k]), dmul(im[k], im[k]));
            if (F.full_power) F.full_power[r * bins + k] = pw;
            if (F.band && k >= F.first_bin && k < F.first_bin + F.kept)
                F.band[r * F.kept + (k - F.first_bin)] = pw;
        }
    } else {
        // direct DFT over the padded sequence (fft_provider.c uwb_dft_real)
        for (int64_t k = threadIdx.x; k < bins; k += blockDim.x) {
            const bool want = F.full_power || (k >= F.first_bin && k < F.first_bin + F.kept);
            if (!want) continue;
            double ar = 0.0, ai = 0.0;
            for (int64_t j = 0; j < L; ++j) {
                const double xj = j < n ? im[j] : 0.0;
                const int64_t mm = (j * k) % L;
                ar = dadd(ar, dmul(xj, F.wr[mm]));
                ai = dadd(ai, dmul(xj, F.wi[mm]));
            }
            const double pw = dadd(dmul(ar, ar), dmul(ai, ai));
            if (F.full_power) F.full_power[r * bins + k] = pw;
            if (F.band && k >= F.first_bin && k < F.first_bin + F.kept)
                F.band[r * F.kept + (k - F.first_bin)] = pw;
        }
    }
}


// ---------------------------------------------------------------------------
// Fused detect() front end for L = 1024 (the batched device detect() path):
// two kernels and no fp64 work frame in HBM.
//
// (f1) frontend_stats_kernel — one warp per 32 traces (columns) of one record:
//      the 32 x m input block is staged in shared memory once, then each lane
//      runs remove_dc's mean (pipeline.cpp:58-69) and detrend_linear's moment
//      sums (:71-98) over its column, serially in the reference's order, and
//      stores (mean, slope, intercept) per column. Non-finite samples are
//      reported here (RadarFrame::validate, pipeline.cpp:27-38).
// (f2) frontend_fft1024_kernel — one warp per range row: the row is read once
//      (coalesced), detrended from the column statistics with the reference's
//      expression, mean-filtered (:100-122) and normalised (:139-155) in
//      registers / shared memory, then transformed by the radix-2 DIT of the
//      FFT provider with the same twiddles and per-element operation order:
//      stages 1..5 as 32-point FFTs in registers (lane t holds bit-reversed
//      elements 32t..32t+31, which are the stride-32 samples starting at
//      rev5(t)), a padded shared-memory transpose, stages 6..10 in registers
//      with lane t holding elements 32a + t, pruned to the butterflies whose
//      outputs reach the band bins (band select, :192-223). Every value that
//      reaches the band map is produced by the same IEEE operations on the same
//      operands as in frontend_rows_kernel, so the band map is bit-identical.
constexpr int kStatGroup = 16;        // rows per cp.async group of the stats kernel's ring
constexpr int kStatRingBytes = 8192;  // ring size (measured: more CTAs per SM beat L2 reuse of the second pass)

// Streams the 32-column block of rows [0, m) through a shared-memory ring
// (cp.async, stat_slots<T>() - 1 groups in flight) and calls use(r, value) in row order.
template <typename T>
__host__ __device__ constexpr int stat_slots() { return kStatRingBytes / (kStatGroup * kWarp * static_cast<int>(sizeof(T))); }

template <typename T, typename Use>
__device__ __forceinline__ void stream_block(const T* base, int64_t n, int64_t m, bool vec, bool ok, T* ring, Use use) {
    const int lane = threadIdx.x;
    const unsigned sb = static_cast<unsigned>(__cvta_generic_to_shared(ring));
    constexpr int kVec = 16 / sizeof(T);         // elements per 16-byte piece
    constexpr int kPieces = kWarp / kVec;        // pieces per 32-element row
    constexpr int kRowsPer = kWarp / kPieces;    // rows per warp-wide copy
    const int64_t ngroups = (m + kStatGroup - 1) / kStatGroup;
    auto issue = [&](int64_t g) {
        if (g < ngroups) {
            const unsigned slot = sb + static_cast<unsigned>((g % stat_slots<T>()) * kStatGroup * kWarp * sizeof(T));
            const int64_t r0 = g * kStatGroup;
            if (vec) {
                const int pr = lane / kPieces, pc = lane % kPieces;
                for (int rr = pr; rr < kStatGroup && r0 + rr < m; rr += kRowsPer)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                     slot + static_cast<unsigned>((rr * kWarp + pc * kVec) * sizeof(T))),
                                 "l"(base + (r0 + rr) * n + pc * kVec)
                                 : "memory");
            } else if (ok) {
                for (int rr = 0; rr < kStatGroup && r0 + rr < m; ++rr)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(
                                     slot + static_cast<unsigned>((rr * kWarp + lane) * sizeof(T))),
                                 "l"(base + (r0 + rr) * n + lane), "n"(sizeof(T))
                                 : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int g = 0; g < stat_slots<T>() - 1; ++g) issue(g);
    for (int64_t g = 0; g < ngroups; ++g) {
        asm volatile("cp.async.wait_group %0;" ::"n"(stat_slots<T>() - 2) : "memory");
        __syncwarp();
        const T* slot = ring + (g % stat_slots<T>()) * kStatGroup * kWarp;
        const int64_t r0 = g * kStatGroup;
        if (r0 + kStatGroup <= m) {
#pragma unroll
            for (int rr = 0; rr < kStatGroup; ++rr) use(r0 + rr, widen(slot[rr * kWarp + lane]));
        } else {
            for (int rr = 0; r0 + rr < m; ++rr) use(r0 + rr, widen(slot[rr * kWarp + lane]));
        }
        __syncwarp(); // the slot is consumed before it is refilled
        issue(g + stat_slots<T>() - 1);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

template <typename T>
__global__ void __launch_bounds__(32) frontend_stats_kernel(FrontendLaunch F) {
    __shared__ __align__(16) T ring[kStatRingBytes / sizeof(T)];
    const int lane = threadIdx.x;
    const int64_t m = F.m, n = F.n, rec = blockIdx.y;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kWarp;
    const int64_t c = c0 + lane;
    const bool ok = c < n;
    const T* base = static_cast<const T*>(F.frame) + rec * m * n + c0;
    const bool vec = c0 + kWarp <= n && (reinterpret_cast<uintptr_t>(base) % 16) == 0 && (n * sizeof(T)) % 16 == 0;
    const double dm = static_cast<double>(m);
    // remove_dc: serial sum over fast time, then the mean (pipeline.cpp:62-66)
    double sum = 0.0;
    int64_t bad = -1;
    stream_block<T>(base, n, m, vec, ok, ring, [&](int64_t r, double v) {
        if (!isfinite(v) && bad < 0) bad = r;
        sum = dadd(sum, v);
    });
    if (ok && bad >= 0 && F.first_nonfinite)
        report_min(F.first_nonfinite + rec, static_cast<unsigned long long>(bad * n + c));
    const double mean = ddiv(sum, dm);
    // detrend_linear on the DC-removed trace (pipeline.cpp:78-93); the second
    // pass over the block is served by L2
    const double sum_r = ddiv(dmul(dm, dsub(dm, 1.0)), 2.0);
    const double sum_rr = ddiv(dmul(dmul(dsub(dm, 1.0), dm), dsub(dmul(2.0, dm), 1.0)), 6.0);
    const double det = dsub(dmul(dm, sum_rr), dmul(sum_r, sum_r));
    double sum_x = 0.0, sum_rx = 0.0;
    __syncwarp();
    stream_block<T>(base, n, m, vec, ok, ring, [&](int64_t r, double x) {
        const double v = dsub(x, mean);
        sum_x = dadd(sum_x, v);
        sum_rx = dadd(sum_rx, dmul(static_cast<double>(r), v));
    });
    if (!ok) return;
    const double slope = ddiv(dsub(dmul(dm, sum_rx), dmul(sum_r, sum_x)), det);
    const double intercept = ddiv(dsub(sum_x, dmul(slope, sum_r)), dm);
    double* st = F.work + rec * 3 * n;
    st[c] = mean;
    st[n + c] = slope;
    st[2 * n + c] = intercept;
}

__host__ __device__ constexpr int rev5(int a) {
    return ((a & 1) << 4) | ((a & 2) << 2) | (a & 4) | ((a & 8) >> 2) | ((a & 16) >> 4);
}

constexpr int kFftWarps = 4;                        // rows per CTA
constexpr int kTw2 = 31 * kWarp;                    // stage 6..10 twiddles, [stage group][lane]
constexpr int kTw1 = 32;                            // stage 1..5 twiddles (31 used)
constexpr int kXpPitch = 33;                        // padded transpose pitch (doubles)
constexpr int kWarpBuf = kXpPitch * kWarp;          // transpose buffer per warp (doubles; re, then im)
constexpr size_t kFftSmem = sizeof(double) * (2 * kTw2 + 2 * kTw1 + kFftWarps * kWarpBuf);

__device__ __forceinline__ void butterfly(double& ur, double& ui, double& br, double& bi, double w_r, double w_i) {
    const double tr = dsub(dmul(w_r, br), dmul(w_i, bi));
    const double ti = dadd(dmul(w_r, bi), dmul(w_i, br));
    br = dsub(ur, tr);
    bi = dsub(ui, ti);
    ur = dadd(ur, tr);
    ui = dadd(ui, ti);
}

// HALF = mean-filter half width (window / 2), or -1: any window (runtime loop)
template <typename T, int HALF>
__global__ void __launch_bounds__(kFftWarps * kWarp, 3) frontend_fft1024_kernel(FrontendLaunch F) {
    extern __shared__ __align__(16) double fz[];
    double* t2r = fz;              // [g * 32 + t]: stage 6 + s, group g = 2^s - 1 + b, element 32 b + t
    double* t2i = t2r + kTw2;
    double* t1r = t2i + kTw2;      // [2^lh - 1 + j]: stage lh + 1, butterfly offset j
    double* t1i = t1r + kTw1;
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    // twiddle index of butterfly offset j at stage lh: j << (bits - lh - 1), bits = 10
    for (int e = threadIdx.x; e < kTw2; e += blockDim.x) {
        const int g = e / kWarp, t = e % kWarp;
        const int sft = 31 - __clz(g + 1);          // stage lh = 5 + sft
        const int b = g + 1 - (1 << sft);
        const int idx = (kWarp * b + t) << (4 - sft);
        t2r[e] = F.wr[idx];
        t2i[e] = F.wi[idx];
    }
    for (int e = threadIdx.x; e < 31; e += blockDim.x) {
        const int lh = 31 - __clz(e + 1);
        const int j = e + 1 - (1 << lh);
        const int idx = j << (9 - lh);
        t1r[e] = F.wr[idx];
        t1i[e] = F.wi[idx];
    }
    __syncthreads();
    const int64_t m = F.m;
    const int n = static_cast<int>(F.n), nn = n;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kFftWarps + warp; // across the batch
    if (row >= m * (F.n_rec > 0 ? F.n_rec : 1)) return;
    const int64_t rec = row / m, r = row % m;
    double* xbuf = fz + 2 * kTw2 + 2 * kTw1 + warp * kWarpBuf;
    double* zb = xbuf; // the row before the transform (n <= 1024 < 33 * 32)
    const double* st = F.work + rec * 3 * n;                 // mean[n], slope[n], intercept[n] of this record

    // ---- detrend from the column statistics: dsub(v, dadd(intercept, dmul(slope, r))) with
    //      v = dsub(x, mean) (pipeline.cpp:66, :93)
    const T* xr = static_cast<const T*>(F.frame) + row * n;
    const double rd = static_cast<double>(r);
    // the whole row is requested before anything waits on it: one DRAM round trip per
    // row instead of one per 8 blocks (the statistics come from L2: 512 rows share them);
    // config 2: 143.7k -> 149.8k records/s
    T xv[kWarp];
#pragma unroll
    for (int j = 0; j < kWarp; ++j) {
        const int c = kWarp * j + lane;
        xv[j] = c < n ? xr[c] : T(0);
    }
#pragma unroll 8
    for (int j = 0; j < kWarp; ++j) {
        const int c = kWarp * j + lane;
        if (c < n) {
            const double v = dsub(widen(xv[j]), __ldg(st + c));
            zb[c] = dsub(v, dadd(__ldg(st + 2 * n + c), dmul(__ldg(st + n + c), rd)));
        }
    }
    __syncwarp();
    // ---- mean_filter_slow (pipeline.cpp:100-122): centred window, shrunk at the edges;
    //      sum = ((0 + x[c-h]) + ...) + x[c+h], then / (2h + 1). In place, one
    //      32-cell block behind the reads (half <= 15, so block j reads no cell
    //      of block j - 2); a small loop body keeps the kernel's code compact.
    const int half = HALF >= 0 ? HALF : static_cast<int>(F.window / 2);
    auto filt = [&](int c) -> double {
        if (HALF == 0) return zb[c];
        if (HALF > 0 && c >= HALF && c + HALF < nn) { // interior: compile-time taps
            double sum = 0.0;
#pragma unroll
            for (int k = -HALF; k <= HALF; ++k) sum = dadd(sum, zb[c + k]);
            return ddiv(sum, static_cast<double>(2 * HALF + 1));
        }
        if (HALF < 0 && half == 0) return zb[c];
        int h = half;
        if (c < h) h = c;
        if (nn - 1 - c < h) h = nn - 1 - c;
        double sum = 0.0;
        for (int k = c - h; k <= c + h; ++k) sum = dadd(sum, zb[k]);
        return ddiv(sum, static_cast<double>(2 * h + 1));
    };
    const int nblk = (nn + kWarp - 1) / kWarp;
    double peak = 0.0, prev = 0.0;
    auto block = [&](const int j, auto interior_tag) {
        constexpr bool kInterior = decltype(interior_tag)::value;
        const int c = kWarp * j + lane;
        double v;
        if constexpr (kInterior) { // every cell of the block has its whole window: compile-time taps only
            double sum = 0.0;
#pragma unroll
            for (int k = -(HALF > 0 ? HALF : 0); k <= (HALF > 0 ? HALF : 0); ++k) sum = dadd(sum, zb[c + k]);
            v = ddiv(sum, static_cast<double>(2 * (HALF > 0 ? HALF : 0) + 1));
        } else {
            v = c < nn ? filt(c) : 0.0;
        }
        __syncwarp(); // block j's reads are done: block j - 1 may be overwritten
        if (j > 0) zb[c - kWarp] = prev;
        if (kInterior || c < nn) peak = fmax(peak, fabs(v)); // normalize_slow's max |x| (pipeline.cpp:143-147)
        prev = v;
    };
    // the edge blocks (shrunk windows, a second division path) run outside the loop, so the
    // loop body is the interior case alone (instruction cache; the kernel is fetch- and
    // latency-bound)
    int j = 0;
    if (HALF > 0) {
        const int j_hi = (nn - HALF) / kWarp - 1; // last block whose cells all have c + HALF < nn
        block(0, std::false_type{});
        j = 1;
#pragma unroll 2
        for (; j <= j_hi; ++j) block(j, std::true_type{});
    }
#pragma unroll 1
    for (; j < nblk; ++j) block(j, std::false_type{});
    if (kWarp * (nblk - 1) + lane < nn) zb[kWarp * (nblk - 1) + lane] = prev;
    // ---- normalize_slow (pipeline.cpp:139-155): divide by max(max |x|, eps)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
    const double scale = peak < F.epsilon ? F.epsilon : peak;
#pragma unroll 4
    for (int j = 0; j < nblk; ++j) {
        const int c = kWarp * j + lane;
        if (c < nn) zb[c] = ddiv(zb[c], scale);
    }
    __syncwarp();
    // ---- bit-reversed load: element 32 t + a = sample 32 rev5(a) + rev5(t) (zero past n)
    double yr[kWarp], yi[kWarp];
    const int rt = rev5(lane);
#pragma unroll
    for (int a = 0; a < kWarp; ++a) {
        const int src = kWarp * rev5(a) + rt;
        yr[a] = src < n ? zb[src] : 0.0;
        yi[a] = 0.0;
    }
    // ---- stages 1..5: butterflies (p, p + 2^lh) inside the lane's 32 elements
    //      (offset j = 0 has the twiddle (1, -0): w * b is b itself for every
    //      nonzero b, and zeros stay zeros, so those butterflies skip the product)
#pragma unroll
    for (int lh = 0; lh < 5; ++lh) {
        const int hf = 1 << lh;
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const int j = b & (hf - 1);
            const int p = ((b >> lh) << (lh + 1)) + j;
            const int q = p + hf;
            if (j == 0) {
                const double ur = yr[p], ui = yi[p];
                yr[p] = dadd(ur, yr[q]);
                yi[p] = dadd(ui, yi[q]);
                yr[q] = dsub(ur, yr[q]);
                yi[q] = dsub(ui, yi[q]);
            } else {
                butterfly(yr[p], yi[p], yr[q], yi[q], t1r[hf - 1 + j], t1i[hf - 1 + j]);
            }
        }
    }
    // ---- transpose (padded pitch: conflict-free both ways): lane t then holds elements 32 a + t
    __syncwarp();
#pragma unroll
    for (int a = 0; a < kWarp; ++a) xbuf[kXpPitch * lane + a] = yr[a];
    __syncwarp();
#pragma unroll
    for (int a = 0; a < kWarp; ++a) yr[a] = xbuf[kXpPitch * a + lane];
    __syncwarp();
#pragma unroll
    for (int a = 0; a < kWarp; ++a) xbuf[kXpPitch * lane + a] = yi[a];
    __syncwarp();
#pragma unroll
    for (int a = 0; a < kWarp; ++a) yi[a] = xbuf[kXpPitch * a + lane];
    // ---- stages 6..10 (pairs a, a + 2^s in registers); the last stage only forms
    //      the outputs at or below L/2 (registers 0..16)
#pragma unroll
    for (int sft = 0; sft < 5; ++sft) {
        const int sb = 1 << sft;
#pragma unroll
        for (int a0 = 0; a0 < kWarp; ++a0) {
            if (a0 & sb) continue;
            const int a1 = a0 + sb;
            const int g = sb - 1 + (a0 & (sb - 1));
            const double w_r = t2r[g * kWarp + lane], w_i = t2i[g * kWarp + lane];
            if (sft < 4 || a1 == 16) {
                butterfly(yr[a0], yi[a0], yr[a1], yi[a1], w_r, w_i);
            } else {
                const double br = yr[a1], bi = yi[a1];
                yr[a0] = dadd(yr[a0], dsub(dmul(w_r, br), dmul(w_i, bi)));
                yi[a0] = dadd(yi[a0], dadd(dmul(w_r, bi), dmul(w_i, br)));
            }
        }
    }
    // ---- |X|^2 of the band bins (pipeline.cpp:183-188, :211-219)
    const int k_lo = static_cast<int>(F.first_bin), k_hi = static_cast<int>(F.first_bin + F.kept); // bins [k_lo, k_hi)
#pragma unroll
    for (int a = 0; a <= 16; ++a) {
        const int k = kWarp * a + lane;
        if (k >= k_lo && k < k_hi) F.band[row * F.kept + (k - k_lo)] = dadd(dmul(yr[a], yr[a]), dmul(yi[a], yi[a]));
    }
}
} // namespace

cudaError_t launch_frontend_columns(const FrontendLaunch& F, cudaStream_t stream) {
    const dim3 blocks(static_cast<unsigned>((F.n + 127) / 128), static_cast<unsigned>(F.n_rec > 0 ? F.n_rec : 1));
    ++g_kernel_launches;
    if (F.dtype == UWB_F32) frontend_columns_kernel<float><<<blocks, 128, 0, stream>>>(F);
    else frontend_columns_kernel<double><<<blocks, 128, 0, stream>>>(F);
    return cudaGetLastError();
}

size_t frontend_rows_smem(int64_t n, int64_t L) {
    const int64_t big = L > n ? L : n;
    return sizeof(double) * static_cast<size_t>(n + L + big);
}

cudaError_t launch_frontend_rows(const FrontendLaunch& F, cudaStream_t stream) {
    const size_t smem = frontend_rows_smem(F.n, F.L);
    cudaError_t e = cudaFuncSetAttribute(frontend_rows_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    ++g_kernel_launches;
    const dim3 grid(static_cast<unsigned>(F.m), static_cast<unsigned>(F.n_rec > 0 ? F.n_rec : 1));
    frontend_rows_kernel<<<grid, 256, smem, stream>>>(F);
    return cudaGetLastError();
}

} // namespace uwb

namespace uwb {

namespace {
template <typename T, int HALF>
cudaError_t launch_fft(const FrontendLaunch& F, dim3 grid, cudaStream_t stream) {
    cudaError_t e = cudaFuncSetAttribute(frontend_fft1024_kernel<T, HALF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kFftSmem));
    if (e != cudaSuccess) return e;
    frontend_fft1024_kernel<T, HALF><<<grid, kFftWarps * kWarp, kFftSmem, stream>>>(F);
    return cudaSuccess;
}
template <typename T>
cudaError_t launch_fft_half(const FrontendLaunch& F, int half, dim3 grid, cudaStream_t stream) {
    switch (half) {
        case 0: return launch_fft<T, 0>(F, grid, stream);
        case 1: return launch_fft<T, 1>(F, grid, stream);
        case 2: return launch_fft<T, 2>(F, grid, stream);
        case 3: return launch_fft<T, 3>(F, grid, stream);
        case 4: return launch_fft<T, 4>(F, grid, stream);
        default: return launch_fft<T, -1>(F, grid, stream);
    }
}
} // namespace

// The fused front end (stats + fft1024) for the whole detect() front end;
// cudaErrorNotSupported when the configuration needs the general kernels.
cudaError_t launch_frontend_fused(const FrontendLaunch& F, cudaStream_t stream) {
    if (const char* e = UWB_KNOB("UWB_FE_FUSED"))
        if (atoi(e) == 0) return cudaErrorNotSupported;
    if (F.L != 1024 || F.n < 2 || F.n > 1024 || F.m < 3 || F.mode != 0 || F.full_power || !F.band || F.kept < 1 ||
        F.first_bin < 0 || F.first_bin + F.kept > F.L / 2 + 1 || F.window < 1 || (F.window & 1) == 0 ||
        F.window > 31)
        return cudaErrorNotSupported;
    const int64_t n_rec = F.n_rec > 0 ? F.n_rec : 1;
    // (f1) column statistics into the work buffer (3 n doubles per record <= m n)
    const dim3 g1(static_cast<unsigned>((F.n + kWarp - 1) / kWarp), static_cast<unsigned>(n_rec));
    cudaError_t e = cudaSuccess;
    ++g_kernel_launches;
    if (F.dtype == UWB_F32) frontend_stats_kernel<float><<<g1, kWarp, 0, stream>>>(F);
    else frontend_stats_kernel<double><<<g1, kWarp, 0, stream>>>(F);
    if (e != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // (f2) rows: detrend, filter, normalise, FFT, band power
    const dim3 g2(static_cast<unsigned>((F.m * n_rec + kFftWarps - 1) / kFftWarps));
    const int half = F.window <= 9 ? static_cast<int>(F.window / 2) : -1;
    e = F.dtype == UWB_F32 ? launch_fft_half<float>(F, half, g2, stream) : launch_fft_half<double>(F, half, g2, stream);
    ++g_kernel_launches;
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

} // namespace uwb
