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
