// Kernel (c): exact summed-area table, replacing build_sat
// (/root/reference/proj/src/sat.cpp:10-37).
//
// The reference evaluates, row by row and left to right,
//     S(r,c) = ((x(r,c) + S(r-1,c)) + S(r,c-1)) - S(r-1,c-1)        (sat.cpp:33)
// Every S depends only on its up, left and up-left neighbours, so any schedule
// that respects those dependencies and performs the same three IEEE additions
// reproduces the reference table bit for bit. This kernel runs that recurrence
// as a systolic wavefront:
//   * a CTA owns a strip of 1024 columns of one table (8 warps x 32 lanes x 4
//     columns); lane l of warp w handles row r at step T = r + 32 w + l, so the
//     lanes of a warp sweep one anti-diagonal band;
//   * S(r, left column) arrives from lane l-1 by a register shuffle of the value
//     it produced one step earlier; warp boundaries hand over through a
//     double-buffered shared-memory slot, one __syncthreads per step;
//   * strips of wider maps are chained through a global edge column and a
//     release/acquire row counter; tiles are claimed from an atomic counter in
//     (table, strip) order, so the strip a CTA waits on is always already running.
// Loads of the source row slice are 16-byte vectors; the table is written in the
// shifted layout (padded element (i,j) at table[i*ld + 1 + j]) so each lane's
// four outputs land as two aligned 16-byte stores. Non-finite inputs are
// reported as the smallest row-major index (sat.cpp:28-32 semantics).
#include "common.cuh"
#include "kernels.cuh"

namespace uwb {

namespace {

constexpr int kSatK = 4;
constexpr int kSatWarps = 8;
constexpr int kSatStripCols = kSatWarps * kWarp * kSatK; // 1024
constexpr int kPublishEvery = 8;

template <typename T>
__device__ __forceinline__ void load_slice(const T* row, int64_t c0, int nvalid, bool vec_ok,
                                           double (&x)[kSatK]);

template <>
__device__ __forceinline__ void load_slice<float>(const float* row, int64_t c0, int nvalid,
                                                  bool vec_ok, double (&x)[kSatK]) {
    if (vec_ok && nvalid == kSatK) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(row + c0));
        x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else {
#pragma unroll
        for (int j = 0; j < kSatK; ++j) x[j] = j < nvalid ? static_cast<double>(__ldg(row + c0 + j)) : 0.0;
    }
}

template <>
__device__ __forceinline__ void load_slice<double>(const double* row, int64_t c0, int nvalid,
                                                   bool vec_ok, double (&x)[kSatK]) {
    if (vec_ok && nvalid == kSatK) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(row + c0));
        const double2 b = __ldg(reinterpret_cast<const double2*>(row + c0 + 2));
        x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
    } else {
#pragma unroll
        for (int j = 0; j < kSatK; ++j) x[j] = j < nvalid ? __ldg(row + c0 + j) : 0.0;
    }
}

template <typename T>
__global__ void __launch_bounds__(kSatWarps * kWarp)
sat_systolic_kernel(SatLaunch L) {
    __shared__ double edge_s[kSatWarps][2];
    __shared__ long long tile_s;

    const int warp = threadIdx.x / kWarp;
    const int lane = threadIdx.x % kWarp;
    const int64_t n_tiles = L.n_jobs * L.strips;

    for (;;) {
        if (threadIdx.x == 0) tile_s = static_cast<long long>(atomicAdd(L.tile_counter, 1u));
        __syncthreads();
        const int64_t tile = tile_s;
        __syncthreads();
        if (tile >= n_tiles) return;

        const int64_t job = tile / L.strips;
        const int strip = static_cast<int>(tile % L.strips);
        const SatJobView J = sat_job(L, job);

        const int64_t c_strip0 = static_cast<int64_t>(strip) * kSatStripCols;
        const int64_t strip_cols = imin(kSatStripCols, L.cols - c_strip0);
        const int nwa = static_cast<int>((strip_cols + kWarp * kSatK - 1) / (kWarp * kSatK));
        const int64_t c0 = c_strip0 + static_cast<int64_t>(warp) * kWarp * kSatK + lane * kSatK;
        const int nvalid = static_cast<int>(imax(0, imin(kSatK, L.cols - c0)));

        double* table = J.table;
        // padded row 0 is identically zero (sat.hpp:11-13)
        for (int64_t c = threadIdx.x; c < strip_cols; c += blockDim.x)
            table[1 + 1 + c_strip0 + c] = 0.0;
        if (strip == 0 && threadIdx.x == 0) table[1] = 0.0;

        const bool has_left = strip > 0;
        const bool has_right = strip + 1 < L.strips;
        const int64_t edge_base = job * L.strips + strip;
        const double* ge_in = has_left ? L.gedge + (edge_base - 1) * L.edge_stride : nullptr;
        const unsigned* prog_in = has_left ? L.gprog + (edge_base - 1) : nullptr;
        double* ge_out = has_right ? L.gedge + edge_base * L.edge_stride : nullptr;
        unsigned* prog_out = has_right ? L.gprog + edge_base : nullptr;
        const bool edge_writer = has_right && warp == kSatWarps - 1 && lane == kWarp - 1;

        double prev[kSatK];
#pragma unroll
        for (int j = 0; j < kSatK; ++j) prev[j] = 0.0;
        double left_prev = 0.0; // S(r-1, left column)
        double my_last = 0.0;   // S(r, my last column), shuffled right next step
        unsigned avail = 0;

        const T* src = static_cast<const T*>(J.src);
        const int64_t steps = J.rows + static_cast<int64_t>(kWarp) * nwa - 1;
        for (int64_t t = 0; t < steps; ++t) {
            const int64_t r = t - static_cast<int64_t>(kWarp) * warp - lane;
            double left = __shfl_up_sync(0xffffffffu, my_last, 1);
            const bool in_rows = r >= 0 && r < J.rows;
            if (lane == 0) {
                if (warp == 0) {
                    left = 0.0;
                    if (has_left && in_rows) {
                        while (avail <= static_cast<unsigned>(r)) avail = ld_acquire_u32(prog_in);
                        left = ge_in[r];
                    }
                } else {
                    left = edge_s[warp - 1][(t - 1) & 1];
                }
            }
            const bool active = warp < nwa && in_rows && nvalid > 0;
            if (active) {
                double x[kSatK];
                load_slice<T>(src + r * L.ld, c0, nvalid, L.vec_ok, x);
                double s_left = left, a_left = left_prev;
#pragma unroll
                for (int j = 0; j < kSatK; ++j) {
                    if (j < nvalid) {
                        if (!isfinite(x[j]))
                            report_min(J.nonfinite, static_cast<unsigned long long>(
                                                        (J.row0 + r) * L.cols + c0 + j));
                        // sat.cpp:33: out[c+1] = v + above[c+1] + out[c] - above[c]
                        const double s = dsub(dadd(dadd(x[j], prev[j]), s_left), a_left);
                        a_left = prev[j];
                        prev[j] = s;
                        s_left = s;
                    }
                }
                double* out = table + (r + 1) * L.table_ld + 1 + 1 + c0;
                if (nvalid == kSatK) {
                    reinterpret_cast<double2*>(out)[0] = make_double2(prev[0], prev[1]);
                    reinterpret_cast<double2*>(out)[1] = make_double2(prev[2], prev[3]);
                } else {
#pragma unroll
                    for (int j = 0; j < kSatK; ++j)
                        if (j < nvalid) out[j] = prev[j];
                }
                if (strip == 0 && warp == 0 && lane == 0) table[(r + 1) * L.table_ld + 1] = 0.0;
                my_last = s_left;
                left_prev = left;
                if (lane == kWarp - 1) edge_s[warp][t & 1] = my_last;
                if (edge_writer) {
                    ge_out[r] = my_last;
                    if ((r + 1) % kPublishEvery == 0 || r + 1 == J.rows)
                        st_release_u32(prog_out, static_cast<unsigned>(r + 1));
                }
            }
            __syncthreads();
        }
    }
}

} // namespace

std::atomic<uint64_t> g_kernel_launches{0};

cudaError_t launch_sat(const SatLaunch& L, int dtype, cudaStream_t stream) {
    const int64_t n_tiles = L.n_jobs * L.strips;
    if (n_tiles == 0) return cudaSuccess;
    ++g_kernel_launches;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (dtype == UWB_F32)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sat_systolic_kernel<float>,
                                                      kSatWarps * kWarp, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sat_systolic_kernel<double>,
                                                      kSatWarps * kWarp, 0);
    const int64_t grid = imin(n_tiles, static_cast<int64_t>(sms) * max(per_sm, 1));
    if (dtype == UWB_F32)
        sat_systolic_kernel<float><<<static_cast<unsigned>(grid), kSatWarps * kWarp, 0, stream>>>(L);
    else
        sat_systolic_kernel<double><<<static_cast<unsigned>(grid), kSatWarps * kWarp, 0, stream>>>(L);
    return cudaGetLastError();
}

int64_t sat_strips(int64_t cols) { return (cols + kSatStripCols - 1) / kSatStripCols; }

} // namespace uwb
