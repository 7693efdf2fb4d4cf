// RFRM ingest: the reference's frame file holds a radar frame
// trace by trace (frame_io.hpp:10-23: "RFRM", u16 version, u32 m_samples,
// u32 n_traces, f64 fast_rate, f64 prf, then n_traces x m_samples f32). The
// detection chain wants it range-major (row = fast-time sample, column = trace,
// RadarFrame::data). The host validates the file image exactly as read_frame
// does (frame_io.cpp:69-122, same FormatError messages); the payloads of a
// batch of files are copied to the device as they lie and transposed there:
// 32 x 32 tiles through shared memory, both the trace-major reads and the
// range-major writes coalesced, each value widened exactly (f32 -> f32/f64),
// and the first non-finite sample of each record reported for
// RadarFrame::validate (pipeline.cpp:27-38).
#include "common.cuh"
#include "kernels.cuh"

namespace uwb {

namespace {

constexpr int kTile = 32;

template <typename Out>
__global__ void __launch_bounds__(kTile * 8) rfrm_transpose_kernel(const float* payload, int64_t m, int64_t n,
                                                                   Out* frames, unsigned long long* first_bad) {
    __shared__ float tile[kTile][kTile + 1];
    const int64_t rec = blockIdx.z;
    const float* in = payload + rec * m * n;          // [trace][sample]
    Out* out = frames + rec * m * n;                  // [sample][trace]
    const int64_t s0 = static_cast<int64_t>(blockIdx.x) * kTile; // samples
    const int64_t t0 = static_cast<int64_t>(blockIdx.y) * kTile; // traces
    const int tx = threadIdx.x % kTile, ty = threadIdx.x / kTile; // 32 x 8 threads
    for (int k = ty; k < kTile; k += 8) {
        const int64_t t = t0 + k, s = s0 + tx;
        float v = 0.0f;
        if (t < n && s < m) {
            v = __ldg(in + t * m + s);
            if (!isfinite(v) && first_bad) report_min(first_bad + rec, static_cast<unsigned long long>(s * n + t));
        }
        tile[k][tx] = v;
    }
    __syncthreads();
    for (int k = ty; k < kTile; k += 8) {
        const int64_t s = s0 + k, t = t0 + tx;
        if (s < m && t < n) out[s * n + t] = static_cast<Out>(tile[tx][k]);
    }
}

} // namespace

cudaError_t launch_rfrm_transpose(const float* payload, int64_t n_rec, int64_t m, int64_t n, int out_dtype,
                                  void* frames, unsigned long long* first_bad, cudaStream_t stream) {
    if (n_rec == 0) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>((m + kTile - 1) / kTile), static_cast<unsigned>((n + kTile - 1) / kTile),
                    static_cast<unsigned>(n_rec));
    ++g_kernel_launches;
    if (out_dtype == UWB_F32)
        rfrm_transpose_kernel<float><<<grid, kTile * 8, 0, stream>>>(payload, m, n, static_cast<float*>(frames),
                                                                       first_bad);
    else
        rfrm_transpose_kernel<double><<<grid, kTile * 8, 0, stream>>>(payload, m, n, static_cast<double*>(frames),
                                                                        first_bad);
    return cudaGetLastError();
}

} // namespace uwb
