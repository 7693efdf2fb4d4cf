// Achievable DRAM rate for the SAT's traffic mix: read 4 bytes, write 8 bytes per
// element (fp32 -> fp64 stream), 16-byte vector loads / stores, grid-stride.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void widen(const float4* __restrict__ in, double2* __restrict__ out, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = in[i];
        out[2 * i] = make_double2(v.x, v.y);
        out[2 * i + 1] = make_double2(v.z, v.w);
    }
}
__global__ void copy4(const float4* __restrict__ in, float4* __restrict__ out, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

int main() {
    const size_t n = size_t(4096) * 1024 * 1024; // config-3 cells
    float4* in;
    double2* out;
    cudaMalloc(&in, n * 4);
    cudaMalloc(&out, n * 8);
    cudaMemset(in, 0, n * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int grid_mult : {4, 8, 16}) {
        const int grid = sms * grid_mult;
        widen<<<grid, 512>>>(in, out, n / 4);
        cudaEventRecord(a);
        for (int k = 0; k < 5; ++k) widen<<<grid, 512>>>(in, out, n / 4);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 5;
        printf("widen f32->f64 (grid %d x 512): %.2f ms, %.0f GB/s (12 B/elem)\n", grid, ms, 12.0 * n / ms / 1e6);
        copy4<<<grid, 512>>>(in, reinterpret_cast<float4*>(out), n / 4);
        cudaEventRecord(a);
        for (int k = 0; k < 5; ++k) copy4<<<grid, 512>>>(in, reinterpret_cast<float4*>(out), n / 4);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        ms /= 5;
        printf("copy f32 (grid %d x 512): %.2f ms, %.0f GB/s (8 B/elem)\n", grid, ms, 8.0 * n / ms / 1e6);
    }
    return 0;
}
