// Dependent-chain latencies on this GPU: DADD (rn), DMUL, SHFL (64-bit as two 32-bit), LDS.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dadd(double* out, long long* cyc, double a, int n) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, a);
    long long t1 = clock64();
    out[0] = x;
    cyc[0] = t1 - t0;
}
__global__ void k_fadd(float* out, long long* cyc, float a, int n) {
    float x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __fadd_rn(x, a);
    long long t1 = clock64();
    out[0] = x;
    cyc[0] = t1 - t0;
}
__global__ void k_shfl(double* out, long long* cyc, double a, int n) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_up_sync(0xffffffffu, x, 1);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl_dadd(double* out, long long* cyc, double a, int n) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(__shfl_up_sync(0xffffffffu, x, 1), a);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double* d; float* f; long long* c;
    cudaMalloc(&d, 1024); cudaMalloc(&f, 1024); cudaMalloc(&c, 64);
    const int n = 4096;
    long long h;
    k_dadd<<<1, 1>>>(d, c, 1.0000001, n); cudaDeviceSynchronize();
    k_dadd<<<1, 1>>>(d, c, 1.0000001, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent: %.2f cycles\n", double(h) / n);
    k_fadd<<<1, 1>>>(f, c, 1.0001f, n); cudaDeviceSynchronize();
    k_fadd<<<1, 1>>>(f, c, 1.0001f, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("FADD dependent: %.2f cycles\n", double(h) / n);
    k_shfl<<<1, 32>>>(d, c, 1.0, n); cudaDeviceSynchronize();
    k_shfl<<<1, 32>>>(d, c, 1.0, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("SHFL.UP f64 dependent: %.2f cycles\n", double(h) / n);
    k_shfl_dadd<<<1, 32>>>(d, c, 1.0, n); cudaDeviceSynchronize();
    k_shfl_dadd<<<1, 32>>>(d, c, 1.0, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("SHFL.UP f64 + DADD dependent: %.2f cycles\n", double(h) / n);
    return 0;
}
