// FP64 add-pipe throughput probe (the denominator of the config-2 front end's
// roofline): independent __dadd_rn chains on every SM, CUDA-event timed.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, double b, int n) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < n; ++i) {
        x0 = __dadd_rn(x0, b); x1 = __dadd_rn(x1, b); x2 = __dadd_rn(x2, b); x3 = __dadd_rn(x3, b);
        x4 = __dadd_rn(x4, b); x5 = __dadd_rn(x5, b); x6 = __dadd_rn(x6, b); x7 = __dadd_rn(x7, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void m(double* out, double b, int n) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < n; ++i) {
        x0 = __dmul_rn(x0, b); x1 = __dmul_rn(x1, b); x2 = __dmul_rn(x2, b); x3 = __dmul_rn(x3, b);
        x4 = __dmul_rn(x4, b); x5 = __dmul_rn(x5, b); x6 = __dmul_rn(x6, b); x7 = __dmul_rn(x7, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, n = 1 << 14;
    double* o; cudaMalloc(&o, sizeof(double) * blocks * threads);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int which = 0; which < 2; ++which) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            if (which == 0) k<<<blocks, threads>>>(o, 1e-3, n); else m<<<blocks, threads>>>(o, 1.0000001, n);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        const double ops = 8.0 * n * blocks * threads;
        printf("{\"op\": \"%s\", \"gops\": %.1f, \"ms\": %.3f, \"sms\": %d}\n", which ? "dmul" : "dadd", ops / (best * 1e-3) / 1e9, best, sms);
    }
    return 0;
}
