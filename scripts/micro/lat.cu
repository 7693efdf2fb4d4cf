// Latency probe: dependent DADD chain, dependent shfl chain, LDS chain (one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = __dadd_rn(x, b); x = __dadd_rn(x, -b); x = __dadd_rn(x, b); x = __dadd_rn(x, -b); }
    long long t1 = clock64();
    double y = a;
    for (int i = 0; i < n; ++i) { y = __shfl_up_sync(0xffffffffu, y, 1) + 0.0; }
    long long t2 = clock64();
    float z = (float)a; 
    for (int i = 0; i < n; ++i) { z = __fadd_rn(z, (float)b); z = __fadd_rn(z, (float)-b); z = __fadd_rn(z, (float)b); z = __fadd_rn(z, (float)-b); }
    long long t3 = clock64();
    int u = (int)a;
    for (int i = 0; i < n; ++i) { u = __shfl_sync(0xffffffffu, u, (threadIdx.x + 1) & 31); }
    long long t4 = clock64();
    out[threadIdx.x] = x + y + z + u;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 64);
    int n = 4096;
    k<<<1, 32>>>(o, c, 1.0, 0.5, n); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 1.0, 0.5, n); cudaDeviceSynchronize();
    printf("DADD dep latency %.2f cyc, shfl_up(f64)+DADD %.2f cyc, FADD %.2f cyc, shfl(u32) %.2f cyc\n",
           c[0] / (4.0 * n), c[1] / (double)n, c[2] / (4.0 * n), c[3] / (double)n);
    return 0;
}
