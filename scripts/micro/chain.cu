// Step-latency probe for the single-map SAT chain (sat_cluster.cu): one warp, the
// dependent chain of one systolic step (64-bit shuffle from the left lane, select,
// 2 x columns dependent DADDs), with the step's side work added piece by piece.
//   v0: shfl_up(f64) + 4 DADD                      (the bare chain, kC = 2)
//   v1: v0 + lane-0 select + second 64-bit shuffle  (edge hand-over broadcast)
//   v2: v1 + LDS.128 source load + 2 off-chain DADDs (x + prev)
//   v3: v2 + STG.128 of the two results
//   v4: v3 with 4 columns per lane (8 dependent DADDs per shuffle)
//   v5: v0 + lane-0 select from a register (no second shuffle)
//   v6: v5 + LDS.128 + off-chain DADDs + STG.128 to a row per lane (the kernel's store pattern)
//   v8: v0 with lane 0's hand-over value added by a predicated DADD pair (no select)
//   v7: v6 + a predicated strong 8-byte store per step (lane 31's hand-over)
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double dadd2(double a, double b) { return __dadd_rn(a, b); }

template <int V>
__global__ void k(double* out, const double* src, long long* cyc, int n, double e) {
    __shared__ double2 ring[64 * 32];
    const int lane = threadIdx.x;
    for (int i = lane; i < 64 * 32; i += 32) ring[i] = make_double2(src[i & 1023], src[(i + 7) & 1023]);
    __syncwarp();
    double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0, lp = 0.0;
    double* o = out + lane * 4;
    double* o2 = out + 2 * lane - 136 * lane + 136 * 40; // lane l writes row i - l
    long long g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < n; ++i) {
        double x0 = 0.25, x1 = 0.5, x2 = 0.125, x3 = 0.75;
        if (V >= 2 && V != 5 && V != 8) {
            const double2 x = ring[((i & 63) << 5) + lane];
            x0 = x.x, x1 = x.y;
        }
        const double a0 = dadd2(x0, p0), a1 = dadd2(x1, p1);
        double left = __shfl_up_sync(0xffffffffu, V == 4 ? p3 : p1, 1);
        if (V >= 5 && V != 8) {
            if (lane == 0) left = e;
        } else if (V >= 1) {
            const double fs = __shfl_sync(0xffffffffu, e, i & 7);
            if (lane == 0) left = fs;
        }
        double t0;
        if (V == 8) {
            // lane 0 adds its hand-over value, the others the shuffled one: two predicated
            // additions into one register instead of a select between the shuffle and the add
            asm volatile(
                "{\n.reg .pred p;\nsetp.eq.u32 p, %4, 0;\n@p add.rn.f64 %0, %1, %2;\n@!p add.rn.f64 %0, %1, %3;\n}"
                : "=d"(t0)
                : "d"(a0), "d"(e), "d"(left), "r"(lane));
        } else {
            t0 = dadd2(a0, left);
        }
        const double s0 = dadd2(t0, -lp);
        const double s1 = dadd2(dadd2(a1, s0), -p0);
        if (V == 4) {
            const double a2 = dadd2(x2, p2), a3 = dadd2(x3, p3);
            const double s2 = dadd2(dadd2(a2, s1), -p1);
            const double s3 = dadd2(dadd2(a3, s2), -p2);
            p2 = s2, p3 = s3;
            if (V >= 3) reinterpret_cast<double2*>(o)[1] = make_double2(s2, s3);
        }
        lp = left, p0 = s0, p1 = s1;
        if (V >= 6 && V != 8) {
            reinterpret_cast<double2*>(o2)[0] = make_double2(s0, s1);
            o2 += 136;
            if (V >= 7)
                asm volatile("{\n.reg .pred p;\nsetp.eq.u32 p, %2, 31;\n@p st.relaxed.gpu.f64 [%0], %1;\n}" ::"l"(out + 8 * i),
                             "d"(s1), "r"(lane));
        } else if (V >= 3 && V != 8) {
            reinterpret_cast<double2*>(o)[0] = make_double2(s0, s1);
            o += 128;
        }
    }
    long long t1 = clock64();
    out[lane] = p0 + p1 + p2 + p3;
    long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (lane == 0) cyc[V] = t1 - t0, cyc[8 + V] = g1 - g0;
}

int main() {
    double *o, *s;
    long long* c;
    const int n = 4096;
    cudaMalloc(&o, sizeof(double) * (136 * (n + 80) + 256));
    cudaMalloc(&s, sizeof(double) * 1024);
    cudaMemset(s, 0, sizeof(double) * 1024);
    cudaMallocManaged(&c, 256);
    for (int rep = 0; rep < 2; ++rep) {
        k<0><<<1, 32>>>(o, s, c, n, 1.0);
        k<1><<<1, 32>>>(o, s, c, n, 1.0);
        k<2><<<1, 32>>>(o, s, c, n, 1.0);
        k<3><<<1, 32>>>(o, s, c, n, 1.0);
        k<4><<<1, 32>>>(o, s, c, n, 1.0);
        k<5><<<1, 32>>>(o, s, c, n, 1.0);
        k<6><<<1, 32>>>(o, s, c, n, 1.0);
        k<7><<<1, 32>>>(o, s, c, n, 1.0);
        k<8><<<1, 32>>>(o, s, c, n, 1.0);
        cudaDeviceSynchronize();
    }
    for (int v = 0; v < 9; ++v)
        printf("v%d: %.1f cycles per step, %.1f ns per step, SM clock %.0f MHz\n", v, c[v] / (double)n,
               c[8 + v] / (double)n, 1e3 * c[v] / (double)c[8 + v]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
