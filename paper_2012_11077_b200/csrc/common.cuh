// Shared device helpers for the uwbvital B200 kernels.
//
// Exactness rule for every kernel in this library: the reference computes in
// IEEE fp64 on x86-64 without FMA contraction, so each sum and product below is
// written with an explicit round-to-nearest intrinsic, in the reference's
// association, and the library is compiled with --fmad=false as a second guard.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "uwbvital_b200.h"

namespace uwb {

constexpr int kWarp = 32;

__host__ __device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

template <typename T>
__device__ __forceinline__ double widen(T v) {
    return static_cast<double>(v);
}

// Row-major cell index used for "first offending cell" reporting
// (sat.cpp:28-32 and cfar.cpp:85-92 report the first cell in row-major order).
__device__ __forceinline__ void report_min(unsigned long long* slot, unsigned long long idx) {
    if (slot) atomicMin(slot, idx);
}

__device__ __forceinline__ double ld_acquire_f64(const double* p) {
    double v;
    asm volatile("ld.acquire.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Streaming loads that should not pollute L1.
__device__ __forceinline__ float4 ldg_stream_f4(const float* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

} // namespace uwb

// Host-side launch-error helper.
#define UWB_CUDA_TRY(expr)                                                                 \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess) return uwb::set_cuda_error(_e, #expr);                      \
    } while (0)

namespace uwb {
// Implemented in capi.cu: records the message for uwb_last_error().
uwb_status set_error(uwb_status s, const char* msg, int64_t row = -1, int64_t col = -1);
uwb_status set_cuda_error(cudaError_t e, const char* what);
} // namespace uwb
