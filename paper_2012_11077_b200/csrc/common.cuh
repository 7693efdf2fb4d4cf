// Shared device helpers for the uwbvital B200 kernels.
//
// Exactness rule for every kernel in this library: the reference computes in
// IEEE fp64 on x86-64 without FMA contraction, so each sum and product below is
// written with an explicit round-to-nearest intrinsic, in the reference's
// association, and the library is compiled with --fmad=false as a second guard.
#pragma once

#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "uwbvital_b200.h"

// Device-side bounds checks (-DUWB_DEVICE_CHECKS, UWB_DEVICE_CHECKS=1 python
// paper_2012_11077_b200/build.py --force): every global / shared index the
// kernels compute on their hot paths is asserted inside its buffer; a failure
// prints the condition and traps. The stand-in for compute-sanitizer, which is
// closed on this GPU pool. Compiled out of the release build.
#ifdef UWB_DEVICE_CHECKS
#include <cstdio>
#define UWB_DCHECK(cond)                                                                   \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            printf("UWB_DCHECK failed at %s:%d: %s (block %d, thread %d)\n", __FILE__, __LINE__, #cond, \
                   static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));           \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define UWB_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

// Tuning knobs (ring depth, occupancy, chunking ...) read from the environment
// exist only in a tuning build (-DUWB_TUNING_KNOBS, scripts/ probes); the
// release library reads no environment variable, so nothing outside the call
// arguments can change what a call computes or how.
#ifdef UWB_TUNING_KNOBS
#include <cstdlib>
#define UWB_KNOB(name) std::getenv(name)
#else
#define UWB_KNOB(name) (static_cast<const char*>(nullptr))
#endif

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
// Spin until *p >= need: relaxed polls (an acquire load per poll invalidates the
// SM's whole L1 each time, which stalls the other warps on the SM), then one
// acquire fence. Returns the value seen.
__device__ __forceinline__ unsigned wait_count_geq(const unsigned* p, unsigned need) {
    unsigned v;
    for (;;) {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
        if (v >= need) break;
        __nanosleep(100);
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// First non-finite cell (row-major) of columns [c, c + n) in source rows [0, rows_end).
template <typename T>
__device__ __noinline__ int first_nonfinite(const T* src, int64_t ld, int c, int n, int rows_end, int* col) {
    for (int r = 0; r < rows_end; ++r)
        for (int k = 0; k < n; ++k)
            if (!isfinite(widen(src[static_cast<int64_t>(r) * ld + c + k]))) {
                *col = c + k;
                return r;
            }
    return INT_MAX;
}

// ---- mbarrier + bulk async copy (TMA engine, 1-D form) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// global -> shared bulk copy completing `bytes` of transaction on `bar`
// (bytes, src and dst 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "UWB_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra UWB_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Blocking parity wait on a shared-window address; the thread may be suspended
// in the barrier unit for up to kHintNs per try.
template <unsigned kHintNs>
__device__ __forceinline__ void mbar_wait_u(unsigned bar, unsigned parity) {
    if constexpr (kHintNs == 0) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "UWB_WAITZ_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            "@!p bra UWB_WAITZ_%=;\n"
            "}\n" ::"r"(bar),
            "r"(parity)
            : "memory");
        return;
    }
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "UWB_WAITU_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra UWB_WAITU_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity), "n"(kHintNs)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_u(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// ---- cp.async (LDGSTS) small copies ----
__device__ __forceinline__ void cp_async_4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_16(unsigned dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
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
