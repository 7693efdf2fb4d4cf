// Per-cell helpers shared by the CFAR kernels.
#pragma once

#include "common.cuh"
#include "kernels.cuh"

namespace uwb {

// cfar.cpp:47-55 (clamped window edges)
__device__ __forceinline__ int clamp_lo32(int c, int rad) {
    const int v = c - rad;
    return v < 0 ? 0 : v;
}
__device__ __forceinline__ int clamp_hi32(int c, int rad, int dim) {
    const int v = c + rad;
    return v >= dim ? dim - 1 : v;
}

// Emits the mask word, optional per-cell outputs and compacted detections for
// one row segment of 32 cells held by a warp (columns 32k .. 32k+31).
__device__ __forceinline__ void emit_cells(const CfarLaunch& L, int64_t map, int r, int c, bool valid, bool hit,
                                           double v, double thr) {
    const unsigned lane = threadIdx.x % kWarp;
    const unsigned bits = __ballot_sync(0xffffffffu, valid && hit);
    if (lane == 0 && L.mask_bits) {
        const int word = c >> 5;
        if (word < L.words_per_row)
            L.mask_bits[map * L.mask_map_stride + (r - L.geo.row_lo) * L.words_per_row + word] = bits;
    }
    if (valid && (L.mask_u8 || L.thresholds)) {
        const int64_t cell = (map * L.geo.out_rows() + (r - L.geo.row_lo)) * L.cols + c;
        if (L.mask_u8) L.mask_u8[cell] = hit ? 1 : 0;
        if (L.thresholds) L.thresholds[cell] = thr;
    }
    if (bits) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(L.det_counts + map, static_cast<unsigned long long>(__popc(bits)));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (valid && hit) {
            const unsigned long long slot = base + __popc(bits & ((1u << lane) - 1u));
            if (slot < static_cast<unsigned long long>(L.det_cap)) {
                uwb_detection d;
                d.row = static_cast<uint64_t>(r);
                d.col = static_cast<uint64_t>(c);
                d.value = v;
                d.threshold = thr;
                L.dets[map * L.det_cap + slot] = d;
            }
        }
    }
}

} // namespace uwb
