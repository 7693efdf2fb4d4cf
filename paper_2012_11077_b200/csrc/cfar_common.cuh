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
    UWB_DCHECK(!valid || (r >= L.geo.row_lo && r < L.geo.row_hi && c >= 0 && c < L.cols &&
                          map >= 0 && map * L.geo.n_slabs < L.n_jobs));
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

// ---- shared by the ring-fed (cfar_ring.cu) and fused (cfar_fused.cu) CFAR kernels ----

// Per-column constants of one output column.
struct ColConst {
    unsigned xa, xb, ya, yb; // byte offsets of the four tap columns within a ring row
    int ow, gw;              // clamped outer / guard widths
    bool ok;
};

__device__ __forceinline__ ColConst col_const(int c, int cols, int hc, int gc, int e_lo) {
    ColConst k;
    k.ok = c < cols;
    const int cc = k.ok ? c : cols - 1;
    const int oc0 = clamp_lo32(cc, hc), oc1 = clamp_hi32(cc, hc, cols);
    const int gc0 = clamp_lo32(cc, gc), gc1 = clamp_hi32(cc, gc, cols);
    k.ow = oc1 - oc0 + 1;
    k.gw = gc1 - gc0 + 1;
    k.xa = 8u * static_cast<unsigned>(kTabShift + oc0 - e_lo);
    k.xb = 8u * static_cast<unsigned>(kTabShift + 1 + oc1 - e_lo);
    k.ya = 8u * static_cast<unsigned>(kTabShift + gc0 - e_lo);
    k.yb = 8u * static_cast<unsigned>(kTabShift + 1 + gc1 - e_lo);
    return k;
}

__device__ __forceinline__ double tap(const char* row, unsigned off) {
    return *reinterpret_cast<const double*>(row + off);
}
// Four-tap sums of one cell: sat.hpp:32-33 for outer and guard, then outer - guard.
__device__ __forceinline__ double train_sum(const ColConst& k, const char* rA, const char* rB, const char* rC,
                                            const char* rD) {
    const double rs_o = dsub(dadd(tap(rA, k.xa), tap(rB, k.xb)), dadd(tap(rA, k.xb), tap(rB, k.xa)));
    const double rs_g = dsub(dadd(tap(rC, k.ya), tap(rD, k.yb)), dadd(tap(rC, k.yb), tap(rD, k.ya)));
    return dsub(rs_o, rs_g);
}

// Mask words, optional per-cell outputs and detections of one thread's block
// (rows r0..r0+RS-1, columns c_first + 32 j); lane k*CPT+j stores word (k, j).
template <int RS, int CPT>
__device__ __forceinline__ void emit_block(const CfarLaunch& L, int64_t map, int r0, int r_last, int c_word0,
                                           int c_first, const bool (&okc)[CPT], const bool (&hit)[RS][CPT],
                                           const double (&v)[RS][CPT], const double (&thr)[RS][CPT],
                                           bool per_cell) {
    const int lane = threadIdx.x % kWarp;
    const int cols = static_cast<int>(L.cols);
    unsigned my_word = 0, any_bits = 0;
#pragma unroll
    for (int k = 0; k < RS; ++k) {
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const unsigned b = __ballot_sync(0xffffffffu, hit[k][j]);
            any_bits |= b;
            if (lane == k * CPT + j) my_word = b;
        }
    }
    const int wk = lane / CPT, wj = lane % CPT;
    const int wc = c_word0 + wj * kWarp; // first column of the word
    if (lane < CPT * RS && r0 + wk <= r_last && wc < cols && L.mask_bits)
        L.mask_bits[map * L.mask_map_stride + (r0 + wk - L.geo.row_lo) * L.words_per_row + (wc >> 5)] = my_word;
    if (per_cell) { // parity runs only
#pragma unroll
        for (int k = 0; k < RS; ++k) {
#pragma unroll
            for (int j = 0; j < CPT; ++j) {
                if (okc[j] && r0 + k <= r_last) {
                    const int64_t cell =
                        (map * L.geo.out_rows() + (r0 + k - L.geo.row_lo)) * cols + c_first + j * kWarp;
                    if (L.mask_u8) L.mask_u8[cell] = hit[k][j] ? 1 : 0;
                    if (L.thresholds) L.thresholds[cell] = thr[k][j];
                }
            }
        }
    }
    if (any_bits) { // detections (about pfa of the cells plus targets)
#pragma unroll
        for (int k = 0; k < RS; ++k) {
#pragma unroll
            for (int j = 0; j < CPT; ++j) {
                const unsigned b = __ballot_sync(0xffffffffu, hit[k][j]);
                if (b) {
                    unsigned long long base = 0;
                    if (lane == 0) base = atomicAdd(L.det_counts + map, static_cast<unsigned long long>(__popc(b)));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (hit[k][j]) {
                        const unsigned long long slot = base + __popc(b & ((1u << lane) - 1u));
                        if (slot < static_cast<unsigned long long>(L.det_cap)) {
                            uwb_detection d;
                            d.row = static_cast<uint64_t>(r0 + k);
                            d.col = static_cast<uint64_t>(c_first + j * kWarp);
                            d.value = v[k][j];
                            d.threshold = thr[k][j];
                            L.dets[map * L.det_cap + slot] = d;
                        }
                    }
                }
            }
        }
    }
}

} // namespace uwb
