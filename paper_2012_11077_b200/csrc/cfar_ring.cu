// Kernel (d), production path: warp-specialised CA-CFAR over shared-memory rings
// of table rows.
//
// Replaces cfar_rows / run_cfar of /root/reference/proj/src/cfar.cpp:109-175 for
// the integral-image backend (cfar2d_integral, cfar.cpp:218-227).
//
// A CTA owns a W-column x 256-row tile of one job (W = 64 x consumer warps).
// One producer warp streams every table row the tile's windows touch into a
// shared-memory ring with the TMA engine (cp.async.bulk global->shared, one
// 16-byte-aligned row segment per copy), and the CUT row segments into a second
// ring; rows move in groups of 4 that complete on one "full" mbarrier. The
// consumer warps (two output columns per thread, c and c+32) wait on "full",
// evaluate 4 output rows, and hand slots back through "empty" mbarriers, so the
// two sides never meet at a CTA barrier. The eight taps of a cell are
// shared-memory reads:
//     RS = (t[r0][c0] + t[r1+1][c1+1]) - (t[r0][c1+1] + t[r1+1][c0])   (sat.hpp:32-33)
// sum = RS(outer) - RS(guard), T = alpha[n] * (sum / n), mask = cut > T
// (cfar.cpp:115-127).
//
// Threshold decision: the IEEE division is skipped on the common path, which
// compares cut with sum * (alpha[n] / n) (within a few ulp of T); a warp takes
// the exact path (the reference expression alpha[n] * (sum / n)) when any lane
// has cut within 1e-13 relative of it, a detection (whose record carries T), or
// when the threshold map is an output. Decisions equal the reference's `cut > T`.
#include <cstdlib>

#include "cfar_common.cuh"

namespace uwb {

namespace {

constexpr int kRingRows = 256;   // output rows per CTA
constexpr int kG = 4;            // rows per group (output step, copy group)
constexpr int kDefaultAhead = 2; // groups of look-ahead (UWB_RING_AHEAD overrides: 1..4)
constexpr int kColsPerThread = 2;

struct RingGeom {
    int ng;     // table row groups in the ring
    int nr;     // table row slots (ng * kG)
    int stride; // doubles per table slot
};

__host__ __device__ inline RingGeom ring_geom(int w, int hr, int hc, int ahead) {
    RingGeom g;
    // output rows r..r+3 read table rows r-hr .. r+4+hr: 2hr+5 rows, spread over
    // at most ceil((2hr+5)/4)+1 groups
    g.ng = (2 * hr + 5 + kG - 1) / kG + 1 + ahead;
    g.nr = g.ng * kG;
    g.stride = w + 2 * hc + 4;
    return g;
}

template <typename T>
inline size_t ring_smem_bytes(int w, int hr, int hc, int ahead) {
    const RingGeom g = ring_geom(w, hr, hc, ahead);
    const int ncg = 1 + ahead;
    return sizeof(double) * static_cast<size_t>(g.nr) * g.stride + sizeof(T) * static_cast<size_t>(ncg) * kG * w +
           2 * sizeof(uint64_t) * (g.ng + ncg + 1) + (sizeof(uint4) + sizeof(int2)) * kRingRows;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ double lds_f64(unsigned addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ float lds_f32(unsigned addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
template <typename T>
__device__ __forceinline__ double lds_cut(unsigned addr);
template <>
__device__ __forceinline__ double lds_cut<float>(unsigned addr) { return static_cast<double>(lds_f32(addr)); }
template <>
__device__ __forceinline__ double lds_cut<double>(unsigned addr) { return lds_f64(addr); }

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

// Four-tap sums of one cell: sat.hpp:32-33 for outer and guard, then outer - guard.
__device__ __forceinline__ double train_sum(const ColConst& k, unsigned rA, unsigned rB, unsigned rC, unsigned rD) {
    const double rs_o = dsub(dadd(lds_f64(rA + k.xa), lds_f64(rB + k.xb)), dadd(lds_f64(rA + k.xb), lds_f64(rB + k.xa)));
    const double rs_g = dsub(dadd(lds_f64(rC + k.ya), lds_f64(rD + k.yb)), dadd(lds_f64(rC + k.yb), lds_f64(rD + k.ya)));
    return dsub(rs_o, rs_g);
}

template <typename T, int NCW, int AHEAD>
__global__ void __launch_bounds__((NCW + 1) * kWarp)
cfar_ws_kernel(CfarLaunch L) {
    constexpr int W = NCW * kWarp * kColsPerThread;
    constexpr int kNcg = 1 + AHEAD; // CUT groups in the ring
    extern __shared__ __align__(16) unsigned char ring_smem[];
    const RingGeom G = ring_geom(W, L.hr, L.hc, AHEAD);
    double* slots = reinterpret_cast<double*>(ring_smem);
    T* cuts = reinterpret_cast<T*>(slots + static_cast<size_t>(G.nr) * G.stride);
    uint64_t* full_t = reinterpret_cast<uint64_t*>(cuts + static_cast<size_t>(kNcg) * kG * W);
    uint64_t* full_c = full_t + G.ng;
    uint64_t* empty_t = full_c + kNcg;
    uint64_t* empty_c = empty_t + G.ng;

    const int64_t job = blockIdx.y;
    const int64_t map = job / L.geo.n_slabs;
    const int64_t slab = job % L.geo.n_slabs;
    const int col_tile = static_cast<int>(blockIdx.x % L.col_tiles);
    const int chunk = static_cast<int>(blockIdx.x / L.col_tiles);
    const int rows = static_cast<int>(L.geo.rows), cols = static_cast<int>(L.cols);
    const int hr = L.hr, hc = L.hc, gr = L.gr, gc = L.gc;
    const int c0 = col_tile * W;
    const int ra = static_cast<int>(L.geo.owned_begin(slab)) + chunk * kRingRows;
    const int rb = min(ra + kRingRows, static_cast<int>(L.geo.owned_end(slab)));
    if (ra >= rb) return;
    const int trow0 = static_cast<int>(L.geo.table_begin(slab));
    const double* tab = L.table + job * L.table_stride;
    const int64_t ld = L.table_ld;
    const T* cut_base = static_cast<const T*>(L.maps) + map * L.map_stride;

    // table columns the strip touches, as a 16-byte aligned storage span
    const int jlo = max(0, c0 - hc);
    const int jhi = min(cols, c0 + W + hc);
    const int e_lo = (kTabShift + jlo) & ~1;
    const int e_hi = kTabShift + jhi;
    const unsigned copy_bytes = static_cast<unsigned>(((e_hi - e_lo) / 2 + 1) * 16);
    const int strip_w = min(W, cols - c0);
    const unsigned cut_bytes = static_cast<unsigned>(((strip_w * static_cast<int>(sizeof(T)) + 15) / 16) * 16);

    // padded table rows needed by output rows [ra, rb), in groups of kG from i_lo
    const int i_lo = max(0, ra - hr);
    const int i_hi = min(rows, rb + hr);
    const int n_steps = (rb - ra + kG - 1) / kG;

    // Per output row of the tile: the ring addresses of its four tap rows and
    // its clamped outer / guard heights, computed once (cfar.cpp:117-120).
    // (the ring, CUT and 2 * (ng + kNcg) barrier regions keep 16-byte alignment)
    uint4* tap_rows = reinterpret_cast<uint4*>(empty_c + kNcg);
    int2* heights = reinterpret_cast<int2*>(tap_rows + kRingRows);
    {
        const unsigned ring_base = smem_u32(slots);
        const unsigned row_bytes = static_cast<unsigned>(G.stride) * 8u;
        auto ring_addr = [&](int i) { return ring_base + static_cast<unsigned>((i - i_lo) % G.nr) * row_bytes; };
        for (int lr = threadIdx.x; lr < rb - ra; lr += blockDim.x) {
            const int r = ra + lr;
            const int iA = clamp_lo32(r, hr), iB = clamp_hi32(r, hr, rows) + 1;
            const int iC = clamp_lo32(r, gr), iD = clamp_hi32(r, gr, rows) + 1;
            tap_rows[lr] = make_uint4(ring_addr(iA), ring_addr(iB), ring_addr(iC), ring_addr(iD));
            heights[lr] = make_int2(iB - iA, iD - iC);
        }
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < G.ng + kNcg; ++s) {
            mbar_init(&full_t[s], 1);
            mbar_init(&empty_t[s], NCW);
        }
        mbar_fence_init();
    }
    __syncthreads();

    const int warp = threadIdx.x / kWarp;
    const int lane = threadIdx.x % kWarp;

    if (warp == NCW) {
        // =========================== producer warp ===========================
        if (lane != 0) return;
        const int last_grp = (i_hi - i_lo) / kG;
        int grp = 0, gslot = 0, gphase = 0; // next table group, its slot and empty-phase
        int cslot = 0, cphase = 0;
        for (int step = 0; step < n_steps; ++step) {
            const int r_last = min(ra + step * kG + kG, rb) - 1;
            const int need = min((clamp_hi32(r_last, hr, rows) + 1 - i_lo) / kG, last_grp);
            for (; grp <= need; ++grp) {
                if (grp >= G.ng) mbar_wait(&empty_t[gslot], static_cast<unsigned>(gphase ^ 1));
                const int first = i_lo + grp * kG;
                const int cnt = min(kG, i_hi + 1 - first);
                mbar_expect_tx(&full_t[gslot], copy_bytes * cnt);
                for (int k = 0; k < cnt; ++k)
                    bulk_g2s(slots + static_cast<size_t>(gslot * kG + k) * G.stride,
                             tab + static_cast<int64_t>(first + k - trow0) * ld + e_lo, copy_bytes, &full_t[gslot]);
                if (++gslot == G.ng) { gslot = 0; gphase ^= 1; }
            }
            if (step >= kNcg) mbar_wait(&empty_c[cslot], static_cast<unsigned>(cphase ^ 1));
            const int first = ra + step * kG;
            const int cnt = min(kG, rb - first);
            mbar_expect_tx(&full_c[cslot], cut_bytes * cnt);
            for (int k = 0; k < cnt; ++k)
                bulk_g2s(cuts + static_cast<size_t>(cslot * kG + k) * W,
                         cut_base + static_cast<int64_t>(first + k) * L.ld + c0, cut_bytes, &full_c[cslot]);
            if (++cslot == kNcg) { cslot = 0; cphase ^= 1; }
        }
        return;
    }

    // ============================ consumer warps ============================
    const unsigned cut_smem = smem_u32(cuts);
    const unsigned tap_smem = smem_u32(tap_rows);
    const unsigned ht_smem = smem_u32(heights);
    const int tc = warp * kWarp * kColsPerThread + lane; // my first column within the tile
    const ColConst K0 = col_const(c0 + tc, cols, hc, gc, e_lo);
    const ColConst K1 = col_const(c0 + tc + kWarp, cols, hc, gc, e_lo);
    const bool exact_always = L.thresholds != nullptr;

    int waited = -1, wslot = 0, wphase = 0; // full_t groups known resident
    int released = -1, rslot = 0;            // table groups handed back
    int cslot = 0, cphase = 0;
    // per-column alpha cache: n is constant over interior rows
    int n0c = -1, n1c = -1;
    double k0 = 0.0, k1 = 0.0;

    for (int step = 0; step < n_steps; ++step) {
        const int r0 = ra + step * kG;
        const int r_last = min(r0 + kG, rb) - 1;
        {
            const int need = (clamp_hi32(r_last, hr, rows) + 1 - i_lo) / kG;
            while (waited < need) {
                mbar_wait(&full_t[wslot], static_cast<unsigned>(wphase));
                ++waited;
                if (++wslot == G.ng) { wslot = 0; wphase ^= 1; }
            }
        }
        mbar_wait(&full_c[cslot], static_cast<unsigned>(cphase));
        const unsigned cut_grp = cut_smem + static_cast<unsigned>(cslot * kG * W) * sizeof(T);
        // phase 1: ring rows and clamped heights of the step's rows (table lookups)
        unsigned RA[kG], RB[kG], RC[kG], RD[kG];
        int HR[kG], HG[kG];
#pragma unroll
        for (int k = 0; k < kG; ++k) {
            const int lr = min(r0 + k, r_last) - ra;
            uint4 t;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w)
                         : "r"(tap_smem + 16u * static_cast<unsigned>(lr)));
            int2 h;
            asm volatile("ld.shared.v2.s32 {%0,%1}, [%2];" : "=r"(h.x), "=r"(h.y) : "r"(ht_smem + 8u * static_cast<unsigned>(lr)));
            RA[k] = t.x; RB[k] = t.y; RC[k] = t.z; RD[k] = t.w;
            HR[k] = h.x;
            HG[k] = h.y;
        }
        // phase 2: every cell of the step (loads first, decisions after)
        double v[kG][2], sum[kG][2], approx[kG][2];
        int n[kG][2];
        bool need_exact[kG][2], hit[kG][2];
        bool any_slow = false;
#pragma unroll
        for (int k = 0; k < kG; ++k) {
            const unsigned cut_row = cut_grp + static_cast<unsigned>(k * W) * sizeof(T);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const ColConst& K = j ? K1 : K0;
                v[k][j] = lds_cut<T>(cut_row + static_cast<unsigned>(tc + j * kWarp) * sizeof(T));
                sum[k][j] = train_sum(K, RA[k], RB[k], RC[k], RD[k]);
                n[k][j] = HR[k] * K.ow - HG[k] * K.gw;
            }
        }
#pragma unroll
        for (int k = 0; k < kG; ++k) {
            const bool row_ok = r0 + k <= r_last;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const ColConst& K = j ? K1 : K0;
                int& nc = j ? n1c : n0c;
                double& kc = j ? k1 : k0;
                if (n[k][j] != nc && row_ok) {
                    nc = n[k][j];
                    kc = ddiv(__ldg(L.alpha + n[k][j]), static_cast<double>(n[k][j]));
                }
                approx[k][j] = dmul(sum[k][j], kc);
                const bool ok = K.ok && row_ok;
                hit[k][j] = ok && v[k][j] > approx[k][j];
                need_exact[k][j] = ok && (exact_always || hit[k][j] || v[k][j] < 0.0 ||
                                          !(fabs(dsub(v[k][j], approx[k][j])) > 1e-13 * fabs(approx[k][j])));
                any_slow |= need_exact[k][j];
            }
        }
        // phase 3: the reference expression where it is needed (rare, warp-uniform branch)
        double thr[kG][2];
#pragma unroll
        for (int k = 0; k < kG; ++k) thr[k][0] = thr[k][1] = 0.0;
        if (__any_sync(0xffffffffu, any_slow)) {
#pragma unroll
            for (int k = 0; k < kG; ++k) {
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    if (need_exact[k][j]) {
                        thr[k][j] = dmul(__ldg(L.alpha + n[k][j]), ddiv(sum[k][j], static_cast<double>(n[k][j])));
                        hit[k][j] = v[k][j] > thr[k][j];
                        if (v[k][j] < 0.0)
                            report_min(L.first_bad + 2 * map + 1,
                                       static_cast<unsigned long long>(static_cast<int64_t>(r0 + k) * cols + c0 + tc +
                                                                       j * kWarp));
                    }
                }
            }
        }
        // phase 4: mask words (lane w stores word w of the 4x2 block), optional
        // per-cell outputs, detections
        {
            unsigned my_word = 0, any_bits = 0;
#pragma unroll
            for (int k = 0; k < kG; ++k) {
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const unsigned b = __ballot_sync(0xffffffffu, hit[k][j]);
                    any_bits |= b;
                    if (lane == k * 2 + j) my_word = b;
                }
            }
            const int wk = lane >> 1, wj = lane & 1;
            const int wc = c0 + warp * kWarp * kColsPerThread + wj * kWarp; // first column of the word
            if (lane < 2 * kG && r0 + wk <= r_last && wc < cols && L.mask_bits)
                L.mask_bits[map * L.mask_map_stride + static_cast<int64_t>(r0 + wk) * L.words_per_row + (wc >> 5)] =
                    my_word;
            if (exact_always || L.mask_u8) { // parity runs only
#pragma unroll
                for (int k = 0; k < kG; ++k) {
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const ColConst& K = j ? K1 : K0;
                        if (K.ok && r0 + k <= r_last) {
                            const int64_t cell = map * L.geo.rows * L.cols + static_cast<int64_t>(r0 + k) * cols +
                                                 c0 + tc + j * kWarp;
                            if (L.mask_u8) L.mask_u8[cell] = hit[k][j] ? 1 : 0;
                            if (L.thresholds) L.thresholds[cell] = thr[k][j];
                        }
                    }
                }
            }
            if (any_bits) { // detections (about pfa of the cells plus targets)
#pragma unroll
                for (int k = 0; k < kG; ++k) {
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const unsigned b = __ballot_sync(0xffffffffu, hit[k][j]);
                        if (b) {
                            unsigned long long base = 0;
                            if (lane == 0)
                                base = atomicAdd(L.det_counts + map, static_cast<unsigned long long>(__popc(b)));
                            base = __shfl_sync(0xffffffffu, base, 0);
                            if (hit[k][j]) {
                                const unsigned long long slot = base + __popc(b & ((1u << lane) - 1u));
                                if (slot < static_cast<unsigned long long>(L.det_cap)) {
                                    uwb_detection d;
                                    d.row = static_cast<uint64_t>(r0 + k);
                                    d.col = static_cast<uint64_t>(c0 + tc + j * kWarp);
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
        // hand back this step's CUT group and the table groups no later step reads
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&empty_c[cslot]);
            if (step + 1 < n_steps) {
                const int keep_row = max(0, r_last + 1 - hr);
                const int done = (keep_row - i_lo) / kG - 1; // groups entirely below keep_row
                while (released < done) {
                    ++released;
                    mbar_arrive(&empty_t[rslot]);
                    if (++rslot == G.ng) rslot = 0;
                }
            }
        }
        if (++cslot == kNcg) { cslot = 0; cphase ^= 1; }
    }
}

template <typename T, int NCW, int AHEAD>
cudaError_t go(const CfarLaunch& L0, size_t smem, cudaStream_t stream) {
    constexpr int W = NCW * kWarp * kColsPerThread;
    CfarLaunch L = L0;
    L.col_tiles = (L.cols + W - 1) / W;
    L.row_chunks = (L.geo.slab_rows + kRingRows - 1) / kRingRows;
    const dim3 grid(static_cast<unsigned>(L.col_tiles * L.row_chunks), static_cast<unsigned>(L.n_jobs), 1);
    cudaError_t e = cudaFuncSetAttribute(cfar_ws_kernel<T, NCW, AHEAD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    ++g_kernel_launches;
    cfar_ws_kernel<T, NCW, AHEAD><<<grid, (NCW + 1) * kWarp, smem, stream>>>(L);
    return cudaGetLastError();
}

template <typename T>
cudaError_t go_cfg(const CfarLaunch& L, int ncw, int ahead, size_t smem, cudaStream_t stream) {
    if (ncw == 4) {
        switch (ahead) {
            case 1: return go<T, 4, 1>(L, smem, stream);
            case 3: return go<T, 4, 3>(L, smem, stream);
            case 4: return go<T, 4, 4>(L, smem, stream);
            default: return go<T, 4, 2>(L, smem, stream);
        }
    }
    switch (ahead) {
        case 1: return go<T, 2, 1>(L, smem, stream);
        case 3: return go<T, 2, 3>(L, smem, stream);
        case 4: return go<T, 2, 4>(L, smem, stream);
        default: return go<T, 2, 2>(L, smem, stream);
    }
}

} // namespace

// Returns cudaErrorNotSupported when the rings do not fit or the layout does
// not allow 16-byte bulk copies of the CUT rows (caller falls back).
cudaError_t launch_cfar_ring(const CfarLaunch& L, int dtype, cudaStream_t stream) {
    if (getenv("UWB_CFAR_SIMPLE")) return cudaErrorNotSupported;
    if (L.geo.rows >= (int64_t(1) << 31) || L.cols >= (int64_t(1) << 30)) return cudaErrorNotSupported;
    const bool f32 = dtype == UWB_F32;
    const size_t esz = f32 ? 4 : 8;
    // CUT rows are bulk-copied in 16-byte units: rows must start 16-byte aligned
    // and the row pitch must keep them so; a partial last strip may read up to
    // 12 bytes past its last cell, which must stay inside the row pitch.
    if ((reinterpret_cast<uintptr_t>(L.maps) % 16) || ((L.ld * esz) % 16) || ((L.map_stride * esz) % 16))
        return cudaErrorNotSupported;
    if (((L.cols * esz) % 16) && L.ld * esz < ((L.cols * esz + 15) / 16) * 16) return cudaErrorNotSupported;
    int ahead = kDefaultAhead;
    if (const char* a = getenv("UWB_RING_AHEAD")) ahead = min(4, max(1, atoi(a)));
    int ncw_pref = 4;
    if (const char* a = getenv("UWB_RING_NCW")) ncw_pref = atoi(a) == 2 ? 2 : 4;
    auto bytes = [&](int w) {
        return f32 ? ring_smem_bytes<float>(w, L.hr, L.hc, ahead) : ring_smem_bytes<double>(w, L.hr, L.hc, ahead);
    };
    const size_t s4 = bytes(256), s2 = bytes(128);
    if (ncw_pref == 4 && s4 <= 113 * 1024 && L.cols > 128)
        return f32 ? go_cfg<float>(L, 4, ahead, s4, stream) : go_cfg<double>(L, 4, ahead, s4, stream);
    if (s2 <= 200 * 1024)
        return f32 ? go_cfg<float>(L, 2, ahead, s2, stream) : go_cfg<double>(L, 2, ahead, s2, stream);
    return cudaErrorNotSupported;
}

} // namespace uwb
