// Kernel (d), production path: warp-specialised CA-CFAR over shared-memory rings
// of table rows, fed by tensor TMA.
//
// Replaces cfar_rows / run_cfar of /root/reference/proj/src/cfar.cpp:109-175 for
// the integral-image backend (cfar2d_integral, cfar.cpp:218-227).
//
// A CTA owns a 128-column x 256-row tile of one job. One producer thread moves
// every table row the tile's windows touch into a shared-memory ring with 3-D
// tensor TMA (cp.async.bulk.tensor: one box = 4 table rows x (128 + pad)
// columns of one job's table), and the CUT rows into a second ring (one box = 4
// map rows x 128 columns); each box completes on one "full" mbarrier. Ring
// slots are handed back through "empty" mbarriers, so producer and consumers
// never meet at a CTA barrier; the producer always issues the load the
// consumers will read first and sleeps only on that load's slot. Both streams are also
// prefetched into L2 kPfGroups boxes ahead. The consumer warps evaluate 4 output
// rows per step; the eight taps of a cell are shared-memory reads
//     RS = (t[r0][c0] + t[r1+1][c1+1]) - (t[r0][c1+1] + t[r1+1][c0])   (sat.hpp:32-33)
// sum = RS(outer) - RS(guard), T = alpha[n] * (sum / n), mask = cut > T
// (cfar.cpp:115-127).
//
// Fast path (all 4 rows have unclamped windows; columns may be clamped, their
// edges and n are per-lane constants): the 4 tap rows of the step are
// consecutive ring slots (the first group is mirrored past the ring's end), so
// every tap is one shared load at a compile-time offset from one of 8 row
// pointers, and n is the column's constant. The IEEE
// division is skipped: a cell with 0 <= cut < sum * (alpha/n) * (1 - 1e-13) is
// certainly below T; any other cell in the warp sends the warp through the
// reference expression alpha[n] * (sum / n). Decisions, thresholds and
// detection records are exactly the reference's.
#include <climits>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>

#include "cfar_common.cuh"

namespace uwb {

namespace {

constexpr int kRingRows = 256;  // output rows per CTA
constexpr int kG = 4;           // rows per group (output step, TMA box height)
constexpr int kW = 128;         // output columns per CTA
constexpr int kCutGroups = 4;   // CUT ring depth (groups) at 3-4 CTAs per SM
// CUT ring depth at `occ` CTAs per SM: each step consumes one CUT group, so a
// CTA runs at most (depth / TMA latency) steps per second; one or two CTAs per
// SM need the deeper ring (measured: consumers starved on full_c at depth 4)
__host__ __device__ constexpr int cut_groups_for(int occ, int esz) {
    return occ == 1 ? (esz == 4 ? 16 : 8) : kCutGroups;
}
constexpr int kMaxAhead = 8;    // most table groups of look-ahead beyond the window
constexpr int kPfGroups = 6;    // L2 prefetch distance of both streams (groups)

struct RingGeom {
    int ng;     // table row groups in the ring
    int nr;     // table row slots (ng * kG); sg mirror groups follow in memory
};

// sg = groups per consumer step (rows per step rs = 4 sg)
__host__ __device__ inline RingGeom ring_geom(int hr, int sg, int ahead) {
    RingGeom g;
    // output rows r..r+rs-1 read table rows r-hr .. r+rs+hr: 2hr+rs+1 rows,
    // spread over at most ceil((2hr+rs+1)/4)+1 groups
    g.ng = (2 * hr + kG * sg + 1 + kG - 1) / kG + 1 + ahead;
    g.nr = g.ng * kG;
    return g;
}

template <typename T>
inline size_t ring_smem_bytes(int hr, int boxc, int sg, int ahead, int ncut) {
    const RingGeom g = ring_geom(hr, sg, ahead);
    return 128 /* alignment slack */ + sizeof(double) * static_cast<size_t>(g.nr + kG * sg) * boxc +
           sizeof(T) * static_cast<size_t>(ncut) * kG * kW + 2 * sizeof(uint64_t) * (g.ng + ncut);
}

// Blocking wait that suspends the thread in the barrier unit (up to hint_ns per
// try) instead of spinning through issue slots the other warps need.
__device__ __forceinline__ void mbar_wait_susp(uint64_t* bar, unsigned parity, unsigned hint_ns) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "UWB_WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra UWB_WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(hint_ns)
        : "memory");
}
// Shared loads on 32-bit shared-window addresses. Volatile keeps them after the
// (volatile) mbarrier waits; no memory clobber, so other work schedules around them.
__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
template <typename T>
__device__ __forceinline__ double lds_widen(unsigned a);
template <>
__device__ __forceinline__ double lds_widen<float>(unsigned a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return static_cast<double>(v);
}
template <>
__device__ __forceinline__ double lds_widen<double>(unsigned a) {
    return lds_f64(a);
}

// 3-D tensor box -> L2 (no shared memory, no completion tracking).
__device__ __forceinline__ void tma_prefetch3(const CUtensorMap* map, int x, int y, int z) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y), "r"(z)
                 : "memory");
}
// 3-D tensor TMA box -> shared memory, completing on `bar`.
__device__ __forceinline__ void tma_box3(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// NCW consumer warps x CPT columns per thread = kW columns; BOXC = ring row
// width in doubles (the table box width, >= kW + 2 hc + 4, multiple of 4).
// NGRP consumer warp groups take alternate steps (NGRP = 2 at one CTA per SM:
// twice the consumer warps on the same ring); every consumer warp hands back
// every table group, each group's CUT groups come back from its NCW warps.
template <typename T, int NCW, int CPT, int BOXC, int SG, int OCC, int NGRP>
__global__ void __launch_bounds__((NCW * NGRP + 1) * kWarp, OCC)
cfar_ws_kernel(const __grid_constant__ CfarLaunch L, const __grid_constant__ CUtensorMap tmap_tab,
               const __grid_constant__ CUtensorMap tmap_cut) {
    static_assert(NCW * CPT * kWarp == kW, "tile width");
    constexpr int kCutG = cut_groups_for(OCC, sizeof(T));
    static_assert(kCutG % SG == 0, "CUT ring depth");
    static_assert(NGRP == 1 || (SG == 1 && kCutG % NGRP == 0), "interleaved steps");
    constexpr int RS = kG * SG; // output rows per consumer step
    constexpr unsigned kRowBytes = 8u * BOXC;
    constexpr unsigned kTabBox = kG * kRowBytes;
    constexpr unsigned kCutBox = kG * kW * sizeof(T);
    extern __shared__ unsigned char ring_raw[];
    unsigned char* ring_smem =
        ring_raw + ((128u - (static_cast<unsigned>(__cvta_generic_to_shared(ring_raw)) & 127u)) & 127u);
    const RingGeom G = ring_geom(L.hr, SG, L.ring_ahead);
    double* slots = reinterpret_cast<double*>(ring_smem);
    const char* ring = reinterpret_cast<const char*>(ring_smem);
    T* cuts = reinterpret_cast<T*>(slots + static_cast<size_t>(G.nr + RS) * BOXC);
    uint64_t* full_t = reinterpret_cast<uint64_t*>(cuts + static_cast<size_t>(kCutG) * kG * kW);
    uint64_t* full_c = full_t + G.ng;
    uint64_t* empty_t = full_c + kCutG;
    uint64_t* empty_c = empty_t + G.ng;

    const int64_t job = blockIdx.y;
    const int64_t map = job / L.geo.n_slabs;
    const int64_t slab = job % L.geo.n_slabs;
    const int col_tile = static_cast<int>(blockIdx.x % L.col_tiles);
    const int chunk = static_cast<int>(blockIdx.x / L.col_tiles);
    const int rows = static_cast<int>(L.geo.rows), cols = static_cast<int>(L.cols);
    const int hr = L.hr, hc = L.hc, gr = L.gr, gc = L.gc;
    const int c0 = col_tile * kW;
    const int ra = static_cast<int>(L.geo.owned_begin(slab)) + chunk * static_cast<int>(L.ring_rows);
    const int rb = min(ra + static_cast<int>(L.ring_rows), static_cast<int>(L.geo.owned_end(slab)));
    if (ra >= rb) return;
    const int trow0 = static_cast<int>(L.geo.table_begin(slab));

    // table storage columns of the ring rows: [e_lo, e_lo + BOXC), 16-byte aligned
    const int e_lo = (kTabShift + max(0, c0 - hc)) & ~1;
    // TMA column / table index of this tile's band table (UWB_SAT_TILE; the
    // job's own table otherwise). Bands own whole 128-column tiles and start on
    // even columns, so the consumers' offsets from e_lo are unchanged.
    const int64_t band = L.geo.band_of(c0);
    const int e_tx = e_lo - static_cast<int>(L.geo.band_c0(band));
    const int z_tab = static_cast<int>(job * L.geo.n_bands + band);
    // padded table rows needed by output rows [ra, rb), in groups of kG from i_lo
    const int i_lo = max(0, ra - hr);
    const int i_hi = min(rows, rb + hr);
    const int n_steps = (rb - ra + RS - 1) / RS;
    const int n_cg = (rb - ra + kG - 1) / kG; // CUT groups

    // ring byte offset of padded table row i (i_lo <= i <= i_hi)
    auto ring_off = [&](int i) { return static_cast<unsigned>((i - i_lo) % G.nr) * kRowBytes; };
    if (threadIdx.x == 0) {
        for (int s = 0; s < G.ng + kCutG; ++s) {
            mbar_init(&full_t[s], 1);
            mbar_init(&empty_t[s], s < G.ng ? NCW * NGRP : NCW);
        }
        mbar_fence_init();
    }
    __syncthreads();

    const int warp = threadIdx.x / kWarp;
    const int lane = threadIdx.x % kWarp;

    if (warp == NCW * NGRP) {
        // =========================== producer thread ===========================
        if (lane != 0) return;
        const int last_grp = (i_hi - i_lo) / kG;
        const int pf = L.pf_groups;
        for (int g = 0; g <= min(last_grp, pf - 1); ++g)
            tma_prefetch3(&tmap_tab, e_tx, i_lo + g * kG - trow0, z_tab);
        const int buf0 = static_cast<int>(L.geo.buf_row0);
        for (int g = 0; g < min(n_cg, pf); ++g)
            tma_prefetch3(&tmap_cut, c0, ra + g * kG - buf0, static_cast<int>(map));
        int grp = 0, gslot = 0, gphase = 0;   // next table group, its slot and empty-phase
        int cstep = 0, cslot = 0, cphase = 0; // next CUT group
        // Issue order: always the load the consumers need first; block (suspended)
        // only on that load's ring slot. Table group grp is first read at step
        // (i_lo + 4 grp - ra - hr - 1) / RS, CUT group cstep at step cstep / SG.
        while (grp <= last_grp || cstep < n_cg) {
            const int need_tab = grp <= last_grp ? max(0, (i_lo + kG * grp - ra - hr - 1)) / RS : INT_MAX;
            const int need_cut = cstep < n_cg ? cstep / SG : INT_MAX;
            if (need_tab <= need_cut) {
                if (grp >= G.ng) mbar_wait_susp(&empty_t[gslot], static_cast<unsigned>(gphase ^ 1), L.sleep_ns);
                const int first = i_lo + grp * kG;
                // the first SG groups are mirrored after the last slot, so RS
                // consecutive ring rows are always contiguous in memory
                mbar_expect_tx(&full_t[gslot], gslot < SG ? 2 * kTabBox : kTabBox);
                tma_box3(slots + static_cast<size_t>(gslot * kG) * BOXC, &tmap_tab, e_tx, first - trow0,
                         z_tab, &full_t[gslot]);
                if (gslot < SG)
                    tma_box3(slots + static_cast<size_t>(G.nr + gslot * kG) * BOXC, &tmap_tab, e_tx, first - trow0,
                             z_tab, &full_t[gslot]);
                if (grp + pf <= last_grp)
                    tma_prefetch3(&tmap_tab, e_tx, first + pf * kG - trow0, z_tab);
                if (++gslot == G.ng) { gslot = 0; gphase ^= 1; }
                ++grp;
            } else {
                if (cstep >= kCutG) mbar_wait_susp(&empty_c[cslot], static_cast<unsigned>(cphase ^ 1), L.sleep_ns);
                const int first = ra + cstep * kG;
                mbar_expect_tx(&full_c[cslot], kCutBox);
                tma_box3(cuts + static_cast<size_t>(cslot) * kG * kW, &tmap_cut, c0, first - buf0,
                         static_cast<int>(map), &full_c[cslot]);
                if (cstep + pf < n_cg)
                    tma_prefetch3(&tmap_cut, c0, first + pf * kG - buf0, static_cast<int>(map));
                if (++cslot == kCutG) { cslot = 0; cphase ^= 1; }
                ++cstep;
            }
        }
        return;
    }

    // ============================ consumer warps ============================
    const int grp_id = warp / NCW;            // my steps: grp_id, grp_id + NGRP, ...
    const int cw = warp % NCW;
    const int wc0 = c0 + cw * kWarp * CPT; // first column of my warp
    const int tc = cw * kWarp * CPT + lane; // my first column within the tile
    ColConst K[CPT];
    bool okc[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        K[j] = col_const(c0 + tc + j * kWarp, cols, hc, gc, e_lo);
        okc[j] = K[j].ok;
    }
    const bool per_cell = L.thresholds != nullptr || L.mask_u8 != nullptr;
    // Fast path: every row of the step has an unclamped window, so n is constant
    // down each column (cfar.cpp:28-32 with full-height windows); clamped
    // column edges are in K[j] and n_col[j].
    const bool fast_cols = !per_cell && wc0 < cols;
    int n_col[CPT];
    double alpha_col[CPT], fast_k[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        n_col[j] = (2 * hr + 1) * K[j].ow - (2 * gr + 1) * K[j].gw;
        alpha_col[j] = n_col[j] > 0 ? __ldg(L.alpha + n_col[j]) : 0.0;
        // 0 <= cut < sum * fast_k  implies  cut < alpha * (sum / n) (relative margin 1e-13)
        fast_k[j] = n_col[j] > 0 ? dmul(ddiv(alpha_col[j], static_cast<double>(n_col[j])), 1.0 - 1e-13) : 0.0;
    }

    // ring slots of the (unclamped) tap rows of output row r0, advanced 4 rows per step
    auto slot0 = [&](int i) { return ((i - i_lo) % G.nr + G.nr) % G.nr; };
    const int rg = ra + grp_id * RS;
    int sA = slot0(rg - hr), sB = slot0(rg + hr + 1), sC = slot0(rg - gr), sD = slot0(rg + gr + 1);
    constexpr unsigned kHint = 20000; // ns a waiting consumer may sleep in the barrier unit
    const unsigned full_t_u = smem_u32(full_t), full_c_u = smem_u32(full_c);
    const unsigned empty_t_u = smem_u32(empty_t), empty_c_u = smem_u32(empty_c);
    // table groups needed through step s: min(last, need_base + s) in the interior
    const int last_grp_c = (i_hi - i_lo) / kG;
    int waited = -1, wslot = 0, wphase = 0; // full_t groups known resident
    int released = -1, rslot = 0;            // table groups handed back
    int cslot = grp_id * SG, cphase = 0;
    // per-column alpha cache for the general path
    int ncache[CPT];
    double kcache[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        ncache[j] = -1;
        kcache[j] = 0.0;
    }

    // Steady run: consecutive fast steps (every row of the step has an unclamped
    // window and the step is full). There each step needs exactly one more table
    // group and one CUT group, and frees one of each, so the bookkeeping is a few
    // increments; the step body is the fast path below.
    const int steady_lo = max(0, (hr - ra + RS - 1) / RS);
    // last steady step: floor division (a negative numerator means no steady step;
    // C++ division would truncate it to 0)
    auto fdiv = [](int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
    const int steady_hi = min(n_steps, min(fdiv(rb - RS - ra, RS), fdiv(rows - RS - hr - ra, RS)) + 1);
    const bool steady = SG == 1 && fast_cols && !(L.debug & 1u) && steady_lo < steady_hi;
    constexpr unsigned kCutBytes = kG * kW * sizeof(T);

    // my first step in the steady run
    const int my_steady_lo = steady_lo + ((grp_id - steady_lo) % NGRP + NGRP) % NGRP;
    for (int step = grp_id; step < n_steps; step += NGRP) {
        if (steady && step == my_steady_lo && step < steady_hi) {
            int need = min(last_grp_c, (ra + step * RS + RS + hr - i_lo) / kG);
            int done = (ra + step * RS + RS - hr - i_lo) / kG - 1;
            while (waited < need - 1) { // catch up; then one group per step
                mbar_wait_u<kHint>(full_t_u + 8u * wslot, static_cast<unsigned>(wphase));
                ++waited;
                if (++wslot == G.ng) { wslot = 0; wphase ^= 1; }
            }
            // 32-bit shared addresses (no generic-to-shared conversions in the loop)
            const unsigned ring_s = smem_u32(ring);
            const unsigned ring_end = static_cast<unsigned>(G.nr) * kRowBytes;
            unsigned oA = static_cast<unsigned>(sA) * kRowBytes, oB = static_cast<unsigned>(sB) * kRowBytes;
            unsigned oC = static_cast<unsigned>(sC) * kRowBytes, oD = static_cast<unsigned>(sD) * kRowBytes;
            unsigned xa[CPT], xb[CPT], ya[CPT], yb[CPT];
#pragma unroll
            for (int j = 0; j < CPT; ++j) {
                xa[j] = ring_s + K[j].xa;
                xb[j] = ring_s + K[j].xb;
                ya[j] = ring_s + K[j].ya;
                yb[j] = ring_s + K[j].yb;
            }
            unsigned cut_s = smem_u32(cuts + tc);
            // opaque: keep these shared-window addresses in registers instead of
            // re-deriving the window base every step
            unsigned ft_u = full_t_u, fc_u = full_c_u, ec_u = empty_c_u, et_u = empty_t_u;
            asm volatile("" : "+r"(cut_s), "+r"(ft_u), "+r"(fc_u), "+r"(ec_u), "+r"(et_u));
#pragma unroll
            for (int j = 0; j < CPT; ++j) asm volatile("" : "+r"(xa[j]), "+r"(xb[j]), "+r"(ya[j]), "+r"(yb[j]));
            // lane k*CPT+j owns mask word (row r0 + k, column word of wc0 + 32 j)
            const bool has_word = L.mask_bits && lane < CPT * RS && wc0 + (lane % CPT) * kWarp < cols;
            uint32_t* mword = has_word ? L.mask_bits + map * L.mask_map_stride +
                                             (ra + step * RS + lane / CPT - L.geo.row_lo) * L.words_per_row +
                                             ((wc0 + (lane % CPT) * kWarp) >> 5)
                                       : nullptr;
            const int64_t mstep = has_word ? RS * L.words_per_row : 0;
            if (lane == 0 && step + 1 < n_steps) { // catch up the hand-backs; then one per step
                while (released < done - 1) {
                    ++released;
                    mbar_arrive_u(empty_t_u + 8u * rslot);
                    if (++rslot == G.ng) rslot = 0;
                }
            }
            for (; step < steady_hi; step += NGRP) {
                const int r0 = ra + step * RS;
#pragma unroll
                for (int q = 0; q < NGRP; ++q) { // one more table group per step
                    if (waited < need) {
                        mbar_wait_u<kHint>(ft_u + 8u * wslot, static_cast<unsigned>(wphase));
                        ++waited;
                        if (++wslot == G.ng) { wslot = 0; wphase ^= 1; }
                    }
                }
                need = min(last_grp_c, need + NGRP);
                mbar_wait_u<kHint>(fc_u + 8u * cslot, static_cast<unsigned>(cphase));
                const unsigned cg = cut_s + cslot * kCutBytes;
                double v[RS][CPT], thr[RS][CPT], sum[RS][CPT];
                bool hit[RS][CPT];
                bool any = false;
#pragma unroll
                for (int k = 0; k < RS; ++k) {
#pragma unroll
                    for (int j = 0; j < CPT; ++j) {
                        const unsigned o = k * kRowBytes;
                        const double rs_o = dsub(dadd(lds_f64(xa[j] + oA + o), lds_f64(xb[j] + oB + o)),
                                                 dadd(lds_f64(xb[j] + oA + o), lds_f64(xa[j] + oB + o)));
                        const double rs_g = dsub(dadd(lds_f64(ya[j] + oC + o), lds_f64(yb[j] + oD + o)),
                                                 dadd(lds_f64(yb[j] + oC + o), lds_f64(ya[j] + oD + o)));
                        sum[k][j] = dsub(rs_o, rs_g);
                        v[k][j] = lds_widen<T>(cg + (k * kW + j * kWarp) * sizeof(T));
                        any |= !(v[k][j] < dmul(sum[k][j], fast_k[j])) || v[k][j] < 0.0;
                    }
                }
                if (__any_sync(0xffffffffu, any)) {
#pragma unroll
                    for (int k = 0; k < RS; ++k) {
#pragma unroll
                        for (int j = 0; j < CPT; ++j) {
                            thr[k][j] = 0.0;
                            hit[k][j] = false;
                            if (!(v[k][j] < dmul(sum[k][j], fast_k[j])) || v[k][j] < 0.0) {
                                thr[k][j] = dmul(alpha_col[j], ddiv(sum[k][j], static_cast<double>(n_col[j])));
                                hit[k][j] = v[k][j] > thr[k][j];
                                if (v[k][j] < 0.0)
                                    report_min(L.first_bad + 2 * map + 1,
                                               static_cast<unsigned long long>(static_cast<int64_t>(r0 + k) * cols +
                                                                               c0 + tc + j * kWarp));
                            }
                        }
                    }
                    emit_block<RS, CPT>(L, map, r0, r0 + RS - 1, wc0, c0 + tc, okc, hit, v, thr, false);
                } else if (has_word) { // no hit in the block: zero mask words
                    *mword = 0u;
                }
                mword += mstep * NGRP;
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive_u(ec_u + 8u * cslot);
                    if (step + 1 < n_steps) {
#pragma unroll
                        for (int q = 0; q < NGRP; ++q) {
                            if (released < done) {
                                ++released;
                                mbar_arrive_u(et_u + 8u * rslot);
                                if (++rslot == G.ng) rslot = 0;
                            }
                        }
                    }
                }
                done += NGRP;
                cslot += NGRP;
                if (cslot >= kCutG) { cslot -= kCutG; cphase ^= 1; }
                constexpr unsigned kAdv = RS * NGRP * kRowBytes;
                oA += kAdv; if (oA >= ring_end) oA -= ring_end;
                oB += kAdv; if (oB >= ring_end) oB -= ring_end;
                oC += kAdv; if (oC >= ring_end) oC -= ring_end;
                oD += kAdv; if (oD >= ring_end) oD -= ring_end;
            }
            sA = static_cast<int>(oA / kRowBytes);
            sB = static_cast<int>(oB / kRowBytes);
            sC = static_cast<int>(oC / kRowBytes);
            sD = static_cast<int>(oD / kRowBytes);
            if (step >= n_steps) break;
        }
        const int r0 = ra + step * RS;
        const int r_last = min(r0 + RS, rb) - 1;
        {
            const int need = min(last_grp_c, (min(r_last + hr, rows - 1) + 1 - i_lo) / kG);
            while (waited < need) {
                mbar_wait_u<kHint>(full_t_u + 8u * wslot, static_cast<unsigned>(wphase));
                ++waited;
                if (++wslot == G.ng) { wslot = 0; wphase ^= 1; }
            }
        }
#pragma unroll
        for (int q = 0; q < SG; ++q)
            if (q == 0 || r0 + q * kG <= r_last)
                mbar_wait_u<kHint>(full_c_u + 8u * (cslot + q), static_cast<unsigned>(cphase));
        const T* cut_grp = cuts + static_cast<size_t>(cslot) * kG * kW;
        double v[RS][CPT], thr[RS][CPT];
        bool hit[RS][CPT];
        if (L.debug & 1u) goto release; // data-movement probe
        {
            const bool fast = fast_cols && r0 - hr >= 0 && r0 + RS - 1 == r_last && r_last + hr <= rows - 1;
            if (fast) {
                // ---- interior step: 8 row pointers, compile-time tap offsets ----
                const char* pA = ring + static_cast<unsigned>(sA) * kRowBytes;
                const char* pB = ring + static_cast<unsigned>(sB) * kRowBytes;
                const char* pC = ring + static_cast<unsigned>(sC) * kRowBytes;
                const char* pD = ring + static_cast<unsigned>(sD) * kRowBytes;
                double sum[RS][CPT];
                bool need = false;
#pragma unroll
                for (int k = 0; k < RS; ++k) {
#pragma unroll
                    for (int j = 0; j < CPT; ++j) {
                        const unsigned o = k * kRowBytes;
                        const double rs_o = dsub(dadd(tap(pA, K[j].xa + o), tap(pB, K[j].xb + o)),
                                                 dadd(tap(pA, K[j].xb + o), tap(pB, K[j].xa + o)));
                        const double rs_g = dsub(dadd(tap(pC, K[j].ya + o), tap(pD, K[j].yb + o)),
                                                 dadd(tap(pC, K[j].yb + o), tap(pD, K[j].ya + o)));
                        sum[k][j] = dsub(rs_o, rs_g);
                        v[k][j] = static_cast<double>(cut_grp[k * kW + tc + j * kWarp]);
                        need |= !(v[k][j] < dmul(sum[k][j], fast_k[j])) || v[k][j] < 0.0;
                    }
                }
                if (__any_sync(0xffffffffu, need)) {
#pragma unroll
                    for (int k = 0; k < RS; ++k) {
#pragma unroll
                        for (int j = 0; j < CPT; ++j) {
                            thr[k][j] = 0.0;
                            hit[k][j] = false;
                            if (!(v[k][j] < dmul(sum[k][j], fast_k[j])) || v[k][j] < 0.0) {
                                thr[k][j] = dmul(alpha_col[j], ddiv(sum[k][j], static_cast<double>(n_col[j])));
                                hit[k][j] = v[k][j] > thr[k][j];
                                if (v[k][j] < 0.0)
                                    report_min(L.first_bad + 2 * map + 1,
                                               static_cast<unsigned long long>(static_cast<int64_t>(r0 + k) * cols +
                                                                               c0 + tc + j * kWarp));
                            }
                        }
                    }
                    emit_block<RS, CPT>(L, map, r0, r_last, wc0, c0 + tc, okc, hit, v, thr, false);
                } else if (lane < CPT * RS && L.mask_bits) { // no hit in the block: zero mask words
                    const int wk = lane / CPT, wc = wc0 + (lane % CPT) * kWarp;
                    if (wc < cols)
                        L.mask_bits[map * L.mask_map_stride + (r0 + wk - L.geo.row_lo) * L.words_per_row +
                                    (wc >> 5)] = 0u;
                }
            } else {
                // ---- general step: clamped windows, per-cell n ----
                const char* RA[RS];
                const char* RB[RS];
                const char* RC[RS];
                const char* RD[RS];
                int HR[RS], HG[RS];
#pragma unroll
                for (int k = 0; k < RS; ++k) {
                    // clamped window rows and heights (cfar.cpp:117-120)
                    const int r = min(r0 + k, r_last);
                    const int iA = clamp_lo32(r, hr), iB = clamp_hi32(r, hr, rows) + 1;
                    const int iC = clamp_lo32(r, gr), iD = clamp_hi32(r, gr, rows) + 1;
                    RA[k] = ring + ring_off(iA);
                    RB[k] = ring + ring_off(iB);
                    RC[k] = ring + ring_off(iC);
                    RD[k] = ring + ring_off(iD);
                    HR[k] = iB - iA;
                    HG[k] = iD - iC;
                }
                double sum[RS][CPT], approx[RS][CPT];
                int n[RS][CPT];
                bool need_exact[RS][CPT];
                bool any_slow = false;
#pragma unroll
                for (int k = 0; k < RS; ++k) {
#pragma unroll
                    for (int j = 0; j < CPT; ++j) {
                        v[k][j] = static_cast<double>(cut_grp[k * kW + tc + j * kWarp]);
                        sum[k][j] = train_sum(K[j], RA[k], RB[k], RC[k], RD[k]);
                        n[k][j] = HR[k] * K[j].ow - HG[k] * K[j].gw;
                    }
                }
#pragma unroll
                for (int k = 0; k < RS; ++k) {
                    const bool row_ok = r0 + k <= r_last;
#pragma unroll
                    for (int j = 0; j < CPT; ++j) {
                        if (n[k][j] != ncache[j] && row_ok) {
                            ncache[j] = n[k][j];
                            kcache[j] = ddiv(__ldg(L.alpha + n[k][j]), static_cast<double>(n[k][j]));
                        }
                        approx[k][j] = dmul(sum[k][j], kcache[j]);
                        const bool ok = K[j].ok && row_ok;
                        hit[k][j] = ok && v[k][j] > approx[k][j];
                        need_exact[k][j] = ok && (per_cell || hit[k][j] || v[k][j] < 0.0 ||
                                                  !(fabs(dsub(v[k][j], approx[k][j])) > 1e-13 * fabs(approx[k][j])));
                        any_slow |= need_exact[k][j];
                        thr[k][j] = 0.0;
                    }
                }
                // the reference expression where it is needed (rare, warp-uniform branch)
                if (__any_sync(0xffffffffu, any_slow)) {
#pragma unroll
                    for (int k = 0; k < RS; ++k) {
#pragma unroll
                        for (int j = 0; j < CPT; ++j) {
                            if (need_exact[k][j]) {
                                thr[k][j] =
                                    dmul(__ldg(L.alpha + n[k][j]), ddiv(sum[k][j], static_cast<double>(n[k][j])));
                                hit[k][j] = v[k][j] > thr[k][j];
                                if (v[k][j] < 0.0)
                                    report_min(L.first_bad + 2 * map + 1,
                                               static_cast<unsigned long long>(static_cast<int64_t>(r0 + k) * cols +
                                                                               c0 + tc + j * kWarp));
                            }
                        }
                    }
                }
                emit_block<RS, CPT>(L, map, r0, r_last, wc0, c0 + tc, okc, hit, v, thr, per_cell);
            }
        }
    release:
        // hand back this step's CUT group and the table groups no later step reads
        __syncwarp();
        if (lane == 0) {
#pragma unroll
            for (int q = 0; q < SG; ++q)
                if (q == 0 || r0 + q * kG <= r_last) mbar_arrive_u(empty_c_u + 8u * (cslot + q));
            if (step + 1 < n_steps) {
                const int keep_row = max(0, r_last + 1 - hr);
                const int done = (keep_row - i_lo) / kG - 1; // groups entirely below keep_row
                while (released < done) {
                    ++released;
                    mbar_arrive_u(empty_t_u + 8u * rslot);
                    if (++rslot == G.ng) rslot = 0;
                }
            }
        }
        cslot += SG * NGRP;
        if (cslot >= kCutG) { cslot -= kCutG; cphase ^= 1; }
        sA += RS * NGRP; if (sA >= G.nr) sA -= G.nr;
        sB += RS * NGRP; if (sB >= G.nr) sB -= G.nr;
        sC += RS * NGRP; if (sC >= G.nr) sC -= G.nr;
        sD += RS * NGRP; if (sD >= G.nr) sD -= G.nr;
    }
}

// ---- host side: tensor maps ----

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

bool encode3(CUtensorMap* m, CUtensorMapDataType dt, size_t esz, const void* base, uint64_t d0, uint64_t d1,
             uint64_t d2, uint64_t s1, uint64_t s2, unsigned b0, unsigned b1) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[3] = {d0, d1, d2};
    const cuuint64_t strides[2] = {s1 * esz, s2 * esz};
    const cuuint32_t box[3] = {b0, b1, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, int NCW, int CPT, int BOXC, int SG, int OCC, int NGRP = 1>
cudaError_t go(const CfarLaunch& L0, cudaStream_t stream) {
    CfarLaunch L = L0;
    L.sleep_ns = 20000;
    if (const char* e = UWB_KNOB("UWB_RING_SLEEP_NS")) L.sleep_ns = static_cast<unsigned>(atoi(e));
    L.pf_groups = kPfGroups;
    if (const char* e = UWB_KNOB("UWB_RING_PF")) L.pf_groups = atoi(e) > 0 ? atoi(e) : kPfGroups;
    L.debug = 0;
#ifdef UWB_PROBE_BUILD // timing probes only: skip the arithmetic (never in the release library)
    if (const char* e = UWB_KNOB("UWB_RING_DEBUG")) L.debug = static_cast<unsigned>(atoi(e));
#endif
    L.col_tiles = (L.cols + kW - 1) / kW;
    // row chunks of kRingRows; a batch too small to give every SM two CTAs
    // (single small maps) takes shorter chunks (each re-reads its window's
    // 2 hr + 1 halo rows, but the chunks' serial steps run in parallel)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // tall windows (config 4: 2 hr + 1 = 73) take 512-row chunks: each chunk
    // re-reads its 2 hr + 1 halo rows and fills its ring before the first step
    // (cfg 4: 1.62 -> 1.48 ms)
    L.ring_rows = 2 * L.hr + 1 > 48 ? 2 * kRingRows : kRingRows;
    auto ctas = [&](int64_t rr) { return L.col_tiles * ((L.geo.slab_rows + rr - 1) / rr) * L.n_jobs; };
    if (const char* e = UWB_KNOB("UWB_RING_ROWS")) L.ring_rows = atoi(e) > 0 ? atoi(e) : kRingRows;
    while (L.ring_rows > 16 && ctas(L.ring_rows) < 2 * sms && !L.fixed_rows && !UWB_KNOB("UWB_RING_FIXED_ROWS")) L.ring_rows /= 2;
    L.row_chunks = (L.geo.slab_rows + L.ring_rows - 1) / L.ring_rows;
    const int64_t n_maps = L.n_jobs / L.geo.n_slabs;
    CUtensorMap tmap_tab, tmap_cut;
    const uint64_t tab_rows = static_cast<uint64_t>(L.table_stride / L.table_ld);
    if (!encode3(&tmap_tab, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, L.table, L.table_ld, tab_rows, L.n_jobs * L.geo.n_bands, L.table_ld,
                 L.table_stride, BOXC, kG))
        return cudaErrorNotSupported;
    // a single map's stride is never used; give the encoder a valid one
    const int64_t mstride = n_maps > 1 ? L.map_stride : (L.ld * L.geo.buf_rows + 1) / 2 * 2;
    if (!encode3(&tmap_cut, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                 sizeof(T), L.maps, L.cols, L.geo.buf_rows, n_maps, L.ld, mstride, kW, kG))
        return cudaErrorNotSupported;
    const size_t smem = ring_smem_bytes<T>(L.hr, BOXC, SG, L.ring_ahead, cut_groups_for(OCC, sizeof(T)));
    if (smem > 227 * 1024) return cudaErrorNotSupported;
    const dim3 grid(static_cast<unsigned>(L.col_tiles * L.row_chunks), static_cast<unsigned>(L.n_jobs), 1);
    cudaError_t e = cudaFuncSetAttribute(cfar_ws_kernel<T, NCW, CPT, BOXC, SG, OCC, NGRP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    ++g_kernel_launches;
    cfar_ws_kernel<T, NCW, CPT, BOXC, SG, OCC, NGRP><<<grid, (NCW * NGRP + 1) * kWarp, smem, stream>>>(L, tmap_tab, tmap_cut);
    return cudaGetLastError();
}

template <typename T, int BOXC>
cudaError_t go_occ(const CfarLaunch& L, cudaStream_t stream) {
    // The most CTAs per SM whose rings fit with one group of look-ahead, then
    // the deepest look-ahead that still fits at that occupancy (measured: CTAs
    // per SM matter more than look-ahead). UWB_RING_OCC pins the occupancy.
    int occ = 0;
    const char* occ_knob = UWB_KNOB("UWB_RING_OCC");
    const int pinned = occ_knob ? atoi(occ_knob) : 0;
    auto fits = [&](int o, int ahead) {
        return ring_smem_bytes<T>(L.hr, BOXC, 1, ahead, cut_groups_for(o, sizeof(T))) <= static_cast<size_t>(233472 / o - 1024);
    };
    for (int o : {4, 3, 2, 1}) {
        if (pinned && o != pinned) continue;
        if (fits(o, 1)) {
            occ = o;
            break;
        }
    }
    if (!occ) return cudaErrorNotSupported;
    CfarLaunch La = L;
    La.ring_ahead = 1;
    while (La.ring_ahead < kMaxAhead && fits(occ, La.ring_ahead + 1)) ++La.ring_ahead;
    switch (occ) {
        case 4: return go<T, 4, 1, BOXC, 1, 4>(La, stream);
        case 3: return go<T, 4, 1, BOXC, 1, 3>(La, stream);
        case 2: return go<T, 4, 1, BOXC, 1, 2>(La, stream);
        default:
            // one CTA per SM (tall windows): two consumer warp groups on alternate steps
            {
                const char* e = UWB_KNOB("UWB_RING_GROUPS");
                const int ngrp = e ? atoi(e) : 2;
                if (ngrp == 4) return go<T, 4, 1, BOXC, 1, 1, 4>(La, stream);
                if (ngrp == 1) return go<T, 4, 1, BOXC, 1, 1>(La, stream);
                return go<T, 4, 1, BOXC, 1, 1, 2>(La, stream);
            }
    }
}

template <typename T>
cudaError_t go_cfg(const CfarLaunch& L, int boxc, cudaStream_t stream) {
    switch (boxc) {
        case 152: return go_occ<T, 152>(L, stream);
        case 160: return go_occ<T, 160>(L, stream);
        case 204: return go_occ<T, 204>(L, stream);
        default: return go_occ<T, 256>(L, stream);
    }
}

} // namespace

// Returns cudaErrorNotSupported when the rings do not fit or the layout does
// not allow tensor copies (caller falls back to the simple kernel).
cudaError_t launch_cfar_ring(const CfarLaunch& L, int dtype, cudaStream_t stream) {
    if (UWB_KNOB("UWB_CFAR_SIMPLE")) return cudaErrorNotSupported;
    if (L.geo.rows >= (int64_t(1) << 31) || L.cols >= (int64_t(1) << 30)) return cudaErrorNotSupported;
    const bool f32 = dtype == UWB_F32;
    const size_t esz = f32 ? 4 : 8;
    // tensor maps: 16-byte aligned base and row / map pitches
    if ((reinterpret_cast<uintptr_t>(L.maps) % 16) || ((L.ld * esz) % 16) ||
        (L.n_jobs / L.geo.n_slabs > 1 && (L.map_stride * esz) % 16))
        return cudaErrorNotSupported;
    // ring row width: kW + 2 hc + 4 doubles at most (16-byte aligned span)
    const int need = kW + 2 * L.hc + 4;
    const int boxc = need <= 152 ? 152 : need <= 160 ? 160 : need <= 204 ? 204 : need <= 256 ? 256 : 0;
    if (!boxc) return cudaErrorNotSupported;
    return f32 ? go_cfg<float>(L, boxc, stream) : go_cfg<double>(L, boxc, stream);
}

} // namespace uwb
