// Kernels (c)+(d) fused: exact summed-area table and CA-CFAR in one pass, with
// the table kept in shared memory (it never reaches HBM).
//
// Replaces build_sat (/root/reference/proj/src/sat.cpp:10-37) followed by
// cfar_rows (/root/reference/proj/src/cfar.cpp:109-175) for cfar2d_integral
// (cfar.cpp:218-227) on whole maps. The two-kernel path (sat.cu + cfar_ring.cu)
// writes 8 bytes of table per cell and reads them back; this kernel reads the
// map once (4 bytes per f32 cell) and writes only the mask bits and detections.
//
// Work unit = one 128-column band of one map (bands claimed from an atomic
// counter in band-major order, so the band to the left was claimed earlier).
// A CTA = 1 SAT warp + 4 CFAR warps sharing a ring of table rows:
//   * the SAT warp runs the systolic wavefront of sat.cu over the band's
//     32*kCpl table columns: padded columns [c0 - hc, c0 - hc + 32 kCpl), i.e.
//     the band plus the hc + 1 columns to its left and hc to its right that the
//     windows of the band's cells tap. Lane l owns kCpl consecutive columns and
//     evaluates row s - l at step s with the reference's three additions
//     (sat.cpp:33); the column left of the band comes, one double per row, from
//     the band to the left (edge buffer + release/acquire row counter, as in
//     sat.cu). It writes each table row into the ring (slot = padded row mod
//     nr; the first 4 slots are mirrored past the end so 4 consecutive rows are
//     always contiguous) and, once lane 31 has finished a group of 4 rows,
//     every lane arrives on that group's "full" mbarrier;
//   * CFAR warp w evaluates columns c0 + 32 w + lane, 4 rows per step, exactly
//     as the ring kernel's consumers (cfar_ring.cu): interior fast path with
//     compile-time tap offsets and the certified bound, clamped windows through
//     the reference expression. The CUT values are read from the map (L2-hot:
//     the SAT warp staged the same rows a few dozen steps earlier). Groups no
//     later step reads are handed back on "empty" mbarriers, which the SAT warp
//     waits on before reusing a slot.
// Every table value is produced by the same operations in the same order as the
// reference's build_sat, so thresholds, masks and detections are bit-identical
// to the two-kernel path and to the reference.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "cfar_common.cuh"

namespace uwb {

namespace {

constexpr int kBandOut = 128;   // output columns per band (unit)
constexpr int kNcw = 4;         // CFAR warps (one column x 4 rows per thread per step)
constexpr int kRs = 4;          // output rows per CFAR step (= ring group)
#ifndef UWB_FUSED_XSLOTS
#define UWB_FUSED_XSLOTS 8
#endif
constexpr int kFXSlots = UWB_FUSED_XSLOTS; // lane-private source ring (copy steps)
constexpr int kFAhead = kFXSlots - 2;      // SAT source staging distance (steps; rows are L2-prefetched)
constexpr int kMirror = kRs - 1; // ring slots mirrored past the end (4 consecutive slots stay contiguous)
constexpr int kFPublish = 64;   // SAT steps between edge hand-overs
constexpr int kFL2Ahead = 24;   // source rows are prefetched into L2 this many steps before staging
#ifndef UWB_FUSED_HINT_S
#define UWB_FUSED_HINT_S 0
#endif
#ifndef UWB_FUSED_HINT_C
#define UWB_FUSED_HINT_C 20000
#endif
// barrier-wait suspend hints (ns; 0 = plain try_wait): the SAT warp (the
// critical path) / the CFAR warps (which would otherwise spin on issue slots)
constexpr unsigned kFHint = UWB_FUSED_HINT_S;
constexpr unsigned kCHint = UWB_FUSED_HINT_C;
#ifndef UWB_FUSED_UNROLL
#define UWB_FUSED_UNROLL 4
#endif
constexpr int kFUnroll = UWB_FUSED_UNROLL; // SAT steps per unrolled body (source slots stay compile-time)

struct FusedLaunch {
    CfarLaunch c;
    double* gedge;          // (n_maps * strips) edge columns of edge_stride doubles
    int64_t edge_stride;
    unsigned* gprog;        // (n_maps * strips) row counters, zeroed before launch
    unsigned* unit_counter; // zeroed before launch
    int64_t strips;         // stride of the per-map edge / counter arrays (>= n_bands)
    int64_t n_maps;
    int64_t n_units;        // n_maps * n_bands
    int n_bands;
    int nr;                 // ring rows (multiple of 4)
};

template <typename T, int kCpl>
struct FusedSmem {
    static constexpr unsigned kRowBytes = kWarp * kCpl * 8u;  // one table row of the band
    static constexpr unsigned kXLane = kCpl * sizeof(T);
    static constexpr unsigned kXSlotBytes = kWarp * kXLane;
    static constexpr unsigned kXRing = kFXSlots * kXSlotBytes;
    // ring (+ mirror rows), source ring, edge staging, unit queue, barriers
    static size_t bytes(int nr) {
        return 128 + static_cast<size_t>(nr + kMirror) * kRowBytes + kXRing + kWarp * 8 + 16 + 8 * 4 +
               2 * 8 * static_cast<size_t>(nr / kRs);
    }
};

__device__ __forceinline__ void st_shared_f64(unsigned a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_shared_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_shared_u32(unsigned a, unsigned v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_shared_u32(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void mbar_init_u(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void cp_elem(unsigned dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_elem(unsigned dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
// One contiguous global range -> L2 (no completion tracking). 16-byte aligned.
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void sts_zero(unsigned a, float*) {
    asm volatile("st.shared.u32 [%0], 0;" ::"r"(a) : "memory");
}
__device__ __forceinline__ void sts_zero(unsigned a, double*) {
    asm volatile("st.shared.u64 [%0], 0;" ::"r"(a) : "memory");
}

template <typename T, int kCpl, int OCC>
__global__ void __launch_bounds__((kNcw + 1) * kWarp, OCC) cfar_fused_kernel(const __grid_constant__ FusedLaunch F) {
    using SM = FusedSmem<T, kCpl>;
    constexpr unsigned kRowBytes = SM::kRowBytes;
    constexpr int kSlotElems = kWarp * kCpl; // doubles per ring slot
    static_assert(kWarp * kCpl >= kBandOut + 1, "band");
    extern __shared__ unsigned char fz_raw[];
    const unsigned raw = smem_u32(fz_raw);
    const unsigned base = (raw + 127u) & ~127u;
    const int nr = F.nr, nq = F.nr / kRs;
    const unsigned ring_u = base;
    const unsigned xring_u = ring_u + static_cast<unsigned>(nr + kMirror) * kRowBytes;
    const unsigned edge_u = xring_u + SM::kXRing;
    const unsigned unitq_u = edge_u + kWarp * 8u;      // 2 unit ids (+ pad)
    const unsigned ubar_u = unitq_u + 16u;             // unit_full[2], unit_empty[2]
    const unsigned full_u = ubar_u + 32u;
    const unsigned empty_u = full_u + 8u * static_cast<unsigned>(nq);
    const CfarLaunch& L = F.c;
    const int warp = threadIdx.x / kWarp;
    const int lane = threadIdx.x % kWarp;
    if (threadIdx.x == 0) {
        for (int q = 0; q < nq; ++q) {
            mbar_init_u(full_u + 8u * q, kWarp);
            mbar_init_u(empty_u + 8u * q, kNcw);
        }
        mbar_init_u(ubar_u, 1);
        mbar_init_u(ubar_u + 8u, 1);
        mbar_init_u(ubar_u + 16u, kNcw);
        mbar_init_u(ubar_u + 24u, kNcw);
        mbar_fence_init();
    }
    __syncthreads();
    const int rows = static_cast<int>(L.geo.rows), cols = static_cast<int>(L.cols);
    const int hr = L.hr, hc = L.hc, gr = L.gr, gc = L.gc;
    // ring slots of a unit: SAT steps -1 .. rows + 30 write slots 0 .. rows + 31
    const int groups = (rows + kWarp + kRs - 1) / kRs;
    const int vstep = (kRs * groups) % nr;

    if (warp == kNcw) {
        // ============================== SAT warp ==============================
        // generic views for plain shared loads / stores (the compiler may schedule them)
        double* ring_w = reinterpret_cast<double*>(fz_raw + (base - raw)) + kCpl * lane; // my columns, slot 0
        const T* x_w = reinterpret_cast<const T*>(fz_raw + (xring_u - raw)) + kCpl * lane;
        const unsigned x_lane = xring_u + lane * SM::kXLane;
        constexpr int kEdgeLane = (kBandOut - 1) / kCpl, kEdgeK = (kBandOut - 1) % kCpl;
        unsigned eslot = 0, epar = 1; // next "empty" group to wait for (first pass passes)
        unsigned fslot = 0;           // next "full" group to arrive on
        int vb = 0;                   // ring slot of the unit's slot 0
        for (int k = 0;; ++k) {
            // claim a unit and hand it to the CFAR warps (2-deep queue)
            long long unit = 0;
            if (lane == 0) unit = static_cast<long long>(atomicAdd(F.unit_counter, 1u));
            unit = __shfl_sync(0xffffffffu, unit, 0);
            const int q = k & 1;
            mbar_wait_u<kFHint>(ubar_u + 16u + 8u * q, static_cast<unsigned>(((k >> 1) & 1) ^ 1));
            if (lane == 0) {
                st_shared_u32(unitq_u + 4u * q, unit < F.n_units ? static_cast<unsigned>(unit) : 0xffffffffu);
                mbar_arrive_u(ubar_u + 8u * q);
            }
            if (unit >= F.n_units) break;
            const int band = static_cast<int>(unit / F.n_maps);
            const int64_t m = unit % F.n_maps;
            const int jb = band * kBandOut - hc;          // padded column of band column 0
            const int mc = jb - 1 + kCpl * lane;          // map column of my first column
            int k_lo = kCpl, k_hi = 0;
#pragma unroll
            for (int j = 0; j < kCpl; ++j)
                if (mc + j >= 0 && mc + j < cols) {
                    k_lo = min(k_lo, j);
                    k_hi = j + 1;
                }
            const int64_t ld = L.ld;
            const T* map0 = static_cast<const T*>(L.maps) + m * L.map_stride;
            const bool has_left = band > 0, has_right = band + 1 < F.n_bands;
            const unsigned* prog_in = has_left ? F.gprog + m * F.strips + band - 1 : nullptr;
            unsigned* prog_out = has_right ? F.gprog + m * F.strips + band : nullptr;
            const double* ge_in = has_left ? F.gedge + (m * F.strips + band - 1) * F.edge_stride : nullptr;
            double* ge_out = has_right ? F.gedge + (m * F.strips + band) * F.edge_stride : nullptr;

            // columns outside the map read as 0: zero them in every source slot
            // once (copies never touch them)
#pragma unroll
            for (int j = 0; j < kCpl; ++j)
                if (j < k_lo || j >= k_hi)
                    for (int sl = 0; sl < kFXSlots; ++sl)
                        sts_zero(x_lane + sl * SM::kXSlotBytes + j * sizeof(T), static_cast<T*>(nullptr));

            // slot 0 (pre-step -1): lane 0's part of padded row 0
            mbar_wait_u<kFHint>(empty_u + 8u * eslot, epar);
            if (++eslot == static_cast<unsigned>(nq)) { eslot = 0; epar ^= 1; }
            if (lane == 0) {
#pragma unroll
                for (int j = 0; j < kCpl; ++j) {
                    ring_w[vb * kSlotElems + j] = 0.0;
                    if (vb < kMirror) ring_w[(nr + vb) * kSlotElems + j] = 0.0;
                }
            }

            unsigned avail = 0;
            auto fetch_left = [&](int b0) {
                double v = 0.0;
                if (prog_in && b0 < rows) {
                    const unsigned need = static_cast<unsigned>(min(rows, b0 + kWarp));
                    if (avail < need) {
                        if (lane == 0)
                            avail = wait_count_geq(prog_in, need);
                        avail = __shfl_sync(0xffffffffu, avail, 0);
                    }
                    if (b0 + lane < rows) v = ge_in[b0 + lane];
                }
                return v;
            };
            // lane l stages at step s its own columns of source row s + kFAhead - l
            const T* xrow = map0 + mc + static_cast<int64_t>(kFAhead - lane) * ld;
            // the band's source row segment, 16-byte aligned inside the row, for the L2 prefetch
            const char* pf_row;
            unsigned pf_bytes;
            {
                const int64_t lo = static_cast<int64_t>(max(0, jb - 1)) * static_cast<int64_t>(sizeof(T));
                const int64_t hi =
                    static_cast<int64_t>(min(cols, jb - 1 + kWarp * kCpl)) * static_cast<int64_t>(sizeof(T));
                const char* row0 = reinterpret_cast<const char*>(map0);
                const uintptr_t a0 = (reinterpret_cast<uintptr_t>(row0 + lo)) & ~static_cast<uintptr_t>(15);
                const uintptr_t a1 = (reinterpret_cast<uintptr_t>(row0 + hi)) & ~static_cast<uintptr_t>(15);
                pf_row = reinterpret_cast<const char*>(a0) + (kFAhead + kFL2Ahead) * ld * static_cast<int64_t>(sizeof(T));
                pf_bytes = static_cast<unsigned>(a1 - a0);
            }
            const bool pf_ok = lane == 0 && pf_bytes > 0 && (ld * sizeof(T)) % 16 == 0;
            auto stage = [&](unsigned slot_off, int row, const T* p, bool checked) {
                if (!checked || (row >= 0 && row < rows)) {
#pragma unroll
                    for (int j = 0; j < kCpl; ++j)
                        if (j >= k_lo && j < k_hi) cp_elem(x_lane + slot_off + j * sizeof(T), p + j);
                }
            };
            if (pf_ok)
                for (int r = 0; r < min(rows, kFAhead + kFL2Ahead); ++r)
                    bulk_prefetch_l2(pf_row + (r - kFAhead - kFL2Ahead) * ld * static_cast<int64_t>(sizeof(T)), pf_bytes);
#pragma unroll
            for (int v = -kFAhead; v < 0; ++v) {
                stage(static_cast<unsigned>(((v + kFXSlots) & (kFXSlots - 1)) * SM::kXSlotBytes), v + kFAhead - lane,
                      xrow + static_cast<int64_t>(v) * ld, true);
                cp_async_commit();
            }

            double prev[kCpl], last[kCpl];
#pragma unroll
            for (int j = 0; j < kCpl; ++j) prev[j] = last[j] = 0.0;
            double left_prev = 0.0;
            bool scanned = false;
            const int steps = rows + kWarp - 1;
            // every lane writes slot vb + s + 1 at step s (its padded row s - lane + 1)
            int wslot = vb + 1 >= nr ? vb + 1 - nr : vb + 1;
            T xn[kCpl];
            double edge_n = 0.0;

            auto step = [&](const int s0, const int uu, auto checked_tag) {
                constexpr bool kChecked = decltype(checked_tag)::value;
                const int s = s0 + uu;
                const int r = s - lane;
                // (0) slot vb + s + 1 opens a new ring group every 4 steps
                if ((uu & 3) == 3) {
                    mbar_wait_u<kFHint>(empty_u + 8u * eslot, epar);
                    if (++eslot == static_cast<unsigned>(nq)) { eslot = 0; epar ^= 1; }
                }
                // (1a) L2 prefetch of source row s + kFAhead + kFL2Ahead (one lane)
                if (pf_ok && s + kFAhead + kFL2Ahead < rows) bulk_prefetch_l2(pf_row, pf_bytes);
                pf_row += ld * static_cast<int64_t>(sizeof(T));
                // (1) stage my source row s + kFAhead - lane into slot s mod kFXSlots
                stage(static_cast<unsigned>((uu & (kFXSlots - 1)) * SM::kXSlotBytes), s + kFAhead - lane, xrow,
                      kChecked);
                cp_async_commit();
                xrow += ld;
                // (2) this step's inputs were loaded one step ahead (copied at step s - kFAhead)
                T x[kCpl];
#pragma unroll
                for (int j = 0; j < kCpl; ++j) x[j] = xn[j];
                const double from_left = edge_n;
                cp_async_wait<kFAhead - 1>();
                {
                    const T* a = x_w + ((uu + 1 - kFAhead + kFXSlots) & (kFXSlots - 1)) * kSlotElems;
#pragma unroll
                    for (int j = 0; j < kCpl; ++j) xn[j] = a[j];
                }
                if (uu + 1 < kWarp) edge_n = ld_shared_f64(edge_u + static_cast<unsigned>(uu + 1) * 8u);
                // (3) S(r, first column - 1): lane l-1's newest value; lane 0: left band
                double left = __shfl_up_sync(0xffffffffu, last[kCpl - 1], 1);
                if (lane == 0) left = from_left;
                // (4) sat.cpp:33
                double sv[kCpl];
                sv[0] = dsub(dadd(dadd(widen(x[0]), prev[0]), left), left_prev);
#pragma unroll
                for (int j = 1; j < kCpl; ++j) sv[j] = dsub(dadd(dadd(widen(x[j]), prev[j]), sv[j - 1]), prev[j - 1]);
                const bool act = !kChecked || (r >= 0 && r < rows);
                double* dst = ring_w + wslot * kSlotElems;
                if (act) {
#pragma unroll
                    for (int j = 0; j < kCpl; ++j) dst[j] = sv[j];
                    if (wslot < kMirror) {
#pragma unroll
                        for (int j = 0; j < kCpl; ++j) dst[nr * kSlotElems + j] = sv[j];
                    }
                    if (lane == kEdgeLane && ge_out) ge_out[r] = sv[kEdgeK];
                    left_prev = left;
#pragma unroll
                    for (int j = 0; j < kCpl; ++j) prev[j] = last[j] = sv[j];
                } else if (kChecked && r == -1) { // my part of padded row 0
#pragma unroll
                    for (int j = 0; j < kCpl; ++j) dst[j] = 0.0;
                    if (wslot < kMirror) {
#pragma unroll
                        for (int j = 0; j < kCpl; ++j) dst[nr * kSlotElems + j] = 0.0;
                    }
                }
                if (++wslot == nr) wslot = 0;
                // (5) close the group of slot vb + s + 1
                const bool close = kChecked ? ((uu & 3) == 2 || s == steps - 1) : (uu & 3) == 2;
                if (close) {
                    mbar_arrive_u(full_u + 8u * fslot);
                    if (++fslot == static_cast<unsigned>(nq)) fslot = 0;
                }
            };

            double e_cur = fetch_left(0);
            double e_next = fetch_left(kWarp);
            cp_async_wait<kFAhead - 1>();
            {
                const T* a = x_w + ((kFXSlots - kFAhead) & (kFXSlots - 1)) * kSlotElems;
#pragma unroll
                for (int j = 0; j < kCpl; ++j) xn[j] = a[j];
            }
            for (int s0 = 0; s0 < steps; s0 += kWarp) {
                __syncwarp();
                st_shared_f64(edge_u + 8u * lane, e_cur);
                __syncwarp();
                edge_n = ld_shared_f64(edge_u);
                e_cur = e_next;
                e_next = fetch_left(s0 + 2 * kWarp);
                const bool fast = s0 >= kWarp && s0 + kWarp + kFAhead <= rows;
                if (fast) {
#pragma unroll kFUnroll
                    for (int uu = 0; uu < kWarp; ++uu) step(s0, uu, std::false_type{});
                } else {
#pragma unroll 1
                    for (int uu = 0; uu < kWarp && s0 + uu < steps; ++uu) step(s0, uu, std::true_type{});
                }
                // non-finite inputs poison every later S of their column (sat.cu)
                bool finite = true;
#pragma unroll
                for (int j = 0; j < kCpl; ++j) finite &= j < k_lo || j >= k_hi || isfinite(last[j]);
                if (!scanned && !finite) {
                    scanned = true;
                    int col = 0;
                    const int bad = first_nonfinite<T>(map0, ld, mc + k_lo, k_hi - k_lo, min(rows, s0 + kWarp), &col);
                    if (bad != INT_MAX && L.first_bad)
                        report_min(L.first_bad + 2 * m, static_cast<unsigned long long>(
                                                            static_cast<int64_t>(bad) * cols + col));
                }
                const int s_end = min(s0 + kWarp, steps);
                if (prog_out && lane == kEdgeLane && ((s_end & (kFPublish - 1)) == 0 || s_end == steps))
                    st_release_u32(prog_out, static_cast<unsigned>(min(rows, max(0, s_end - kEdgeLane))));
            }
            cp_async_wait<0>();
            __syncwarp();
            vb += vstep;
            if (vb >= nr) vb -= nr;
        }
        return;
    }

    // ============================== CFAR warps ==============================
    // Ring slot of table entry (padded row i, band column t): vb + i + t / kCpl
    // (the SAT lane owning column t wrote it at step i + t / kCpl - 1).
    const bool per_cell = L.thresholds != nullptr || L.mask_u8 != nullptr;
    const char* ring = reinterpret_cast<const char*>(fz_raw) + (base - raw); // generic view of the ring
    const unsigned ring_bytes = static_cast<unsigned>(nr) * kRowBytes;
    unsigned wslot = 0, wpar = 0; // next "full" group to wait for
    unsigned rslot = 0;           // next "empty" group to hand back
    int vb = 0;
    const int n_steps = (rows + kRs - 1) / kRs;
    // steps whose 4 rows have unclamped windows: hr <= r0 and r0 + 3 + hr <= rows - 1
    const int t_fast_lo = (hr + kRs - 1) / kRs;
    const int t_fast_hi = rows - 1 - hr - (kRs - 1) >= 0 ? (rows - 1 - hr - (kRs - 1)) / kRs + 1 : 0;
    const int64_t ld = L.ld;
    const int64_t wpr = L.words_per_row;
    for (int k = 0;; ++k) {
        const int q = k & 1;
        mbar_wait_u<kCHint>(ubar_u + 8u * q, static_cast<unsigned>((k >> 1) & 1));
        const unsigned unit = ld_shared_u32(unitq_u + 4u * q);
        __syncwarp();
        if (lane == 0) mbar_arrive_u(ubar_u + 16u + 8u * q);
        if (unit == 0xffffffffu) break;
        const int band = static_cast<int>(unit / F.n_maps);
        const int64_t map = unit % F.n_maps;
        const int c0 = band * kBandOut;
        const int jb = c0 - hc;
        const int wc0 = c0 + warp * kWarp;
        const int c = wc0 + lane;
        const ColConst K = col_const(c, cols, hc, gc, jb + kTabShift);
        const bool okc[1] = {K.ok};
        // SAT lanes of my four tap columns, and the warp's lane range
        const int l_xa = static_cast<int>(K.xa / 8u) / kCpl, l_xb = static_cast<int>(K.xb / 8u) / kCpl;
        const int l_ya = static_cast<int>(K.ya / 8u) / kCpl, l_yb = static_cast<int>(K.yb / 8u) / kCpl;
        const int l_hi = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(l_xb));
        const int l_lo = static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(l_xa)));
        // a warp right of the map only keeps the barrier protocol (so does every
        // warp under the UWB_FUSED_DEBUG=1 probe)
        const bool warp_live = wc0 < cols && !(L.debug & 1u);
        // Rows with unclamped windows take the fast path in every column: the
        // clamped column edges are in K, and n is constant down a column there
        // (cfar.cpp:28-32 with full-height windows).
        const bool fast_cols = !per_cell;
        const int n_col = (2 * hr + 1) * K.ow - (2 * gr + 1) * K.gw;
        const double alpha_col = n_col > 0 ? __ldg(L.alpha + n_col) : 0.0;
        // 0 <= cut < sum * fast_k  implies  cut < alpha * (sum / n) (relative margin 1e-13)
        const double fast_k = n_col > 0 ? dmul(ddiv(alpha_col, static_cast<double>(n_col)), 1.0 - 1e-13) : 0.0;
        const T* cp = static_cast<const T*>(L.maps) + map * L.map_stride + (K.ok ? c : 0); // CUT, row r0 + 4
        uint32_t* mrow = L.mask_bits ? L.mask_bits + map * L.mask_map_stride + (wc0 >> 5) : nullptr;
        auto slot_of = [&](int i) { return ((vb + i) % nr + nr) % nr; };
        auto tap_at = [&](int i, unsigned xoff, int lt) {
            return *reinterpret_cast<const double*>(ring + static_cast<unsigned>(slot_of(i + lt)) * kRowBytes + xoff);
        };
        // fast-path tap pointers: window rows A = r0 - hr, B = r0 + hr + 1, C = r0 - gr, D = r0 + gr + 1
        auto wrap = [&](unsigned o) { return o >= ring_bytes ? o - ring_bytes : o; };
        unsigned oAa = wrap(static_cast<unsigned>(slot_of(-hr + l_xa)) * kRowBytes);
        unsigned oAb = wrap(static_cast<unsigned>(slot_of(-hr + l_xb)) * kRowBytes);
        unsigned oBa = wrap(static_cast<unsigned>(slot_of(hr + 1 + l_xa)) * kRowBytes);
        unsigned oBb = wrap(static_cast<unsigned>(slot_of(hr + 1 + l_xb)) * kRowBytes);
        unsigned oCa = wrap(static_cast<unsigned>(slot_of(-gr + l_ya)) * kRowBytes);
        unsigned oCb = wrap(static_cast<unsigned>(slot_of(-gr + l_yb)) * kRowBytes);
        unsigned oDa = wrap(static_cast<unsigned>(slot_of(gr + 1 + l_ya)) * kRowBytes);
        unsigned oDb = wrap(static_cast<unsigned>(slot_of(gr + 1 + l_yb)) * kRowBytes);
        int waited = -1, released = -1; // unit groups known full / handed back
        int ncache = -1;
        double kcache = 0.0;
        // CUT values of the next step (loaded one step ahead, widened at use)
        T vn[kRs];
#pragma unroll
        for (int kk = 0; kk < kRs; ++kk) vn[kk] = (K.ok && kk < rows) ? cp[kk * ld] : T(0);
        cp += kRs * ld;

        for (int step = 0; step < n_steps; ++step) {
            const int r0 = step * kRs;
            const int r_last = min(r0 + kRs, rows) - 1;
            {
                // newest entry read: padded row min(rows, r_last + hr + 1) in SAT lane l_hi
                const int need = (min(rows, r_last + hr + 1) + l_hi) / kRs;
                while (waited < need) {
                    mbar_wait_u<kCHint>(full_u + 8u * wslot, wpar);
                    ++waited;
                    if (++wslot == static_cast<unsigned>(nq)) { wslot = 0; wpar ^= 1; }
                }
            }
            double v[kRs][1], thr[kRs][1];
            bool hit[kRs][1];
#pragma unroll
            for (int kk = 0; kk < kRs; ++kk) v[kk][0] = widen(vn[kk]);
            if (step + 1 < n_steps) {
                if (K.ok && r0 + 2 * kRs <= rows) {
#pragma unroll
                    for (int kk = 0; kk < kRs; ++kk) vn[kk] = cp[kk * ld];
                } else {
#pragma unroll
                    for (int kk = 0; kk < kRs; ++kk) vn[kk] = (K.ok && r0 + kRs + kk < rows) ? cp[kk * ld] : T(0);
                }
                cp += kRs * ld;
            }
            if (!warp_live) {
                // nothing to evaluate
            } else if (fast_cols && step >= t_fast_lo && step < t_fast_hi) {
                const char* pAa = ring + oAa + K.xa;
                const char* pAb = ring + oAb + K.xb;
                const char* pBa = ring + oBa + K.xa;
                const char* pBb = ring + oBb + K.xb;
                const char* pCa = ring + oCa + K.ya;
                const char* pCb = ring + oCb + K.yb;
                const char* pDa = ring + oDa + K.ya;
                const char* pDb = ring + oDb + K.yb;
                double sum[kRs];
                bool need = false;
#pragma unroll
                for (int kk = 0; kk < kRs; ++kk) {
                    const unsigned o = kk * kRowBytes;
                    const double rs_o = dsub(dadd(tap(pAa, o), tap(pBb, o)), dadd(tap(pAb, o), tap(pBa, o)));
                    const double rs_g = dsub(dadd(tap(pCa, o), tap(pDb, o)), dadd(tap(pCb, o), tap(pDa, o)));
                    sum[kk] = dsub(rs_o, rs_g);
                    need |= !(v[kk][0] < dmul(sum[kk], fast_k)) || v[kk][0] < 0.0;
                }
                if (__any_sync(0xffffffffu, need)) {
#pragma unroll
                    for (int kk = 0; kk < kRs; ++kk) {
                        thr[kk][0] = 0.0;
                        hit[kk][0] = false;
                        if (!(v[kk][0] < dmul(sum[kk], fast_k)) || v[kk][0] < 0.0) {
                            thr[kk][0] = dmul(alpha_col, ddiv(sum[kk], static_cast<double>(n_col)));
                            hit[kk][0] = v[kk][0] > thr[kk][0];
                            if (v[kk][0] < 0.0 && L.first_bad)
                                report_min(L.first_bad + 2 * map + 1,
                                           static_cast<unsigned long long>(static_cast<int64_t>(r0 + kk) * cols + c));
                        }
                    }
                    emit_block<kRs, 1>(L, map, r0, r_last, wc0, c, okc, hit, v, thr, false);
                } else if (lane < kRs && mrow) {
                    mrow[(r0 + lane) * wpr] = 0u;
                }
            } else {
                // clamped windows, per-cell n (cfar.cpp:117-127)
                double sum[kRs], approx[kRs];
                int n[kRs];
                bool need_exact[kRs];
                bool any_slow = false;
#pragma unroll
                for (int kk = 0; kk < kRs; ++kk) {
                    const int r = min(r0 + kk, r_last);
                    const int iA = clamp_lo32(r, hr), iB = clamp_hi32(r, hr, rows) + 1;
                    const int iC = clamp_lo32(r, gr), iD = clamp_hi32(r, gr, rows) + 1;
                    const double rs_o = dsub(dadd(tap_at(iA, K.xa, l_xa), tap_at(iB, K.xb, l_xb)),
                                             dadd(tap_at(iA, K.xb, l_xb), tap_at(iB, K.xa, l_xa)));
                    const double rs_g = dsub(dadd(tap_at(iC, K.ya, l_ya), tap_at(iD, K.yb, l_yb)),
                                             dadd(tap_at(iC, K.yb, l_yb), tap_at(iD, K.ya, l_ya)));
                    sum[kk] = dsub(rs_o, rs_g);
                    n[kk] = (iB - iA) * K.ow - (iD - iC) * K.gw;
                }
#pragma unroll
                for (int kk = 0; kk < kRs; ++kk) {
                    const bool row_ok = r0 + kk <= r_last;
                    if (n[kk] != ncache && row_ok) {
                        ncache = n[kk];
                        kcache = ddiv(__ldg(L.alpha + n[kk]), static_cast<double>(n[kk]));
                    }
                    approx[kk] = dmul(sum[kk], kcache);
                    const bool ok = K.ok && row_ok;
                    hit[kk][0] = ok && v[kk][0] > approx[kk];
                    need_exact[kk] = ok && (per_cell || hit[kk][0] || v[kk][0] < 0.0 ||
                                            !(fabs(dsub(v[kk][0], approx[kk])) > 1e-13 * fabs(approx[kk])));
                    any_slow |= need_exact[kk];
                    thr[kk][0] = 0.0;
                }
                if (__any_sync(0xffffffffu, any_slow)) {
#pragma unroll
                    for (int kk = 0; kk < kRs; ++kk) {
                        if (need_exact[kk]) {
                            thr[kk][0] = dmul(__ldg(L.alpha + n[kk]), ddiv(sum[kk], static_cast<double>(n[kk])));
                            hit[kk][0] = v[kk][0] > thr[kk][0];
                            if (v[kk][0] < 0.0 && L.first_bad)
                                report_min(L.first_bad + 2 * map + 1,
                                           static_cast<unsigned long long>(static_cast<int64_t>(r0 + kk) * cols + c));
                        }
                    }
                }
                emit_block<kRs, 1>(L, map, r0, r_last, wc0, c, okc, hit, v, thr, per_cell);
            }
            // hand back the groups no later step of this unit reads: entries of
            // padded rows < keep_row in lanes >= l_lo, i.e. slots < keep_row + l_lo
            __syncwarp();
            if (step + 1 < n_steps) {
                const int done = (max(0, r_last + 1 - hr) + l_lo) / kRs - 1;
                while (released < done) {
                    ++released;
                    if (lane == 0) mbar_arrive_u(empty_u + 8u * rslot);
                    if (++rslot == static_cast<unsigned>(nq)) rslot = 0;
                }
            }
            constexpr unsigned kAdv = kRs * kRowBytes;
            oAa = wrap(oAa + kAdv); oAb = wrap(oAb + kAdv); oBa = wrap(oBa + kAdv); oBb = wrap(oBb + kAdv);
            oCa = wrap(oCa + kAdv); oCb = wrap(oCb + kAdv); oDa = wrap(oDa + kAdv); oDb = wrap(oDb + kAdv);
        }
        // every group of the unit is waited for and handed back once
        while (waited < groups - 1) {
            mbar_wait_u<kCHint>(full_u + 8u * wslot, wpar);
            ++waited;
            if (++wslot == static_cast<unsigned>(nq)) { wslot = 0; wpar ^= 1; }
        }
        __syncwarp();
        while (released < groups - 1) {
            ++released;
            if (lane == 0) mbar_arrive_u(empty_u + 8u * rslot);
            if (++rslot == static_cast<unsigned>(nq)) rslot = 0;
        }
        vb += vstep;
        if (vb >= nr) vb -= nr;
    }
}

template <typename T, int kCpl, int OCC>
cudaError_t go_fused(const FusedLaunch& F, cudaStream_t stream) {
    const size_t smem = FusedSmem<T, kCpl>::bytes(F.nr);
    cudaError_t e = cudaFuncSetAttribute(cfar_fused_kernel<T, kCpl, OCC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cfar_fused_kernel<T, kCpl, OCC>, (kNcw + 1) * kWarp, smem);
    if (per_sm < 1) return cudaErrorNotSupported;
    const int64_t grid = imin(F.n_units, static_cast<int64_t>(sms) * per_sm);
    ++g_kernel_launches;
    cfar_fused_kernel<T, kCpl, OCC><<<static_cast<unsigned>(grid), (kNcw + 1) * kWarp, smem, stream>>>(F);
    return cudaGetLastError();
}

template <typename T, int kCpl>
cudaError_t go_fused_occ(FusedLaunch F, cudaStream_t stream) {
    // The ring must hold, for every CFAR warp, the window (2 hr + 1 rows) plus
    // the SAT lanes its taps span (the wavefront skew between them), plus
    // group alignment on both sides (see the deadlock bound in DESIGN.md);
    // more slots only add look-ahead.
    // Deadlock bound: the SAT opens slot group 4G' while the CFAR warps still
    // need the group it replaces until they have passed rows 2 hr + (l_hi - l_lo)
    // + 14 further on, so nr >= 2 hr + (l_hi - l_lo) + 14, with l_hi - l_lo the
    // SAT lanes one CFAR warp's taps span; one group of margin on top.
    const int span_lanes = (kWarp + 2 * F.c.hc + 1 + kCpl - 1) / kCpl + 2;
    const int need = ((2 * F.c.hr + span_lanes + 14 + kRs - 1) / kRs + 1) * kRs;
    int pinned = 0;
    if (const char* e = UWB_KNOB("UWB_FUSED_OCC")) pinned = atoi(e);
    for (int occ : {3, 2, 1}) {
        if (pinned && occ != pinned) continue;
        const size_t budget = static_cast<size_t>(233472 / occ - 1024);
        int nr = need;
        if (FusedSmem<T, kCpl>::bytes(nr) > budget) continue;
        while (FusedSmem<T, kCpl>::bytes(nr + kRs) <= budget && nr + kRs <= need + 64) nr += kRs;
        if (const char* e = UWB_KNOB("UWB_FUSED_RING")) nr = std::max(need, atoi(e) / kRs * kRs);
        F.nr = nr;
        switch (occ) {
            case 3: return go_fused<T, kCpl, 3>(F, stream);
            case 2: return go_fused<T, kCpl, 2>(F, stream);
            default: return go_fused<T, kCpl, 1>(F, stream);
        }
    }
    return cudaErrorNotSupported;
}

template <typename T>
cudaError_t go_fused_cpl(const FusedLaunch& F, cudaStream_t stream) {
    const int span = kBandOut + 2 * F.c.hc + 1; // band columns the windows tap
    if (span <= kWarp * 5) return go_fused_occ<T, 5>(F, stream);
    if (span <= kWarp * 6) return go_fused_occ<T, 6>(F, stream);
    if (span <= kWarp * 8) return go_fused_occ<T, 8>(F, stream);
    return cudaErrorNotSupported;
}

} // namespace

// Whole-map batches only (no row window / slabs). Returns cudaErrorNotSupported
// when the geometry does not qualify (the caller runs SAT + CFAR instead).
cudaError_t launch_cfar_fused(const SatLaunch& S, const CfarLaunch& C, int dtype, cudaStream_t stream) {
    if (const char* e = UWB_KNOB("UWB_FUSED"))
        if (atoi(e) == 0) return cudaErrorNotSupported;
    const JobGeometry& g = C.geo;
    if (g.n_slabs != 1 || g.n_bands != 1 || g.row_lo != 0 || g.row_hi != g.rows || g.buf_row0 != 0 || g.buf_rows != g.rows)
        return cudaErrorNotSupported;
    if (g.rows < 1 || g.rows >= (int64_t(1) << 30) || C.cols < 1 || C.cols >= (int64_t(1) << 30))
        return cudaErrorNotSupported;
    FusedLaunch F{};
    F.c = C;
    F.n_maps = C.n_jobs;
    F.n_bands = static_cast<int>((C.cols + kBandOut - 1) / kBandOut);
    F.n_units = F.n_maps * F.n_bands;
    if (F.n_units >= (int64_t(1) << 32) - 1) return cudaErrorNotSupported;
    F.strips = S.strips;
    if (F.n_bands > 1 && (S.strips < F.n_bands || !S.gedge || S.edge_stride < g.rows)) return cudaErrorNotSupported;
    F.gedge = S.gedge;
    F.edge_stride = S.edge_stride;
    F.gprog = S.gprog;
    F.unit_counter = S.tile_counter;
    F.c.debug = 0;
#ifdef UWB_PROBE_BUILD // timing probes only: skip the arithmetic (never in the release library)
    if (const char* e = UWB_KNOB("UWB_FUSED_DEBUG")) F.c.debug = static_cast<unsigned>(atoi(e));
#endif
    return dtype == UWB_F32 ? go_fused_cpl<float>(F, stream) : go_fused_cpl<double>(F, stream);
}

} // namespace uwb
