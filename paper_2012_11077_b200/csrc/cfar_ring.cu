// Kernel (d), production path: warp-specialised CA-CFAR over shared-memory rings
// of table rows.
//
// Replaces cfar_rows / run_cfar of /root/reference/proj/src/cfar.cpp:109-175 for
// the integral-image backend (cfar2d_integral, cfar.cpp:218-227).
//
// A CTA owns a W-column x 256-row tile of one job (W = 32 x consumer warps).
// One producer warp streams every table row the tile's windows touch into a
// shared-memory ring with the TMA engine (cp.async.bulk global->shared, one
// 16-byte-aligned row segment per copy), and the CUT row segments into a second
// ring; rows move in groups of 4 that complete on one "full" mbarrier. The
// consumer warps (one output column per thread) wait on "full", evaluate 4
// output rows, and hand slots back through "empty" mbarriers, so the two sides
// never meet at a CTA barrier. The eight taps of a cell are shared-memory reads:
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
constexpr int kAheadGroups = 3;  // groups of look-ahead

struct RingGeom {
    int ng;     // table row groups in the ring
    int nr;     // table row slots (ng * kG)
    int stride; // doubles per table slot
    int ncg;    // CUT row groups
};

__host__ __device__ inline RingGeom ring_geom(int w, int hr, int hc) {
    RingGeom g;
    // output rows r..r+3 read table rows r-hr .. r+4+hr: 2hr+5 rows, spread over
    // at most ceil((2hr+5)/4)+1 groups
    g.ng = (2 * hr + 5 + kG - 1) / kG + 1 + kAheadGroups;
    g.nr = g.ng * kG;
    g.stride = w + 2 * hc + 4;
    g.ncg = 1 + kAheadGroups;
    return g;
}

template <typename T>
inline size_t ring_smem_bytes(int w, int hr, int hc) {
    const RingGeom g = ring_geom(w, hr, hc);
    return sizeof(double) * static_cast<size_t>(g.nr) * g.stride + sizeof(T) * static_cast<size_t>(g.ncg) * kG * w +
           2 * sizeof(uint64_t) * (g.ng + g.ncg);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename T, int NCW>
__global__ void __launch_bounds__((NCW + 1) * kWarp)
cfar_ws_kernel(CfarLaunch L) {
    constexpr int W = NCW * kWarp;
    extern __shared__ __align__(16) unsigned char ring_smem[];
    const RingGeom G = ring_geom(W, L.hr, L.hc);
    double* slots = reinterpret_cast<double*>(ring_smem);
    T* cuts = reinterpret_cast<T*>(slots + static_cast<size_t>(G.nr) * G.stride);
    uint64_t* full_t = reinterpret_cast<uint64_t*>(cuts + static_cast<size_t>(G.ncg) * kG * W);
    uint64_t* full_c = full_t + G.ng;
    uint64_t* empty_t = full_c + G.ncg;
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
    const unsigned cut_bytes = static_cast<unsigned>(strip_w * static_cast<int>(sizeof(T)));
    const bool cut_bulk = (cut_bytes % 16 == 0) && (reinterpret_cast<uintptr_t>(cut_base + c0) % 16 == 0) &&
                          ((L.ld * sizeof(T)) % 16 == 0);

    // padded table rows needed by output rows [ra, rb), in groups of kG from i_lo
    const int i_lo = max(0, ra - hr);
    const int i_hi = min(rows, rb + hr);
    const int n_steps = (rb - ra + kG - 1) / kG;
    auto need_grp = [&](int step) { // last table group read by output step `step`
        const int r_last = min(ra + step * kG + kG, rb) - 1;
        return (clamp_hi32(r_last, hr, rows) + 1 - i_lo) / kG;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < G.ng + G.ncg; ++s) {
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
        int grp = 0;  // next table group to issue
        const int last_grp = (i_hi - i_lo) / kG;
        for (int step = 0; step < n_steps; ++step) {
            const int need = min(need_grp(step), last_grp);
            for (; grp <= need; ++grp) {
                const int s = grp % G.ng;
                if (grp >= G.ng) mbar_wait(&empty_t[s], static_cast<unsigned>((grp / G.ng - 1) & 1));
                const int first = i_lo + grp * kG;
                const int cnt = min(kG, i_hi + 1 - first);
                mbar_expect_tx(&full_t[s], copy_bytes * cnt);
                for (int k = 0; k < cnt; ++k)
                    bulk_g2s(slots + static_cast<size_t>(s * kG + k) * G.stride,
                             tab + static_cast<int64_t>(first + k - trow0) * ld + e_lo, copy_bytes, &full_t[s]);
            }
            if (cut_bulk) {
                const int s = step % G.ncg;
                if (step >= G.ncg) mbar_wait(&empty_c[s], static_cast<unsigned>((step / G.ncg - 1) & 1));
                const int first = ra + step * kG;
                const int cnt = min(kG, rb - first);
                mbar_expect_tx(&full_c[s], cut_bytes * cnt);
                for (int k = 0; k < cnt; ++k)
                    bulk_g2s(cuts + static_cast<size_t>(s * kG + k) * W,
                             cut_base + static_cast<int64_t>(first + k) * L.ld + c0, cut_bytes, &full_c[s]);
            }
        }
        return;
    }

    // ============================ consumer warps ============================
    const int c = c0 + static_cast<int>(threadIdx.x);
    const bool col_ok = c < cols;
    const int ring_len = G.nr * G.stride;
    int waited = -1;          // table groups [0, waited] known resident
    int released = -1;        // table groups [0, released] handed back
    // tap rows and their ring offsets (doubles)
    int iA = clamp_lo32(ra, hr), iB = clamp_hi32(ra, hr, rows) + 1;
    int iC = clamp_lo32(ra, gr), iD = clamp_hi32(ra, gr, rows) + 1;
    int oA = ((iA - i_lo) % G.nr) * G.stride, oB = ((iB - i_lo) % G.nr) * G.stride;
    int oC = ((iC - i_lo) % G.nr) * G.stride, oD = ((iD - i_lo) % G.nr) * G.stride;

    // per-column constants
    const int oc0 = clamp_lo32(c, hc), oc1 = clamp_hi32(c, hc, cols);
    const int gc0 = clamp_lo32(c, gc), gc1 = clamp_hi32(c, gc, cols);
    const int ow = oc1 - oc0 + 1, gw = gc1 - gc0 + 1;
    const int xa = kTabShift + oc0 - e_lo, xb = kTabShift + 1 + oc1 - e_lo;
    const int ya = kTabShift + gc0 - e_lo, yb = kTabShift + 1 + gc1 - e_lo;
    const bool exact_always = L.thresholds != nullptr;

    int n_cached = -1;
    double k_cached = 0.0; // alpha[n] / n for the fast comparison

    for (int step = 0; step < n_steps; ++step) {
        const int r0 = ra + step * kG;
        const int r_last = min(r0 + kG, rb) - 1;
        {
            const int need = need_grp(step);
            while (waited < need) {
                ++waited;
                mbar_wait(&full_t[waited % G.ng], static_cast<unsigned>((waited / G.ng) & 1));
            }
        }
        const int cs = step % G.ncg;
        if (cut_bulk) mbar_wait(&full_c[cs], static_cast<unsigned>((step / G.ncg) & 1));
        const T* cut_grp = cuts + static_cast<size_t>(cs) * kG * W;
#pragma unroll
        for (int k = 0; k < kG; ++k) {
            const int r = r0 + k;
            if (r > r_last) break; // uniform
            {   // advance the tap cursors (each moves by 0 or 1 row per output row)
                const int nA = clamp_lo32(r, hr), nB = clamp_hi32(r, hr, rows) + 1;
                const int nC = clamp_lo32(r, gr), nD = clamp_hi32(r, gr, rows) + 1;
                if (nA != iA) { iA = nA; oA += G.stride; if (oA == ring_len) oA = 0; }
                if (nB != iB) { iB = nB; oB += G.stride; if (oB == ring_len) oB = 0; }
                if (nC != iC) { iC = nC; oC += G.stride; if (oC == ring_len) oC = 0; }
                if (nD != iD) { iD = nD; oD += G.stride; if (oD == ring_len) oD = 0; }
            }
            double v = 0.0, sum = 0.0, approx = 0.0;
            int n = 1;
            bool need_exact = false, hit = false;
            if (col_ok) {
                v = cut_bulk ? static_cast<double>(cut_grp[k * W + threadIdx.x])
                             : static_cast<double>(cut_base[static_cast<int64_t>(r) * L.ld + c]);
                const double* pA = slots + oA;
                const double* pB = slots + oB;
                const double* pC = slots + oC;
                const double* pD = slots + oD;
                const double rs_o = dsub(dadd(pA[xa], pB[xb]), dadd(pA[xb], pB[xa]));
                const double rs_g = dsub(dadd(pC[ya], pD[yb]), dadd(pC[yb], pD[ya]));
                sum = dsub(rs_o, rs_g);
                n = (iB - iA) * ow - (iD - iC) * gw;
                if (n != n_cached) {
                    n_cached = n;
                    k_cached = ddiv(__ldg(L.alpha + n), static_cast<double>(n));
                }
                approx = dmul(sum, k_cached);
                hit = v > approx;
                need_exact = exact_always || hit || !(fabs(dsub(v, approx)) > 1e-13 * fabs(approx));
                if (v < 0.0)
                    report_min(L.first_bad + 2 * map + 1,
                               static_cast<unsigned long long>(static_cast<int64_t>(r) * cols + c));
            }
            double thr = 0.0;
            if (__any_sync(0xffffffffu, need_exact)) {
                if (need_exact) {
                    thr = dmul(__ldg(L.alpha + n), ddiv(sum, static_cast<double>(n)));
                    hit = v > thr;
                }
            }
            emit_cells(L, map, r, c, col_ok, hit, v, thr);
        }
        // hand back this step's CUT group and the table groups no later step reads
        __syncwarp();
        if (lane == 0) {
            if (cut_bulk) mbar_arrive(&empty_c[cs]);
            if (step + 1 < n_steps) {
                const int keep_row = max(0, r_last + 1 - hr);
                const int done = (keep_row - i_lo) / kG - 1; // groups entirely below keep_row
                for (; released < done; ) {
                    ++released;
                    mbar_arrive(&empty_t[released % G.ng]);
                }
            }
        }
    }
}

template <typename T, int NCW>
cudaError_t go(const CfarLaunch& L0, size_t smem, cudaStream_t stream) {
    constexpr int W = NCW * kWarp;
    CfarLaunch L = L0;
    L.col_tiles = (L.cols + W - 1) / W;
    L.row_chunks = (L.geo.slab_rows + kRingRows - 1) / kRingRows;
    const dim3 grid(static_cast<unsigned>(L.col_tiles * L.row_chunks), static_cast<unsigned>(L.n_jobs), 1);
    cudaError_t e = cudaFuncSetAttribute(cfar_ws_kernel<T, NCW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    ++g_kernel_launches;
    cfar_ws_kernel<T, NCW><<<grid, (NCW + 1) * kWarp, smem, stream>>>(L);
    return cudaGetLastError();
}

} // namespace

// Returns cudaErrorNotSupported when the rings do not fit (caller falls back).
cudaError_t launch_cfar_ring(const CfarLaunch& L, int dtype, cudaStream_t stream) {
    if (getenv("UWB_CFAR_SIMPLE")) return cudaErrorNotSupported;
    if (L.geo.rows >= (int64_t(1) << 31) || L.cols >= (int64_t(1) << 30)) return cudaErrorNotSupported;
    const bool f32 = dtype == UWB_F32;
    const size_t s256 = f32 ? ring_smem_bytes<float>(256, L.hr, L.hc) : ring_smem_bytes<double>(256, L.hr, L.hc);
    const size_t s128 = f32 ? ring_smem_bytes<float>(128, L.hr, L.hc) : ring_smem_bytes<double>(128, L.hr, L.hc);
    if (s256 <= 113 * 1024 && L.cols > 128)
        return f32 ? go<float, 8>(L, s256, stream) : go<double, 8>(L, s256, stream);
    if (s128 <= 200 * 1024)
        return f32 ? go<float, 4>(L, s128, stream) : go<double, 4>(L, s128, stream);
    return cudaErrorNotSupported;
}

} // namespace uwb
