// Certified-decision CA-CFAR: the throughput path of the integral-image backend.
//
// Replaces cfar_rows / run_cfar (/root/reference/proj/src/cfar.cpp:109-175) for
// batches that want masks and detection lists (no per-cell threshold map), with
// results identical to the two-kernel path (SAT + cfar_ws_kernel) and therefore
// to cfar2d_integral (cfar.cpp:218-227) bit for bit.
//
// The reference decides cut > T with T = alpha[n] * ((RS(outer) - RS(guard)) / n)
// evaluated from the fp64 summed-area table (sat.cpp:33, sat.hpp:32-33). Almost
// every cell is far below T, so the exact table value is only needed near T:
//
//  1. cert_kernel reads the map once. Each input value is quantised to a grid of
//     2^-s (q = round(x * 2^s), error <= 2^-(s+1)); window sums of q are exact in
//     32-bit integer arithmetic (sliding sums, wrap-around cancels). The
//     reference's table rounding is bounded a priori: every table entry is a
//     sum of non-negative cells below S = cells * X_lim, so each of the three
//     additions of sat.cpp:33 errs by at most 4u*S per cell and the ring sum of
//     n cells by (4n + 11) u S (region-sum association of sat.hpp:32-33, the
//     final subtraction, u = 2^-53). A cell with
//         (cut_q + 2^-(s+1)) * n / alpha[n] * (1 + 4e-6) < Q - n 2^-(s+1) - (4n+11) u S
//     (directed rounding in every float operation) is certainly not a detection
//     and lies outside the 1e-6 tie band. Every other cell is a candidate
//     (about Pfa of the cells plus the targets).
//  2. cert_mark_kernel marks the eight table taps of every candidate in a bitmap.
//  3. The SAT kernel (sat.cu) runs the exact recurrence over the whole map but
//     stores only the marked 32-byte table segments (sparse mode).
//  4. cert_resolve_kernel evaluates each candidate exactly as cfar.cpp:115-127
//     from those taps: mask bit, detection record {row, col, value, threshold},
//     tie-band cell (|cut - T| <= 1e-6 T).
// A map with a value outside [0, X_lim) (X_lim = 2^9 by default), or more
// candidates than the list holds, is flagged and runs the exact two-kernel path
// instead (full table for that map + cfar_ws_kernel restricted to flagged maps),
// inside the same stream-ordered call.
//
// HBM per cell: 4 B (map) here + 4 B (map) in the sparse SAT, against 24.125 B
// for materialising the table and reading it back.
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "cfar_common.cuh"

namespace uwb {

namespace {

// ---- geometry --------------------------------------------------------------
// The map is cut into 2x2 tiles (tile-row I = rows 2I, 2I+1). Per axis, a cell
// at 2I + a (a = 0, 1) with outer half-width h and guard half-width g has its
// outer window fully covering tiles I + [so(a), eo(a)] and its guard window
// inside tiles I + [sg(a), eg(a)]; the tile box minus the guard tile box lies
// inside the cell's training ring, so its sum is a lower bound of the ring sum.
constexpr int kTB = 8;         // tile-rows per phase
constexpr int kTW = 128;       // output tile-columns per CTA (256 columns)
constexpr int kItemTiles = 8;  // tiles per horizontal item
constexpr int kPT = 8;         // tile-rows of register prefetch
constexpr int kL2AheadT = 24;  // tile-rows of L2 prefetch
constexpr int kStage = 64;     // cells of passing tiles staged per phase (shared memory)
constexpr int kCandLocal = 384; // candidates a CTA collects in shared memory before its one global append (cfg 5: ~260 per CTA)

__host__ __device__ constexpr int fdiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }
__host__ __device__ constexpr int cdiv(int a, int b) { return -fdiv(-a, b); }
__host__ __device__ constexpr int imn(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int imx(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int rup(int a, int b) { return (a + b - 1) / b * b; }

struct TileAxis {
    int so0, so1, eo0, eo1, lo; // outer tile box per parity, length
    int sg0, sg1, eg0, eg1, lg; // guard tile box per parity, length
    int hl, hh;                 // tiles needed below / above a tile
};
__host__ __device__ constexpr TileAxis tile_axis(int h, int g) {
    TileAxis t{};
    t.so0 = cdiv(-h, 2), t.so1 = cdiv(1 - h, 2), t.eo0 = fdiv(h - 1, 2), t.eo1 = fdiv(h, 2);
    t.lo = t.eo0 - t.so0 + 1;
    t.sg0 = cdiv(-g - 1, 2), t.sg1 = cdiv(-g, 2), t.eg0 = fdiv(g, 2), t.eg1 = fdiv(g + 1, 2);
    t.lg = t.eg0 - t.sg0 + 1;
    t.hl = -imn(imn(t.so0, t.so1), imn(t.sg0, t.sg1));
    t.hh = imx(imx(t.eo0, t.eo1), imx(t.eg0, t.eg1));
    return t;
}

template <int HR, int GR, int HC, int GC, int ESZ>
struct CertGeo {
    static constexpr TileAxis R = tile_axis(HR, GR), C = tile_axis(HC, GC);
    static_assert(R.eo1 - R.so1 + 1 == R.lo && R.eg1 - R.sg1 + 1 == R.lg, "row tile boxes");
    static_assert(C.eo1 - C.so1 + 1 == C.lo && C.eg1 - C.sg1 + 1 == C.lg, "column tile boxes");
    static_assert(R.so0 <= R.sg0 && R.so1 <= R.sg1 && R.eg0 <= R.eo0 && R.eg1 <= R.eo1, "guard inside outer");
    static_assert(C.so0 <= C.sg0 && C.so1 <= C.sg1 && C.eg0 <= C.eo0 && C.eg1 <= C.eo1, "guard inside outer");
    static constexpr int NT = rup(kTW + C.hl + C.hh, 32); // one thread per input tile-column
    static constexpr int LAG = cdiv(kTB + R.hl + R.hh, kTB); // phases between a tile-row's Z and its test
    static constexpr int SOMIN = imn(R.so0, R.so1), SGMIN = imn(R.sg0, R.sg1);
    // shared rings of window sums (slot = completion step mod NB) and tile maxima:
    // one barrier per phase, so the rows read by phase p's items must survive
    // phase p + 1's vertical writes
    static constexpr int NBO = rup(kTB * LAG + 2 * kTB + 1 - R.hl - SOMIN - R.lo, 8);
    static constexpr int NBG = rup(kTB * LAG + 2 * kTB + 1 - R.hl - SGMIN - R.lg, 8);
    static constexpr int NBC = rup(kTB * LAG + 2 * kTB - R.hl, 8);
    static constexpr int SW = NT + 1; // ring row stride (words), == 1 (mod 32) with NT % 32 == 0
    // tile maxima are 16-bit upper bounds (the top half of the float, rounded up)
    static constexpr int SWC = rup(SW, 2) / 2 + 1; // words per tile-max row (odd)
    static constexpr size_t smem =
        sizeof(uint32_t) * (static_cast<size_t>(NBO + NBG) * SW + static_cast<size_t>(NBC) * SWC + 2 * (3 * kStage + 1) +
                            2 * kCandLocal + 4);
    static constexpr int OCC = smem * 3 <= 220 * 1024 ? 3 : 2;
};

__device__ __align__(16) float g_cert_zero[4]; // source of the tile-columns outside the map

template <typename T>
struct CertIO;

template <>
struct CertIO<float> {
    using Raw = uint32_t;
    using Raw2 = uint2;
    static __device__ __forceinline__ uint2 load2(const void* p) {
        uint2 v;
        asm volatile("ld.global.nc.L1::no_allocate.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
        return v;
    }
    static __device__ __forceinline__ uint2 zero2() { return make_uint2(0u, 0u); }
    // q' = bits(x + M) = bits(M) + round(x 2^s) for 0 <= x < X_lim <= M
    static __device__ __forceinline__ uint32_t quant(Raw b, const CertLaunch& L) {
        return __float_as_uint(__fadd_rn(__uint_as_float(b), L.magic));
    }
    static __device__ __forceinline__ Raw mx2(uint2 v) { return max(v.x, v.y); }
    static __device__ __forceinline__ Raw lo(uint2 v) { return v.x; }
    static __device__ __forceinline__ Raw hi(uint2 v) { return v.y; }
    // every value outside [0, X_lim) (negative, -0, NaN, Inf, too large) has bits >= bits(X_lim)
    static __device__ __forceinline__ bool in_range(Raw mx, const CertLaunch& L) { return mx < L.xlim_bits; }
    static __device__ __forceinline__ uint32_t cut_bits(Raw b) { return b; } // float bits of an upper bound
    static __device__ __forceinline__ double value(Raw b) { return static_cast<double>(__uint_as_float(b)); }
};

template <>
struct CertIO<double> {
    using Raw = unsigned long long;
    using Raw2 = ulonglong2;
    static __device__ __forceinline__ ulonglong2 load2(const void* p) {
        ulonglong2 v;
        asm volatile("ld.global.nc.L1::no_allocate.v2.b64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
        return v;
    }
    static __device__ __forceinline__ ulonglong2 zero2() { return make_ulonglong2(0ull, 0ull); }
    static __device__ __forceinline__ uint32_t quant(Raw b, const CertLaunch& L) {
        const double d = __longlong_as_double(static_cast<long long>(b));
        return static_cast<uint32_t>(__double2uint_rn(__dmul_rn(d, L.scale))) + L.bits_magic;
    }
    static __device__ __forceinline__ Raw mx2(ulonglong2 v) { return max(v.x, v.y); }
    static __device__ __forceinline__ Raw lo(ulonglong2 v) { return v.x; }
    static __device__ __forceinline__ Raw hi(ulonglong2 v) { return v.y; }
    static __device__ __forceinline__ bool in_range(Raw mx, const CertLaunch& L) {
        return mx < static_cast<Raw>(__double_as_longlong(L.xlim));
    }
    static __device__ __forceinline__ uint32_t cut_bits(Raw b) {
        return __float_as_uint(__double2float_ru(__longlong_as_double(static_cast<long long>(b))));
    }
    static __device__ __forceinline__ double value(Raw b) { return __longlong_as_double(static_cast<long long>(b)); }
};

// A value outside [0, X_lim): non-finite and negative cells are the reference's
// input errors (sat.cpp:28-32, cfar.cpp:85-92, first row-major cell); -0.0 is a
// valid zero; anything else is out of the certified range (the map runs exact).
__device__ __noinline__ void cert_classify(const CertLaunch& L, int64_t map, int row, int col, double v) {
    if (v == 0.0 || (v > 0.0 && v < L.xlim)) return;
    const unsigned long long cell =
        static_cast<unsigned long long>(static_cast<int64_t>(row) * L.geo.map_cols + col);
    if (!isfinite(v)) {
        report_min(L.first_bad + 2 * map, cell);
    } else if (v < 0.0) {
        report_min(L.first_bad + 2 * map + 1, cell);
    }
    atomicOr(L.status + map, 2u);
}

__device__ __forceinline__ uint32_t lds1(unsigned a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts1(unsigned a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

template <int I, int N, typename F>
__device__ __forceinline__ void static_for_impl(F&& f) {
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        static_for_impl<I + 1, N>(f);
    }
}
template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
    static_for_impl<0, N>(f);
}

// Sliding sums over L consecutive words of one ring row: out[m] = sum of words
// [m, m + L) (word address `row` + 4 * first column), m = 0 .. N-1.
template <int L, int N>
__device__ __forceinline__ void row_windows(unsigned row, uint32_t (&out)[N]) {
    uint32_t h = 0;
#pragma unroll
    for (int m = 0; m < L; ++m) h += lds1(row + 4u * m);
    out[0] = h;
#pragma unroll
    for (int m = 1; m < N; ++m) {
        h += lds1(row + 4u * (m + L - 1)) - lds1(row + 4u * (m - 1));
        out[m] = h;
    }
}

// Exact candidate test of one cell whose tile passed the tile test (rare): its
// own n (clamped windows, cfar.cpp:28-32), its own tile bound and its exact CUT.
template <typename T>
__device__ __forceinline__ bool cert_cell_test(const CertLaunch& L, int64_t map, int r, int c, uint32_t lb) {
    const int R = static_cast<int>(L.geo.rows), C = static_cast<int>(L.cols);
    const int n = (min(r + L.hr, R - 1) - max(r - L.hr, 0) + 1) * (min(c + L.hc, C - 1) - max(c - L.hc, 0) + 1) -
                  (min(r + L.gr, R - 1) - max(r - L.gr, 0) + 1) * (min(c + L.gc, C - 1) - max(c - L.gc, 0) + 1);
    const float4 ke = __ldg(L.ke + n);
    const T* src = static_cast<const T*>(L.maps) + map * L.map_stride + (r - L.geo.buf_row0) * L.ld + c;
    const float x = sizeof(T) == 4 ? static_cast<float>(__ldg(src)) : __double2float_ru(static_cast<double>(__ldg(src)));
    // cut >= T_ref (1 - 4e-6) is impossible when x K_n < LB 2^-s - E_n (see the header)
    return __fmul_ru(x, ke.x) >= __fmaf_rd(__uint2float_rd(lb), L.inv_scale, -ke.z);
}

// Candidates are collected per CTA in shared memory (cs[0 .. kCandLocal), count *cn) and
// appended to the map's list once, at the end of the kernel: a global atomic with a
// returned slot per candidate cost the service warp - for which the whole CTA waits at the
// next barrier - an L2 round trip each (certify pass 5.90 -> see DESIGN.md).
__device__ __forceinline__ void cert_append_global(const CertLaunch& L, int64_t map, int2 rc) {
    const unsigned slot = atomicAdd(L.cand_count + map, 1u);
    if (slot < static_cast<unsigned>(L.cand_cap))
        L.cand[map * L.cand_cap + slot] = rc;
    else
        atomicOr(L.status + map, 1u);
}
__device__ __forceinline__ void cert_append(const CertLaunch& L, int64_t map, int r, int c, int2* cs, unsigned* cn) {
    const unsigned i = atomicAdd(cn, 1u);
    if (i < static_cast<unsigned>(kCandLocal))
        cs[i] = make_int2(r, c);
    else
        cert_append_global(L, map, make_int2(r, c)); // local list full (rare)
}

// Cells of passing tiles are staged in shared memory by the item threads and
// tested by the CTA's service warp (threads >= 128, idle during the item pass)
// one phase later, so no item thread waits on a global load.
// Service warp: exact tests of the cells staged in the previous phase, then
// empties the buffer (it is refilled two phases later, after two barriers).
template <typename T>
__device__ __noinline__ void cert_service(const CertLaunch& L, int64_t map, uint32_t* stg, int2* cs, unsigned* cn) {
    const int lane = threadIdx.x & 31;
    const unsigned n = min(stg[0], static_cast<unsigned>(kStage));
    for (unsigned i = lane; i < n; i += 32) {
        const int r = static_cast<int>(stg[1 + i]), c = static_cast<int>(stg[1 + kStage + i]);
        if (cert_cell_test<T>(L, map, r, c, stg[1 + 2 * kStage + i])) cert_append(L, map, r, c, cs, cn);
    }
    __syncwarp();
    if (lane == 0) stg[0] = 0;
}

// A passing tile's 4 cells (rows r0, r0+1, columns c0, c0+1; lb per cell in
// the order (0,0), (0,1), (1,0), (1,1)) into the phase's staging buffer; when
// the buffer is full, tested right here.
template <typename T>
__device__ __noinline__ void cert_stage_tile(const CertLaunch& L, int64_t map, uint32_t* stg, int2* cs, unsigned* cn, int r0,
                                             int c0, int r_s, int r_e, int cols, uint32_t lb0, uint32_t lb1, uint32_t lb2,
                                             uint32_t lb3) {
    const uint32_t lb[4] = {lb0, lb1, lb2, lb3};
#pragma unroll
    for (int cell = 0; cell < 4; ++cell) {
        const int r = r0 + (cell >> 1), c = c0 + (cell & 1);
        if (r >= r_s && r < r_e && c < cols) {
            const unsigned i = atomicAdd(stg, 1u);
            if (i < static_cast<unsigned>(kStage)) {
                stg[1 + i] = static_cast<uint32_t>(r);
                stg[1 + kStage + i] = static_cast<uint32_t>(c);
                stg[1 + 2 * kStage + i] = lb[cell];
            } else if (cert_cell_test<T>(L, map, r, c, lb[cell])) {
                cert_append(L, map, r, c, cs, cn); // staging full (rare)
            }
        }
    }
}

template <typename T, int HR, int GR, int HC, int GC>
__global__ void __launch_bounds__(CertGeo<HR, GR, HC, GC, sizeof(T)>::NT, CertGeo<HR, GR, HC, GC, sizeof(T)>::OCC)
cert_kernel(const __grid_constant__ CertLaunch L) {
    using G = CertGeo<HR, GR, HC, GC, sizeof(T)>;
    using IO = CertIO<T>;
    using Raw = typename IO::Raw;
    using Raw2 = typename IO::Raw2;
    constexpr int SW = G::SW, LAG = G::LAG;
    extern __shared__ __align__(16) uint32_t cert_sm[];
    const unsigned sO = smem_u32(cert_sm);
    const unsigned sG = sO + 4u * G::NBO * SW;
    const unsigned sC = sG + 4u * G::NBG * SW;
    // staging of cells of passing tiles, double-buffered by phase parity:
    // [count, r[kStage], c[kStage], lb[kStage]]
    uint32_t* stage = cert_sm + (G::NBO + G::NBG) * SW + G::NBC * G::SWC;
    // the CTA's candidate list: [count, base slot] + kCandLocal entries (8-byte aligned)
    unsigned* cand_n = reinterpret_cast<unsigned*>(
        (reinterpret_cast<uintptr_t>(stage + 2 * (3 * kStage + 1)) + 7) & ~static_cast<uintptr_t>(7));
    int2* cand_sm = reinterpret_cast<int2*>(cand_n + 2);
    if (threadIdx.x < 2) stage[threadIdx.x * (3 * kStage + 1)] = 0;
    if (threadIdx.x < 2) cand_n[threadIdx.x] = 0;

    const int64_t map = blockIdx.y;
    const int band = static_cast<int>(blockIdx.x % L.col_ctas);
    const int chunk = static_cast<int>(blockIdx.x / L.col_ctas);
    const int cols = static_cast<int>(L.cols);
    const int r_s = static_cast<int>(L.geo.row_lo) + chunk * static_cast<int>(L.row_chunk);
    const int r_e = min(r_s + static_cast<int>(L.row_chunk), static_cast<int>(L.geo.row_hi));
    if (r_s >= r_e) return;
    const int I_s = r_s >> 1, I_e = (r_e + 1) >> 1; // output tile-rows
    const int K0 = I_s - G::R.hl;                     // first tile-row of the vertical pass
    const int n_k = (I_e - I_s) + G::R.hl + G::R.hh;    // vertical steps
    const int J_s = band * kTW;                     // first output tile-column
    const int t = threadIdx.x;
    const int J_in = J_s - G::C.hl + t;               // my input tile-column (columns 2J, 2J+1)
    const bool col_ok = t < kTW + G::C.hl + G::C.hh && J_in >= 0 && 2 * J_in < cols; // cols is even
    const int rb_lo = static_cast<int>(max(int64_t(0), L.geo.buf_row0));
    const int rb_hi = static_cast<int>(min(L.geo.rows, L.geo.buf_row0 + L.geo.buf_rows));
    const uint32_t ld_t = col_ok ? static_cast<uint32_t>(L.ld * sizeof(T)) : 0u; // bytes per row
    const char* col0 = col_ok ? reinterpret_cast<const char*>(static_cast<const T*>(L.maps) + map * L.map_stride +
                                                              (int64_t(0) - L.geo.buf_row0) * L.ld + 2 * J_in)
                              : reinterpret_cast<const char*>(g_cert_zero);
    auto row_ptr = [&](int rho) { return col0 + static_cast<int64_t>(rho) * ld_t; };
    auto load_tile_row = [&](int K, Raw2& a, Raw2& b) { // rows 2K, 2K+1 (checked)
        const int r0 = 2 * K;
        a = (r0 >= rb_lo && r0 < rb_hi) ? IO::load2(row_ptr(r0)) : IO::zero2();
        b = (r0 + 1 >= rb_lo && r0 + 1 < rb_hi) ? IO::load2(row_ptr(r0 + 1)) : IO::zero2();
    };
    const unsigned a_me = 4u * t;

    Raw2 ra[kPT], rb[kPT]; // register prefetch: tile-rows K .. K + kPT - 1
#pragma unroll
    for (int u = 0; u < kPT; ++u) load_tile_row(K0 + u, ra[u], rb[u]);
    // tile-sum history of my column: hz[i] = Z(k0 - lo + i) for i < lo at the
    // start of a phase; the phase appends Z(k0 .. k0 + 7) and shifts by 8
    constexpr int LO = G::R.lo, LG = G::R.lg;
    uint32_t hz[LO + kTB];
#pragma unroll
    for (int i = 0; i < LO; ++i) hz[i] = 4u * L.bits_magic; // tiles before K0: zero cells
    uint32_t vo = LO * 4u * L.bits_magic, vg = LG * 4u * L.bits_magic;
    Raw mx = 0; // largest raw value: out-of-range values compare >= bits(X_lim)
    const float4 kin = __ldg(L.ke + L.n_int); // interior constants (the largest K_n and E_n)
    const int l2t = L.l2_ahead_t;             // L2 prefetch distance (tile-rows)
    const char* pnext = row_ptr(2 * (K0 + kPT)); // the tile-row the next step prefetches
    const int n_items = I_e - I_s;
    const int n_phases = LAG + (n_items + kTB - 1) / kTB;

#pragma unroll 1
    for (int p = 0; p < n_phases; ++p) {
        const int k0 = kTB * p;
        // ---- vertical: tile-rows k0 .. k0 + 7 of my tile-column ----
        if (k0 < n_k) {
            const char* pblk = pnext;
            pnext += static_cast<int64_t>(2 * kTB) * ld_t;
            const unsigned wO = sO + 4u * SW * static_cast<unsigned>(k0 % G::NBO) + a_me;
            const unsigned wG = sG + 4u * SW * static_cast<unsigned>(k0 % G::NBG) + a_me;
            const unsigned wC = sC + 4u * G::SWC * static_cast<unsigned>(k0 % G::NBC) + 2u * t;
            const int r_pf = 2 * (K0 + k0 + kPT); // first row this phase prefetches
            const bool safe = r_pf >= rb_lo && r_pf + 2 * kTB <= rb_hi; // every prefetched row in the buffer
            auto vertical = [&](auto safe_tag) {
                constexpr bool kSafe = decltype(safe_tag)::value;
#pragma unroll
            for (int u = 0; u < kTB; ++u) {
                // consume tile-row K (loaded kPT steps ago) before its slot is reloaded,
                // so the slot keeps one register across phases
                const Raw2 a = ra[u], b = rb[u];
                const Raw mt = max(IO::mx2(a), IO::mx2(b));
                mx = max(mx, mt);
                const uint32_t z = IO::quant(IO::lo(a), L) + IO::quant(IO::hi(a), L) + IO::quant(IO::lo(b), L) +
                                   IO::quant(IO::hi(b), L);
                const int r0 = r_pf + 2 * u; // (warp-uniform bounds)
                const char* pu = pblk + static_cast<uint32_t>(2 * u) * ld_t;
                if (kSafe) {
                    ra[u] = IO::load2(pu);
                    rb[u] = IO::load2(pu + ld_t);
                    if ((u & 3) == 0 && col_ok && l2t > 0 && r0 + 2 * l2t < rb_hi)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(pu + 2 * l2t * ld_t));
                } else {
                    ra[u] = (r0 >= rb_lo && r0 < rb_hi) ? IO::load2(pu) : IO::zero2();
                    rb[u] = (r0 + 1 >= rb_lo && r0 + 1 < rb_hi) ? IO::load2(pu + ld_t) : IO::zero2();
                }
                hz[LO + u] = z;
                vo += z - hz[u];
                vg += z - hz[LO + u - LG];
                const unsigned row = 4u * SW * static_cast<unsigned>(u);
                sts1(wO + row, vo);
                sts1(wG + row, vg);
                asm volatile("st.shared.u16 [%0], %1;" ::"r"(wC + 4u * G::SWC * static_cast<unsigned>(u)),
                             "h"(static_cast<unsigned short>((IO::cut_bits(mt) + 0xFFFFu) >> 16))
                             : "memory");
            }
            };
            // the checked variant (chunk edges) as its own copy, out of the hot path's instruction lines
            if (safe) vertical(std::true_type{});
            else vertical(std::false_type{});
#pragma unroll
            for (int i = 0; i < LO; ++i) hz[i] = hz[i + kTB];
        }
        __syncthreads();
        // ---- horizontal: output tile-row block q, one item = 1 tile-row x 8 tiles ----
        const int q = p - LAG;
        if (q >= 0 && t < kTW) {
            const int ir = t & (kTB - 1), grp = t >> 3;
            const int I = I_s + kTB * q + ir;
            const int J0 = J_s + kItemTiles * grp;
            if (I < I_e && 2 * J0 < cols) {
                const int kI = kTB * q + ir + G::R.hl; // vertical step of tile-row I
                constexpr int CO = G::C.so1 - G::C.so0, CG = G::C.sg1 - G::C.sg0; // 0 or 1 extra window
                constexpr int NO = kItemTiles + CO, NG = kItemTiles + CG;
                constexpr int SOC = imn(G::C.so0, G::C.so1), SGC = imn(G::C.sg0, G::C.sg1);
                // ring rows of the outer / guard tile boxes of both row parities
                auto rowO = [&](int so) {
                    const int k = kI + so + G::R.lo - 1;
                    return sO + 4u * (SW * static_cast<unsigned>(k % G::NBO) + static_cast<unsigned>(J0 + SOC - J_s + G::C.hl));
                };
                auto rowG = [&](int sg) {
                    const int k = kI + sg + G::R.lg - 1;
                    return sG + 4u * (SW * static_cast<unsigned>(k % G::NBG) + static_cast<unsigned>(J0 + SGC - J_s + G::C.hl));
                };
                uint32_t ho0[NO], ho1[NO], hg0[NG], hg1[NG];
                row_windows<G::C.lo, NO>(rowO(G::R.so0), ho0);
                if constexpr (G::R.so1 != G::R.so0) row_windows<G::C.lo, NO>(rowO(G::R.so1), ho1);
                row_windows<G::C.lg, NG>(rowG(G::R.sg0), hg0);
                if constexpr (G::R.sg1 != G::R.sg0) row_windows<G::C.lg, NG>(rowG(G::R.sg1), hg1);
                const unsigned cC = sC + 4u * G::SWC * static_cast<unsigned>(kI % G::NBC) +
                                    2u * static_cast<unsigned>(J0 - J_s + G::C.hl);
                const uint32_t off = L.ring_off;
                uint32_t lbs[kItemTiles][4]; // per tile, cells (a, b) = (0,0), (0,1), (1,0), (1,1)
                unsigned pass = 0;
#pragma unroll
                for (int j = 0; j < kItemTiles; ++j) {
#pragma unroll
                    for (int a = 0; a < 2; ++a) {
#pragma unroll
                        for (int b = 0; b < 2; ++b) {
                            const int io = j + (b ? G::C.so1 : G::C.so0) - SOC;
                            const int ig = j + (b ? G::C.sg1 : G::C.sg0) - SGC;
                            const uint32_t o = (a && G::R.so1 != G::R.so0) ? ho1[io] : ho0[io];
                            const uint32_t g = (a && G::R.sg1 != G::R.sg0) ? hg1[ig] : hg0[ig];
                            lbs[j][2 * a + b] = o - g - off;
                        }
                    }
                    const uint32_t lbmin = min(min(lbs[j][0], lbs[j][1]), min(lbs[j][2], lbs[j][3]));
                    unsigned short cm16;
                    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(cm16) : "r"(cC + 2u * j));
                    const float cmax = __uint_as_float(static_cast<uint32_t>(cm16) << 16); // >= the tile's max CUT
                    // tile test with the largest K_n, E_n (n_int): no cell of the tile can reach T
                    if (__fmul_ru(cmax, kin.x) >= __fmaf_rd(__uint2float_rd(lbmin), L.inv_scale, -kin.z))
                        pass |= 1u << j;
                }
                // rare: exact per-cell tests of the tiles that passed, staged by an
                // out-of-line function (keeps the unrolled item code small for the
                // instruction cache); static indices keep lbs in registers
                if (pass) {
                    uint32_t* stg = stage + (p & 1) * (3 * kStage + 1);
                    static_for<kItemTiles>([&](auto jc) {
                        constexpr int j = decltype(jc)::value;
                        if (pass & (1u << j))
                            cert_stage_tile<T>(L, map, stg, cand_sm, cand_n, 2 * I, 2 * (J0 + j), r_s, r_e, cols, lbs[j][0],
                                               lbs[j][1], lbs[j][2], lbs[j][3]);
                    });
                }
            }
        } else if (t >= kTW && t < kTW + 32 && p > 0) {
            cert_service<T>(L, map, stage + ((p - 1) & 1) * (3 * kStage + 1), cand_sm, cand_n);
        }
    }
    __syncthreads();
    if (t >= kTW && t < kTW + 32) cert_service<T>(L, map, stage + ((n_phases - 1) & 1) * (3 * kStage + 1), cand_sm, cand_n);
    __syncthreads();
    { // the CTA's candidates: one reservation in the map's list, then a coalesced copy
        const unsigned n_loc = min(cand_n[0], static_cast<unsigned>(kCandLocal));
        if (t == 0 && n_loc) cand_n[1] = atomicAdd(L.cand_count + map, n_loc);
        __syncthreads();
        const unsigned base = cand_n[1];
        for (unsigned i = t; i < n_loc; i += blockDim.x) {
            if (base + i < static_cast<unsigned>(L.cand_cap))
                L.cand[map * L.cand_cap + base + i] = cand_sm[i];
            else
                atomicOr(L.status + map, 1u);
        }
    }
    // A value outside [0, X_lim) somewhere in this CTA's input: classify every
    // such cell of my two columns (rare: input errors or the exact fallback).
    if (__syncthreads_or(!IO::in_range(mx, L)) && col_ok) {
        const int lo = max(rb_lo, 2 * K0), hi = min(rb_hi, 2 * (K0 + n_k));
        for (int rho = lo; rho < hi; ++rho) {
            const Raw2 v = IO::load2(row_ptr(rho));
            if (!IO::in_range(IO::lo(v), L)) cert_classify(L, map, rho, 2 * J_in, IO::value(IO::lo(v)));
            if (!IO::in_range(IO::hi(v), L)) cert_classify(L, map, rho, 2 * J_in + 1, IO::value(IO::hi(v)));
        }
    }
}

// Per n: {K_n, K_n 2^-(s+1), E_n} (value units), rounded away from the decision.
__global__ void cert_table_kernel(CertLaunch L, float4* ke, int n_max) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n > n_max) return;
    if (n == 0) {
        ke[0] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
    const double a = L.alpha[n];
    const double k = (static_cast<double>(n) / a) * (1.0 + 4e-6);
    const double e = static_cast<double>(n) * 0.5 * L.inv_scale_d +
                     (4.0 * n + 11.0) * 0x1p-53 * L.s_bound * (1.0 + 1e-6);
    ke[n] = make_float4(__double2float_ru(k), __double2float_ru(k * 0.5 * L.inv_scale_d), __double2float_ru(e), 0.f);
}

// Table tap (global padded (i, j)) of the candidate's table; row/col 0 are zero.
struct TapView {
    const double* tab;
    int64_t ld;
    int i0, j0; // global source row / column of the table's row / column 0
    __device__ __forceinline__ double operator()(int i, int j) const {
        const int il = i - i0, jl = j - j0;
        UWB_DCHECK(il >= 0 && jl >= 0 && kTabShift + jl < ld);
        return (il == 0 || jl == 0) ? 0.0 : tab[static_cast<int64_t>(il) * ld + kTabShift + jl];
    }
};

struct CandGeo {
    int64_t sat_job;
    int i0, j0;
    int or0, or1, oc0, oc1, gr0, gr1, gc0, gc1;
};

__device__ __forceinline__ CandGeo cand_geo(const CertLaunch& L, int64_t map, int r, int c) {
    CandGeo g;
    const int64_t s = (r - L.geo.row_lo) / L.geo.slab_rows;
    const int64_t k = L.geo.band_of(c);
    g.sat_job = (map * L.geo.n_slabs + s) * L.geo.n_bands + k;
    g.i0 = static_cast<int>(L.geo.table_begin(s));
    g.j0 = static_cast<int>(L.geo.band_c0(k));
    const int R = static_cast<int>(L.geo.rows), C = static_cast<int>(L.cols);
    g.or0 = clamp_lo32(r, L.hr);
    g.or1 = clamp_hi32(r, L.hr, R);
    g.oc0 = clamp_lo32(c, L.hc);
    g.oc1 = clamp_hi32(c, L.hc, C);
    g.gr0 = clamp_lo32(r, L.gr);
    g.gr1 = clamp_hi32(r, L.gr, R);
    g.gc0 = clamp_lo32(c, L.gc);
    g.gc1 = clamp_hi32(c, L.gc, C);
    return g;
}

__global__ void cert_mark_kernel(const __grid_constant__ CertLaunch L) {
    const int64_t map = blockIdx.x;
    if (L.status[map]) return; // flagged: the SAT writes the whole table
    const unsigned n = min(L.cand_count[map], static_cast<unsigned>(L.cand_cap));
    const int span = 32 * L.cpl;
    for (unsigned k = blockIdx.y * blockDim.x + threadIdx.x; k < n; k += gridDim.y * blockDim.x) {
        const int2 rc = L.cand[map * L.cand_cap + k];
        const CandGeo g = cand_geo(L, map, rc.x, rc.y);
        // the eight taps of sat.hpp:32-33 for the outer and the guard rectangle
        const int ti[8] = {g.or0, g.or0, g.or1 + 1, g.or1 + 1, g.gr0, g.gr0, g.gr1 + 1, g.gr1 + 1};
        const int tj[8] = {g.oc0, g.oc1 + 1, g.oc0, g.oc1 + 1, g.gc0, g.gc1 + 1, g.gc0, g.gc1 + 1};
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const int il = ti[a] - g.i0, jl = tj[a] - g.j0;
            if (il <= 0 || jl <= 0) continue; // padded row / column 0 is zero
            const int dr = il - 1, dc = jl - 1;
            const int strip = dc / span, bit = (dc % span) / L.cpl;
            UWB_DCHECK(strip >= 0 && strip < L.strips && dr >= 0 && dr < L.need_rows && g.sat_job >= 0 &&
                       g.sat_job < L.n_maps * L.geo.n_slabs * L.geo.n_bands);
            atomicOr(L.need + (g.sat_job * L.strips + strip) * L.need_rows + dr, 1u << bit);
        }
    }
}

template <typename T>
__global__ void cert_resolve_kernel(const __grid_constant__ CertLaunch L) {
    const int64_t map = blockIdx.x;
    if (L.status[map]) { // the exact path decides this map (launch_cfar_integral_filtered)
        if (blockIdx.y == 0 && threadIdx.x == 0) {
            if (L.tie_counts) L.tie_counts[map] = ~0ull;
            L.flagged[atomicAdd(L.flagged_count, 1u)] = static_cast<unsigned>(map);
        }
        return;
    }
    const unsigned n_c = min(L.cand_count[map], static_cast<unsigned>(L.cand_cap));
    const T* src = static_cast<const T*>(L.maps) + map * L.map_stride;
    for (unsigned k = blockIdx.y * blockDim.x + threadIdx.x; k < n_c; k += gridDim.y * blockDim.x) {
        const int2 rc = L.cand[map * L.cand_cap + k];
        const int r = rc.x, c = rc.y;
        const CandGeo g = cand_geo(L, map, r, c);
        TapView tv;
        tv.tab = L.table + g.sat_job * L.table_stride;
        tv.ld = L.table_ld;
        tv.i0 = g.i0;
        tv.j0 = g.j0;
        // sat.hpp:32-33 for outer and guard, cfar.cpp:115-127
        const double rs_o = dsub(dadd(tv(g.or0, g.oc0), tv(g.or1 + 1, g.oc1 + 1)),
                                 dadd(tv(g.or0, g.oc1 + 1), tv(g.or1 + 1, g.oc0)));
        const double rs_g = dsub(dadd(tv(g.gr0, g.gc0), tv(g.gr1 + 1, g.gc1 + 1)),
                                 dadd(tv(g.gr0, g.gc1 + 1), tv(g.gr1 + 1, g.gc0)));
        const int n = (g.or1 - g.or0 + 1) * (g.oc1 - g.oc0 + 1) - (g.gr1 - g.gr0 + 1) * (g.gc1 - g.gc0 + 1);
        const double sum = dsub(rs_o, rs_g);
        const double mean = ddiv(sum, static_cast<double>(n));
        const double thr = dmul(__ldg(L.alpha + n), mean);
        const double v = widen(__ldg(src + (r - L.geo.buf_row0) * L.ld + c));
        UWB_DCHECK(r >= L.geo.row_lo && r < L.geo.row_hi && c >= 0 && c < L.cols);
        if (v > thr) { // cfar.cpp:125, ties -> H0
            atomicOr(L.mask_bits + map * L.mask_map_stride + (r - L.geo.row_lo) * L.words_per_row + (c >> 5),
                     1u << (c & 31));
            const unsigned long long slot = atomicAdd(L.det_counts + map, 1ull);
            if (slot < static_cast<unsigned long long>(L.det_cap)) {
                uwb_detection d;
                d.row = static_cast<uint64_t>(r);
                d.col = static_cast<uint64_t>(c);
                d.value = v;
                d.threshold = thr;
                L.dets[map * L.det_cap + slot] = d;
            }
        }
        if (L.tie_counts && fabs(v - thr) <= 1e-6 * thr) {
            const unsigned long long slot = atomicAdd(L.tie_counts + map, 1ull);
            if (L.ties && slot < static_cast<unsigned long long>(L.tie_cap)) {
                uwb_detection d;
                d.row = static_cast<uint64_t>(r);
                d.col = static_cast<uint64_t>(c);
                d.value = v;
                d.threshold = thr;
                L.ties[map * L.tie_cap + slot] = d;
            }
        }
    }
}

// row chunks (even): every chunk re-reads its halo tile-rows; at least two CTAs per SM
void chunk_rows(CertLaunch& L) {
    const int64_t owned = L.geo.row_hi - L.geo.row_lo;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t chunk = 1024;
    while (chunk > 64 && L.col_ctas * ((owned + chunk - 1) / chunk) * L.n_maps < 2 * sms) chunk /= 2;
    L.row_chunk = chunk;
    L.row_chunks = (owned + chunk - 1) / chunk;
}

template <typename T, int HR, int GR, int HC, int GC>
cudaError_t go_cert(CertLaunch L, cudaStream_t stream) {
    using Geo = CertGeo<HR, GR, HC, GC, sizeof(T)>;
    L.col_ctas = (L.cols / 2 + kTW - 1) / kTW;
    // every tile sum carries 4 bits(M) (cells quantised as bits(x + M))
    L.ring_off = static_cast<uint32_t>(static_cast<uint64_t>(Geo::R.lo * Geo::C.lo - Geo::R.lg * Geo::C.lg) * 4u *
                                       L.bits_magic);
    chunk_rows(L);
    L.l2_ahead_t = kL2AheadT;
    if (const char* e = UWB_KNOB("UWB_CERT_L2AHEAD")) L.l2_ahead_t = atoi(e);
    auto kern = cert_kernel<T, HR, GR, HC, GC>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Geo::smem));
    if (e != cudaSuccess) return e;
    const dim3 grid(static_cast<unsigned>(L.col_ctas * L.row_chunks), static_cast<unsigned>(L.n_maps), 1);
    ++g_kernel_launches;
    kern<<<grid, Geo::NT, Geo::smem, stream>>>(L);
    return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch_cert(const CertLaunch& L, cudaStream_t stream) {
    const int key[4] = {L.hr, L.gr, L.hc, L.gc};
    auto is = [&](int a, int b, int c, int d) { return key[0] == a && key[1] == b && key[2] == c && key[3] == d; };
    if (is(10, 2, 10, 2)) return go_cert<T, 10, 2, 10, 2>(L, stream);   // configs 1, 3
    if (is(5, 1, 5, 1)) return go_cert<T, 5, 1, 5, 1>(L, stream);       // config 2
    if (is(36, 4, 36, 4)) return go_cert<T, 36, 4, 36, 4>(L, stream);   // config 4
    if (is(5, 1, 19, 3)) return go_cert<T, 5, 1, 19, 3>(L, stream);     // config 5 (1,3,4,16)
    if (is(19, 3, 5, 1)) return go_cert<T, 19, 3, 5, 1>(L, stream);     // config 5 (3,1,16,4)
    return cudaErrorNotSupported;
}

} // namespace

bool cert_supported(int hr, int gr, int hc, int gc) {
    const int k[5][4] = {{10, 2, 10, 2}, {5, 1, 5, 1}, {36, 4, 36, 4}, {5, 1, 19, 3}, {19, 3, 5, 1}};
    for (const auto& v : k)
        if (v[0] == hr && v[1] == gr && v[2] == hc && v[3] == gc) return true;
    return false;
}

// Quantisation and bound constants of a launch (host side).
void cert_prepare(CertLaunch& L, int range_log2) {
    const int64_t n_full = static_cast<int64_t>(2 * L.hr + 1) * (2 * L.hc + 1) -
                           static_cast<int64_t>(2 * L.gr + 1) * (2 * L.gc + 1);
    const int64_t n_outer = static_cast<int64_t>(2 * L.hr + 1) * (2 * L.hc + 1);
    int lg = 0;
    while ((int64_t(1) << lg) <= n_outer) ++lg; // 2^lg > n_outer
    // q < 2^(range + s) <= 2^23 (magic-number rounding) and n_outer q < 2^32
    int s = 32 - lg - range_log2;
    if (s > 23 - range_log2) s = 23 - range_log2;
    L.s_bits = s;
    L.scale = std::ldexp(1.0, s);
    L.inv_scale_d = std::ldexp(1.0, -s);
    L.inv_scale = static_cast<float>(L.inv_scale_d);
    L.magic = std::ldexp(1.0f, 23 - s);
    uint32_t mb;
    std::memcpy(&mb, &L.magic, 4);
    L.bits_magic = mb;
    const float xl = std::ldexp(1.0f, range_log2);
    std::memcpy(&L.xlim_bits, &xl, 4);
    L.xlim = static_cast<double>(xl);
    L.ring_off = static_cast<uint32_t>(static_cast<uint64_t>(n_full) * mb);
    L.s_bound = static_cast<double>(L.geo.rows) * static_cast<double>(L.geo.map_cols) * L.xlim;
}

cudaError_t launch_cert_table(const CertLaunch& L, float4* ke, int n_max, cudaStream_t stream) {
    ++g_kernel_launches;
    cert_table_kernel<<<(n_max + 1 + 255) / 256, 256, 0, stream>>>(L, ke, n_max);
    return cudaGetLastError();
}

cudaError_t launch_cert(const CertLaunch& L, int dtype, cudaStream_t stream) {
    if (L.n_maps > 65535) return cudaErrorInvalidValue;
    return dtype == UWB_F32 ? dispatch_cert<float>(L, stream) : dispatch_cert<double>(L, stream);
}

static unsigned cand_grid_y(const CertLaunch& L) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (4 * sms + L.n_maps - 1) / L.n_maps;
    return static_cast<unsigned>(want < 1 ? 1 : want > 1024 ? 1024 : want);
}

cudaError_t launch_cert_mark(const CertLaunch& L, cudaStream_t stream) {
    ++g_kernel_launches;
    cert_mark_kernel<<<dim3(static_cast<unsigned>(L.n_maps), cand_grid_y(L)), 128, 0, stream>>>(L);
    return cudaGetLastError();
}

cudaError_t launch_cert_resolve(const CertLaunch& L, int dtype, cudaStream_t stream) {
    ++g_kernel_launches;
    const dim3 grid(static_cast<unsigned>(L.n_maps), cand_grid_y(L));
    if (dtype == UWB_F32) cert_resolve_kernel<float><<<grid, 128, 0, stream>>>(L);
    else cert_resolve_kernel<double><<<grid, 128, 0, stream>>>(L);
    return cudaGetLastError();
}

} // namespace uwb
