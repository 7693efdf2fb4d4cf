// Kernel (c): exact summed-area table, replacing build_sat
// (/root/reference/proj/src/sat.cpp:10-37).
//
// The reference evaluates, row by row and left to right,
//     S(r,c) = ((x(r,c) + S(r-1,c)) + S(r,c-1)) - S(r-1,c-1)        (sat.cpp:33)
// Every S depends only on its up, left and up-left neighbours, so any schedule
// that respects those dependencies and performs the same three IEEE additions
// reproduces the reference table bit for bit. This kernel runs the recurrence
// as a systolic wavefront:
//   * the unit of work is one warp on a 128-column strip of one table; lane l
//     owns columns 4l..4l+3 and handles row r = s - l at step s, so the warp
//     sweeps an anti-diagonal band down the whole strip. Warps are
//     independent (no CTA barrier). Per step a lane evaluates its 4 cells left
//     to right (12 additions); S(r, 4l-1) comes from lane l-1 by a register
//     shuffle of the value it produced one step earlier, and lane 0 takes it
//     from the edge column of the strip to the left, fetched 32 rows at a time;
//   * lanes form 4 groups of 8. Group g stages, with 16-byte cp.async per lane,
//     the row its lanes need kAhead..kAhead+7 steps later (one 128-byte
//     segment per group and step) into lane-private slots of a 16-step ring
//     (slot = copy step mod 16), so no lane ever reads data another lane
//     copied. Results go through a lane-private 8-row delay ring; group g
//     writes back row s - 8g - 8, so each group stores two whole 128-byte lines
//     of the table per step;
//   * all ring slots used inside the 32-step unrolled block are compile-time
//     offsets or one ADD/AND away from a per-lane base;
//   * strips are claimed from an atomic counter in strip-major order, so the
//     strip a warp depends on was claimed earlier and is running or finished;
//     the dependency is a release/acquire count of rows the left strip has
//     handed over through the edge buffer.
// The table uses the shifted layout of kernels.cuh (padded (i, j) at
// table[i*ld + kTabShift + j]), which makes every group's flush line-aligned.
// Non-finite inputs are reported as the smallest row-major index (sat.cpp:28-32):
// a non-finite input makes every later S of its column non-finite, so each lane
// checks its last S once per block and, the first time it is not finite,
// rescans its own columns for the first offending row.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <type_traits>
#include <vector>
#include <cstdio>

#include "common.cuh"
#include "kernels.cuh"

namespace uwb {

namespace {

constexpr int kWarpsPerCta = 4;         // independent warps per CTA
constexpr int kAhead = 8;               // staging distance in steps (<= kXSlots - 8)
constexpr int kXSlots = 16;             // lane-private source ring (copy steps)
constexpr int kOSlots = 8;              // lane-private result delay ring (rows)
constexpr int kPublishEvery = 64;       // steps between edge hand-overs
constexpr int kL2Ahead = 0;             // sparse mode: L2 prefetch distance (rows); measured: 0 best (48: +3%, 96: +26%)
constexpr int kSatCtasPerSm = 3;        // occupancy target (registers and shared memory)
constexpr int kSatCtasPerSmSparse = 4;  // sparse mode: no result ring, <= 128 registers
constexpr int kSatCtasPerSmSparseRun = 4; // all 4 resident (3 measured faster until the first block shrank: 4.17 vs 3.84 ms at cfg 3)
#ifndef UWB_POLL_SLEEP_NS
#define UWB_POLL_SLEEP_NS 200
#endif
constexpr unsigned kPollSleepNs = UWB_POLL_SLEEP_NS; // back-off between edge polls

// Shared memory per CTA: the warps' source rings, the result rings and the
// edge staging.
template <typename T, int kCpl, bool kSparse = false>
struct SatSmem {
    static constexpr unsigned kXLane = kCpl * sizeof(T);              // source bytes per lane and row
    static constexpr unsigned kXSlotBytes = kWarp * kXLane;
    static constexpr unsigned kXRing = kXSlots * kXSlotBytes;        // 8 KB (f32) / 16 KB (f64)
    static constexpr unsigned kOLane = kCpl * sizeof(double);
    static constexpr unsigned kOSlotBytes = kWarp * kOLane;
    static constexpr unsigned kORing = kSparse ? 0u : kOSlots * kOSlotBytes; // 8 KB (none when sparse)
    static constexpr size_t bytes() {
        return 16 /* alignment slack */ + kWarpsPerCta * (kXRing + kORing + kWarp * sizeof(double));
    }
};

// cp.async of a lane's kCpl source values (16-byte pieces; 4 / 8 bytes when that is all)
template <typename T, int kCpl>
__device__ __forceinline__ void cp_async_lane(unsigned dst, const T* src) {
    constexpr unsigned kBytes = kCpl * sizeof(T);
    if constexpr (kBytes == 4) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
    } else if constexpr (kBytes == 8) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
    } else {
#pragma unroll
        for (unsigned q = 0; q < kBytes / 16; ++q)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * q),
                         "l"(reinterpret_cast<const char*>(src) + 16u * q)
                         : "memory");
    }
}
__device__ __forceinline__ void cp_async_one(unsigned dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_one(unsigned dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
template <int kCpl>
__device__ __forceinline__ void lds_lane(unsigned addr, float (&x)[kCpl]) {
    if constexpr (kCpl == 1) {
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x[0]) : "r"(addr));
    } else if constexpr (kCpl % 4 == 0) {
#pragma unroll
        for (int q = 0; q < kCpl / 4; ++q)
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(x[4 * q]), "=f"(x[4 * q + 1]), "=f"(x[4 * q + 2]), "=f"(x[4 * q + 3])
                         : "r"(addr + 16u * q));
    } else {
#pragma unroll
        for (int q = 0; q < kCpl / 2; ++q)
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x[2 * q]), "=f"(x[2 * q + 1]) : "r"(addr + 8u * q));
    }
}
template <int kCpl>
__device__ __forceinline__ void lds_lane(unsigned addr, double (&x)[kCpl]) {
    if constexpr (kCpl == 1) {
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x[0]) : "r"(addr));
    } else {
#pragma unroll
        for (int q = 0; q < kCpl / 2; ++q)
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x[2 * q]), "=d"(x[2 * q + 1]) : "r"(addr + 16u * q));
    }
}
// Result delay ring: a lane's kCpl doubles of one row are split into 16-byte
// halves stored kOHalf apart, so each 16-byte access of the warp is one
// contiguous 512-byte run (no bank conflicts; a 32-byte lane stride conflicts 2-way).
constexpr unsigned kOHalf = kWarp * 16u;

template <int kCpl>
__device__ __forceinline__ void sts_out(unsigned addr, const double (&v)[kCpl]) {
    if constexpr (kCpl == 1) {
        asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v[0]) : "memory");
    } else {
#pragma unroll
        for (int q = 0; q < kCpl / 2; ++q)
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr + kOHalf * q), "d"(v[2 * q]), "d"(v[2 * q + 1])
                         : "memory");
    }
}
template <int kCpl>
__device__ __forceinline__ void lds_out(unsigned addr, double (&v)[kCpl]) {
    if constexpr (kCpl == 1) {
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v[0]) : "r"(addr) : "memory");
    } else {
#pragma unroll
        for (int q = 0; q < kCpl / 2; ++q)
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[2 * q]), "=d"(v[2 * q + 1]) : "r"(addr + kOHalf * q)
                         : "memory");
    }
}
// Edge hand-over stores: strong (relaxed, gpu scope) so that the next strip's
// ld.relaxed.gpu polling is a race-free morally-strong pair under the PTX
// memory model; each 8-byte element is single-copy atomic.
__device__ __forceinline__ void st_edge(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ void st_edge2_if(double* p, double a, double b, bool on) {
    asm volatile(
        "{\n"
        ".reg .pred q;\n"
        "setp.ne.u32 q, %3, 0;\n"
        "@q st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};\n"
        "}\n" ::"l"(p),
        "d"(a), "d"(b), "r"(static_cast<unsigned>(on))
        : "memory");
}

__device__ __forceinline__ double lds_d(unsigned addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}

// Zero source for the virtual rows r < 0 of a strip's first block (see step()).
__device__ __align__(16) double g_sat_zero[4];

__device__ __forceinline__ double canon_edge(double v) {
    return __double_as_longlong(v) == -1LL ? __longlong_as_double(0x7ff8000000000000LL) : v;
}

// Lane 31 (which produced the strip's edge column) releases the row count.
__device__ __noinline__ void publish_rows(unsigned* prog, int rows_done, int lane) {
    if (lane == kWarp - 1 && rows_done > 0) st_release_u32(prog, static_cast<unsigned>(rows_done));
    __syncwarp();
}

// kSparse: certified-CFAR mode (see kernels.cuh SatLaunch::need): the same
// recurrence, but only the table segments marked in the tap bitmap are stored,
// straight from registers (no delay ring, no zero row / column).
template <typename T, int kCpl, bool kSparse>
__global__ void __launch_bounds__(kWarpsPerCta * kWarp, kSparse ? kSatCtasPerSmSparse : kSatCtasPerSm)
sat_systolic_kernel(SatLaunch L) {
    constexpr int kStripCols = kCpl * kWarp;
    extern __shared__ __align__(16) unsigned char sat_smem_raw[];
    using SM = SatSmem<T, kCpl, kSparse>;
    constexpr unsigned kXSlotBytes = SM::kXSlotBytes;
    constexpr unsigned kOSlotBytes = SM::kOSlotBytes;
    const int warp = threadIdx.x / kWarp;
    const int lane = threadIdx.x % kWarp;
    const int grp = lane >> 3; // lane group: stages and flushes together
    const unsigned raw = smem_u32(sat_smem_raw);
    const unsigned base = (raw + 15u) & ~15u;
    const unsigned x_lane = base + warp * SM::kXRing + lane * SM::kXLane; // slot 0, my columns
    const unsigned o_lane = base + kWarpsPerCta * SM::kXRing + warp * SM::kORing + lane * (kCpl == 1 ? 8u : 16u);
    const unsigned edge_smem = base + kWarpsPerCta * (SM::kXRing + SM::kORing) + warp * kWarp * sizeof(double);
    const int64_t n_tiles = L.n_jobs * L.strips;
    const int cols = static_cast<int>(L.cols);
    // flags bit 3: one strip warp per SM (a batch of at most one strip per SM is
    // latency-bound on its dependent chain, which co-resident warps slow down)
    if ((L.flags & 8u) && warp != 0) return;

    for (;;) {
        long long tile = 0;
        if (lane == 0) tile = static_cast<long long>(atomicAdd(L.tile_counter, 1u));
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= n_tiles) return;

        // strip-major claim order: every job's strip k precedes any job's strip k+1
        const int strip = static_cast<int>(tile / L.n_jobs);
        const int64_t job = tile % L.n_jobs;
        const SatJobView J = sat_job(L, job);
        const int rows = static_cast<int>(J.rows);
        const int c = strip * kStripCols + kCpl * lane;   // my first column
        const int nvalid = max(0, min(kCpl, cols - c));    // my columns inside the map
        double* table = J.table;
        const int64_t tld = L.table_ld;
        const int64_t ld = L.ld;
        const T* src = static_cast<const T*>(J.src);

        // sparse mode: this strip's tap bitmap (one word per row, bit = lane);
        // a flagged map stores its whole table (the exact CFAR reads it)
        const unsigned* need_col = kSparse ? L.need + (job * L.strips + strip) * L.need_rows : nullptr;
#ifdef UWB_TUNING_KNOBS
        const int l2_ahead = L.l2_ahead;
#else
        constexpr int l2_ahead = kL2Ahead; // release build: no prefetch instructions in the step at all
#endif
        const bool store_all = kSparse && L.map_full && L.map_full[job / L.jobs_per_map] != 0;
        const bool dense = !kSparse || store_all;
        // sparse mode: need words of the previous / current / next block of rows
        // (lane j: row base + j), fetched one block ahead so no step waits on them
        unsigned need_prev = 0u, need_cur = 0u, need_next = 0u;
        if (kSparse && !store_all && lane < J.rows) need_next = __ldg(need_col + lane);
        if (dense) {
            for (int k = 0; k < nvalid; ++k) table[kTabShift + 1 + c + k] = 0.0; // padded row 0 is zero
            if (strip == 0 && lane == 0) table[kTabShift] = 0.0;
        }

        const unsigned* prog_in = strip > 0 ? L.gprog + job * L.strips + strip - 1 : nullptr;
        unsigned* prog_out = strip + 1 < L.strips ? L.gprog + job * L.strips + strip : nullptr;
        // S(r, last column) of the strip to the left / of this strip, one double
        // per row (contiguous, so 32 rows are fetched as one 256-byte segment)
        const double* ge_in = prog_in ? L.gedge + (job * L.strips + strip - 1) * L.edge_stride : nullptr;
        double* ge_out = prog_out ? L.gedge + (job * L.strips + strip) * L.edge_stride : nullptr;
        unsigned avail = 0;
        // flags bit 4: the edge buffer holds a sentinel (all-ones NaN) until a
        // row's value is stored, so a lane polls its own row's value and no row
        // counter, fence or release is needed (low-latency chains)
        const bool sentinel = (L.flags & 16u) != 0;
        const bool poll_sleep = (L.flags & 128u) == 0; // flags bit 7: spin without back-off
        // left-strip edge for rows [base, base+32) (lane k: row base + k)
        auto fetch_left = [&](int base) {
            double v = 0.0;
            if (sentinel) {
                if (prog_in && base + lane < rows) {
                    const double* p = ge_in + base + lane;
                    for (;;) { // back off between polls: spinning warps would load L2
                        asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
                        if (__double_as_longlong(v) != -1LL) break;
                        if (poll_sleep) __nanosleep(kPollSleepNs);
                    }
                }
                __syncwarp(); // reconverge: lanes whose rows came early must not run ahead alone
                return v;
            }
            if (prog_in && base < rows) { // warp-uniform
                const unsigned need = static_cast<unsigned>(min(rows, base + kWarp));
                if (avail < need) { // lane 0 acquires; the warp barrier extends the ordering
                    if (lane == 0)
                        avail = wait_count_geq(prog_in, need);
                    avail = __shfl_sync(0xffffffffu, avail, 0);
                }
                if (base + lane < rows) v = ge_in[base + lane];
            }
            return v;
        };

        // staging: group g copies, at step s, source row s + kAhead - 8g
        constexpr unsigned kVecAlign = SM::kXLane >= 16 ? 16 : SM::kXLane;
        const bool vec_ok = nvalid == kCpl && (reinterpret_cast<uintptr_t>(src + c) % kVecAlign) == 0 &&
                            ((ld * sizeof(T)) % kVecAlign) == 0;
        const bool warp_fast = __all_sync(0xffffffffu, vec_ok);
        const T* xrow = src + c + static_cast<int64_t>(kAhead - 8 * grp) * ld; // row staged at step 0
        // a copy issued at step s lands in slot s mod 16
        const T* zero_src = reinterpret_cast<const T*>(g_sat_zero);
        auto stage = [&](unsigned slot_off, int row, const T* p, bool checked) {
            const unsigned dst = x_lane + slot_off;
            if (!checked) {
                cp_async_lane<T, kCpl>(dst, p);
            } else if (row >= 0 && row < rows) {
                if (warp_fast) {
                    cp_async_lane<T, kCpl>(dst, p);
                } else {
                    for (int k = 0; k < nvalid; ++k) cp_async_one(dst + k * sizeof(T), p + k);
                }
            }
        };
        // mode-2 first block: every source slot starts as zero (virtual rows of
        // lanes whose first slot is read before any copy lands in it)
        const bool first_fast = kWarp + kAhead <= rows && warp_fast && !(L.flags & 64u);
        if (first_fast) {
            for (int sl = 0; sl < kXSlots; ++sl)
                for (unsigned q = 0; q < SM::kXLane; q += 4)
                    asm volatile("st.shared.u32 [%0], 0;" ::"r"(x_lane + sl * kXSlotBytes + q) : "memory");
        }
        // prologue: virtual steps -kAhead..-1 stage rows -8g .. kAhead-1-8g
#pragma unroll
        for (int v = -kAhead; v < 0; ++v) {
            const int row = v + kAhead - 8 * grp;
            stage(static_cast<unsigned>(((v + kXSlots) & (kXSlots - 1)) * kXSlotBytes), row,
                  xrow + static_cast<int64_t>(v) * ld, true);
            cp_async_commit();
        }

        double prev[kCpl];       // S(r-1, c + k)
        double last[kCpl];       // S(r, c + k), newest; last[kCpl-1] is shuffled right
#pragma unroll
        for (int k = 0; k < kCpl; ++k) prev[k] = last[k] = 0.0;
        double left_prev = 0.0;  // S(r-1, c-1)
        bool scanned = false;    // non-finite rescan done
        // write-back pointer: table row rf + 1 for rf = s - 8g - 8 (my columns)
        double* tflush = table + static_cast<int64_t>(1 - 8 * grp - 8) * tld + kTabShift + 1 + c;
        const int steps = rows + kWarp;
        // lane l needs at step s the row copied at step s - kAhead - (l mod 8)
        const unsigned x_rbase_lane = static_cast<unsigned>(2 * kXSlots - kAhead - (lane & 7));
        const unsigned o_rbase_lane = static_cast<unsigned>(kWarp - lane); // (u - l) mod 8
        const bool edge_lane = lane == kWarp - 1 && ge_out != nullptr;
        // ge_edge = ge_out + (row of lane 31 at the current even step); advanced by the
        // fast / first blocks' paired stores (2 rows per store), resynchronised per block
        double* ge_edge = ge_out;
        T xn[kCpl];          // source values of the next step (loaded one step ahead)
        double edge_n = 0.0; // lane 0: left strip's edge for the next step

        // One systolic step. Mode 0: interior block, no checks. Mode 1: range
        // checks on rows (last block, short maps). Mode 2: the first block as
        // straight-line code: a lane whose row r = s - lane is still negative
        // computes a virtual row of zeros (its source slots read zero: the ring
        // is zeroed at the tile start and rows < 0 copy from a zero buffer; its
        // state is zero, so S stays 0), and only the table and edge stores are
        // predicated.
        auto step = [&](const int s0, const int u, auto mode_tag) {
            constexpr int kMode = decltype(mode_tag)::value;
            constexpr bool kChecked = kMode == 1, kFirst = kMode == 2;
            const int s = s0 + u;
            const int r = s - lane;
            // (1) group g writes back row s - 8g - 8 (slot u mod 8, stored >= 1 step ago)
            const int rf = s - 8 * grp - 8;
            if (!kSparse && (kFirst ? rf >= 0 : (!kChecked || (rf >= 0 && rf < rows)))) {
                UWB_DCHECK(rf >= 0 && rf < rows && tflush == table + static_cast<int64_t>(rf + 1) * tld + kTabShift + 1 + c);
                double o[kCpl];
                lds_out<kCpl>(o_lane + static_cast<unsigned>(u & (kOSlots - 1)) * kOSlotBytes, o);
                if (!kChecked || nvalid == kCpl) {
                    if constexpr (kCpl == 1) {
                        *tflush = o[0];
                    } else {
#pragma unroll
                        for (int q = 0; q < kCpl / 2; ++q)
                            reinterpret_cast<double2*>(tflush)[q] = make_double2(o[2 * q], o[2 * q + 1]);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < kCpl; ++k)
                        if (k < nvalid) tflush[k] = o[k];
                }
            }
            if constexpr (!kSparse) tflush += tld;
            // (2) stage source row s + kAhead - 8g into slot u (s0 is a multiple of 32)
            if (kFirst) {
                const int row = s + kAhead - 8 * grp;
                cp_async_lane<T, kCpl>(x_lane + static_cast<unsigned>((u & (kXSlots - 1)) * kXSlotBytes),
                                       row >= 0 ? xrow : zero_src);
            } else {
                stage(static_cast<unsigned>((u & (kXSlots - 1)) * kXSlotBytes), s + kAhead - 8 * grp, xrow, kChecked);
            }
            cp_async_commit();
            // sparse mode is read-bound: pull the row kL2Ahead steps later into L2
            // (the 16-step staging ring alone does not cover the DRAM latency)
            if (kSparse && kMode == 0 && l2_ahead > 0 && s + kAhead - 8 * grp + l2_ahead < rows) // interior steps
                asm volatile("prefetch.global.L2 [%0];" ::"l"(xrow + l2_ahead * ld));
            xrow += ld;
            // (3) this step's inputs were loaded one step ahead; load the next step's
            T x[kCpl];
#pragma unroll
            for (int k = 0; k < kCpl; ++k) x[k] = xn[k];
            const double from_left_strip = edge_n;
            cp_async_wait<kAhead - 1>();
            lds_lane<kCpl>(x_lane + ((static_cast<unsigned>(u + 1) + x_rbase_lane) & (kXSlots - 1)) * kXSlotBytes, xn);
            if (u + 1 < kWarp) edge_n = lds_d(edge_smem + static_cast<unsigned>(u + 1) * 8u);
            // (4) left neighbour S(r, c-1): lane l-1's newest S(., c+kCpl-1); lane 0: left strip's edge
            double left = __shfl_up_sync(0xffffffffu, last[kCpl - 1], 1);
            if (lane == 0) left = from_left_strip;
            // (5) sat.cpp:33 for each of my columns: out[c+1] = v + above[c+1] + out[c] - above[c]
            double sv[kCpl];
            sv[0] = dsub(dadd(dadd(widen(x[0]), prev[0]), left), left_prev);
#pragma unroll
            for (int k = 1; k < kCpl; ++k) sv[k] = dsub(dadd(dadd(widen(x[k]), prev[k]), sv[k - 1]), prev[k - 1]);
            // sparse mode: need word of row r = s0 + u - lane from the block's words
            // (lane j holds rows s0 + j and s0 - 32 + j; see the block loop),
            // shuffled while the warp is converged
            unsigned w_need = 0u;
            (void)w_need;
            if constexpr (kSparse)
                w_need = __shfl_sync(0xffffffffu, lane <= u ? need_cur : need_prev, (u - lane) & (kWarp - 1));
            const bool act = !kChecked || (r >= 0 && r < rows);
            if (act) {
                // (6) edge column for the strip to the right (two rows per 16-byte store)
                if (kChecked) {
                    if (edge_lane) {
                        // the all-ones NaN is the sentinel of flags bit 4; any NaN marks
                        // a non-finite input, which the call reports as an error
                        const double e_new = canon_edge(sv[kCpl - 1]), e_prev = canon_edge(prev[kCpl - 1]);
                        UWB_DCHECK(r >= 0 && r < L.edge_stride);
                        st_edge(ge_out + r, e_new);
                        if (u == 0 && r >= 1) st_edge(ge_out + r - 1, e_prev); // row a fast block left unstored
                    }
                } else if ((u & 1) == 0) { // r = s - 31 is odd: two rows per 16-byte store
                    // one predicated store, no branch: the whole warp used to run lane 31's
                    // branch (values are made canonical only for the sentinel hand-over)
                    double e_new = sv[kCpl - 1], e_prev = prev[kCpl - 1];
                    if (sentinel) e_new = canon_edge(e_new), e_prev = canon_edge(e_prev); // (warp-uniform)
                    UWB_DCHECK(!edge_lane || (kFirst && r < 1) || (r >= 1 && r < L.edge_stride));
                    st_edge2_if(ge_edge - 1, e_prev, e_new, edge_lane && (!kFirst || r >= 1));
                    ge_edge += 2;
                }
                left_prev = left;
#pragma unroll
                for (int k = 0; k < kCpl; ++k) prev[k] = last[k] = sv[k];
                if constexpr (!kSparse) {
                    sts_out<kCpl>(o_lane + ((static_cast<unsigned>(u) + o_rbase_lane) & (kOSlots - 1)) * kOSlotBytes, sv);
                } else if (!kFirst || r >= 0) {
                    // marked taps of row r: S(r, c..c+kCpl-1) = padded (r+1, c+1..)
                    const unsigned w = store_all ? ~0u : w_need;
                    if ((w >> lane) & 1u) {
                        UWB_DCHECK(r >= 0 && r < rows && c >= 0 && c + nvalid <= cols && kTabShift + 1 + c + nvalid <= tld);
                        double* dst = table + static_cast<int64_t>(r + 1) * tld + kTabShift + 1 + c;
                        if (kCpl >= 2 && nvalid == kCpl) {
#pragma unroll
                            for (int q = 0; q < kCpl / 2; ++q)
                                reinterpret_cast<double2*>(dst)[q] = make_double2(sv[2 * q], sv[2 * q + 1]);
                        } else {
#pragma unroll
                            for (int k = 0; k < kCpl; ++k)
                                if (k < nvalid) dst[k] = sv[k];
                        }
                    }
                }
            }
        };

        // left-strip edge values, one block ahead (lane k: row s0 + k)
        // (low-latency mode, for batches too small to fill the GPU: one block
        // ahead and hand-overs every 32 steps, which shortens the strip chain)
        const bool low_latency = (L.flags & 2u) != 0;
        // flags bit 5: fetch the next block's edge at the end of the block (shorter
        // chain lag, the fetch latency exposed once per block)
        const bool late_fetch = low_latency && (L.flags & 32u) != 0;
        double e_cur = fetch_left(0);
        double e_next = low_latency ? 0.0 : fetch_left(kWarp);
        cp_async_wait<kAhead - 1>();
        lds_lane<kCpl>(x_lane + (x_rbase_lane & (kXSlots - 1)) * kXSlotBytes, xn);
        for (int s0 = 0; s0 < steps; s0 += kWarp) {
            if constexpr (kSparse) {
                need_prev = need_cur;
                need_cur = need_next;
                const int rn = s0 + kWarp + lane;
                need_next = (!store_all && rn < rows) ? __ldg(need_col + rn) : 0u;
            }
            // left-strip edge values for rows [s0, s0 + 32) (lane 0 reads row s at step s)
            __syncwarp();
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(edge_smem + 8u * lane), "d"(e_cur) : "memory");
            __syncwarp();
            edge_n = lds_d(edge_smem);
            if (low_latency) {
                if (!late_fetch) e_cur = fetch_left(s0 + kWarp);
            } else {
                e_cur = e_next;
                e_next = fetch_left(s0 + 2 * kWarp);
            }
            // padded column 0 of the rows group 0 writes back in this block
            if (dense && strip == 0 && s0 - 8 + lane >= 0 && s0 - 8 + lane < rows)
                table[static_cast<int64_t>(s0 - 8 + lane + 1) * tld + kTabShift] = 0.0;
            const bool fast = s0 >= kWarp && s0 + kWarp + kAhead <= rows && warp_fast;
            ge_edge = ge_out + (s0 - (kWarp - 1)); // lane 31's row at step s0 (meaningful only when ge_out != nullptr)
            if (fast) {
                // unrolled by 8, not 16: half the code, the instruction cache decides
#pragma unroll 8
                for (int u = 0; u < kWarp; ++u) step(s0, u, std::integral_constant<int, 0>{});
            } else if (first_fast && s0 == 0) {
                // the first block at interior speed (it is on every later strip's
                // critical path in a chain); unrolled by 2 only: with 12 warps per SM in
                // different blocks the instruction cache decides (cfg 3 sparse SAT:
                // unroll 16 4.40 ms, 8 4.32, 4 4.24, 2 4.17, 1 4.20; the marked-tap
                // store as an out-of-line function: 4.58 ms, the call's register traffic)
#pragma unroll 2
                for (int u = 0; u < kWarp; ++u) step(s0, u, std::integral_constant<int, 2>{});
            } else {
#pragma unroll 1
                for (int u = 0; u < kWarp && s0 + u < steps; ++u) step(s0, u, std::integral_constant<int, 1>{});
            }
            // non-finite inputs poison every later S of their column (see header)
            bool finite = true;
#pragma unroll
            for (int k = 0; k < kCpl; ++k) finite &= k >= nvalid || isfinite(last[k]);
            if (!scanned && nvalid > 0 && !finite) {
                scanned = true;
                int col = c;
                const int bad = first_nonfinite<T>(src, ld, c, nvalid, min(rows, s0 + kWarp), &col);
                if (bad != INT_MAX)
                    report_min(J.nonfinite, static_cast<unsigned long long>((J.row0 + bad) * L.geo.map_cols + J.col0 + col));
            }
            if (late_fetch) e_cur = fetch_left(s0 + kWarp);
            // hand over the edge rows stored so far (warp-uniform); a fast block
            // leaves its last row for the next block's paired store
            const int s_end = min(s0 + kWarp, steps);
            const int every = low_latency ? kWarp : kPublishEvery;
            if (!sentinel && prog_out && ((s_end & (every - 1)) == 0 || s_end == steps))
                publish_rows(prog_out, min(rows, s_end - (kWarp - 1) - (fast ? 1 : 0)), lane);
        }
        cp_async_wait<0>();
        __syncwarp();
    }
}

// ---- small batches: one CTA per table, strips hand over through shared memory
//
// A batch of a few maps cannot fill the GPU, and the strip chain of the kernel
// above (one warp per strip, edges handed over through global memory 32 rows at
// a time, one warp per SM) is latency-bound. Here one CTA owns a whole table:
// warp w runs strip w of the same systolic schedule, kCtaSkew steps behind
// warp w-1 (lane l: row s - l at local step s = t - kCtaSkew w); lane 31 of warp
// w leaves S(r, last column) in a shared-memory ring and lane 0 of warp w+1
// reads it kCtaSync + 1 steps later, one __syncthreads every kCtaSync steps
// ordering the ring. Lanes own 16 bytes of source per row (4 fp32 / 2 fp64
// columns: the shortest dependent chain per step that keeps the loads whole
// lines), and global memory is touched only in whole 128-byte lines: lane group
// g (8 lanes) stages, with cp.async, the row its lanes need kCtaAhead..+7 steps
// later into lane-private slots, and writes back, from a lane-private 8-row
// delay ring, the row it finished 8..15 steps earlier. The same three additions
// per cell in the same order (sat.cpp:33): bit-identical tables.
constexpr int kCtaSync = 8;                      // steps per block (one CTA barrier each)
constexpr int kCtaSkew = kWarp + kCtaSync;       // steps between adjacent strips
constexpr int kCtaEdgeRing = 64;                 // edge ring rows (>= kCtaSkew + kCtaSync, power of 2)
constexpr int kCtaXSlots = 24;                   // lane-private source slots (copy index mod 24)
constexpr int kCtaOSlots = 16;                   // lane-private result slots (step mod 16)
constexpr int kCtaMaxWarps = 12;                 // launch bound; the shared memory caps fp64 / fp32 at 11 / 7
constexpr size_t kCtaSmemCap = 227 * 1024;
static_assert(kCtaEdgeRing >= kCtaSkew + kCtaSync && kCtaSync < kWarp, "edge ring / barrier spacing");
static_assert(kCtaSkew % kCtaSync == 0, "block alignment");

template <typename T>
__host__ __device__ constexpr int cta_cpl() { return 16 / static_cast<int>(sizeof(T)); }
template <typename T>
constexpr size_t cta_smem_per_warp() {
    return kCtaXSlots * kWarp * 16 + kCtaOSlots * kWarp * cta_cpl<T>() * sizeof(double) +
           kCtaEdgeRing * sizeof(double);
}
constexpr size_t kCtaSmemExtra = 16 + 2 * kCtaEdgeRing * sizeof(double); // alignment, zero and scratch edge rows
template <typename T>
constexpr int cta_max_warps() {
    return static_cast<int>((kCtaSmemCap - kCtaSmemExtra) / cta_smem_per_warp<T>()) < kCtaMaxWarps
               ? static_cast<int>((kCtaSmemCap - kCtaSmemExtra) / cta_smem_per_warp<T>())
               : kCtaMaxWarps;
}

// Per block of kCtaSync steps a warp (i) issues, per lane group g, the cp.async
// copies of the 8 rows it needs in the next block (copy index q: group g copies
// row q - 8g into slot q mod 24; lane j of the group reads index s - j at step
// s; indices s0 - 7 .. s0 + 15 are live during a block), (ii) runs 8 systolic steps whose only shared-memory traffic is plain
// loads / stores of lane-private slots, so the compiler is free to overlap
// consecutive steps (no asm memory clobber inside), and (iii) writes back the 8
// rows its groups finished (group g: rows s0 - 8g - 7 .. s0 - 8g), 128-byte
// lines per group.
template <typename T>
__global__ void __launch_bounds__(kCtaMaxWarps * kWarp, 1) sat_cta_kernel(SatLaunch L) {
    constexpr int kC = cta_cpl<T>();
    extern __shared__ __align__(16) unsigned char cta_smem_raw[];
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const int grp = lane >> 3, j = lane & 7;
    const int n_warps = blockDim.x / kWarp; // == strips of this table
    unsigned char* sm = cta_smem_raw + ((16u - (smem_u32(cta_smem_raw) & 15u)) & 15u);
    // x ring [warp][slot][lane] of 16 bytes; o ring [warp][slot][lane] of kC doubles; edge ring [warp][row]
    T* xr = reinterpret_cast<T*>(sm) + (static_cast<size_t>(warp) * kCtaXSlots * kWarp + lane) * kC;
    double* orr = reinterpret_cast<double*>(sm + static_cast<size_t>(n_warps) * kCtaXSlots * kWarp * 16) +
                  (static_cast<size_t>(warp) * kCtaOSlots * kWarp + lane) * kC;
    double* edge = reinterpret_cast<double*>(sm + static_cast<size_t>(n_warps) *
                                                      (kCtaXSlots * kWarp * 16 + kCtaOSlots * kWarp * kC * 8));
    constexpr int kXStride = kWarp * kC; // elements between x slots of a lane
    constexpr int kOStride = kWarp * kC; // doubles between o slots of a lane
    const SatJobView J = sat_job(L, blockIdx.x);
    const int rows = static_cast<int>(J.rows);
    const int cols = static_cast<int>(L.cols);
    const int c = (warp * kWarp + lane) * kC;
    const int nvalid = max(0, min(kC, cols - c));
    const T* src = static_cast<const T*>(J.src) + c;
    const int64_t ld = L.ld, tld = L.table_ld;
    double* table = J.table;
    for (int k = 0; k < nvalid; ++k) table[kTabShift + 1 + c + k] = 0.0; // padded row 0
    if (warp == 0 && lane == 0) table[kTabShift] = 0.0;
    const bool vec = nvalid == kC && L.vec_ok;
    // edge rings: row r of strip w at edge[w][r mod 64]; strip 0 reads the zero
    // row (slot n_warps), the last strip writes a scratch row (slot n_warps + 1)
    double* zero_row = edge + n_warps * kCtaEdgeRing;
    const double* edge_in = warp > 0 ? edge + (warp - 1) * kCtaEdgeRing : zero_row;
    double* edge_out = warp + 1 < n_warps ? edge + warp * kCtaEdgeRing : zero_row + kCtaEdgeRing;
    for (int i = threadIdx.x; i < kCtaEdgeRing; i += blockDim.x) zero_row[i] = 0.0;
    __syncthreads();
    const unsigned x_smem = smem_u32(xr);
    auto mod_x = [](int q) { // q mod kCtaXSlots for q >= -kCtaXSlots
        const int m = q % kCtaXSlots;
        return m < 0 ? m + kCtaXSlots : m;
    };
    // copies of indices [q0, q0 + 8) by my group: row q - 8g, slot q mod 24
    // (checked: rows outside the map are skipped; a lane with fewer than kC
    // columns inside the map copies element by element)
    auto stage8 = [&](int q0, auto checked_tag) {
        constexpr bool kChecked = decltype(checked_tag)::value;
        const int slot0 = mod_x(q0);
        const int r0 = q0 - 8 * grp;
        const T* p = src + static_cast<int64_t>(r0) * ld;
        unsigned dst = x_smem + static_cast<unsigned>(slot0) * kXStride * sizeof(T);
        constexpr unsigned kSlotBytes = kXStride * sizeof(T);
#pragma unroll
        for (int u = 0; u < kCtaSync; ++u) {
            const bool row_ok = !kChecked || (r0 + u >= 0 && r0 + u < rows);
            if (row_ok && vec) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(p) : "memory");
            } else if (row_ok) {
                for (int k = 0; k < nvalid; ++k) cp_async_one(dst + k * sizeof(T), p + k);
            }
            p += ld;
            dst = slot0 + u + 1 == kCtaXSlots ? dst + kSlotBytes - kCtaXSlots * kSlotBytes : dst + kSlotBytes;
        }
        cp_async_commit();
    };
    double prev[kC];
#pragma unroll
    for (int k = 0; k < kC; ++k) prev[k] = 0.0;
    double left_prev = 0.0;
    // local steps from -8 (the first copies: index 0 = group 0's row 0) to the
    // last write-back (row rows - 1 of group 3 after step rows - 1 + 31)
    const int s_first = -kCtaSync;
    const int s_end = rows + kWarp + kCtaSync;
    const int skew = kCtaSkew * warp;
    const int n_blocks = (s_end - s_first + kCtaSkew * (n_warps - 1) + kCtaSync - 1) / kCtaSync;

    // 8 systolic steps: branch-free (state updates by select, stores by
    // predicate), so the compiler overlaps a step's loads and x + S(r-1, .) adds
    // with the previous step's dependent chain
    auto steps8 = [&](const int s0, auto checked_tag) {
        constexpr bool kChecked = decltype(checked_tag)::value;
        const int xbase = mod_x(s0 - j); // slot of step s0
#pragma unroll
        for (int u = 0; u < kCtaSync; ++u) {
            const int s = s0 + u;
            const int r = s - lane;
            const bool act = !kChecked || (r >= 0 && r < rows);
            const int xslot = xbase + u < kCtaXSlots ? xbase + u : xbase + u - kCtaXSlots;
            UWB_DCHECK(xslot >= 0 && xslot < kCtaXSlots);
            const T* xs = xr + xslot * kXStride;
            double a[kC]; // x + S(r-1, .): independent of the left neighbour
#pragma unroll
            for (int k = 0; k < kC; ++k) a[k] = dadd(widen(xs[k]), prev[k]);
            double left = __shfl_up_sync(0xffffffffu, prev[kC - 1], 1);
            const double e = edge_in[s & (kCtaEdgeRing - 1)]; // lane 0's row is s (broadcast load)
            if (lane == 0) left = e;
            if (kChecked && !act) left = 0.0;
            double sv[kC];
            sv[0] = dsub(dadd(a[0], left), left_prev);
#pragma unroll
            for (int k = 1; k < kC; ++k) sv[k] = dsub(dadd(a[k], sv[k - 1]), prev[k - 1]);
            double* o = orr + (s & (kCtaOSlots - 1)) * kOStride;
            if (act) {
#pragma unroll
                for (int k = 0; k < kC; ++k) o[k] = sv[k];
            }
            if (lane == kWarp - 1 && act) edge_out[r & (kCtaEdgeRing - 1)] = sv[kC - 1];
            left_prev = act ? left : left_prev;
#pragma unroll
            for (int k = 0; k < kC; ++k) prev[k] = act ? sv[k] : prev[k];
        }
    };
    // write back the rows my group finished: s0 - 8g - 7 .. s0 - 8g (row r of lane
    // 8g + j sits in slot (r + 8g + j) mod 16)
    auto flush8 = [&](const int s0, auto checked_tag) {
        constexpr bool kChecked = decltype(checked_tag)::value;
        const int rf0 = s0 - 8 * grp - 7;
        double* dst = table + static_cast<int64_t>(rf0 + 1) * tld + kTabShift + 1 + c;
#pragma unroll
        for (int u = 0; u < kCtaSync; ++u) {
            const int rf = rf0 + u;
            if (!kChecked || (rf >= 0 && rf < rows)) {
                UWB_DCHECK(rf >= 0 && rf < rows && dst == table + static_cast<int64_t>(rf + 1) * tld + kTabShift + 1 + c);
                const double* o = orr + ((rf + lane) & (kCtaOSlots - 1)) * kOStride;
                if (nvalid == kC) {
#pragma unroll
                    for (int q = 0; q < kC / 2; ++q)
                        reinterpret_cast<double2*>(dst)[q] = reinterpret_cast<const double2*>(o)[q];
                } else {
                    for (int k = 0; k < nvalid; ++k) dst[k] = o[k];
                }
                if (warp == 0 && lane == 0) dst[-1] = 0.0; // padded column 0
            }
            dst += tld;
        }
    };
#pragma unroll 1
    for (int b = 0; b < n_blocks; ++b) {
        const int s0 = s_first + b * kCtaSync - skew; // my first local step in this block
        if (s0 + kCtaSync > s_first && s0 < s_end) {
            // staged rows s0 + 8 - 24 .. s0 + 15, computed rows s0 - 31 .. s0 + 7,
            // written-back rows s0 - 31 .. s0 all inside [0, rows)
            const bool interior = s0 >= kWarp && s0 + 2 * kCtaSync <= rows;
            if (interior) stage8(s0 + kCtaSync, std::integral_constant<bool, false>{}); // used in the next block
            else stage8(s0 + kCtaSync, std::integral_constant<bool, true>{});
            cp_async_wait<1>(); // this block's copies may still fly
            __syncwarp();
            if (interior) steps8(s0, std::integral_constant<bool, false>{});
            else steps8(s0, std::integral_constant<bool, true>{});
            __syncwarp();
            if (interior) flush8(s0, std::integral_constant<bool, false>{});
            else flush8(s0, std::integral_constant<bool, true>{});
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    // non-finite inputs poison every later S of their column (see the header)
    bool finite = true;
#pragma unroll
    for (int k = 0; k < kC; ++k) finite &= k >= nvalid || isfinite(prev[k]);
    if (!finite && J.nonfinite) {
        int col = c;
        const int bad = first_nonfinite<T>(static_cast<const T*>(J.src), ld, c, nvalid, rows, &col);
        if (bad != INT_MAX)
            report_min(J.nonfinite, static_cast<unsigned long long>((J.row0 + bad) * L.geo.map_cols + J.col0 + col));
    }
}

} // namespace
bool sat_cta_eligible(int64_t n_jobs, int64_t cols, int dtype);
namespace {

// One CTA per table when the batch is too small to fill the GPU and every
// table's strips fit one CTA (dense tables only).
template <typename T>
static bool launch_sat_cta(const SatLaunch& L, cudaStream_t stream, cudaError_t* err) {
    if (L.need || !sat_cta_eligible(L.n_jobs, L.cols, sizeof(T) == 4 ? UWB_F32 : UWB_F64)) return false;
    const int warps = static_cast<int>((L.cols + kWarp * cta_cpl<T>() - 1) / (kWarp * cta_cpl<T>()));
    const size_t smem = kCtaSmemExtra + static_cast<size_t>(warps) * cta_smem_per_warp<T>();
    *err = cudaFuncSetAttribute(sat_cta_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (*err != cudaSuccess) return true;
    ++g_kernel_launches;
    sat_cta_kernel<T><<<static_cast<unsigned>(L.n_jobs), warps * kWarp, smem, stream>>>(L);
    *err = cudaGetLastError();
    return true;
}

template <typename T, int kCpl, bool kSparse>
static cudaError_t launch_sat_t(const SatLaunch& L, cudaStream_t stream) {
    const int64_t n_tiles = L.n_jobs * L.strips;
    const size_t smem = SatSmem<T, kCpl, kSparse>::bytes();
    auto kern = sat_systolic_kernel<T, kCpl, kSparse>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarpsPerCta * kWarp, smem);
    // leave room for a concurrent CFAR on another stream (UWB_SAT_CTAS_PER_SM)
    if (kSparse) per_sm = std::min(per_sm, kSatCtasPerSmSparseRun);
    SatLaunch Lp = L;
    Lp.l2_ahead = kL2Ahead;
    if (const char* e = UWB_KNOB("UWB_SAT_L2AHEAD")) Lp.l2_ahead = atoi(e);
    if (const char* e = UWB_KNOB("UWB_SAT_CTAS_PER_SM")) per_sm = std::min(per_sm, std::max(1, atoi(e)));
    const int64_t ctas = (n_tiles + kWarpsPerCta - 1) / kWarpsPerCta;
    int64_t grid = imin(ctas, static_cast<int64_t>(sms) * (per_sm > 0 ? per_sm : 1));
    SatLaunch L2 = Lp;
    // batches that cannot fill the resident warps are latency-bound on the strip chain
    if (n_tiles < 2LL * sms * (per_sm > 0 ? per_sm : 1) * kWarpsPerCta) L2.flags |= 2u;
    // at most one strip per SM: each strip gets an SM to itself
    if (n_tiles <= sms) L2.flags |= 8u;
    if (const char* f = UWB_KNOB("UWB_SAT_FLAGS")) L2.flags = static_cast<unsigned>(atoi(f));
    // low-latency chains hand edges over through sentinel-initialised values
    // (and, one strip per SM, fetch each block's left edge at the end of the
    // previous block: 32 steps less lag per strip, measured 6% faster on 128 strips)
    if ((L2.flags & 2u) && L.strips > 1 && !UWB_KNOB("UWB_SAT_FLAGS")) L2.flags |= (L2.flags & 8u) ? 48u : 16u;
    if (L2.flags & 8u) grid = imin(n_tiles, sms);
    if ((L2.flags & 16u) && L.strips > 1) {
        const cudaError_t me = cudaMemsetAsync(L.gedge, 0xff, sizeof(double) * L.n_jobs * L.strips * L.edge_stride, stream);
        if (me != cudaSuccess) return me;
    }
    ++g_kernel_launches;
    kern<<<static_cast<unsigned>(grid), kWarpsPerCta * kWarp, smem, stream>>>(L2);
    return cudaGetLastError();
}

template <typename T>
static cudaError_t launch_sat_cpl(const SatLaunch& L, cudaStream_t stream) {
    cudaError_t e = cudaSuccess;
    constexpr int kDtype = sizeof(T) == 4 ? UWB_F32 : UWB_F64;
    if (!(L.flags & 256u) && sat_cluster_eligible(L, kDtype)) return launch_sat_cluster(L, kDtype, stream);
    if (launch_sat_cta<T>(L, stream, &e)) return e;
    if (L.need) {
        switch (L.cpl) {
            case 1: return launch_sat_t<T, 1, true>(L, stream);
            case 2: return launch_sat_t<T, 2, true>(L, stream);
            default: return launch_sat_t<T, 4, true>(L, stream);
        }
    }
    switch (L.cpl) {
        case 1: return launch_sat_t<T, 1, false>(L, stream);
        case 2: return launch_sat_t<T, 2, false>(L, stream);
        default: return launch_sat_t<T, 4, false>(L, stream);
    }
}

} // namespace

std::atomic<uint64_t> g_kernel_launches{0};

cudaError_t launch_sat(const SatLaunch& L, int dtype, cudaStream_t stream) {
    if (L.n_jobs * L.strips == 0) return cudaSuccess;
    if (L.geo.rows >= (int64_t(1) << 31) - 4096 || L.cols >= (int64_t(1) << 30)) return cudaErrorInvalidValue;
    if (L.strips != sat_strips(L.cols, L.cpl)) return cudaErrorInvalidValue;
    return dtype == UWB_F32 ? launch_sat_cpl<float>(L, stream) : launch_sat_cpl<double>(L, stream);
}

// Columns per lane. 4 (128-column strips) is best measured for every batch
// shape: for large batches it needs the fewest per-cell operations, and for a
// single map the strip chain (strips x hand-over lag + rows) is shortest with
// the fewest strips; 32- and 64-column strips (UWB_SAT_CPL=1/2) stay available.
int sat_cpl_for(int64_t n_jobs, int64_t cols) {
    (void)n_jobs;
    (void)cols;
    if (const char* e = UWB_KNOB("UWB_SAT_CPL")) {
        const int c = atoi(e);
        if (c == 1 || c == 2 || c == 4) return c;
    }
    return 4;
}

bool sat_cta_eligible(int64_t n_jobs, int64_t cols, int dtype) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t strip_cols = kWarp * (dtype == UWB_F32 ? cta_cpl<float>() : cta_cpl<double>());
    const int max_warps = dtype == UWB_F32 ? cta_max_warps<float>() : cta_max_warps<double>();
    return n_jobs >= 1 && n_jobs <= sms && (cols + strip_cols - 1) / strip_cols <= max_warps;
}

int64_t sat_strips(int64_t cols, int cpl) { return (cols + kWarp * cpl - 1) / (kWarp * cpl); }

} // namespace uwb
