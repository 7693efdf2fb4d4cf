// Kernel (c): exact summed-area table, replacing build_sat
// (/root/reference/proj/src/sat.cpp:10-37).
//
// The reference evaluates, row by row and left to right,
//     S(r,c) = ((x(r,c) + S(r-1,c)) + S(r,c-1)) - S(r-1,c-1)        (sat.cpp:33)
// Every S depends only on its up, left and up-left neighbours, so any schedule
// that respects those dependencies and performs the same three IEEE additions
// reproduces the reference table bit for bit. This kernel runs the recurrence
// as a systolic wavefront:
//   * the unit of work is one warp on a 32-column strip of one table; lane l
//     owns column l of the strip and handles row r = s - l at step s, so the
//     warp sweeps an anti-diagonal band down the whole strip. Warps are
//     independent (no CTA barrier);
//   * S(r, left column) comes from lane l-1 by a register shuffle of the value
//     it produced one step earlier; lane 0 takes it from the table column the
//     strip to the left has already written, 32 rows at a time (one load per
//     lane, handed over by shuffle);
//   * global traffic stays coalesced although every lane works on a different
//     row: the warp streams its 32 source columns row by row into a shared
//     ring with cp.async (one 128-byte row segment per step, 8 rows ahead), and
//     every lane delays its results through a 32-row shared ring so the
//     completed row s-31 leaves as one 256-byte segment per step;
//   * strips are claimed from an atomic counter in pair-major order: strips
//     2p and 2p+1 of a table are claimed back to back (so the two halves of
//     each 256-byte source segment are read close together and stay in L2),
//     and every table's pair p precedes any table's pair p+1. The strip a warp
//     depends on is therefore already running or finished; the dependency is a
//     release/acquire count of rows the left strip has flushed.
// The table uses the shifted layout of kernels.cuh (padded (i, j) at
// table[i*ld + kTabShift + j]), which makes every 32-column flush line-aligned.
// Non-finite inputs are reported as the smallest row-major index (sat.cpp:28-32).
#include <climits>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace uwb {

namespace {

constexpr int kStripCols = kWarp;          // 32 columns per unit of work
constexpr int kWarpsPerCta = 4;            // independent warps per CTA
constexpr int kAhead = 8;                  // source rows prefetched ahead
constexpr int kInSlots = kWarp + kAhead;   // source ring depth (rows)
constexpr int kPublishEvery = 64;

template <typename T>
struct WarpSmem {
    T xin[kInSlots][kWarp];
    double sout[kWarp][kWarp];
};

template <typename T>
__device__ __forceinline__ void cp_async_cell(unsigned dst, const T* src);
template <>
__device__ __forceinline__ void cp_async_cell<float>(unsigned dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
template <>
__device__ __forceinline__ void cp_async_cell<double>(unsigned dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
template <typename T>
__device__ __forceinline__ double lds_x(unsigned addr);
template <>
__device__ __forceinline__ double lds_x<float>(unsigned addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return static_cast<double>(v);
}
template <>
__device__ __forceinline__ double lds_x<double>(unsigned addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts_f64(unsigned addr, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ double lds_f64(unsigned addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}

// Lane 31 (which flushed the strip's last column) releases the flushed-row count.
__device__ __noinline__ void publish_rows(unsigned* prog, int flushed, int lane) {
    if (lane == kWarp - 1 && flushed > 0) st_release_u32(prog, static_cast<unsigned>(flushed));
    __syncwarp();
}

template <typename T>
__global__ void __launch_bounds__(kWarpsPerCta * kWarp)
sat_systolic_kernel(SatLaunch L) {
    extern __shared__ __align__(16) unsigned char sat_smem_raw[];
    const int warp = threadIdx.x / kWarp;
    const int lane = threadIdx.x % kWarp;
    WarpSmem<T>& sm = reinterpret_cast<WarpSmem<T>*>(sat_smem_raw)[warp];
    const unsigned xin_base = smem_u32(&sm.xin[0][lane]);
    const unsigned xin_end = xin_base + kInSlots * kWarp * sizeof(T);
    const unsigned sout_base = smem_u32(&sm.sout[0][lane]);
    const int64_t n_tiles = L.n_jobs * L.strips;
    const int cols = static_cast<int>(L.cols);

    for (;;) {
        long long tile = 0;
        if (lane == 0) tile = static_cast<long long>(atomicAdd(L.tile_counter, 1u));
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= n_tiles) return;

        // pair-major claim order: (pair, job, half)
        const int64_t pair = tile / (2 * L.n_jobs);
        const int64_t rem = tile % (2 * L.n_jobs);
        int64_t job;
        int strip;
        if (2 * pair + 1 < L.strips) {
            job = rem / 2;
            strip = static_cast<int>(2 * pair + (rem & 1));
        } else { // odd strip count: the last layer holds single strips
            job = rem;
            strip = static_cast<int>(2 * pair);
        }
        const SatJobView J = sat_job(L, job);
        const int rows = static_cast<int>(J.rows);
        const int c = strip * kStripCols + lane;
        const bool live = c < cols;
        double* table = J.table;
        const int64_t tld = L.table_ld;

        if (live) table[kTabShift + 1 + c] = 0.0; // padded row 0 is identically zero
        if (strip == 0 && lane == 0) table[kTabShift] = 0.0;

        const unsigned* prog_in = strip > 0 ? L.gprog + job * L.strips + strip - 1 : nullptr;
        unsigned* prog_out = strip + 1 < L.strips ? L.gprog + job * L.strips + strip : nullptr;
        // S(r, last column) of the strip to the left / of this strip, one double
        // per row (contiguous, so 32 rows are fetched as one 256-byte segment)
        const double* ge_in = prog_in ? L.gedge + (job * L.strips + strip - 1) * L.edge_stride : nullptr;
        double* ge_out = prog_out ? L.gedge + (job * L.strips + strip) * L.edge_stride : nullptr;
        unsigned avail = 0;
        // left values for rows [blk, blk+32) live in lane k's register (row blk + k)
        auto fetch_left = [&](int base) -> double {
            if (!prog_in || base >= rows) return 0.0; // warp-uniform
            const unsigned need = static_cast<unsigned>(min(rows, base + kWarp));
            if (avail < need) { // lane 0 acquires; the warp barrier extends the ordering to all lanes
                if (lane == 0)
                    while (avail < need) avail = ld_acquire_u32(prog_in);
                avail = __shfl_sync(0xffffffffu, avail, 0);
            }
            const int rr = base + lane;
            return rr < rows ? ge_in[rr] : 0.0;
        };
        double lcur = fetch_left(0);
        double lnext = fetch_left(kWarp);

        const int64_t ld = L.ld;
        const T* xsrc = static_cast<const T*>(J.src) + c; // row 0 of my column
        // full strips with 16-byte aligned rows stage each row segment with
        // 16-byte copies by the first 32*sizeof(T)/16 lanes
        constexpr int kVecLanes = kWarp * static_cast<int>(sizeof(T)) / 16;
        constexpr int kElemsPerVec = 16 / static_cast<int>(sizeof(T));
        const bool vec = (strip + 1) * kStripCols <= cols && (ld * sizeof(T)) % 16 == 0 &&
                         (reinterpret_cast<uintptr_t>(J.src) % 16) == 0;
        const bool vec_lane = lane < kVecLanes;
        const unsigned vdst_off = (16u - static_cast<unsigned>(sizeof(T))) * static_cast<unsigned>(lane);
        const int vsrc_off = lane * (kElemsPerVec - 1);
        auto stage = [&](unsigned dst, const T* src) { // source row segment -> ring slot
            if (vec) {
                if (vec_lane) cp_async_16(dst + vdst_off, src + vsrc_off);
            } else if (live) {
                cp_async_cell<T>(dst, src);
            }
        };
#pragma unroll
        for (int u = 0; u < kAhead; ++u) {
            if (u < rows) stage(xin_base + u * kWarp * sizeof(T), xsrc + u * ld);
            cp_async_commit();
        }
        const T* xnext = xsrc + kAhead * ld;                                // row s + kAhead
        unsigned xin_next = xin_base + kAhead * kWarp * sizeof(T);          // its ring slot
        unsigned xin_cur = xin_base + ((kInSlots - lane) % kInSlots) * kWarp * sizeof(T); // slot of row s - lane
        double* tflush = table + tld + kTabShift + 1 + c;                   // table row rf + 1, rf = s - 31
        double* zflush = table + tld + kTabShift;                           // padded column 0

        double prev = 0.0;      // S(r-1, c)
        double left_prev = 0.0; // S(r-1, c-1)
        double my_last = 0.0;   // S(r, c), shuffled right next step
        int first_bad = INT_MAX; // first row of my column holding a non-finite value
        const bool corner = strip == 0 && lane == 0;
        const int steps = rows + kWarp;

        // One systolic step. kSteady: every lane's row and the flushed row are
        // inside the table and the prefetched row exists (no range checks).
        auto step = [&](const int s, const int u, auto steady_tag) {
            constexpr bool kSteady = decltype(steady_tag)::value;
            const int r = s - lane;
            // stream in source row s + kAhead
            if (kSteady || s + kAhead < rows) stage(xin_next, xnext);
            cp_async_commit();
            xnext += ld;
            xin_next += kWarp * sizeof(T);
            if (xin_next == xin_end) xin_next = xin_base;
            cp_async_wait<kAhead>();
            __syncwarp(); // rows staged by other lanes' 16-byte copies
            const double from_left_strip = __shfl_sync(0xffffffffu, lcur, u);
            double left = __shfl_up_sync(0xffffffffu, my_last, 1);
            if (lane == 0) left = from_left_strip;
            const double v = lds_x<T>(xin_cur);
            // sat.cpp:33: out[c+1] = v + above[c+1] + out[c] - above[c]
            const double sv = dsub(dadd(dadd(v, prev), left), left_prev);
            const bool act = kSteady ? live : (live && r >= 0 && r < rows);
            if (act) {
                first_bad = (!isfinite(v) && r < first_bad) ? r : first_bad;
                prev = sv;
                left_prev = left;
                my_last = sv;
                sts_f64(sout_base + static_cast<unsigned>(r & (kWarp - 1)) * kWarp * 8u, sv);
                if (lane == kWarp - 1 && ge_out) ge_out[r] = sv;
            }
            xin_cur += kWarp * sizeof(T);
            if (xin_cur == xin_end) xin_cur = xin_base;
            // flush the completed row rf = s - 31 (own column; the warp stores one segment)
            const int rf = s - (kWarp - 1);
            if (kSteady || (rf >= 0 && rf < rows)) {
                if (live) *tflush = lds_f64(sout_base + static_cast<unsigned>(rf & (kWarp - 1)) * kWarp * 8u);
                if (corner) *zflush = 0.0;
            }
            if (kSteady || rf >= 0) {
                tflush += tld;
                zflush += tld;
            }
        };

        for (int s0 = 0; s0 < steps; s0 += kWarp) {
            if (s0 > 0) { // left-strip values for rows [s0, s0 + 32) come from the previous fetch
                lcur = lnext;
                lnext = fetch_left(s0 + kWarp);
            }
            if (s0 >= kWarp && s0 + kWarp + kAhead <= rows) {
#pragma unroll
                for (int u = 0; u < kWarp; ++u) step(s0 + u, u, std::true_type{});
            } else {
#pragma unroll 1
                for (int u = 0; u < kWarp && s0 + u < steps; ++u) step(s0 + u, u, std::false_type{});
            }
            // publish the flushed row count for the strip to the right (warp-uniform)
            const int s_end = min(s0 + kWarp, steps);
            if ((s_end & (kPublishEvery - 1)) == 0 || s_end == steps) {
                if (prog_out) publish_rows(prog_out, min(rows, s_end - (kWarp - 1)), lane);
            }
        }
        cp_async_wait<0>();
        if (first_bad != INT_MAX)
            report_min(J.nonfinite, static_cast<unsigned long long>((J.row0 + first_bad) * L.cols + c));
        __syncwarp();
    }
}

} // namespace

std::atomic<uint64_t> g_kernel_launches{0};

template <typename T>
static cudaError_t launch_sat_t(const SatLaunch& L, cudaStream_t stream) {
    const int64_t n_tiles = L.n_jobs * L.strips;
    const size_t smem = sizeof(WarpSmem<T>) * kWarpsPerCta;
    cudaError_t e = cudaFuncSetAttribute(sat_systolic_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sat_systolic_kernel<T>, kWarpsPerCta * kWarp, smem);
    const int64_t ctas = (n_tiles + kWarpsPerCta - 1) / kWarpsPerCta;
    const int64_t grid = imin(ctas, static_cast<int64_t>(sms) * (per_sm > 0 ? per_sm : 1));
    ++g_kernel_launches;
    sat_systolic_kernel<T><<<static_cast<unsigned>(grid), kWarpsPerCta * kWarp, smem, stream>>>(L);
    return cudaGetLastError();
}

cudaError_t launch_sat(const SatLaunch& L, int dtype, cudaStream_t stream) {
    if (L.n_jobs * L.strips == 0) return cudaSuccess;
    if (L.geo.rows >= (int64_t(1) << 31) - 4096 || L.cols >= (int64_t(1) << 30)) return cudaErrorInvalidValue;
    return dtype == UWB_F32 ? launch_sat_t<float>(L, stream) : launch_sat_t<double>(L, stream);
}

int64_t sat_strips(int64_t cols) { return (cols + kStripCols - 1) / kStripCols; }

} // namespace uwb
