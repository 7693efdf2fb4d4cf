// Kernel (c), latency path: exact summed-area table of a few small maps, one
// thread-block cluster per table (replacing build_sat,
// /root/reference/proj/src/sat.cpp:10-37, for single-map calls: the paper's
// Table I shape and BASELINE config 1).
//
// A single table is bound by the dependent chain of the recurrence
//     S(r,c) = ((x(r,c) + S(r-1,c)) + S(r,c-1)) - S(r-1,c-1)        (sat.cpp:33)
// not by bandwidth: the wavefront needs rows + columns dependent steps whatever
// the machine. This kernel keeps each step as close to that chain as it can:
//   * a strip of 32 lanes x 16 source bytes (64 fp64 / 128 fp32 columns) is
//     swept by ONE compute warp that has a scheduler of its own: lane l owns
//     its 2 / 4 columns and handles row s - l at step s (the systolic schedule
//     of sat.cu); per step a lane issues one 16-byte shared load of x, the
//     x + S(r-1, .) additions (off the chain), one 64-bit shuffle and the
//     2 x columns dependent additions of sat.cpp:33 in the reference's
//     association, and stores its S values straight from registers (the table
//     of a small map lives in L2, so 16-byte scattered stores cost nothing
//     and no write-back ring, barrier or second pass sits on the chain).
//     Steps run in straight-line blocks of 32 (a block end costs ~190 cycles
//     of branches and barrier tests: measured 62 -> 43 ns per step against
//     8-step blocks; scripts/micro/chain.cu has the bare chain at 22 ns);
//   * the strips of a table are the CTAs of one thread-block cluster (up to 8
//     CTAs x up to 3 strips). Lane 31 of strip w stores S(r, last column)
//     into the shared memory of the CTA that runs strip w + 1 (a relaxed
//     remote store through DSMEM); that strip reads the 8 values of its next
//     group of steps one group ahead with broadcast shared loads (every lane
//     the same 64 bytes: no shuffle, no divergence) and polls them when the
//     group starts if they had not arrived. Every 8-byte value is its own
//     flag: the edge column starts as a signalling-NaN sentinel (no IEEE
//     addition returns one, so no S - not even one poisoned by a NaN input -
//     can look like "not yet written"), and a whole column of `rows` values
//     is kept, so there is no ring to recycle, no counter, no fence and no
//     back-pressure: the chain is self-timed, strip w + 1 runs 32 + 8 steps
//     plus the hand-over latency behind strip w (measured ~75 steps);
//   * a table wider than 24 strips is a CHAIN of clusters (config 4's global
//     table: 128 strips, one per SM): the last strip
//     of a cluster stores its edge column into a global boundary column, and
//     a relay warp of the next cluster's first CTA polls that column and
//     copies arrived values into the strip's shared edge column, so the
//     compute warps are the same in both cases. Clusters are dispatched in
//     block-index order, so a cluster never waits on one that has not started;
//     the cluster size (8, 4, 2, 1) is the largest for which
//     cudaOccupancyMaxActiveClusters keeps the whole chain resident (config 4
//     with 8-CTA clusters whatever the occupancy: 2.55 ms, the last clusters
//     waiting for SMs; with the resident size: 1.93 ms);
//   * a helper warp per strip feeds the source ring with the TMA engine's 1-D
//     bulk copies (one 512-byte row segment per lane, 32 rows per mbarrier
//     phase, a 128-row ring), so the compute warp never computes a global
//     address for its inputs.
// The same three additions per cell in the same order: bit-identical tables.
#include <climits>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace uwb {

namespace {

#ifndef UWB_CL_PROBE
#define UWB_CL_PROBE 0 // timing probes (scripts/cl_probe.sh): 1 no table stores, 2 no hand-over shuffle, 4 no source waits
#endif
#ifndef UWB_CL_BLOCK
#define UWB_CL_BLOCK 32
#endif
constexpr int kClBlock = UWB_CL_BLOCK;             // steps per block = rows per staged chunk
constexpr int kClRingRows = 128;                   // source ring rows per strip
constexpr int kClChunks = kClRingRows / kClBlock;  // chunks of the ring
constexpr int kClGroup = 8;                        // hand-over values polled per group of steps
constexpr int kClBack = (kWarp - 1 + kClBlock - 1) / kClBlock; // chunks behind the newest that are still read
constexpr int kClRowBytes = kWarp * 16;            // 512 bytes of source per strip row
constexpr unsigned kClRingBytes = kClRingRows * kClRowBytes; // 64 KB per strip
constexpr int kClMaxSpc = 3;                       // strips per CTA
constexpr int kClMaxCtas = 8;                      // portable cluster size
constexpr size_t kClSmemCap = 227 * 1024;
constexpr unsigned kClBarBytes = 2 * kClChunks * sizeof(uint64_t);
constexpr unsigned kClZeroBytes = 128;             // strip 0's "hand-over values"

__device__ __forceinline__ unsigned cluster_ctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Hand-over pair: a relaxed cluster-scope store into the neighbour's shared
// memory against relaxed cluster-scope polls (morally strong, single-copy
// atomic per 8-byte value). The store is predicated, not branched: only lane
// 31 of a strip with a right neighbour stores.
#ifndef UWB_CL_SLACK
#define UWB_CL_SLACK 0 // rows of slack a strip starts with behind its left neighbour (beyond the first group)
#endif
#ifndef UWB_CL_HANDOVER
#define UWB_CL_HANDOVER 0 // 0: st.relaxed.cluster, 1: atom.exch (result unused)
#endif
__device__ __forceinline__ void st_edge_dsmem(unsigned addr, double v, unsigned on) {
#if UWB_CL_HANDOVER == 1
    // An exchange, not a store: a plain remote store may sit in the sender's write path
    // for ~2 us before the neighbour sees it (measured: a strip that had caught up with
    // its left neighbour advanced 8 rows per ~2.3 us); an atomic is performed at the
    // destination at once (~180 ns one way, scripts/micro/dsmem_pingpong.cu).
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        ".reg .b64 old;\n"
        "setp.ne.u32 p, %2, 0;\n"
        "@p atom.relaxed.cluster.shared::cluster.exch.b64 old, [%0], %1;\n"
        "}\n" ::"r"(addr),
        "l"(__double_as_longlong(v)), "r"(on));
#else
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.u32 p, %2, 0;\n"
        "@p st.relaxed.cluster.shared::cluster.f64 [%0], %1;\n"
        "}\n" ::"r"(addr),
        "d"(v), "r"(on)); // no memory clobber: ordered against the other volatile asm only
#endif
}
// ... and into the boundary column of a chain (global memory, polled by the next cluster's relay warp)
__device__ __forceinline__ void st_edge_global(unsigned long long addr, double v, unsigned on) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.u32 p, %2, 0;\n"
        "@p st.relaxed.gpu.global.f64 [%0], %1;\n"
        "}\n" ::"l"(addr),
        "d"(v), "r"(on));
}
// shared-window address of `local_s` (an address in my shared memory) in CTA `rank` of the cluster
__device__ __forceinline__ unsigned map_to_cta_s(unsigned local_s, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_s), "r"(rank));
    return r;
}
// two consecutive rows per load; every 8-byte element is its own single-copy atomic access
__device__ __forceinline__ void ld_edge_poll2(unsigned addr, double& a, double& b) {
    // volatile = relaxed at system scope (PTX memory model), and on my own shared memory it is a
    // plain LDS (~30 cycles); ld.relaxed.cluster.shared::cluster compiles to a generic strong load
    // whose round trip (~1 us) was added to every strip's lag
    asm volatile("ld.volatile.shared::cta.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(addr) : "memory");
}
// "Not yet written": a signalling NaN. Every S is the result of an IEEE
// addition, and an addition never returns a signalling NaN (a NaN result is
// quiet whatever the inputs), so no table value can equal the sentinel.
constexpr long long kClSentinel = 0x7ff0000000000001LL;
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename T>
struct XVec;
template <>
struct XVec<double> {
    using type = double2;
    static __device__ __forceinline__ void get(const double2& v, double (&x)[2]) {
        x[0] = v.x;
        x[1] = v.y;
    }
    static __device__ __forceinline__ double2 lds(unsigned addr) {
        double2 v;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
        return v;
    }
};
template <>
struct XVec<float> {
    using type = float4;
    static __device__ __forceinline__ void get(const float4& v, float (&x)[4]) {
        x[0] = v.x;
        x[1] = v.y;
        x[2] = v.z;
        x[3] = v.w;
    }
    static __device__ __forceinline__ float4 lds(unsigned addr) {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
        return v;
    }
};

template <typename T>
__global__ void __launch_bounds__((kClMaxSpc * 2 + 1) * kWarp, 1)
sat_cluster_kernel(SatLaunch L, int spc, int csize, int chain, unsigned edge_bytes) {
    constexpr int kC = 16 / static_cast<int>(sizeof(T));
    constexpr int kStripCols = kWarp * kC;
    extern __shared__ __align__(128) unsigned char cl_smem[];
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const unsigned rank = cluster_ctarank();
    // a table wider than one cluster's strips is a chain of `chain` clusters (cluster q
    // of a job owns strips [q, q + 1) * csize * spc); clusters are dispatched in
    // block-index order, so the cluster a strip waits on started earlier
    const int cl = static_cast<int>(blockIdx.x) / csize;
    const int q_cl = cl % chain;
    const int64_t job = cl / chain;
    const bool relay = warp == 2 * spc;                 // one extra warp: the global hand-over's relay
    const bool helper = warp >= spc && !relay;
    const int j = relay ? 0 : (helper ? warp - spc : warp); // my strip inside the CTA
    const int g = (q_cl * csize + static_cast<int>(rank)) * spc + j; // my strip of the table
    const int cols = static_cast<int>(L.cols);
    const int strips = (cols + kStripCols - 1) / kStripCols;
    const bool live = g < strips;
    const SatJobView J = sat_job(L, job);
    const int rows = static_cast<int>(J.rows);
    const int64_t ld = L.ld, tld = L.table_ld;
    double* table = J.table;

    unsigned char* ring = cl_smem + static_cast<size_t>(j) * kClRingBytes;
    unsigned char* edges = cl_smem + static_cast<size_t>(spc) * kClRingBytes;
    double* edge_in = reinterpret_cast<double*>(edges + static_cast<size_t>(j) * edge_bytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(edges + static_cast<size_t>(spc) * edge_bytes +
                                                 static_cast<size_t>(j) * kClBarBytes);
    uint64_t* empty = full + kClChunks;
    unsigned char* zeros = edges + static_cast<size_t>(spc) * (edge_bytes + kClBarBytes); // kClZeroBytes
    const unsigned zero_s = smem_u32(zeros);

    // every edge value starts as the sentinel; barriers: one arrival per phase
    for (unsigned i = threadIdx.x; i < static_cast<unsigned>(spc) * edge_bytes / 8; i += blockDim.x)
        reinterpret_cast<long long*>(edges)[i] = kClSentinel;
    if (threadIdx.x < kClZeroBytes / 8) reinterpret_cast<long long*>(zeros)[threadIdx.x] = 0;
    if (!helper && lane == 0) {
        for (int i = 0; i < kClChunks; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_fence_init();
    }
    __syncthreads();
    cluster_sync_all(); // nobody stores into a neighbour before its sentinels are in place

    const int n_chunks = (rows + kClBlock - 1) / kClBlock;
    if (relay) {
        // The first strip of a chained cluster takes its left edge from the previous
        // cluster through global memory: this warp polls that column (lane l: rows
        // l, l + 32, ...; the same sentinel, written by fill_sentinel_kernel) and stores
        // every value that has arrived into the strip's shared edge column, so the
        // compute warp polls shared memory like every other strip.
        if (rank == 0 && q_cl > 0 && live) {
            const double* ge = L.gedge + (job * L.strips + (q_cl - 1)) * L.edge_stride;
            const unsigned dst = smem_u32(edge_in);
            for (int r = lane; r < rows; r += kWarp) {
                UWB_DCHECK(r < L.edge_stride && static_cast<unsigned>(r) * 8u < edge_bytes && q_cl - 1 < L.strips);
                double v;
                for (;;) {
                    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(ge + r) : "memory");
                    if (__double_as_longlong(v) != kClSentinel) break;
                    __nanosleep(64);
                }
                asm volatile("st.relaxed.cluster.shared::cta.f64 [%0], %1;" ::"r"(dst + 8u * static_cast<unsigned>(r)), "d"(v)
                             : "memory");
            }
        }
    } else if (helper) {
        if (live) {
            const int c0 = g * kStripCols;
            const unsigned row_bytes =
                static_cast<unsigned>(min(kStripCols, cols - c0)) * static_cast<unsigned>(sizeof(T));
            const T* src = static_cast<const T*>(J.src) + c0;
            const bool bulk_ok = L.vec_ok && (static_cast<int64_t>(cols) * sizeof(T)) % 16 == 0;
            for (int q = 0; q < n_chunks; ++q) {
                const int slot = q & (kClChunks - 1);
                // sleeping between tries: a spinning try_wait loop shares the SM's shared-memory
                // pipeline with the compute warp's shuffles and loads and stretches every step
                if (q >= kClChunks) {
                    const unsigned par = static_cast<unsigned>(((q / kClChunks) - 1) & 1);
                    while (!mbar_test(&empty[slot], par)) __nanosleep(256);
                }
                const int nr = min(kClBlock, rows - kClBlock * q);
                if (bulk_ok) {
                    if (lane == 0) mbar_expect_tx(&full[slot], static_cast<unsigned>(nr) * row_bytes);
                    __syncwarp();
                    const int r = kClBlock * q + lane;
                    if (lane < nr)
                        bulk_g2s(ring + static_cast<size_t>(r & (kClRingRows - 1)) * kClRowBytes,
                                 src + static_cast<int64_t>(r) * ld, row_bytes, &full[slot]);
                } else {
                    // rows that are not 16-byte aligned or whole 16-byte pieces (the reference
                    // pipeline's band maps: 7 fp64 columns): the warp copies them element by
                    // element, zero-fills the rest of the strip row, and releases the phase
                    // (16 rows of loads in flight per lane: two memory round trips per chunk)
                    const int nc = min(kStripCols, cols - c0);
                    constexpr int kSub = 16;
                    for (int i0 = 0; i0 < nr; i0 += kSub) {
                        T v[kSub][kC];
#pragma unroll
                        for (int i = 0; i < kSub; ++i) {
                            const T* sr = src + static_cast<int64_t>(kClBlock * q + i0 + i) * ld;
#pragma unroll
                            for (int k = 0; k < kC; ++k) {
                                const int e = lane + kWarp * k;
                                v[i][k] = (i0 + i < nr && e < nc) ? sr[e] : T(0);
                            }
                        }
#pragma unroll
                        for (int i = 0; i < kSub; ++i) {
                            const int r = kClBlock * q + i0 + i;
                            T* dst = reinterpret_cast<T*>(ring + static_cast<size_t>(r & (kClRingRows - 1)) * kClRowBytes);
#pragma unroll
                            for (int k = 0; k < kC; ++k)
                                if (i0 + i < nr) dst[lane + kWarp * k] = v[i][k];
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&full[slot]); // (release: the copies above are visible to the waiter)
                }
            }
            // padded column 0 (the compute lanes write padded row 0)
            if (g == 0)
                for (int r = lane; r <= rows; r += kWarp) table[static_cast<int64_t>(r) * tld + kTabShift] = 0.0;
        }
    } else if (live) {
        const int c = g * kStripCols + lane * kC;
        const int nvalid = max(0, min(kC, cols - c)); // my columns inside the map
        // The one lane that straddles the last column (odd widths) stores its whole 16-byte
        // group like every other lane: its columns past the map read as zeros, and the row
        // pitch has room for them (checked by sat_cluster_eligible), so the step has no
        // second store path.
        const bool valid = nvalid > 0;
#pragma unroll
        for (int k = 0; k < kC; ++k)
            if (k < nvalid) table[kTabShift + 1 + c + k] = 0.0; // padded row 0
        const bool has_in = g > 0, has_out = g + 1 < strips;
        // S(r, my last column) of lane 31 goes to edge_out + 8 r: the right neighbour's shared
        // edge column (same cluster) or boundary column q_cl of the chain (global memory)
        unsigned edge_out_s = 0;
        unsigned long long edge_out_g = 0;
        bool out_dsmem = false;
        if (has_out) {
            const int gn = g + 1, per_cluster = spc * csize;
            out_dsmem = gn / per_cluster == q_cl;
            if (out_dsmem)
                edge_out_s = map_to_cta_s(smem_u32(edges + static_cast<size_t>(gn % spc) * edge_bytes),
                                          static_cast<unsigned>((gn % per_cluster) / spc));
            else
                edge_out_g = reinterpret_cast<unsigned long long>(L.gedge + (job * L.strips + q_cl) * L.edge_stride);
        }
        const unsigned edge_lane_s = has_out && out_dsmem && lane == kWarp - 1 ? 1u : 0u;
        const unsigned edge_lane_g = has_out && !out_dsmem && lane == kWarp - 1 ? 1u : 0u;
        edge_out_s -= 8u * static_cast<unsigned>(lane); // + 8 s = row s - lane
        edge_out_g -= 8ull * static_cast<unsigned>(lane);
        const unsigned edge_in_s = smem_u32(edge_in);
        // every shared address of the loop is a 32-bit shared-window address held in a
        // register (a generic pointer would be converted again in every block)
        const unsigned xbase = smem_u32(ring) + 16u * static_cast<unsigned>(lane);
        unsigned xoff = (static_cast<unsigned>(-lane) & (kClRingRows - 1)) * kClRowBytes; // ring row of my step-0 row
        double prev[kC]; // S(r-1, c + k)
#pragma unroll
        for (int k = 0; k < kC; ++k) prev[k] = 0.0;
        double left_prev = 0.0; // S(r-1, c-1)
        // table row of my current row r = s - lane (padded row r + 1)
        double* trow = table + kTabShift + 1 + c + static_cast<int64_t>(1 - lane) * tld;
        const int steps = rows + kWarp - 1;
        const int n_blocks = (steps + kClBlock - 1) / kClBlock;
        using XV = typename XVec<T>::type;
        XV xn; // source values of the next step (loaded one step ahead inside a block)

        // Hand-over values: f[i] = the left strip's S(row, last column) for the 8 rows
        // of a group of steps, fn[] the next group's, read one group ahead. Every lane
        // reads the same 64 bytes (a broadcast: no shuffle, no divergence, no staging
        // between the hand-over and lane 0's additions); a value still equal to the
        // sentinel is polled when its group starts. Strip 0 reads a block of zeros
        // (S(r, -1) = 0) with a stride of 0, so the loop has no "first strip" branch.
        double f[kClGroup], fn[kClGroup];
        unsigned ep = has_in ? edge_in_s : zero_s;          // address of the next group to load
        const unsigned ep_step = has_in ? 8u * kClGroup : 0u;
        auto load_group = [&](const unsigned p, double (&v)[kClGroup]) {
            UWB_DCHECK(!has_in || (p >= edge_in_s && p + 8u * kClGroup <= edge_in_s + edge_bytes));
#pragma unroll
            for (int i = 0; i < kClGroup; i += 2) ld_edge_poll2(p + 8u * i, v[i], v[i + 1]);
        };
        load_group(ep, fn);

        // One block of 32 steps. Mode 0: interior (every lane's row is inside the map).
        // Mode 2: the first block (rows >= 32): a lane whose row r = s - lane is still
        // negative computes a virtual row of zeros (its x reads as zero and its state is
        // zero, so every S stays +0) - only the stores are predicated, nothing
        // conditional sits on the dependent chain. Every strip's first 39 steps are the
        // lag of the strip to its right, so this block is on the critical path of the
        // whole table. Mode 3: the last blocks (r >= 0 everywhere): lanes past the last
        // row keep adding zeros, unstored; a non-finite S of the last row stays
        // non-finite, a finite one stays finite, so the check after the loop holds (and
        // does not start a column rescan on stale ring contents).
        // Mode 1: maps shorter than a block (state updates conditional).
        auto block = [&](const int s0, auto mode_tag) {
            constexpr int kMode = decltype(mode_tag)::value;
            constexpr bool kRowCheck = kMode == 1 || kMode == 3; // rows >= `rows` exist in this block
#pragma unroll
            for (int u = 0; u < kClBlock; ++u) {
                if (u % kClGroup == 0) {
                    bool miss = false;
#pragma unroll
                    for (int i = 0; i < kClGroup; ++i) {
                        f[i] = fn[i];
                        miss |= (!kRowCheck || s0 + u + i < rows) && __double_as_longlong(f[i]) == kClSentinel;
                    }
                    while (miss) { // warp-uniform: every lane reads the same values
#ifdef UWB_CL_POLL_SLEEP
                        __nanosleep(UWB_CL_POLL_SLEEP);
#endif
                        load_group(ep, f);
                        miss = false;
#pragma unroll
                        for (int i = 0; i < kClGroup; ++i)
                            miss |= (!kRowCheck || s0 + u + i < rows) && __double_as_longlong(f[i]) == kClSentinel;
                    }
                    if (kMode == 3) { // rows past the map: lane 0 adds zeros, not the sentinel (a NaN)
#pragma unroll
                        for (int i = 0; i < kClGroup; ++i) f[i] = s0 + u + i < rows ? f[i] : 0.0;
                    }
                    ep += ep_step;
                    if (!kRowCheck || s0 + u + kClGroup < rows) load_group(ep, fn); // (never past the edge column)
                }
                const int r = s0 + u - lane;
                const bool in_map = kMode == 0 || (kMode == 2 ? r >= 0 : kMode == 3 ? r < rows : (r >= 0 && r < rows));
                T x[kC];
                XVec<T>::get(xn, x);
                if (kMode == 2 || kMode == 3) { // rows outside the map read as zeros (stale ring rows may hold NaNs)
#pragma unroll
                    for (int k = 0; k < kC; ++k) x[k] = in_map ? x[k] : T(0);
                }
                xoff = (xoff + kClRowBytes) & (kClRingBytes - 1u);
                if (u + 1 < kClBlock) xn = XVec<T>::lds(xbase + xoff);
                double a[kC]; // x + S(r-1, .): independent of the left neighbour
#pragma unroll
                for (int k = 0; k < kC; ++k) a[k] = dadd(widen(x[k]), prev[k]);
                double left = __shfl_up_sync(0xffffffffu, prev[kC - 1], 1);
#if !(UWB_CL_PROBE & 2)
                if (lane == 0) left = f[u % kClGroup];
#endif
                double sv[kC];
                sv[0] = dsub(dadd(a[0], left), left_prev);
#pragma unroll
                for (int k = 1; k < kC; ++k) sv[k] = dsub(dadd(a[k], sv[k - 1]), prev[k - 1]);
                if (in_map) {
                    if (valid && !(UWB_CL_PROBE & 1)) {
                        UWB_DCHECK(r >= 0 && r < rows && c < cols && kTabShift + 1 + c + kC <= tld &&
                                   trow == table + static_cast<int64_t>(r + 1) * tld + kTabShift + 1 + c);
#pragma unroll
                        for (int q = 0; q < kC / 2; ++q)
                            reinterpret_cast<double2*>(trow)[q] = make_double2(sv[2 * q], sv[2 * q + 1]);
                    }
                    UWB_DCHECK(!(edge_lane_s | edge_lane_g) || static_cast<unsigned>(r) * 8u < edge_bytes);
                    UWB_DCHECK(!edge_lane_g || (r < L.edge_stride && q_cl < L.strips));
                }
                st_edge_dsmem(edge_out_s + 8u * static_cast<unsigned>(s0 + u), sv[kC - 1], in_map ? edge_lane_s : 0u);
                st_edge_global(edge_out_g + 8ull * static_cast<unsigned>(s0 + u), sv[kC - 1], in_map ? edge_lane_g : 0u);
                if (kMode != 1 || in_map) {
                    left_prev = left;
#pragma unroll
                    for (int k = 0; k < kC; ++k) prev[k] = sv[k];
                }
                trow += tld;
            }
        };

#if UWB_CL_SLACK > 0
        // start with some slack behind the left strip (see UWB_CL_SLACK)
        if (has_in) {
            const unsigned p = edge_in_s + 8u * static_cast<unsigned>(min(kClGroup - 1 + UWB_CL_SLACK, rows - 1) & ~1);
            double v0, v1;
            do {
                ld_edge_poll2(p, v0, v1);
            } while (__double_as_longlong(v0) == kClSentinel);
        }
#endif
#pragma unroll 1
        for (int b = 0; b < n_blocks; ++b) {
            const int s0 = b * kClBlock;
            // this block reads rows s0 - 31 .. s0 + 31: chunks b - 1 (waited for) and b
            if (!(UWB_CL_PROBE & 4) && s0 < rows)
                mbar_wait(&full[b & (kClChunks - 1)], static_cast<unsigned>((b / kClChunks) & 1));
            xn = XVec<T>::lds(xbase + xoff);
            if (s0 >= kWarp - 1 && s0 + kClBlock <= rows) block(s0, std::integral_constant<int, 0>{});
            else if (s0 == 0 && rows >= kClBlock) block(s0, std::integral_constant<int, 2>{});
            else if (s0 >= kWarp - 1) block(s0, std::integral_constant<int, 3>{});
            else block(s0, std::integral_constant<int, 1>{});
            // the next block reads rows >= s0 + 1: chunk b - 1 may be refilled
            if (b >= kClBack && b - kClBack + kClChunks < n_chunks) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[(b - kClBack) & (kClChunks - 1)]);
            }
        }
        // non-finite inputs poison every later S of their column (sat.cu header)
        bool finite = true;
#pragma unroll
        for (int k = 0; k < kC; ++k) finite &= k >= nvalid || isfinite(prev[k]);
        if (nvalid > 0 && !finite && J.nonfinite) {
            int col = c;
            const int bad = first_nonfinite<T>(static_cast<const T*>(J.src), ld, c, nvalid, rows, &col);
            if (bad != INT_MAX)
                report_min(J.nonfinite,
                           static_cast<unsigned long long>((J.row0 + bad) * L.geo.map_cols + J.col0 + col));
        }
    }
    __syncthreads();
    cluster_sync_all(); // a CTA's shared memory must outlive its neighbour's stores
}

struct ClShape {
    int spc, csize, chain;
    unsigned edge_bytes;
    size_t smem;
};

template <typename T>
__global__ void sat_cluster_kernel(SatLaunch L, int spc, int csize, int chain, unsigned edge_bytes);

// Clusters of `csize` CTAs with this much shared memory that the device keeps
// resident at once (the GPCs limit how many 8-CTA clusters fit: a chain whose last
// clusters only start when the first ones finish would double its time).
static int max_active_clusters(int elem, int csize, int spc, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int, size_t>, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(dev, elem, csize, spc, smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(csize), 1, 1);
    cfg.blockDim = dim3(static_cast<unsigned>((2 * spc + 1) * kWarp), 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(csize);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e;
    if (elem == 4) {
        e = cudaFuncSetAttribute(sat_cluster_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveClusters(&n, sat_cluster_kernel<float>, &cfg);
    } else {
        e = cudaFuncSetAttribute(sat_cluster_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveClusters(&n, sat_cluster_kernel<double>, &cfg);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    cache[key] = n;
    return n;
}

// Strips per CTA, CTAs per cluster and clusters per table, in the order measured
// fastest (1024-row fp32 maps): one strip per CTA in one cluster (8 strips 121 us),
// two per CTA (16 strips 160 us), a chain of one-strip clusters (32 strips 227 us,
// 128 strips 642 us), and only then three strips per CTA (24 strips 240 us: three
// compute warps, their helpers and the relay share four schedulers). A chain's
// cluster size (8, 4, 2, 1) is the largest that keeps every cluster resident.
static bool cluster_shape(int64_t cols, int64_t rows, int elem, int64_t n_jobs, int sms, ClShape* S,
                          bool single_only = false) {
    const int64_t strip_cols = kWarp * (16 / elem);
    const int64_t strips = (cols + strip_cols - 1) / strip_cols;
    if (strips < 1 || rows < 1 || rows > 16384 || n_jobs < 1) return false;
    // one group past the last row is read ahead (and stays a sentinel)
    S->edge_bytes = static_cast<unsigned>((rows * 8 + 8 * kClGroup + 127) / 128 * 128);
    const size_t per_strip = kClRingBytes + S->edge_bytes + kClBarBytes;
    auto take = [&](int spc, bool chained) {
        const size_t smem = spc * per_strip + kClZeroBytes;
        if (smem > kClSmemCap) return false;
        const int64_t ctas = (strips + spc - 1) / spc;
        if (!chained) {
            if (ctas > kClMaxCtas || n_jobs * ctas > sms) return false;
            *S = ClShape{spc, static_cast<int>(ctas), 1, S->edge_bytes, smem};
            return true;
        }
        if (single_only || ctas <= kClMaxCtas) return false;
        for (int csize = kClMaxCtas; csize >= 1; csize /= 2) {
            const int64_t chain = (ctas + csize - 1) / csize;
            if (n_jobs * chain * csize > sms || max_active_clusters(elem, csize, spc, smem) < n_jobs * chain) continue;
            *S = ClShape{spc, csize, static_cast<int>(chain), S->edge_bytes, smem};
            return true;
        }
        return false;
    };
    return take(1, false) || take(2, false) || take(1, true) || take(2, true) || take(3, false) || take(3, true);
}

static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

__global__ void fill_sentinel_kernel(double* gedge, int64_t strips, int64_t edge_stride, int chain, int64_t rows) {
    // boundary column q of job blockIdx.y: (job * strips + q) * edge_stride
    const int64_t q = blockIdx.x % chain, part = blockIdx.x / chain, parts = gridDim.x / chain;
    long long* col = reinterpret_cast<long long*>(gedge + (static_cast<int64_t>(blockIdx.y) * strips + q) * edge_stride);
    for (int64_t r = part * blockDim.x + threadIdx.x; r < rows; r += parts * blockDim.x) col[r] = kClSentinel;
}

} // namespace

// One cluster (or, with `allow_chain`, a chain of clusters) per table when every
// CTA of the batch is resident at once (dense tables, 16-byte aligned rows whose
// length is a multiple of 16 bytes).
bool sat_cluster_fits(int64_t n_jobs, int64_t cols, int64_t max_rows, int dtype, bool allow_chain) {
    const int elem = dtype == UWB_F32 ? 4 : 8;
    ClShape S;
    return n_jobs >= 1 && cluster_shape(cols, max_rows, elem, n_jobs, sm_count(), &S, !allow_chain);
}

bool sat_cluster_eligible(const SatLaunch& L, int dtype) {
    // (rows that the TMA bulk copy cannot take - unaligned or not whole 16-byte pieces - are
    // copied by the helper warp itself)
    const int elem = dtype == UWB_F32 ? 4 : 8;
    const int64_t kc = 16 / elem;
    if (kTabShift + 1 + (L.cols + kc - 1) / kc * kc > L.table_ld) return false; // room for the straddling lane's group
    ClShape S;
    // without an edge buffer (one-strip plans) only single clusters
    const bool single_only = L.gedge == nullptr;
    if (!cluster_shape(L.cols, L.geo.max_table_rows(), elem, L.n_jobs, sm_count(), &S, single_only)) return false;
    // a sparse-mode call (certified path) only reaches here with a table too wide for
    // the small-batch exact path (cert_applies): the chain writes the whole table, a
    // superset of the marked taps, far faster than the one-warp-per-strip chain of sat.cu
    if (L.need) {
        ClShape S1;
        return !cluster_shape(L.cols, L.geo.max_table_rows(), elem, L.n_jobs, sm_count(), &S1, true);
    }
    return true;
}

template <typename T>
static cudaError_t launch_sat_cluster_t(const SatLaunch& L, const ClShape& S, cudaStream_t stream) {
    auto kern = sat_cluster_kernel<T>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(S.smem));
    if (e != cudaSuccess) return e;
    if (S.chain > 1) {
        // the boundary columns between the clusters of a chain start as sentinels
        ++g_kernel_launches;
        fill_sentinel_kernel<<<dim3(static_cast<unsigned>(S.chain * 4), static_cast<unsigned>(L.n_jobs)), 256, 0, stream>>>(
            L.gedge, L.strips, L.edge_stride, S.chain, L.geo.max_table_rows());
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(L.n_jobs * S.chain * S.csize), 1, 1);
    cfg.blockDim = dim3(static_cast<unsigned>((2 * S.spc + 1) * kWarp), 1, 1);
    cfg.dynamicSmemBytes = S.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(S.csize);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ++g_kernel_launches;
    return cudaLaunchKernelEx(&cfg, kern, L, S.spc, S.csize, S.chain, S.edge_bytes);
}

cudaError_t launch_sat_cluster(const SatLaunch& L, int dtype, cudaStream_t stream) {
    ClShape S;
    if (!cluster_shape(L.cols, L.geo.max_table_rows(), dtype == UWB_F32 ? 4 : 8, L.n_jobs, sm_count(), &S,
                       L.gedge == nullptr))
        return cudaErrorInvalidValue;
    if (S.chain > 1 && (!L.gedge || S.chain > L.strips || L.geo.max_table_rows() > L.edge_stride)) return cudaErrorInvalidValue;
    return dtype == UWB_F32 ? launch_sat_cluster_t<float>(L, S, stream) : launch_sat_cluster_t<double>(L, S, stream);
}

} // namespace uwb
