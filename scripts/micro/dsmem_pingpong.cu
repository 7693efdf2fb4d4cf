// One-way latency of a value handed from one CTA of a cluster to the next through
// distributed shared memory (the cluster SAT's strip hand-over): a 2-CTA cluster
// plays ping-pong with 8-byte values that are their own flags; time per round / 2.
//   v0: st.relaxed.cluster.shared::cluster.f64   (the kernel's store)
//   v1: st.weak (plain) shared::cluster store
//   v2: st.async ... mbarrier::complete_tx::bytes (value polled, barrier unused)
//   v3: atom.exch.relaxed.cluster.shared::cluster.b64
//   v4: v0 while the same thread also streams 16-byte global stores (the table rows)
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}

template <int V>
__global__ void __cluster_dims__(2, 1, 1) k(long long* out, double* sink, int n) {
    __shared__ __align__(16) unsigned long long slot[2];
    __shared__ __align__(8) unsigned long long bar;
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        slot[0] = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0) {
        const unsigned mine = smem_u32(&slot[0]);
        const unsigned peer = mapa(mine, rank ^ 1u), peer_bar = mapa(smem_u32(&bar), rank ^ 1u);
        long long t0 = 0, t1 = 0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (unsigned long long i = 1; i <= static_cast<unsigned long long>(n); ++i) {
            if (rank == 0) { // send i, wait for the echo
                if (V == 0 || V == 4) asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(peer), "l"(i) : "memory");
                if (V == 1) asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(peer), "l"(i) : "memory");
                if (V == 2)
                    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.u64 [%0], %1, [%2];" ::"r"(peer), "l"(i),
                                 "r"(peer_bar)
                                 : "memory");
                if (V == 3) {
                    unsigned long long old;
                    asm volatile("atom.relaxed.cluster.shared::cluster.exch.b64 %0, [%1], %2;" : "=l"(old) : "r"(peer), "l"(i) : "memory");
                }
                if (V == 4) reinterpret_cast<double2*>(sink)[i & 4095] = make_double2(1.0, 2.0);
                unsigned long long v;
                do {
                    asm volatile("ld.volatile.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(mine) : "memory");
                } while (v != i);
            } else { // wait for i, echo it
                unsigned long long v;
                do {
                    asm volatile("ld.volatile.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(mine) : "memory");
                } while (v != i);
                if (V == 0 || V == 4) asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(peer), "l"(i) : "memory");
                if (V == 1) asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(peer), "l"(i) : "memory");
                if (V == 2)
                    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.u64 [%0], %1, [%2];" ::"r"(peer), "l"(i),
                                 "r"(peer_bar)
                                 : "memory");
                if (V == 3) {
                    unsigned long long old;
                    asm volatile("atom.relaxed.cluster.shared::cluster.exch.b64 %0, [%1], %2;" : "=l"(old) : "r"(peer), "l"(i) : "memory");
                }
                if (V == 4) reinterpret_cast<double2*>(sink)[4096 + (i & 4095)] = make_double2(1.0, 2.0);
            }
        }
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (rank == 0) out[V] = t1 - t0;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main() {
    long long* c;
    double* sink;
    const int n = 2000;
    cudaMallocManaged(&c, 64);
    cudaMalloc(&sink, 16 * 8192);
    for (int rep = 0; rep < 2; ++rep) {
        k<0><<<2, 32>>>(c, sink, n);
        k<1><<<2, 32>>>(c, sink, n);
        k<2><<<2, 32>>>(c, sink, n);
        k<3><<<2, 32>>>(c, sink, n);
        k<4><<<2, 32>>>(c, sink, n);
        cudaDeviceSynchronize();
    }
    const char* names[5] = {"st.relaxed.cluster", "st.weak", "st.async", "atom.exch", "st.relaxed + global stores"};
    for (int v = 0; v < 5; ++v) printf("v%d %-28s one-way %.0f ns\n", v, names[v], c[v] / (2.0 * n));
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
