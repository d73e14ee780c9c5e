// mbar_bench.cu — microbenchmark of the handshake latencies the tcgen05 kernels depend on
// (sm_100a): an mbarrier ping-pong between two warps (a) in one CTA with local arrives, (b) across
// the two CTAs of a cluster with remote (shared::cluster) arrives, and (c) a tcgen05.commit
// "accumulator full" signal (no MMA in flight) answered by a local arrive.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbar_bench tools/mbar_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint32_t b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c) : "memory");
}
__device__ __forceinline__ void arrive(uint32_t b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t b, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(b), "r"(rank));
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}
__device__ __forceinline__ void wait(uint32_t b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(b), "r"(ph) : "memory");
}
__device__ __forceinline__ uint32_t crank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// mode 0: local ping-pong; mode 1: cross-CTA ping-pong (warp 0 of CTA 0 <-> warp 0 of CTA 1);
// mode 2: tcgen05.commit ping (warp 1 commits, warp 0 waits + arrives back locally)
__global__ void __cluster_dims__(2, 1, 1) pingpong(int mode, int iters, unsigned long long* out) {
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = crank();
    if (threadIdx.x == 0) {
        init(s32(&bar[0]), 1);
        init(s32(&bar[1]), mode == 3 ? 2 : 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (mode == 2 && warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(s32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (mode == 3 && warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(s32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    __syncthreads();
    csync();
    unsigned long long t0 = clock64();
    if (mode == 0 && rank == 0 && lane == 0) {
        for (int i = 0; i < iters; ++i) {
            if (warp == 0) { arrive(s32(&bar[0])); wait(s32(&bar[1]), i & 1); }
            else if (warp == 1) { wait(s32(&bar[0]), i & 1); arrive(s32(&bar[1])); }
        }
    } else if (mode == 1 && warp == 0 && lane == 0) {
        for (int i = 0; i < iters; ++i) {
            if (rank == 0) { arrive_remote(s32(&bar[0]), 1); wait(s32(&bar[1]), i & 1); }
            else { wait(s32(&bar[0]), i & 1); arrive_remote(s32(&bar[1]), 0); }
        }
    } else if (mode == 2 && rank == 0 && lane == 0) {
        for (int i = 0; i < iters; ++i) {
            if (warp == 1) {
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(&bar[0])) : "memory");
                wait(s32(&bar[1]), i & 1);
            } else if (warp == 0) {
                wait(s32(&bar[0]), i & 1);
                arrive(s32(&bar[1]));
            }
        }
    }
    else if (mode == 3 && lane == 0) {
        // leader warp 1 multicasts a cta_group::2 commit to bar[0] of both CTAs; warp 0 of each
        // CTA waits and arrives remotely on the leader's bar[1] (count 1 -> re-init with 2)
        for (int i = 0; i < iters; ++i) {
            if (rank == 0 && warp == 1) {
                asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(s32(&bar[0])), "h"((uint16_t)3) : "memory");
                wait(s32(&bar[1]), i & 1);
            } else if (warp == 0) {
                wait(s32(&bar[0]), i & 1);
                arrive_remote(s32(&bar[1]), 0);
            }
        }
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) out[mode] = (t1 - t0) / iters;
    __syncthreads();
    csync();
    if (mode == 2 && warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tslot));
    if (mode == 3 && warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 32;" ::"r"(tslot));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    cudaMemset(d, 0, 64);
    const char* names[4] = {"local mbarrier ping-pong", "cross-CTA (cluster) ping-pong",
                            "tcgen05.commit -> wait -> local arrive",
                            "cta_group::2 multicast commit -> 2 remote arrivals"};
    for (int mode = 0; mode < 4; ++mode) {
        pingpong<<<2, 64>>>(mode, 2000, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("mode %d err %s\n", mode, cudaGetErrorString(e)); return 1; }
    }
    unsigned long long h[4];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int m = 0; m < 4; ++m) printf("%-40s %6llu cycles per round trip\n", names[m], h[m]);
    return 0;
}
