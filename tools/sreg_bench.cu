// sreg_bench.cu — latency of a few instructions the pair kernel's row-block loop depends on
// (sm_100a, cluster of 2): special-register reads (%cluster_ctarank, %tid, clusterid) and a
// kernel-parameter read forced through ld.param, each measured as a dependent chain.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sreg_bench tools/sreg_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct P { int a[64]; };

__global__ void __cluster_dims__(2, 1, 1) k(P p, int iters, unsigned long long* out, int* sink) {
    uint32_t acc = threadIdx.x;
    unsigned long long t0, t1;
    // 0: %cluster_ctarank chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t r;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
        acc = acc * 3 + r;
    }
    t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
    // 1: %tid.x chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t r;
        asm volatile("mov.u32 %0, %%tid.x;" : "=r"(r));
        acc = acc * 3 + r;
    }
    t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (t1 - t0) / iters;
    // 2: shared-window base (cvta of a static shared array) chain
    __shared__ int sh[256];
    sh[threadIdx.x & 255] = threadIdx.x;
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        volatile int* q = sh;
        acc = acc * 3 + q[(acc + i) & 255];
    }
    t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[2] = (t1 - t0) / iters;
    // 3: param read chain (index depends on acc so it cannot be hoisted)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) acc = acc * 3 + p.a[acc & 63];
    t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[3] = (t1 - t0) / iters;
    // 4: global store issue rate (independent stores)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) sink[(blockIdx.x * 64 + (i & 63)) * 32 + (threadIdx.x & 31)] = acc + i;
    t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[4] = (t1 - t0) / iters;
    sink[blockIdx.x * 1024 + threadIdx.x] += acc;
}

int main() {
    unsigned long long* d;
    int* sink;
    cudaMalloc(&d, 64);
    cudaMalloc(&sink, 1 << 24);
    P p;
    for (int i = 0; i < 64; ++i) p.a[i] = i;
    k<<<2, 128>>>(p, 1000, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long h[5];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const char* nm[5] = {"cluster_ctarank chain", "tid.x chain", "lds chain", "param (indexed) chain",
                         "global store issue"};
    for (int i = 0; i < 5; ++i) printf("%-24s %llu cycles/iter\n", nm[i], h[i]);
    return 0;
}
