// tmem_bench.cu — microbenchmark: tcgen05.ld (32x32b.x32) latency and throughput per SM on
// sm_100a. One CTA per SM allocates 512 TMEM columns; `warps` warps each issue `iters` loads,
// either load+wait each (latency-bound) or `batch` loads then one wait (throughput).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}

__global__ void bench(int iters, int batch, unsigned long long* cycles, float* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
    float acc = 0.f;
    uint32_t r[32];
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i += batch) {
        for (int b = 0; b < batch; ++b) {
            ld32(base + ((i + b) * 32) % 512, r);
            acc += __uint_as_float(r[0]) + __uint_as_float(r[17]) + __uint_as_float(r[31]);
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    }
    const unsigned long long t1 = clock64();
    if (lane == 0) atomicAdd(cycles, t1 - t0);
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    unsigned long long* d_cyc;
    float* sink;
    cudaMalloc(&d_cyc, 8);
    cudaMalloc(&sink, 148 * 1024 * 4);
    const int iters = 4096;
    for (int warps : {1, 4, 8, 16}) {
        for (int batch : {1, 4}) {
            cudaMemset(d_cyc, 0, 8);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            bench<<<148, warps * 32>>>(iters, batch, d_cyc, sink);
            cudaEventRecord(b);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            unsigned long long cyc;
            cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost);
            const double cyc_per_warp = (double)cyc / (148.0 * warps);
            const double bytes = 148.0 * warps * iters * 4096.0;
            printf("warps=%2d batch=%d  cycles/load/warp=%7.1f  TMEM->RF %.1f TB/s (%.0f B/clk/SM @1.9GHz)\n",
                   warps, batch, cyc_per_warp / iters, bytes / (ms * 1e-3) / 1e12,
                   bytes / (ms * 1e-3) / 148 / 1.9e9);
        }
    }
    return 0;
}
