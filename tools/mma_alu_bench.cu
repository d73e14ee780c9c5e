// mma_alu_bench.cu — does a busy tensor pipe slow down CUDA-core ALU work on the same SM?
// One CTA per SM. Warp 0 (one elected lane) keeps tcgen05 busy with M=128 x N=256 x K=16 fp16
// MMAs (operands: garbage in shared memory, accumulator in TMEM), double-buffered commits.
// Warps 4..11 run the distance-fold instruction mix (FFMA imm, set.geu, FMNMX, FFMA) on
// registers. Reports ALU cycles per warp-column with and without the MMA stream.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_alu_bench tools/mma_alu_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint32_t b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t@!P1 bra W_%=;\n\t}" ::"r"(b), "r"(ph), "r"(0x989680) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__global__ void __launch_bounds__(384, 1) k(int mma_on, int iters, int alu_iters, unsigned long long* out, float* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bars[2];
    __shared__ uint32_t tslot;
    __shared__ int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { bar_init(s32(&bars[0]), 1); bar_init(s32(&bars[1]), 1); stop = 0; }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (warp == 0) {
        if (mma_on) {
            const uint32_t idesc = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            const uint32_t a = s32(sm), b = s32(sm + 32768);
            for (int i = 0; i < iters; ++i) {
                const int buf = i & 1;
                if (i >= 2) bar_wait(s32(&bars[buf]), ((i - 2) >> 1) & 1);
                if (lane == 0) {
                    for (int kk = 0; kk < 8; ++kk) {
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                     ::"r"(tmem + buf * 256), "l"(desc(a + kk * 32)), "l"(desc(b + kk * 32)), "r"(idesc), "r"(kk));
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(&bars[buf])) : "memory");
                }
                __syncwarp();
                if (*(volatile int*)&stop) break;
            }
            bar_wait(s32(&bars[0]), 0); // drain (best effort)
        }
    } else if (warp >= 4) {
        float v[8], s[8], x0 = lane * 0.001f, acc = 0.f;
        for (int c = 0; c < 8; ++c) { v[c] = 1e30f; s[c] = -1.f; }
        const unsigned long long t0 = clock64();
        for (int i = 0; i < alu_iters; ++i) {
#pragma unroll
            for (int e = 0; e < 32; ++e) {
                const float x = fmaf(x0 + e, -2.0f, (float)i);
                float nf;
                asm("set.geu.f32.f32 %0, %1, %2;" : "=f"(nf) : "f"(x), "f"(v[e & 7]));
                v[e & 7] = fminf(v[e & 7], x);
                s[e & 7] = fmaf(s[e & 7], nf, -1.0f);
            }
            x0 += 1e-7f;
        }
        const unsigned long long t1 = clock64();
        for (int c = 0; c < 8; ++c) acc += v[c] + s[c];
        sink[blockIdx.x * 384 + threadIdx.x] = acc;
        if (lane == 0) atomicAdd(out, (t1 - t0));
        if (warp == 4 && lane == 0) stop = 1;
    }
    __syncthreads();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 8);
    cudaMalloc(&sink, 148 * 384 * 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    const int alu_iters = 2000;
    for (int on = 0; on < 2; ++on) {
        cudaMemset(d, 0, 8);
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        k<<<148, 384, 65536 + 1024>>>(on, 1 << 30, alu_iters, d, sink);
        cudaEventRecord(b);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        float ms; cudaEventElapsedTime(&ms, a, b);
        unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        const double per_warp = (double)cyc / (148.0 * 8);
        printf("mma_on=%d  ALU: %.2f cycles per warp-column (8 fold warps/SM, 2 per SMSP), kernel %.3f ms\n",
               on, per_warp / (alu_iters * 32.0), ms);
    }
    return 0;
}
