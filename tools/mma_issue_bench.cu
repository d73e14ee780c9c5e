// mma_issue_bench.cu — issue cost vs execution time of back-to-back tcgen05.mma (cta_group::1,
// M = 128, fp16 K = 16 / E5M2 K = 32, N = 256 or 128; operands: garbage in shared memory,
// accumulator in TMEM). One CTA per SM; warp 0's elected lane issues `count` MMAs into one
// accumulator and commits once. Reports, per MMA, the cycles the issuing thread spends in the
// issue loop and the cycles until the commit's mbarrier completes — i.e. whether the MMA issuer
// or the tensor pipe bounds the pair kernel's tile (8 fp16 or 4 E5M2 MMAs per 256-column tile).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_issue_bench tools/mma_issue_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
    // K-major, 128-byte swizzle, SBO 1024 B (8 rows x 128 B), sm100 descriptor version bits
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

template <bool F8>
__global__ void __launch_bounds__(128, 1) k(int count, int n_cols, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(s32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (warp == 0) {
        uint32_t pred;
        asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
        if (pred) {
            // instruction descriptor: f32 accumulate, A/B format, K-major, N, M = 128
            const uint32_t fmt = F8 ? 1u : 0u;   // E5M2 in kind::f8f6f4, fp16 in kind::f16
            const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) |
                                   ((uint32_t)(n_cols >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            const uint64_t a = desc(s32(sm)), b = desc(s32(sm + 32768));
            const long long t0 = clock64();
            for (int i = 0; i < count; ++i) {
                const uint64_t ad = a + (uint64_t)((i & 3) * 2), bd = b + (uint64_t)((i & 3) * 2);
                if (F8)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(i));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(i));
            }
            const long long t1 = clock64();
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         ::"r"(s32(&bar)) : "memory");
            asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}"
                         ::"r"(s32(&bar)) : "memory");
            const long long t2 = clock64();
            if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
        }
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    unsigned long long h[2];
    const int smem = 65536 + 1024;
    cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int f8 = 0; f8 < 2; ++f8)
        for (int n : {256, 128})
            for (int count : {8, 64, 512}) {
                for (int rep = 0; rep < 2; ++rep) {
                    if (f8) k<true><<<148, 128, smem>>>(count, n, d);
                    else k<false><<<148, 128, smem>>>(count, n, d);
                }
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                const double work = 2.0 * 128 * n * (f8 ? 32 : 16) / (f8 ? 16384.0 : 8192.0);
                printf("%s N=%d count=%4d: issue %.1f cycles/MMA, issue+complete %.1f cycles/MMA "
                       "(tensor work at the nominal dense rate: %.0f cycles/MMA)\n",
                       f8 ? "e5m2 K=32" : "fp16 K=16", n, count, (double)h[0] / count,
                       (double)h[1] / count, work);
            }
    return 0;
}
