// op_rate_bench.cu — per-SMSP throughput of the fold's candidate instructions on sm_100a:
// 8 warps per SM (2 per SMSP), 8 independent chains per warp, cycles per warp-instruction.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/op_rate_bench tools/op_rate_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(int iters, unsigned long long* out, float* sink) {
    const int lane = threadIdx.x & 31;
    float v[8], s[8];
    float x = lane * 0.001f;
    for (int c = 0; c < 8; ++c) { v[c] = 1.0f + c; s[c] = -1.f - c; }
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            float& a = v[e & 7];
            float& b = s[e & 7];
            if (MODE == 0) {          // FMNMX
                a = fminf(a, x + (float)e);      // FADD folded? keep x const per e
            } else if (MODE == 1) {   // FSET.BF
                float r;
                asm volatile("set.geu.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
                a = r;
            } else if (MODE == 2) {   // FFMA imm
                a = fmaf(a, -2.0f, b);
            } else if (MODE == 3) {   // FSETP + FSEL (old chain update, value part)
                const bool p = b < a;
                a = p ? b : a;
                b = b + 1.0f;
            } else if (MODE == 4) {   // FMNMX on two registers (no FADD)
                a = fminf(a, b);
                b = fmaxf(b, a);
            } else if (MODE == 6) {   // FSET + FMNMX on the same inputs (chain update core)
                float r;
                asm volatile("set.geu.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(x), "f"(a));
                a = fminf(a, x);
                b = b + r;
            } else if (MODE == 7) {   // FSET + FMNMX, no FADD (flags accumulate via FMNMX)
                float r;
                asm volatile("set.geu.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(b), "f"(a));
                a = fminf(a, b);
                b = fmaxf(r, b);
            } else if (MODE == 8) {   // FFMA2 alone (two lanes of fp32x2)
                uint64_t a2 = ((uint64_t)__float_as_uint(b) << 32) | __float_as_uint(a), d2;
                asm volatile("fma.rn.f32x2 %0, %1, %2, %1;" : "=l"(d2) : "l"(a2), "l"(0xC0000000C0000000ull));
                a = __uint_as_float((uint32_t)d2); b = __uint_as_float((uint32_t)(d2 >> 32));
            } else if (MODE == 9) {   // 1 FFMA2 + 2 FMNMX (the fold's pipe mix without FSET)
                uint64_t a2 = ((uint64_t)__float_as_uint(b) << 32) | __float_as_uint(a), d2;
                asm volatile("fma.rn.f32x2 %0, %1, %2, %1;" : "=l"(d2) : "l"(a2), "l"(0xC0000000C0000000ull));
                const float lo = __uint_as_float((uint32_t)d2), hi = __uint_as_float((uint32_t)(d2 >> 32));
                a = fminf(a, lo);
                b = fminf(b, hi);
            } else if (MODE == 10) {  // 1 FFMA (imm) + 2 FMNMX
                const float lo = fmaf(a, -2.0f, b);
                a = fminf(a, lo);
                b = fminf(b, lo + 1.0f);
            } else if (MODE == 11) {  // the fold's chain update on two chains (chain_step_x2)
                // per element pair: FFMA2 x, 2 FSET, 2 FMNMX, FFMA2 s
                static_assert(true, "");
                uint64_t acc2 = ((uint64_t)__float_as_uint(x + e) << 32) | __float_as_uint(x - e);
                mpk::tcdev::chain_step_x2(acc2, 0x3F8000003F800000ull, 0xC0000000C0000000ull,
                                          v[e & 7], v[(e + 1) & 7], *reinterpret_cast<uint64_t*>(&s[(e & 3) * 2]),
                                          0xBF800000BF800000ull);
            } else if (MODE == 12) {  // FMNMX3 alone (independent chains)
                float r;
                asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(x));
                a = r;
            } else if (MODE == 13) {  // FMNMX3 + 2 FSET (the reverse fold's alu mix, 2 columns)
                float r, p0, p1;
                asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(x));
                asm volatile("set.gtu.f32.f32 %0, %1, %2;" : "=f"(p0) : "f"(b), "f"(a));
                asm volatile("set.gtu.f32.f32 %0, %1, %2;" : "=f"(p1) : "f"(x), "f"(r));
                a = r;
                b = fmaf(fmaf(b, p0, -1.0f), p1, -1.0f);
            } else if (MODE == 14) {  // chain_pair_x2 (4 columns: 2 chains x 2 groups)
                uint64_t xa = ((uint64_t)__float_as_uint(x + e) << 32) | __float_as_uint(x - e);
                uint64_t xb = ((uint64_t)__float_as_uint(x * e) << 32) | __float_as_uint(x + 2 * e);
                mpk::tcdev::chain_pair_x2(xa, xb, v[e & 7], v[(e + 1) & 7],
                                          *reinterpret_cast<uint64_t*>(&s[(e & 3) * 2]),
                                          0xBF800000BF800000ull);
            } else if (MODE == 5) {   // SEL int
                int ia = __float_as_int(a), ib = __float_as_int(b);
                ia = (ia & 1) ? ib : ia;
                a = __int_as_float(ia + 1);
            }
        }
        x += 1e-7f;
    }
    const unsigned long long t1 = clock64();
    float acc = 0.f;
    for (int c = 0; c < 8; ++c) acc += v[c] + s[c];
    sink[blockIdx.x * 256 + threadIdx.x] = acc;
    if (lane == 0) atomicAdd(out, t1 - t0);
}

template <int MODE>
void run(const char* name) {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 8);
    cudaMalloc(&sink, 148 * 256 * 4);
    cudaMemset(d, 0, 8);
    const int iters = 4000;
    k<MODE><<<148, 256>>>(iters, d, sink);
    cudaDeviceSynchronize();
    unsigned long long cyc;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %.2f cycles per warp-iteration-element (2 warps/SMSP)\n", name,
           (double)cyc / (148.0 * 8) / (iters * 32.0));
    cudaFree(d);
    cudaFree(sink);
}

int main() {
    run<0>("FADD + FMNMX");
    run<1>("FSET.BF");
    run<2>("FFMA imm");
    run<3>("FSETP + FSEL + FADD");
    run<4>("FMNMX + FMNMX");
    run<5>("LOP/SEL/IADD int");
    run<6>("FSET + FMNMX + FADD");
    run<7>("FSET + FMNMX + FMNMX");
    run<8>("FFMA2 (per 2 fp32)");
    run<9>("FFMA2 + 2 FMNMX");
    run<10>("FFMA imm + FADD + 2 FMNMX");
    run<11>("chain_step_x2 (2 columns)");
    run<12>("FMNMX3");
    run<13>("FMNMX3 + 2 FSET + 2 FFMA");
    run<14>("chain_pair_x2 (4 columns)");
    return 0;
}
