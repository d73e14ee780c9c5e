// fold_bench.cu — the pair kernel's fold (fold32_x2 / fold32) in isolation: 8 warps per SM
// (2 per SM sub-partition), register "accumulators", ||c||^2 from shared memory as in the
// kernel. Cycles per 32-column chunk per warp vs the alu-pipe model (64 alu ops x 2 = 128).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_12208_b200/csrc \
//        -o tools/fold_bench tools/fold_bench.cu
#include <cstdio>
#include "common.cuh"
#include "tc_common.cuh"

using namespace mpk::tcdev;

// Variants of fold_rev_m3 for the pipe-mix experiments: XP / SP = packed (FFMA2) or scalar
// (FFMA) value / offset updates; LDS = ||c||^2 from shared memory (else registers).
template <bool XP, bool SP, bool LDS>
__device__ __forceinline__ void fold_var(const uint32_t (&v)[32], const float* cn_s, int j0,
                                         float (&cv)[NCH], uint64_t (&s2)[NCH / 2], float creg) {
    const uint64_t m1 = pack2(-1.0f, -1.0f);
    const uint64_t mm = pack2(-2.0f, -2.0f);
    const uint32_t cn_a = smem_u32(cn_s + j0);
#pragma unroll
    for (int gp = 1; gp >= 0; --gp) {
        float x[2][8];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int g = 2 * gp + 1 - h;
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
                const int col = 8 * g + 4 * qq;
                float4 cc = make_float4(creg, creg + 1.f, creg + 2.f, creg + 3.f);
                if (LDS) cc = lds_f4(cn_a + 4 * col);
                if (XP) {
                    uint64_t a = fma2(pack2u(v[col + 0], v[col + 1]), mm, pack2(cc.x, cc.y));
                    uint64_t b = fma2(pack2u(v[col + 2], v[col + 3]), mm, pack2(cc.z, cc.w));
                    unpack2(a, x[h][4 * qq + 0], x[h][4 * qq + 1]);
                    unpack2(b, x[h][4 * qq + 2], x[h][4 * qq + 3]);
                } else {
                    x[h][4 * qq + 0] = fmaf(__uint_as_float(v[col + 0]), -2.f, cc.x);
                    x[h][4 * qq + 1] = fmaf(__uint_as_float(v[col + 1]), -2.f, cc.y);
                    x[h][4 * qq + 2] = fmaf(__uint_as_float(v[col + 2]), -2.f, cc.z);
                    x[h][4 * qq + 3] = fmaf(__uint_as_float(v[col + 3]), -2.f, cc.w);
                }
            }
        }
#pragma unroll
        for (int m = 0; m < NCH / 2; ++m) {
            if (SP) {
                chain_pair_x2(pack2(x[0][2 * m], x[0][2 * m + 1]), pack2(x[1][2 * m], x[1][2 * m + 1]),
                              cv[2 * m], cv[2 * m + 1], s2[m], m1);
            } else {
                float lo, hi;
                unpack2(s2[m], lo, hi);
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int c = 2 * m + u;
                    float& s = u ? hi : lo;
                    float w, na, nb;
                    asm("min.f32 %0, %1, %2, %3;" : "=f"(w) : "f"(cv[c]), "f"(x[0][c]), "f"(x[1][c]));
                    asm("set.gtu.f32.f32 %0, %1, %2;" : "=f"(na) : "f"(x[0][c]), "f"(cv[c]));
                    asm("set.gtu.f32.f32 %0, %1, %2;" : "=f"(nb) : "f"(x[1][c]), "f"(w));
                    cv[c] = w;
                    s = fmaf(fmaf(s, na, -1.f), nb, -1.f);
                }
                s2[m] = pack2(lo, hi);
            }
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned long long* out, float* sink) {
    __shared__ __align__(16) float cn_s[1024];
    for (int j = threadIdx.x; j < 1024; j += blockDim.x) cn_s[j] = 0.5f * j;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t va[32], vb[32];
    for (int e = 0; e < 32; ++e) { va[e] = __float_as_uint(lane * 0.25f + e); vb[e] = va[e] ^ 3; }
    float cv[NCH], cs[NCH], c2[NCH], cv2[NCH], cs2_[NCH], c22[NCH];
    chains_init(cv, cs, c2);
    chains_init(cv2, cs2_, c22);
    uint64_t s2[NCH / 2], s22[NCH / 2];
    for (int m = 0; m < NCH / 2; ++m) { s2[m] = pack2(-1.f, -1.f); s22[m] = s2[m]; }
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const int j0 = (i * 32) & 1023;
        if (MODE == 0 || MODE == 2) fold32_x2<false>(va, cn_s, cn_s, -2.f, j0, cv, s2);
        else if (MODE == 1) fold32<false, false>(va, cn_s, cn_s, -2.f, j0, cv, cs, c2);
        else if (MODE == 4) fold_rev_m3<4, false>(va, cn_s, cn_s, -2.f, j0, cv, s2);
        else if (MODE == 5) fold_var<true, true, false>(va, cn_s, j0, cv, s2, (float)i);
        else if (MODE == 6) fold_var<false, true, true>(va, cn_s, j0, cv, s2, 0.f);
        else if (MODE == 7) fold_var<true, false, true>(va, cn_s, j0, cv, s2, 0.f);
        else if (MODE == 8) fold_var<false, false, true>(va, cn_s, j0, cv, s2, 0.f);
        else if (MODE == 9) fold_var<false, false, false>(va, cn_s, j0, cv, s2, (float)i);
        else {   // MODE 3: two chunks interleaved into two independent chain sets
            fold32_x2<false>(va, cn_s, cn_s, -2.f, j0, cv, s2);
            fold32_x2<false>(vb, cn_s, cn_s, -2.f, (j0 + 32) & 1023, cv2, s22);
            ++i;
        }
        va[0] ^= (uint32_t)i; vb[1] ^= (uint32_t)i; va[17] += 1u; vb[29] += 3u;   // keep the data live / varying
    }
    const unsigned long long t1 = clock64();
    float acc = 0.f;
    for (int c = 0; c < NCH; ++c) acc += cv[c] + cs[c] + cv2[c];
    for (int m = 0; m < NCH / 2; ++m)   // both halves of the packed offsets stay live
        acc += __uint_as_float((uint32_t)s2[m]) + __uint_as_float((uint32_t)(s2[m] >> 32)) +
               __uint_as_float((uint32_t)s22[m]) + __uint_as_float((uint32_t)(s22[m] >> 32));
    sink[blockIdx.x * 512 + threadIdx.x] = acc;
    if (lane == 0) atomicAdd(out, t1 - t0);
}

template <int MODE>
void run(const char* nm, int threads = 256) {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 8);
    cudaMalloc(&sink, 148 * 512 * 4);
    cudaMemset(d, 0, 8);
    const int iters = 20000;
    k<MODE><<<148, threads>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double per_warp = (double)c / (148.0 * (threads / 32)) / iters;
    const double per_smsp_chunk = per_warp / ((threads / 32) / 4) / (MODE == 3 ? 2 : 1);
    printf("%-36s %.1f cycles per chunk per SMSP (alu floor 128)\n", nm, per_smsp_chunk);
}

int main() {
    run<0>("fold32_x2, 2 warps/SMSP");
    run<1>("fold32 scalar, 2 warps/SMSP");
    run<2>("fold32_x2, 4 warps/SMSP", 512);
    run<3>("fold32_x2 x2 interleaved, 2 warps/SMSP");
    run<4>("fold_rev_m3 (alu floor 96), 2 warps/SMSP");
    run<4>("fold_rev_m3, 4 warps/SMSP", 512);
    run<5>("rev: packed x, packed s, no LDS");
    run<6>("rev: scalar x, packed s, LDS");
    run<7>("rev: packed x, scalar s, LDS");
    run<8>("rev: scalar x, scalar s, LDS");
    run<9>("rev: scalar x, scalar s, no LDS");
    run<9>("rev: scalar x, scalar s, no LDS, 4 warps/SMSP", 512);
    return 0;
}
