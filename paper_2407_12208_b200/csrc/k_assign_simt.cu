// k_assign_simt.cu — CUDA-core distance + argmin kernels.
//
// K6  assign_simt: generic register-tiled kernel for every precision pair. The operands are the
//     stored low-precision values widened exactly to the accumulation type; the dot product
//     x~_i . c~_j accumulates in fp32 FMA for fp32/fp16/bf16/E5M2 operands (the tensor-core
//     model of reading Z2/Z3) and in fp64 for fp64 operands. Epilogue (working precision):
//         v_ij = fma(-2 s_i s_j, dot_ij, ||c_j||^2)        (eq:dist-eval, PAPER.md:193-196;
//                                                           Alg 4 line 6)
//     ||x_i||^2 is row-constant and is added only to the minimum (SSE_t). Running argmin over
//     j with (value, index) ordering: lowest j on ties, NaN never wins (readings Z12, Z13).
//     Also the final working-precision assignment (Alg 3 step 7).
// K5  smalld_fused: d <= 4, k <= 8 (image segmentation): one pass over X
//     in working precision per iteration computes x~ on the fly, assigns, and accumulates the
//     per-cluster sums in fp64 registers -> warp shuffles -> block smem -> one global fp64
//     atomic per (block, value): the update of eq:center fused in.
// K10 final_sse: sum_i ||x_i - c_{l_i}||^2 by the direct formula (eq:dist-eval-alternative,
//     PAPER.md:189-192) in fp64.
#include "common.cuh"
#include "internal.h"

#include <stdlib.h>

namespace mpk {

namespace {

constexpr int BM = 64, BN = 64, BK = 32, NT = 256;

template <typename LT, typename AT, typename W>
__global__ void __launch_bounds__(NT)
assign_simt_kernel(Problem p, const LT* __restrict__ Xl, const W* __restrict__ xn,
                   const W* __restrict__ sx, const LT* __restrict__ Cl,
                   const W* __restrict__ cn, const W* __restrict__ sc,
                   int32_t* __restrict__ labels, double* acc_sse, double* acc_changed,
                   const int* __restrict__ rows) {
    __shared__ AT Xs[BK][BM];
    __shared__ AT Cs[BK][BN];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t row0 = (int64_t)blockIdx.x * BM;

    W bestv[4];
    int bestj[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) { bestv[r] = (W)INFINITY; bestj[r] = 0; }
    W srow[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int64_t li = row0 + ty * 4 + r;   // list index; the row is rows[li] if listed
        const int64_t row = (rows && li < p.n) ? (int64_t)rows[li] : li;
        srow[r] = (p.guard && sx && li < p.n) ? sx[row] : (W)1;
    }

    for (int n0 = 0; n0 < p.k; n0 += BN) {
        AT acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[r][c] = (AT)0;
        for (int k0 = 0; k0 < p.d; k0 += BK) {
#pragma unroll
            for (int e = 0; e < (BM * BK) / NT; ++e) {
                int idx = tid + e * NT;
                int r = idx / BK, kk = idx % BK;
                const int64_t li = row0 + r;
                int col = k0 + kk;
                AT v = (AT)0;
                if (li < p.n && col < p.d) {
                    const int64_t row = rows ? (int64_t)rows[li] : li;
                    v = (AT)widen(Xl[row * p.d_pad + col]);
                }
                Xs[kk][r] = v;
                int cj = n0 + r;
                AT w = (AT)0;
                if (cj < p.k && col < p.d) w = (AT)widen(Cl[(int64_t)cj * p.d_pad + col]);
                Cs[kk][r] = w;
            }
            __syncthreads();
#pragma unroll 8
            for (int kk = 0; kk < BK; ++kk) {
                AT a[4], b[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) a[r] = Xs[kk][ty * 4 + r];
#pragma unroll
                for (int c = 0; c < 4; ++c) b[c] = Cs[kk][tx * 4 + c];
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
            }
            __syncthreads();
        }
        // epilogue for this centroid tile: ascending j per thread
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            int j = n0 + tx * 4 + c;
            if (j < p.k) {
                W cnj = cn[j];
                W scj = (p.guard && sc) ? sc[j] : (W)1;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    W m2 = (W)-2 * (srow[r] * scj);
                    W v = fma(m2, (W)acc[r][c], cnj);
                    if (v < bestv[r]) { bestv[r] = v; bestj[r] = j; }
                }
            }
        }
    }
    // reduce across the 16 threads (tx) that share rows: lanes ty*16 .. ty*16+15
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            W v2 = __shfl_xor_sync(0xffffffffu, bestv[r], o);
            int j2 = __shfl_xor_sync(0xffffffffu, bestj[r], o);
            argmin_merge(bestv[r], bestj[r], v2, j2);
        }
    }
    double my_sse = 0.0, my_changed = 0.0;
    if (tx == 0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t li = row0 + ty * 4 + r;
            if (li < p.n) {
                const int64_t row = rows ? (int64_t)rows[li] : li;
                if (acc_changed && labels[row] != bestj[r]) my_changed += 1.0;
                labels[row] = bestj[r];
                if (acc_sse) {
                    double md = (double)xn[row] + (double)bestv[r];
                    my_sse += md > 0.0 ? md : 0.0;
                }
            }
        }
    }
    if (acc_sse || acc_changed) {
        my_sse = warp_sum(my_sse);
        my_changed = warp_sum(my_changed);
        __shared__ double red[2][NT / 32];
        if ((tid & 31) == 0) { red[0][tid >> 5] = my_sse; red[1][tid >> 5] = my_changed; }
        __syncthreads();
        if (tid == 0) {
            double a = 0, b = 0;
            for (int w = 0; w < NT / 32; ++w) { a += red[0][w]; b += red[1][w]; }
            if (acc_sse) atomicAdd(acc_sse, a);
            if (acc_changed && b != 0.0) atomicAdd(acc_changed, b);
        }
    }
}

// ------------------------------------------------------------------------------------------
// K6m: Alg 4's per-pair precision switch (Alg 5 step 3). For each pair
// the condition eq:prec-delta is evaluated division-free in fp64,
//     max(xn_i, cn_j) >= delta^2 min(xn_i, cn_j)           (reading R5, same as oracle O4m),
// and the distance is the scaled low-precision value when it holds (Alg 4 lines 1-6: the dot of
// the stored low operands, fp32 accumulation, v = fma(-2 s_i s_j, dot, cn_j)) and the
// working-precision value otherwise (line 8: the dot of the working operands accumulated in
// the working precision, v = fma(-2, dot, cn_j)). Both dot products are formed for every pair
// (CUDA cores; the tensor-core variant is future work); triggered pairs are
// counted (eq:xi-low-prec-ratio). Same argmin / SSE / changed bookkeeping as K6.
// ------------------------------------------------------------------------------------------
constexpr int MBK = 16;

template <typename LT, typename W>
__global__ void __launch_bounds__(NT)
assign_mixed_kernel(Problem p, double delta2, const LT* __restrict__ Xl,
                    const W* __restrict__ Xw, const W* __restrict__ xn,
                    const W* __restrict__ sx, const LT* __restrict__ Cl,
                    const W* __restrict__ Cw, const W* __restrict__ cn,
                    const W* __restrict__ sc, int32_t* __restrict__ labels, double* acc_sse,
                    double* acc_changed, unsigned long long* n_low) {
    __shared__ float Xs[MBK][BM];
    __shared__ float Cs[MBK][BN];
    __shared__ W Xws[MBK][BM];
    __shared__ W Cws[MBK][BN];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t row0 = (int64_t)blockIdx.x * BM;

    W bestv[4];
    int bestj[4];
    W srow[4], xrow[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        bestv[r] = (W)INFINITY;
        bestj[r] = 0;
        const int64_t row = row0 + ty * 4 + r;
        srow[r] = (sx && row < p.n) ? sx[row] : (W)1;
        xrow[r] = row < p.n ? xn[row] : (W)0;
    }
    unsigned long long trig_count = 0;

    for (int n0 = 0; n0 < p.k; n0 += BN) {
        float acc[4][4];
        W accw[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) { acc[r][c] = 0.0f; accw[r][c] = (W)0; }
        for (int k0 = 0; k0 < p.d; k0 += MBK) {
#pragma unroll
            for (int e = 0; e < (BM * MBK) / NT; ++e) {
                const int idx = tid + e * NT;
                const int r = idx / MBK, kk = idx % MBK;
                const int64_t row = row0 + r;
                const int col = k0 + kk;
                float v = 0.0f;
                W vw = (W)0;
                if (row < p.n && col < p.d) {
                    v = (float)widen(Xl[row * p.d_pad + col]);
                    vw = Xw[row * p.d + col];
                }
                Xs[kk][r] = v;
                Xws[kk][r] = vw;
                const int cj = n0 + r;
                float w = 0.0f;
                W ww = (W)0;
                if (cj < p.k && col < p.d) {
                    w = (float)widen(Cl[(int64_t)cj * p.d_pad + col]);
                    ww = Cw[(int64_t)cj * p.d + col];
                }
                Cs[kk][r] = w;
                Cws[kk][r] = ww;
            }
            __syncthreads();
#pragma unroll 4
            for (int kk = 0; kk < MBK; ++kk) {
                float a[4], b[4];
                W aw[4], bw[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) { a[r] = Xs[kk][ty * 4 + r]; aw[r] = Xws[kk][ty * 4 + r]; }
#pragma unroll
                for (int c = 0; c < 4; ++c) { b[c] = Cs[kk][tx * 4 + c]; bw[c] = Cws[kk][tx * 4 + c]; }
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
                        accw[r][c] = fma(aw[r], bw[c], accw[r][c]);
                    }
            }
            __syncthreads();
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int j = n0 + tx * 4 + c;
            if (j < p.k) {
                const W cnj = cn[j];
                const W scj = sc ? sc[j] : (W)1;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (row0 + ty * 4 + r >= p.n) continue;
                    const double a = (double)xrow[r], b = (double)cnj;
                    const double mx = (a > b) ? a : b, mn = (a > b) ? b : a;
                    const bool trig = mx >= delta2 * mn;
                    W v;
                    if (trig) {
                        v = fma((W)-2 * (srow[r] * scj), (W)acc[r][c], cnj);
                        ++trig_count;
                    } else {
                        v = fma((W)-2, accw[r][c], cnj);
                    }
                    if (v < bestv[r]) { bestv[r] = v; bestj[r] = j; }
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            const W v2 = __shfl_xor_sync(0xffffffffu, bestv[r], o);
            const int j2 = __shfl_xor_sync(0xffffffffu, bestj[r], o);
            argmin_merge(bestv[r], bestj[r], v2, j2);
        }
    }
    double my_sse = 0.0, my_changed = 0.0;
    if (tx == 0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t row = row0 + ty * 4 + r;
            if (row < p.n) {
                if (acc_changed && labels[row] != bestj[r]) my_changed += 1.0;
                labels[row] = bestj[r];
                if (acc_sse) {
                    const double md = (double)xn[row] + (double)bestv[r];
                    my_sse += md > 0.0 ? md : 0.0;
                }
            }
        }
    }
    my_sse = warp_sum(my_sse);
    my_changed = warp_sum(my_changed);
    trig_count = warp_sum(trig_count);
    __shared__ double red[2][NT / 32];
    __shared__ unsigned long long redt[NT / 32];
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = my_sse;
        red[1][tid >> 5] = my_changed;
        redt[tid >> 5] = trig_count;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0, b = 0;
        unsigned long long t = 0;
        for (int w = 0; w < NT / 32; ++w) { a += red[0][w]; b += red[1][w]; t += redt[w]; }
        if (acc_sse) atomicAdd(acc_sse, a);
        if (acc_changed && b != 0.0) atomicAdd(acc_changed, b);
        if (n_low && t) atomicAdd(n_low, t);
    }
}

template <typename LT, typename W>
static cudaError_t mixed_launch(const Problem& p, double delta2, const void* Xl, const void* Xw,
                                const void* xn, const void* sx, const void* Cl, const void* Cw,
                                const void* cn, const void* sc, int32_t* labels,
                                double* acc_sse, double* acc_changed, unsigned long long* n_low,
                                cudaStream_t s) {
    const int64_t blocks = (p.n + BM - 1) / BM;
    assign_mixed_kernel<LT, W><<<(unsigned)blocks, NT, 0, s>>>(
        p, delta2, (const LT*)Xl, (const W*)Xw, (const W*)xn, (const W*)sx, (const LT*)Cl,
        (const W*)Cw, (const W*)cn, (const W*)sc, labels, acc_sse, acc_changed, n_low);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K6b: register-tiled (8 x 8 per thread, 128 x 128 per block) CUDA-core variant for fp32
// accumulation — the fp32 working mode and the final pass's CUDA-core rows. Same arithmetic as
// K6: products summed in order t = 0..d-1 by fp32 FMA, v = fma(-2 s_i s_j, dot, ||c_j||^2),
// (value, index) argmin with lowest index on ties.
// ------------------------------------------------------------------------------------------
constexpr int B2M = 128, B2N = 128, B2K = 16, B2T = 256;

template <typename LT, typename W>
__global__ void __launch_bounds__(B2T)
assign_simt_big_kernel(Problem p, const LT* __restrict__ Xl, const W* __restrict__ xn,
                       const W* __restrict__ sx, const LT* __restrict__ Cl,
                       const W* __restrict__ cn, const W* __restrict__ sc,
                       int32_t* __restrict__ labels, double* acc_sse, double* acc_changed,
                       const int* __restrict__ rows) {
    __shared__ __align__(16) float As[B2K][B2M + 4];
    __shared__ __align__(16) float Bs[B2K][B2N + 4];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t row0 = (int64_t)blockIdx.x * B2M;

    float bestv[8];
    int bestj[8];
    W srow[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        bestv[r] = INFINITY;
        bestj[r] = 0;
        const int64_t li = row0 + ty * 8 + r;
        const int64_t row = (rows && li < p.n) ? (int64_t)rows[li] : li;
        srow[r] = (p.guard && sx && li < p.n) ? sx[row] : (W)1;
    }
    // source rows of this block's A tile (each thread loads rows tid/16 + 16 e, column tid%16)
    int64_t arow[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int64_t li = row0 + (tid >> 4) + 16 * e;
        arow[e] = li < p.n ? (rows ? (int64_t)rows[li] : li) : -1;
    }
    for (int n0 = 0; n0 < p.k; n0 += B2N) {
        float acc[8][8];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[r][c] = 0.0f;
        for (int k0 = 0; k0 < p.d; k0 += B2K) {
            const int kk = tid & 15;
            const int col = k0 + kk;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int r = (tid >> 4) + 16 * e;
                As[kk][r] = (arow[e] >= 0 && col < p.d) ? (float)widen(Xl[arow[e] * p.d_pad + col]) : 0.0f;
                const int cj = n0 + r;
                Bs[kk][r] = (cj < p.k && col < p.d) ? (float)widen(Cl[(int64_t)cj * p.d_pad + col]) : 0.0f;
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < B2K; ++q) {
                const float4 a0 = *reinterpret_cast<const float4*>(&As[q][ty * 8]);
                const float4 a1 = *reinterpret_cast<const float4*>(&As[q][ty * 8 + 4]);
                const float4 b0 = *reinterpret_cast<const float4*>(&Bs[q][tx * 8]);
                const float4 b1 = *reinterpret_cast<const float4*>(&Bs[q][tx * 8 + 4]);
                const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int r = 0; r < 8; ++r)
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int j = n0 + tx * 8 + c;
            if (j < p.k) {
                const W cnj = cn[j];
                const W scj = (p.guard && sc) ? sc[j] : (W)1;
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const W m2 = (W)-2 * (srow[r] * scj);
                    const float v = (float)fma(m2, (W)acc[r][c], cnj);
                    if (v < bestv[r]) { bestv[r] = v; bestj[r] = j; }
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            const float v2 = __shfl_xor_sync(0xffffffffu, bestv[r], o);
            const int j2 = __shfl_xor_sync(0xffffffffu, bestj[r], o);
            argmin_merge(bestv[r], bestj[r], v2, j2);
        }
    }
    double my_sse = 0.0, my_changed = 0.0;
    if (tx == 0) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int64_t li = row0 + ty * 8 + r;
            if (li < p.n) {
                const int64_t row = rows ? (int64_t)rows[li] : li;
                if (acc_changed && labels[row] != bestj[r]) my_changed += 1.0;
                labels[row] = bestj[r];
                if (acc_sse) {
                    const double md = (double)xn[row] + (double)bestv[r];
                    my_sse += md > 0.0 ? md : 0.0;
                }
            }
        }
    }
    if (acc_sse || acc_changed) {
        my_sse = warp_sum(my_sse);
        my_changed = warp_sum(my_changed);
        __shared__ double red[2][B2T / 32];
        if ((tid & 31) == 0) { red[0][tid >> 5] = my_sse; red[1][tid >> 5] = my_changed; }
        __syncthreads();
        if (tid == 0) {
            double a = 0, b = 0;
            for (int w = 0; w < B2T / 32; ++w) { a += red[0][w]; b += red[1][w]; }
            if (acc_sse) atomicAdd(acc_sse, a);
            if (acc_changed && b != 0.0) atomicAdd(acc_changed, b);
        }
    }
}

// ------------------------------------------------------------------------------------------
// K6b for d <= 4 (the image rows; the final pass of the small-d loop): one
// row per thread, the centres in shared memory. K6b's 128 x 128 tile left almost every lane
// idle at d = 3, k = 6. Same arithmetic per value as K6b: dot = fma over t = 0..d-1 from 0
// (K6b's zero-padded columns add exact zeros), v = fma(-2 (s_i s_j), dot, ||c_j||^2), and the
// ascending-j scan with strict < gives K6b's (value, index) minimum, lowest index on ties.
// ------------------------------------------------------------------------------------------
constexpr int kSmallK = 256;

template <typename LT, typename W, int D>
__global__ void __launch_bounds__(256)
assign_simt_small_kernel(Problem p, const LT* __restrict__ Xl, const W* __restrict__ xn,
                         const W* __restrict__ sx, const LT* __restrict__ Cl,
                         const W* __restrict__ cn, const W* __restrict__ sc,
                         int32_t* __restrict__ labels, double* acc_sse, double* acc_changed,
                         const int* __restrict__ rows) {
    __shared__ float Cs[kSmallK][D];
    __shared__ W cns[kSmallK], scs[kSmallK];
    for (int j = threadIdx.x; j < p.k; j += blockDim.x) {
#pragma unroll
        for (int t = 0; t < D; ++t) Cs[j][t] = (float)widen(Cl[(int64_t)j * p.d_pad + t]);
        cns[j] = cn[j];
        scs[j] = (p.guard && sc) ? sc[j] : (W)1;
    }
    __syncthreads();
    double my_sse = 0.0, my_changed = 0.0;
    for (int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; li < p.n;
         li += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = rows ? (int64_t)rows[li] : li;
        float x[D];
#pragma unroll
        for (int t = 0; t < D; ++t) x[t] = (float)widen(Xl[row * p.d_pad + t]);
        const W srow = (p.guard && sx) ? sx[row] : (W)1;
        float bestv = INFINITY;
        int bestj = 0;
        for (int j = 0; j < p.k; ++j) {
            float dot = 0.0f;
#pragma unroll
            for (int t = 0; t < D; ++t) dot = fmaf(x[t], Cs[j][t], dot);
            const W m2 = (W)-2 * (srow * scs[j]);
            const float v = (float)fma(m2, (W)dot, cns[j]);
            if (v < bestv) { bestv = v; bestj = j; }
        }
        if (acc_changed && labels[row] != bestj) my_changed += 1.0;
        labels[row] = bestj;
        if (acc_sse) {
            const double md = (double)xn[row] + (double)bestv;
            my_sse += md > 0.0 ? md : 0.0;
        }
    }
    if (acc_sse || acc_changed) {
        my_sse = warp_sum(my_sse);
        my_changed = warp_sum(my_changed);
        __shared__ double red[2][8];
        const int tid = threadIdx.x;
        if ((tid & 31) == 0) { red[0][tid >> 5] = my_sse; red[1][tid >> 5] = my_changed; }
        __syncthreads();
        if (tid == 0) {
            double a = 0, b = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a += red[0][w]; b += red[1][w]; }
            if (acc_sse) atomicAdd(acc_sse, a);
            if (acc_changed && b != 0.0) atomicAdd(acc_changed, b);
        }
    }
}

// ------------------------------------------------------------------------------------------
// K6m-b: Alg 4's per-pair precision switch for fp32 work on K6b's 128 x 128 tiles (8 x 8 per
// thread). Per centroid tile, the rows' and columns' norm ranges classify the tile in fp64
// (monotone, so the classification agrees with every per-pair decision):
//   no pair triggered   <=  xmax < d2 cmin  and  cmax < d2 xmin
//   every pair triggered <= xmin >= d2 cmax  or   cmin >= d2 xmax
// and only the dot products a tile needs are formed (z-scored data at delta = 2 is almost
// entirely "no pair triggered": one fp32 GEMM instead of two). A mixed tile runs the low
// GEMM (triggered pairs) and then the working GEMM (the others); the argmin merges by (value,
// index), so the result equals K6m's ascending-j scan. Same arithmetic per value as K6m:
// dot products accumulated t = 0..d-1 by fp32 FMA, v = fma(-2 s_i s_j, dot_l, cn_j) or
// fma(-2, dot_w, cn_j).
// ------------------------------------------------------------------------------------------
template <typename LT, bool LOWP>
MPK_DEV void mixed_tile_gemm(const Problem& p, const void* __restrict__ Xsrc,
                             const void* __restrict__ Csrc, int64_t row0, int n0, int tid,
                             int tx, int ty, const int64_t (&arow)[8], float (&As)[B2K][B2M + 4],
                             float (&Bs)[B2K][B2N + 4], float (&acc)[8][8]) {
    const int stride = LOWP ? p.d_pad : p.d;
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = 0.0f;
    for (int k0 = 0; k0 < p.d; k0 += B2K) {
        const int kk = tid & 15;
        const int col = k0 + kk;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int r = (tid >> 4) + 16 * e;
            float a = 0.0f, b = 0.0f;
            if (arow[e] >= 0 && col < p.d) {
                a = LOWP ? (float)widen(((const LT*)Xsrc)[arow[e] * stride + col])
                         : ((const float*)Xsrc)[arow[e] * stride + col];
            }
            const int cj = n0 + r;
            if (cj < p.k && col < p.d) {
                b = LOWP ? (float)widen(((const LT*)Csrc)[(int64_t)cj * stride + col])
                         : ((const float*)Csrc)[(int64_t)cj * stride + col];
            }
            As[kk][r] = a;
            Bs[kk][r] = b;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < B2K; ++q) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[q][ty * 8]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[q][ty * 8 + 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[q][tx * 8]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[q][tx * 8 + 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
        }
        __syncthreads();
    }
}

#ifndef MPK_MIXB_MINB
#define MPK_MIXB_MINB 2
#endif
template <typename LT>
__global__ void __launch_bounds__(B2T, MPK_MIXB_MINB)
assign_mixed_big_kernel(Problem p, double delta2, const LT* __restrict__ Xl,
                        const float* __restrict__ Xw, const float* __restrict__ xn,
                        const float* __restrict__ sx, const LT* __restrict__ Cl,
                        const float* __restrict__ Cw, const float* __restrict__ cn,
                        const float* __restrict__ sc, int32_t* __restrict__ labels,
                        double* acc_sse, double* acc_changed, unsigned long long* n_low) {
    __shared__ __align__(16) float As[B2K][B2M + 4];
    __shared__ __align__(16) float Bs[B2K][B2N + 4];
    __shared__ float red_f[4][B2T / 32];
    __shared__ int red_nan[B2T / 32];
    __shared__ float tile_rng[6];   // xmin, xmax, cmin, cmax, row-NaN, col-NaN
    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t row0 = (int64_t)blockIdx.x * B2M;

    float bestv[8], srow[8], xrow[8];
    int bestj[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int64_t row = row0 + ty * 8 + r;
        bestv[r] = INFINITY;
        bestj[r] = 0;
        srow[r] = (sx && row < p.n) ? sx[row] : 1.0f;
        xrow[r] = row < p.n ? xn[row] : 0.0f;
    }
    int64_t arow[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int64_t li = row0 + (tid >> 4) + 16 * e;
        arow[e] = li < p.n ? li : -1;
    }
    // row norm range of this block (thread t < 128 owns row t)
    {
        float lo = INFINITY, hi = -INFINITY;
        int nan = 0;
        if (tid < B2M && row0 + tid < p.n) {
            const float v = xn[row0 + tid];
            if (isnan(v)) nan = 1;
            else { lo = v; hi = v; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
            nan |= __shfl_xor_sync(0xffffffffu, nan, o);
        }
        if (lane == 0) { red_f[0][wid] = lo; red_f[1][wid] = hi; red_nan[wid] = nan; }
        __syncthreads();
        if (tid == 0) {
            float a = INFINITY, b = -INFINITY;
            int c = 0;
            for (int w = 0; w < B2T / 32; ++w) { a = fminf(a, red_f[0][w]); b = fmaxf(b, red_f[1][w]); c |= red_nan[w]; }
            tile_rng[0] = a; tile_rng[1] = b; tile_rng[4] = (float)c;
        }
        __syncthreads();
    }
    const double xmin = tile_rng[0], xmax = tile_rng[1];
    const bool row_nan = tile_rng[4] != 0.0f;
    unsigned long long trig_count = 0;
    float acc[8][8];

    for (int n0 = 0; n0 < p.k; n0 += B2N) {
        // column norm range of this centroid tile
        {
            float lo = INFINITY, hi = -INFINITY;
            int nan = 0;
            if (tid < B2N && n0 + tid < p.k) {
                const float v = cn[n0 + tid];
                if (isnan(v)) nan = 1;
                else { lo = v; hi = v; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
                hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
                nan |= __shfl_xor_sync(0xffffffffu, nan, o);
            }
            if (lane == 0) { red_f[2][wid] = lo; red_f[3][wid] = hi; red_nan[wid] = nan; }
            __syncthreads();
            if (tid == 0) {
                float a = INFINITY, b = -INFINITY;
                int c = 0;
                for (int w = 0; w < B2T / 32; ++w) { a = fminf(a, red_f[2][w]); b = fmaxf(b, red_f[3][w]); c |= red_nan[w]; }
                tile_rng[2] = a; tile_rng[3] = b; tile_rng[5] = (float)c;
            }
            __syncthreads();
        }
        const double cmin = tile_rng[2], cmax = tile_rng[3];
        const bool any_nan = row_nan || tile_rng[5] != 0.0f;
        const bool none_trig = !any_nan && xmax < delta2 * cmin && cmax < delta2 * xmin;
        const bool all_trig = !any_nan && (xmin >= delta2 * cmax || cmin >= delta2 * xmax);
        __syncthreads();   // tile_rng is rewritten by the next tile
        for (int phase = 0; phase < 2; ++phase) {
            const bool low = phase == 0;
            if (low && none_trig) continue;
            if (!low && all_trig) continue;
            if (low) mixed_tile_gemm<LT, true>(p, Xl, Cl, row0, n0, tid, tx, ty, arow, As, Bs, acc);
            else mixed_tile_gemm<LT, false>(p, Xw, Cw, row0, n0, tid, tx, ty, arow, As, Bs, acc);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int j = n0 + tx * 8 + c;
                if (j >= p.k) continue;
                const float cnj = cn[j];
                const float scj = sc ? sc[j] : 1.0f;
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    if (row0 + ty * 8 + r >= p.n) continue;
                    bool trig;
                    if (all_trig) trig = true;
                    else if (none_trig) trig = false;
                    else {
                        const double a = (double)xrow[r], b = (double)cnj;
                        const double mx = (a > b) ? a : b, mn = (a > b) ? b : a;
                        trig = mx >= delta2 * mn;
                    }
                    if (trig != low) continue;
                    float v;
                    if (low) {
                        v = fmaf(-2.0f * (srow[r] * scj), acc[r][c], cnj);
                        ++trig_count;
                    } else {
                        v = fmaf(-2.0f, acc[r][c], cnj);
                    }
                    argmin_merge(bestv[r], bestj[r], v, j);
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            const float v2 = __shfl_xor_sync(0xffffffffu, bestv[r], o);
            const int j2 = __shfl_xor_sync(0xffffffffu, bestj[r], o);
            argmin_merge(bestv[r], bestj[r], v2, j2);
        }
    }
    double my_sse = 0.0, my_changed = 0.0;
    if (tx == 0) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int64_t row = row0 + ty * 8 + r;
            if (row < p.n) {
                // an all-NaN/+inf row keeps label 0 (bestj stays 0)
                if (acc_changed && labels[row] != bestj[r]) my_changed += 1.0;
                labels[row] = bestj[r];
                if (acc_sse) {
                    const double md = (double)xn[row] + (double)bestv[r];
                    my_sse += md > 0.0 ? md : 0.0;
                }
            }
        }
    }
    my_sse = warp_sum(my_sse);
    my_changed = warp_sum(my_changed);
    trig_count = warp_sum(trig_count);
    __shared__ double red[2][B2T / 32];
    __shared__ unsigned long long redt[B2T / 32];
    if (lane == 0) { red[0][wid] = my_sse; red[1][wid] = my_changed; redt[wid] = trig_count; }
    __syncthreads();
    if (tid == 0) {
        double a = 0, b = 0;
        unsigned long long t = 0;
        for (int w = 0; w < B2T / 32; ++w) { a += red[0][w]; b += red[1][w]; t += redt[w]; }
        if (acc_sse) atomicAdd(acc_sse, a);
        if (acc_changed && b != 0.0) atomicAdd(acc_changed, b);
        if (n_low && t) atomicAdd(n_low, t);
    }
}

// ------------------------------------------------------------------------------------------
// K5 small-d fused assign + update.
// ------------------------------------------------------------------------------------------
constexpr int SD_D = 4, SD_K = 8, SD_T = 256;

template <typename W, int DIST>
__global__ void __launch_bounds__(SD_T)
smalld_kernel(Problem p, const W* __restrict__ X, const typename low_type<DIST>::T* __restrict__ Cl,
              const W* __restrict__ cn, const W* __restrict__ sc, int32_t* __restrict__ labels,
              double* __restrict__ acc, AccLayout L) {
    using AT = typename std::conditional<DIST == KMEANS_FP64, double, float>::type;
    constexpr int WORK = sizeof(W) == 8 ? KMEANS_FP64 : KMEANS_FP32;
    constexpr bool same = (DIST == WORK);
    __shared__ AT cl_s[SD_K][SD_D];
    __shared__ W cn_s[SD_K], sc_s[SD_K];
    const int tid = threadIdx.x;
    if (tid < SD_K * SD_D) {
        int j = tid / SD_D, t = tid % SD_D;
        cl_s[j][t] = (j < p.k && t < p.d) ? (AT)widen(Cl[(int64_t)j * p.d_pad + t]) : (AT)0;
    }
    if (tid < SD_K) {
        cn_s[tid] = tid < p.k ? cn[tid] : (W)0;
        sc_s[tid] = (tid < p.k && p.guard && sc) ? sc[tid] : (W)1;
    }
    __syncthreads();

    double sums[SD_K][SD_D];
    double cnts[SD_K];
#pragma unroll
    for (int j = 0; j < SD_K; ++j) {
        cnts[j] = 0.0;
#pragma unroll
        for (int t = 0; t < SD_D; ++t) sums[j][t] = 0.0;
    }
    double my_sse = 0.0, my_changed = 0.0;

    for (int64_t i = (int64_t)blockIdx.x * SD_T + tid; i < p.n; i += (int64_t)gridDim.x * SD_T) {
        W x[SD_D];
        double nrm = 0.0, amax = 0.0;
#pragma unroll
        for (int t = 0; t < SD_D; ++t) {
            x[t] = t < p.d ? X[i * p.d + t] : (W)0;
            double v = (double)x[t];
            nrm = __dadd_rn(nrm, __dmul_rn(v, v));
            amax = fmax(amax, fabs(v));
        }
        W xn = rounder<WORK>::from(nrm);
        W s = (W)1;
        if (p.guard && !same) s = (W)guard_scale((W)amax, p.guard);
        AT xl[SD_D];
#pragma unroll
        for (int t = 0; t < SD_D; ++t) {
            W q = (s == (W)1) ? x[t] : x[t] / s;
            xl[t] = (AT)widen(rounder<DIST>::from(q));
        }
        W best = (W)INFINITY;
        int bj = 0;
#pragma unroll
        for (int j = 0; j < SD_K; ++j) {
            if (j < p.k) {
                AT dot = (AT)0;
#pragma unroll
                for (int t = 0; t < SD_D; ++t) dot = fma(xl[t], cl_s[j][t], dot);
                W v = fma((W)-2 * (s * sc_s[j]), (W)dot, cn_s[j]);
                if (v < best) { best = v; bj = j; }
            }
        }
        if (labels[i] != bj) my_changed += 1.0;
        labels[i] = bj;
        double md = (double)xn + (double)best;
        my_sse += md > 0.0 ? md : 0.0;
#pragma unroll
        for (int j = 0; j < SD_K; ++j) {
            const bool hit = (bj == j);
            cnts[j] += hit ? 1.0 : 0.0;
#pragma unroll
            for (int t = 0; t < SD_D; ++t) sums[j][t] += hit ? (double)x[t] : 0.0;
        }
    }
    // warp -> block -> global
    constexpr int NV = SD_K * SD_D + SD_K + 2;
    __shared__ double red[SD_T / 32][NV];
    const int lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int j = 0; j < SD_K; ++j) {
#pragma unroll
        for (int t = 0; t < SD_D; ++t) {
            double v = warp_sum(sums[j][t]);
            if (lane == 0) red[w][j * SD_D + t] = v;
        }
        double c = warp_sum(cnts[j]);
        if (lane == 0) red[w][SD_K * SD_D + j] = c;
    }
    my_sse = warp_sum(my_sse);
    my_changed = warp_sum(my_changed);
    if (lane == 0) { red[w][NV - 2] = my_sse; red[w][NV - 1] = my_changed; }
    __syncthreads();
    if (tid < NV) {
        double a = 0.0;
        for (int q = 0; q < SD_T / 32; ++q) a += red[q][tid];
        double* dst = nullptr;
        if (tid < SD_K * SD_D) {
            int j = tid / SD_D, t = tid % SD_D;
            if (j < p.k && t < p.d) dst = acc + L.sums() + (int64_t)j * p.d + t;
        } else if (tid < SD_K * SD_D + SD_K) {
            int j = tid - SD_K * SD_D;
            if (j < p.k) dst = acc + L.counts() + j;
        } else if (tid == NV - 2) {
            dst = acc + L.sse();
        } else {
            dst = acc + L.changed();
        }
        if (dst && a != 0.0) atomicAdd(dst, a);
    }
}

// ------------------------------------------------------------------------------------------
// K10 final SSE, direct formula in fp64: one warp per row.
// ------------------------------------------------------------------------------------------
template <typename W>
__global__ void final_sse_kernel(const W* __restrict__ X, int64_t n, int d,
                                 const W* __restrict__ C, const int32_t* __restrict__ labels,
                                 double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // 4 rows per warp per step: their labels and first column chunks are loaded together so
    // the pass is bandwidth- rather than latency-bound.
    constexpr int RW = 4;
    double acc = 0.0;
    for (int64_t i0 = warp * RW; i0 < n; i0 += nwarps * RW) {
        int lab[RW];
#pragma unroll
        for (int r = 0; r < RW; ++r) lab[r] = (i0 + r < n) ? labels[i0 + r] : 0;
        for (int t = lane; t < d; t += 32) {
            W xv[RW], cv[RW];
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                const bool ok = i0 + r < n;
                xv[r] = ok ? X[(i0 + r) * d + t] : (W)0;
                cv[r] = ok ? C[(int64_t)lab[r] * d + t] : (W)0;
            }
            if constexpr (sizeof(W) == 4) {
                // fp32 differences, squares split exactly (p + e), one conversion per step
                float s = 0.0f, comp = 0.0f;
#pragma unroll
                for (int r = 0; r < RW; ++r) {
                    const float df = xv[r] - cv[r];
                    const float p2 = df * df;
                    const float e2 = fmaf(df, df, -p2);
                    const float t = s + p2;
                    const float z = t - s;
                    comp += (s - (t - z)) + (p2 - z) + e2;
                    s = t;
                }
                acc += (double)s + (double)comp;
            } else {
#pragma unroll
                for (int r = 0; r < RW; ++r) {
                    const double df = (double)xv[r] - (double)cv[r];
                    acc = fma(df, df, acc);
                }
            }
        }
    }
    acc = warp_sum(acc);
    __shared__ double red[8];
    if (lane == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += red[w];
        atomicAdd(out, a);
    }
}

// fp32, d <= 32 * TQ: the same sums in the same order as final_sse_kernel<float>, with every
// load of the RW rows issued before the arithmetic (the runtime-length column loop issued one
// column step's loads at a time: four HBM round trips per row group at d = 128).
template <int TQ>
__global__ void final_sse_fast_kernel(const float* __restrict__ X, int64_t n, int d,
                                      const float* __restrict__ C,
                                      const int32_t* __restrict__ labels,
                                      double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int RW = 4;
    double acc = 0.0;
    for (int64_t i0 = warp * RW; i0 < n; i0 += nwarps * RW) {
        int lab[RW];
#pragma unroll
        for (int r = 0; r < RW; ++r) lab[r] = (i0 + r < n) ? labels[i0 + r] : 0;
        float xv[TQ][RW], cv[TQ][RW];
#pragma unroll
        for (int q = 0; q < TQ; ++q) {
            const int t = lane + 32 * q;
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                const bool ok = i0 + r < n && t < d;
                xv[q][r] = ok ? X[(i0 + r) * d + t] : 0.0f;
                cv[q][r] = ok ? C[(int64_t)lab[r] * d + t] : 0.0f;
            }
        }
#pragma unroll
        for (int q = 0; q < TQ; ++q) {
            if (lane + 32 * q >= d) break;
            float s = 0.0f, comp = 0.0f;
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                const float df = xv[q][r] - cv[q][r];
                const float p2 = df * df;
                const float e2 = fmaf(df, df, -p2);
                const float t = s + p2;
                const float z = t - s;
                comp += (s - (t - z)) + (p2 - z) + e2;
                s = t;
            }
            acc += (double)s + (double)comp;
        }
    }
    acc = warp_sum(acc);
    __shared__ double red[8];
    if (lane == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += red[w];
        atomicAdd(out, a);
    }
}

// fp32, d <= 4: a row per thread. Per row the exact products (df^2 = p2 + e2) are summed over
// the D columns with the same compensated fp32 TwoSum as final_sse_fast_kernel (which runs it
// over 4 rows of one column), then added in fp64: the same accuracy class, without 29 of 32
// lanes idle at d = 3.
template <int D>
__global__ void __launch_bounds__(256)
final_sse_small_kernel(const float* __restrict__ X, int64_t n, const float* __restrict__ C,
                       const int32_t* __restrict__ labels, double* __restrict__ out) {
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int lab = labels[i];
        float s = 0.0f, comp = 0.0f;
#pragma unroll
        for (int t = 0; t < D; ++t) {
            const float df = X[i * D + t] - C[(int64_t)lab * D + t];
            const float p2 = df * df;
            const float e2 = fmaf(df, df, -p2);
            const float u = s + p2;
            const float z = u - s;
            comp += (s - (u - z)) + (p2 - z) + e2;
            s = u;
        }
        acc += (double)s + (double)comp;
    }
    acc = warp_sum(acc);
    __shared__ double red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += red[w];
        atomicAdd(out, a);
    }
}

// fp32 rows of 128 / 256 columns (V float4 groups per lane): one 16-byte load of x and of its
// centre per row and group, RW rows in flight per warp; per column the same exact-product TwoSum
// over the RW rows as final_sse_fast_kernel, then fp64.
template <int V>
__global__ void __launch_bounds__(256)
final_sse_vec_kernel(const float* __restrict__ X, int64_t n, int d, const float* __restrict__ C,
                     const int32_t* __restrict__ labels, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int RW = 8 / V;
    double acc = 0.0;
    // the labels of the next row group are fetched one group ahead (the centre loads depend on
    // them); lane r < RW holds label r of a group, broadcast by shuffles
    int nlab = (warp * RW + lane < n && lane < RW) ? __ldg(labels + warp * RW + lane) : 0;
    for (int64_t i0 = warp * RW; i0 < n; i0 += nwarps * RW) {
        int lab[RW];
#pragma unroll
        for (int r = 0; r < RW; ++r) lab[r] = __shfl_sync(0xffffffffu, nlab, r);
        {
            const int64_t j = i0 + nwarps * RW + lane;
            nlab = (lane < RW && j < n) ? __ldg(labels + j) : 0;
        }
        float4 xv[V][RW], cv[V][RW];
#pragma unroll
        for (int w = 0; w < V; ++w)
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                const bool ok = i0 + r < n;
                xv[w][r] = ok ? __ldg(reinterpret_cast<const float4*>(X + (i0 + r) * d + 128 * w) + lane)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
                cv[w][r] = ok ? __ldg(reinterpret_cast<const float4*>(C + (int64_t)lab[r] * d + 128 * w) + lane)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
        for (int w = 0; w < V; ++w)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float sum = 0.0f, comp = 0.0f;
#pragma unroll
                for (int r = 0; r < RW; ++r) {
                    const float xa = e == 0 ? xv[w][r].x : e == 1 ? xv[w][r].y : e == 2 ? xv[w][r].z : xv[w][r].w;
                    const float ca = e == 0 ? cv[w][r].x : e == 1 ? cv[w][r].y : e == 2 ? cv[w][r].z : cv[w][r].w;
                    const float df = xa - ca;
                    const float p2 = df * df;
                    const float e2 = fmaf(df, df, -p2);
                    const float t = sum + p2;
                    const float z = t - sum;
                    comp += (sum - (t - z)) + (p2 - z) + e2;
                    sum = t;
                }
                acc += (double)sum + (double)comp;
            }
    }
    acc = warp_sum(acc);
    __shared__ double red[8];
    if (lane == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += red[w];
        atomicAdd(out, a);
    }
}

template <typename LT, typename W>
cudaError_t simt_dispatch_acc(int dist, const Problem& p, const void* Xl, const void* xn,
                              const void* sx, const void* Cl, const void* cn, const void* sc,
                              int32_t* labels, double* acc_sse, double* acc_changed,
                              cudaStream_t s, const int* rows) {
    if (p.n <= 0) return cudaSuccess;
    if constexpr (!std::is_same<LT, double>::value && std::is_same<W, float>::value) {
        if (p.d <= 4 && p.k <= kSmallK && !getenv("MPK_SIMT_NO_SMALL")) {
            // d <= 4: a row per thread (MPK_SIMT_NO_SMALL=1: K6b, for A/B and tests)
            int64_t want = (p.n + 255) / 256;
            const int g = (int)(want < 1 ? 1 : (want > kNumSMs * 8 ? kNumSMs * 8 : want));
#define SIMT_SMALL(DV)                                                                             \
            assign_simt_small_kernel<LT, W, DV><<<g, 256, 0, s>>>(                                 \
                p, (const LT*)Xl, (const W*)xn, (const W*)sx, (const LT*)Cl, (const W*)cn,         \
                (const W*)sc, labels, acc_sse, acc_changed, rows);
            switch (p.d) {
                case 1: SIMT_SMALL(1) break;
                case 2: SIMT_SMALL(2) break;
                case 3: SIMT_SMALL(3) break;
                default: SIMT_SMALL(4) break;
            }
#undef SIMT_SMALL
            return cudaGetLastError();
        }
        // fp32 accumulation with fp32 working precision: the 8 x 8 register-tiled kernel
        const int64_t b2 = (p.n + B2M - 1) / B2M;
        assign_simt_big_kernel<LT, W><<<(unsigned)b2, B2T, 0, s>>>(
            p, (const LT*)Xl, (const W*)xn, (const W*)sx, (const LT*)Cl, (const W*)cn,
            (const W*)sc, labels, acc_sse, acc_changed, rows);
        return cudaGetLastError();
    }
    int64_t blocks = (p.n + BM - 1) / BM;
    // fp64 operands accumulate in fp64; every other operand type in fp32 (reading Z2/Z3)
    using AT = typename std::conditional<std::is_same<LT, double>::value, double, float>::type;
    assign_simt_kernel<LT, AT, W><<<(unsigned)blocks, NT, 0, s>>>(
        p, (const LT*)Xl, (const W*)xn, (const W*)sx, (const LT*)Cl, (const W*)cn, (const W*)sc,
        labels, acc_sse, acc_changed, rows);
    return cudaGetLastError();
}

template <typename W>
cudaError_t simt_dispatch(int dist, const Problem& p, const void* Xl, const void* xn,
                          const void* sx, const void* Cl, const void* cn, const void* sc,
                          int32_t* labels, double* acc_sse, double* acc_changed,
                          cudaStream_t s, const int* rows) {
#define MPK_SIMT(LT) \
    simt_dispatch_acc<LT, W>(dist, p, Xl, xn, sx, Cl, cn, sc, labels, acc_sse, acc_changed, s, rows)
    switch (dist) {
        case KMEANS_FP64: return MPK_SIMT(double);
        case KMEANS_FP32: return MPK_SIMT(float);
        case KMEANS_FP16: return MPK_SIMT(__half);
        case KMEANS_BF16: return MPK_SIMT(__nv_bfloat16);
        case KMEANS_E5M2: return MPK_SIMT(e5m2_t);
    }
#undef MPK_SIMT
    return cudaErrorInvalidValue;
}

template <typename W>
cudaError_t smalld_dispatch(int dist, const Problem& p, const W* X, const void* Cl,
                            const W* cn, const W* sc, int32_t* labels, double* acc, AccLayout L,
                            cudaStream_t s) {
    int64_t want = (p.n + SD_T * 4 - 1) / (SD_T * 4);
    int grid = (int)(want < 1 ? 1 : (want > kNumSMs * 4 ? kNumSMs * 4 : want));
    switch (dist) {
        case KMEANS_FP64:
            smalld_kernel<W, KMEANS_FP64><<<grid, SD_T, 0, s>>>(p, X, (const double*)Cl, cn, sc,
                                                                labels, acc, L);
            break;
        case KMEANS_FP32:
            smalld_kernel<W, KMEANS_FP32><<<grid, SD_T, 0, s>>>(p, X, (const float*)Cl, cn, sc,
                                                                labels, acc, L);
            break;
        case KMEANS_FP16:
            smalld_kernel<W, KMEANS_FP16><<<grid, SD_T, 0, s>>>(p, X, (const __half*)Cl, cn, sc,
                                                                labels, acc, L);
            break;
        case KMEANS_BF16:
            smalld_kernel<W, KMEANS_BF16><<<grid, SD_T, 0, s>>>(
                p, X, (const __nv_bfloat16*)Cl, cn, sc, labels, acc, L);
            break;
        case KMEANS_E5M2:
            smalld_kernel<W, KMEANS_E5M2><<<grid, SD_T, 0, s>>>(p, X, (const e5m2_t*)Cl, cn, sc,
                                                                labels, acc, L);
            break;
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_assign_simt(int work, int dist, const Problem& p, const void* Xl,
                               const void* xn, const void* sx, const void* Cl, const void* cn,
                               const void* sc, int32_t* labels, double* acc_sse,
                               double* acc_changed, cudaStream_t s, const int* row_list) {
    launches_add(1);
    if (work == KMEANS_FP64)
        return simt_dispatch<double>(dist, p, Xl, xn, sx, Cl, cn, sc, labels, acc_sse,
                                     acc_changed, s, row_list);
    return simt_dispatch<float>(dist, p, Xl, xn, sx, Cl, cn, sc, labels, acc_sse, acc_changed, s,
                                row_list);
}

bool smalld_supported(int d, int k) { return d <= SD_D && k <= SD_K; }

cudaError_t launch_smalld_fused(int work, int dist, const Problem& p, const void* Xw,
                                const void* Cl, const void* cn, const void* sc, int32_t* labels,
                                double* acc, AccLayout L, cudaStream_t s) {
    launches_add(1);
    if (work == KMEANS_FP64)
        return smalld_dispatch<double>(dist, p, (const double*)Xw, Cl, (const double*)cn,
                                       (const double*)sc, labels, acc, L, s);
    return smalld_dispatch<float>(dist, p, (const float*)Xw, Cl, (const float*)cn,
                                  (const float*)sc, labels, acc, L, s);
}

cudaError_t launch_final_sse(int work, const void* Xw, int64_t n, int d, const void* Cw,
                             const int32_t* labels, double* sse_out, cudaStream_t s) {
    launches_add(1);
    int64_t want = (n * 32 + 255) / 256;
    int grid = (int)(want < 1 ? 1 : (want > kNumSMs * 8 ? kNumSMs * 8 : want));
    const bool vec_ok = (d == 128 || d == 256) && ((((uintptr_t)Xw) | ((uintptr_t)Cw)) & 15) == 0;
    if (work == KMEANS_FP64)
        final_sse_kernel<double><<<grid, 256, 0, s>>>((const double*)Xw, n, d, (const double*)Cw,
                                                     labels, sse_out);
    else if (d <= 4 && !getenv("MPK_SIMT_NO_SMALL")) {
        const int64_t wr = (n + 255) / 256;
        const int gs = (int)(wr < 1 ? 1 : (wr > kNumSMs * 8 ? kNumSMs * 8 : wr));
        switch (d) {
            case 1: final_sse_small_kernel<1><<<gs, 256, 0, s>>>((const float*)Xw, n, (const float*)Cw, labels, sse_out); break;
            case 2: final_sse_small_kernel<2><<<gs, 256, 0, s>>>((const float*)Xw, n, (const float*)Cw, labels, sse_out); break;
            case 3: final_sse_small_kernel<3><<<gs, 256, 0, s>>>((const float*)Xw, n, (const float*)Cw, labels, sse_out); break;
            default: final_sse_small_kernel<4><<<gs, 256, 0, s>>>((const float*)Xw, n, (const float*)Cw, labels, sse_out); break;
        }
    } else if (vec_ok && d == 128)
        final_sse_vec_kernel<1><<<grid, 256, 0, s>>>((const float*)Xw, n, d, (const float*)Cw, labels, sse_out);
    else if (vec_ok)
        final_sse_vec_kernel<2><<<grid, 256, 0, s>>>((const float*)Xw, n, d, (const float*)Cw, labels, sse_out);
    else if (d <= 32)
        final_sse_fast_kernel<1><<<grid, 256, 0, s>>>((const float*)Xw, n, d, (const float*)Cw, labels, sse_out);
    else if (d <= 64)
        final_sse_fast_kernel<2><<<grid, 256, 0, s>>>((const float*)Xw, n, d, (const float*)Cw, labels, sse_out);
    else if (d <= 128)
        final_sse_fast_kernel<4><<<grid, 256, 0, s>>>((const float*)Xw, n, d, (const float*)Cw, labels, sse_out);
    else if (d <= 256)
        final_sse_fast_kernel<8><<<grid, 256, 0, s>>>((const float*)Xw, n, d, (const float*)Cw, labels, sse_out);
    else
        final_sse_kernel<float><<<grid, 256, 0, s>>>((const float*)Xw, n, d, (const float*)Cw,
                                                    labels, sse_out);
    return cudaGetLastError();
}

cudaError_t launch_assign_mixed(int work, int dist, const Problem& p, double delta, const void* Xl,
                                const void* Xw, const void* xn, const void* sx, const void* Cl,
                                const void* Cw, const void* cn, const void* sc, int32_t* labels,
                                double* acc_sse, double* acc_changed, unsigned long long* n_low,
                                cudaStream_t s) {
    launches_add(1);
    if (p.n <= 0) return cudaSuccess;
    const double delta2 = delta * delta;
    if (work == KMEANS_FP64) {
        switch (dist) {
            case KMEANS_FP64: return mixed_launch<double, double>(p, delta2, Xl, Xw, xn, sx, Cl, Cw, cn, sc, labels, acc_sse, acc_changed, n_low, s);
            case KMEANS_FP32: return mixed_launch<float, double>(p, delta2, Xl, Xw, xn, sx, Cl, Cw, cn, sc, labels, acc_sse, acc_changed, n_low, s);
            case KMEANS_FP16: return mixed_launch<__half, double>(p, delta2, Xl, Xw, xn, sx, Cl, Cw, cn, sc, labels, acc_sse, acc_changed, n_low, s);
            case KMEANS_BF16: return mixed_launch<__nv_bfloat16, double>(p, delta2, Xl, Xw, xn, sx, Cl, Cw, cn, sc, labels, acc_sse, acc_changed, n_low, s);
            case KMEANS_E5M2: return mixed_launch<e5m2_t, double>(p, delta2, Xl, Xw, xn, sx, Cl, Cw, cn, sc, labels, acc_sse, acc_changed, n_low, s);
        }
    } else if (getenv("MPK_MIXED_SMALL") == nullptr) {
        // fp32 work: K6b-sized tiles, per-tile classification (K6m-b)
        const int64_t blocks = (p.n + B2M - 1) / B2M;
#define MIXB(LT) assign_mixed_big_kernel<LT><<<(unsigned)blocks, B2T, 0, s>>>(p, delta2, (const LT*)Xl, (const float*)Xw, (const float*)xn, (const float*)sx, (const LT*)Cl, (const float*)Cw, (const float*)cn, (const float*)sc, labels, acc_sse, acc_changed, n_low)
        switch (dist) {
            case KMEANS_FP32: MIXB(float); return cudaGetLastError();
            case KMEANS_FP16: MIXB(__half); return cudaGetLastError();
            case KMEANS_BF16: MIXB(__nv_bfloat16); return cudaGetLastError();
            case KMEANS_E5M2: MIXB(e5m2_t); return cudaGetLastError();
        }
#undef MIXB
    } else {
        switch (dist) {
            case KMEANS_FP32: return mixed_launch<float, float>(p, delta2, Xl, Xw, xn, sx, Cl, Cw, cn, sc, labels, acc_sse, acc_changed, n_low, s);
            case KMEANS_FP16: return mixed_launch<__half, float>(p, delta2, Xl, Xw, xn, sx, Cl, Cw, cn, sc, labels, acc_sse, acc_changed, n_low, s);
            case KMEANS_BF16: return mixed_launch<__nv_bfloat16, float>(p, delta2, Xl, Xw, xn, sx, Cl, Cw, cn, sc, labels, acc_sse, acc_changed, n_low, s);
            case KMEANS_E5M2: return mixed_launch<e5m2_t, float>(p, delta2, Xl, Xw, xn, sx, Cl, Cw, cn, sc, labels, acc_sse, acc_changed, n_low, s);
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace mpk
