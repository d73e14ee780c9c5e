// k_final.cu — the final pass's candidate path (Alg 3 step 7, R2).
//
// After the certified tensor-core filter (launch_final_tc), an uncertified row r has a threshold
// T_r = v^(1) + 2 (E + B32): every column whose working-precision (fp32) distance could be the
// row's minimum — including every column tied with it — has v^_j <= T_r. launch_cand_tc lists
// those columns from the same low-precision operands; this file holds
//   * the gather of the uncertified rows' operands into a dense matrix for that pass, and
//   * the exact stage: each listed column re-evaluated in fp32 with the arithmetic of the CUDA-core
//     kernel (k_assign_simt.cu: dot accumulated t = 0..d-1 by FMA, v = fma(-2, dot, ||c_j||^2))
//     and the (value, lowest index) argmin — an atomicMin over orderable 64-bit keys — written
//     as the label.
// Rows without candidates (non-finite values) or with more than cand_q of them are returned for
// the full CUDA-core evaluation, so the labels are those the full evaluation would produce.
#include "common.cuh"
#include "internal.h"

namespace mpk {
namespace {

__global__ void gather_rows_kernel(const uint8_t* __restrict__ src, int row_bytes,
                                   const int* __restrict__ rows, int nr, uint8_t* __restrict__ dst,
                                   const float* __restrict__ vsrc, float* __restrict__ vdst) {
    const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (warp >= nr) return;
    const int64_t r = rows[warp];
    const int4* s = reinterpret_cast<const int4*>(src + r * row_bytes);
    int4* o = reinterpret_cast<int4*>(dst + (int64_t)warp * row_bytes);
    for (int i = lane; i < row_bytes / 16; i += 32) o[i] = s[i];
    if (vdst && lane == 0) vdst[warp] = vsrc[r];
}

// Orderable key of (value, column): smaller value first, then smaller column (the CUDA-core
// kernel's (value, lowest index) rule); NaN values are never keys (the kernel ignores them).
MPK_DEV unsigned long long cand_key(float v, int j) {
    const uint32_t b = __float_as_uint(v);
    const uint32_t u = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return ((unsigned long long)u << 32) | (uint32_t)j;
}

// One thread per (candidate slot i, gathered row r), slot-major so that a warp takes 32
// consecutive rows for the same slot (uncertified rows have ~2 candidates: a warp per row left
// 30 of 32 lanes idle). The dot product is the CUDA-core kernel's: t = 0..d-1, fp32 FMA.
__global__ void cand_exact_kernel(const float* __restrict__ Xw, const float* __restrict__ Cw,
                                  const float* __restrict__ cn, int d,
                                  const int* __restrict__ rows, int nr,
                                  const int* __restrict__ cand_cnt, const int* __restrict__ cand,
                                  int cand_q, unsigned long long* __restrict__ keys) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nr * cand_q) return;
    const int i = (int)(t / nr);
    const int r = (int)(t - (int64_t)i * nr);
    const int cnt = cand_cnt[r];
    if (i >= cnt || cnt > cand_q) return;
    const int j = cand[(int64_t)r * cand_q + i];
    const float* x = Xw + (int64_t)rows[r] * d;
    const float* c = Cw + (int64_t)j * d;
    float dot = 0.0f;
    if ((d & 3) == 0) {
#pragma unroll 8
        for (int q = 0; q < d; q += 4) {
            const float4 xv = *reinterpret_cast<const float4*>(x + q);
            const float4 cv = *reinterpret_cast<const float4*>(c + q);
            dot = fmaf(xv.x, cv.x, dot);
            dot = fmaf(xv.y, cv.y, dot);
            dot = fmaf(xv.z, cv.z, dot);
            dot = fmaf(xv.w, cv.w, dot);
        }
    } else {
        for (int q = 0; q < d; ++q) dot = fmaf(x[q], c[q], dot);
    }
    const float v = fmaf(-2.0f, dot, cn[j]);
    if (!isnan(v)) atomicMin(keys + r, cand_key(v, j));
}

// Labels from the keys; rows without candidates or with overflow go to the full evaluation.
__global__ void cand_finalize_kernel(const int* __restrict__ rows, int nr,
                                     const int* __restrict__ cand_cnt, int cand_q,
                                     const unsigned long long* __restrict__ keys,
                                     int32_t* __restrict__ labels, int* left_count,
                                     int* left_rows) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nr) return;
    const int cnt = cand_cnt[r];
    if (cnt <= 0 || cnt > cand_q) {
        left_rows[atomicAdd(left_count, 1)] = rows[r];
        return;
    }
    const unsigned long long k = keys[r];
    // all candidate values NaN: the CUDA-core kernel keeps label 0
    labels[rows[r]] = k == ~0ull ? 0 : (int32_t)(uint32_t)k;
}

}  // namespace

cudaError_t launch_gather_rows(const void* src, int row_bytes, const int* rows, int nr, void* dst,
                               const float* vsrc, float* vdst, cudaStream_t s) {
    if (nr <= 0) return cudaSuccess;
    if (row_bytes % 16) return cudaErrorInvalidValue;
    const int threads = 256;
    const int64_t blocks = ((int64_t)nr * 32 + threads - 1) / threads;
    launches_add(1);
    gather_rows_kernel<<<(unsigned)blocks, threads, 0, s>>>((const uint8_t*)src, row_bytes, rows,
                                                            nr, (uint8_t*)dst, vsrc, vdst);
    return cudaGetLastError();
}

cudaError_t launch_cand_exact(const float* Xw, const float* Cw, const float* cn, int d,
                              const int* rows, int nr, const int* cand_cnt, const int* cand,
                              int cand_q, int32_t* labels, int* left_count, int* left_rows,
                              unsigned long long* keys, cudaStream_t s) {
    if (nr <= 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(keys, 0xff, (size_t)nr * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    const int threads = 256;
    const int64_t total = (int64_t)nr * cand_q;
    launches_add(2);
    cand_exact_kernel<<<(unsigned)((total + threads - 1) / threads), threads, 0, s>>>(
        Xw, Cw, cn, d, rows, nr, cand_cnt, cand, cand_q, keys);
    cand_finalize_kernel<<<(unsigned)((nr + threads - 1) / threads), threads, 0, s>>>(
        rows, nr, cand_cnt, cand_q, keys, labels, left_count, left_rows);
    return cudaGetLastError();
}

}  // namespace mpk
