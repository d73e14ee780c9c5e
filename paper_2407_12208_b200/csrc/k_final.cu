// k_final.cu — the final pass's candidate path (Alg 3 step 7, R2).
//
// After the certified tensor-core filter (launch_final_tc), an uncertified row r has a threshold
// T_r = v^(1) + 2 (E + B32): every column whose working-precision (fp32) distance could be the
// row's minimum — including every column tied with it — has v^_j <= T_r. launch_cand_tc lists
// those columns from the same low-precision operands; this file holds
//   * the gather of the uncertified rows' operands into a dense matrix for that pass, and
//   * the exact stage: each listed column re-evaluated in fp32 with the arithmetic of the CUDA-core
//     kernel (k_assign_simt.cu: dot accumulated t = 0..d-1 by FMA, v = fma(-2, dot, ||c_j||^2))
//     and the (value, lowest index) argmin written as the label.
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

// One warp per gathered row; lane l evaluates candidates l, l+32, ...
__global__ void cand_exact_kernel(const float* __restrict__ Xw, const float* __restrict__ Cw,
                                  const float* __restrict__ cn, int d,
                                  const int* __restrict__ rows, int nr,
                                  const int* __restrict__ cand_cnt, const int* __restrict__ cand,
                                  int cand_q, int32_t* __restrict__ labels, int* left_count,
                                  int* left_rows) {
    const int r = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= nr) return;
    const int64_t row = rows[r];
    const int cnt = cand_cnt[r];
    if (cnt <= 0 || cnt > cand_q) {
        if (lane == 0) left_rows[atomicAdd(left_count, 1)] = (int)row;
        return;
    }
    const float* x = Xw + row * d;
    float bv = INFINITY;
    int bj = 0x7fffffff;
    for (int i = lane; i < cnt; i += 32) {
        const int j = cand[(int64_t)r * cand_q + i];
        const float* c = Cw + (int64_t)j * d;
        float dot = 0.0f;
        if ((d & 3) == 0) {
            for (int t = 0; t < d; t += 4) {
                const float4 xv = *reinterpret_cast<const float4*>(x + t);
                const float4 cv = *reinterpret_cast<const float4*>(c + t);
                dot = fmaf(xv.x, cv.x, dot);
                dot = fmaf(xv.y, cv.y, dot);
                dot = fmaf(xv.z, cv.z, dot);
                dot = fmaf(xv.w, cv.w, dot);
            }
        } else {
            for (int t = 0; t < d; ++t) dot = fmaf(x[t], c[t], dot);
        }
        const float v = fmaf(-2.0f, dot, cn[j]);
        argmin_merge(bv, bj, v, j);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const int j2 = __shfl_xor_sync(0xffffffffu, bj, o);
        argmin_merge(bv, bj, v2, j2);
    }
    // the CUDA-core kernel keeps label 0 when no value is < +inf; a certified-failed row with a
    // finite threshold always has a finite candidate (its own v^(1) column), so bj is set here
    if (lane == 0) labels[row] = bj == 0x7fffffff ? 0 : bj;
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
                              cudaStream_t s) {
    if (nr <= 0) return cudaSuccess;
    const int threads = 256;
    const int64_t blocks = ((int64_t)nr * 32 + threads - 1) / threads;
    launches_add(1);
    cand_exact_kernel<<<(unsigned)blocks, threads, 0, s>>>(Xw, Cw, cn, d, rows, nr, cand_cnt, cand,
                                                           cand_q, labels, left_count, left_rows);
    return cudaGetLastError();
}

}  // namespace mpk
