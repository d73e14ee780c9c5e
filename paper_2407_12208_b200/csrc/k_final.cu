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

// ------------------------------------------------------------------------------------------
// Alg 4 / Alg 5 on the tensor cores (kmeans_set_delta with tcgen05 operands; R10):
// the certified filter of the final pass runs on the loop's guarded low-precision operands and
// every uncertified row's candidate columns are evaluated with Alg 4's per-pair switch, exactly
// as the CUDA-core kernel K6m-b evaluates them (trigger in fp64, the chosen dot accumulated
// t = 0..d-1 by fp32 FMA).
// ------------------------------------------------------------------------------------------
namespace mpk {
namespace {

// eq:prec-delta as K6m-b evaluates it (reading R5): max(xn, cn) >= delta^2 min(xn, cn) in fp64
MPK_DEV bool mixed_trigger(float xn, float cn, double delta2) {
    const double a = (double)xn, b = (double)cn;
    const double mx = (a > b) ? a : b, mn = (a > b) ? b : a;
    return mx >= delta2 * mn;
}

template <typename LT>
__global__ void cand_exact_mixed_kernel(const LT* __restrict__ Xl, const float* __restrict__ Xw,
                                        const LT* __restrict__ Cl, const float* __restrict__ Cw,
                                        const float* __restrict__ xn, const float* __restrict__ sx,
                                        const float* __restrict__ cn, const float* __restrict__ sc,
                                        int d, int d_pad, double delta2,
                                        const int* __restrict__ rows, int nr,
                                        const int* __restrict__ cand_cnt,
                                        const int* __restrict__ cand, int cand_q,
                                        unsigned long long* __restrict__ keys) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nr * cand_q) return;
    const int i = (int)(t / nr);
    const int r = (int)(t - (int64_t)i * nr);
    const int cnt = cand_cnt[r];
    if (i >= cnt || cnt > cand_q) return;
    const int j = cand[(int64_t)r * cand_q + i];
    const int64_t row = rows[r];
    float v;
    if (mixed_trigger(xn[row], cn[j], delta2)) {
        // Alg 4 lines 1-6: the scaled low-precision operands
        const LT* x = Xl + row * d_pad;
        const LT* c = Cl + (int64_t)j * d_pad;
        float dot = 0.0f;
        for (int q = 0; q < d; ++q) dot = fmaf((float)widen(x[q]), (float)widen(c[q]), dot);
        v = fmaf(-2.0f * (sx[row] * sc[j]), dot, cn[j]);
    } else {
        // Alg 4 line 8: the working-precision dot product
        const float* x = Xw + row * d;
        const float* c = Cw + (int64_t)j * d;
        float dot = 0.0f;
        for (int q = 0; q < d; ++q) dot = fmaf(x[q], c[q], dot);
        v = fmaf(-2.0f, dot, cn[j]);
    }
    if (!isnan(v)) atomicMin(keys + r, cand_key(v, j));
}

// The k centroid norms in increasing order (NaN last) in one block, for the trigger counts.
__global__ void sort_norms_kernel(const float* __restrict__ cn, int k, int kp, float* __restrict__ out) {
    extern __shared__ float sv[];
    for (int j = threadIdx.x; j < kp; j += blockDim.x) {
        float v = j < k ? cn[j] : NAN;
        sv[j] = v;
    }
    __syncthreads();
    // bitonic sort on keys where NaN is the largest
    auto key = [](float v) { return isnan(v) ? INFINITY : v; };
    for (int size = 2; size <= kp; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int j = threadIdx.x; j < kp; j += blockDim.x) {
                const int p = j ^ stride;
                if (p > j) {
                    const bool up = (j & size) == 0;
                    const float a = sv[j], b = sv[p];
                    const bool a_nan = isnan(a), b_nan = isnan(b);
                    const bool gt = a_nan ? !b_nan : (!b_nan && key(a) > key(b));
                    if (gt == up) { sv[j] = b; sv[p] = a; }
                }
            }
            __syncthreads();
        }
    }
    for (int j = threadIdx.x; j < kp; j += blockDim.x) out[j] = sv[j];
}

// Number of pairs of each row that eq:prec-delta sends to the low precision, from the sorted
// norms: {c < xn : xn >= delta^2 c} is a prefix and {c >= xn : c >= delta^2 xn} a suffix of the
// sorted order (both conditions are monotone in c), so two binary searches replace k tests.
__global__ void mixed_count_kernel(const float* __restrict__ xn, int64_t n,
                                   const float* __restrict__ cs, int k, double delta2,
                                   unsigned long long* __restrict__ n_low) {
    unsigned long long cnt = 0;
    int kv = k;                                   // non-NaN norms occupy cs[0 .. kv)
    {
        int lo = 0, hi = k;
        while (lo < hi) { const int m = (lo + hi) >> 1; if (isnan(cs[m])) hi = m; else lo = m + 1; }
        kv = lo;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float x = xn[i];
        if (isnan(x)) continue;
        // prefix: largest p with cs[p-1] < x && x >= delta2 * cs[p-1]
        int lo = 0, hi = kv;
        while (lo < hi) {
            const int m = (lo + hi) >> 1;
            const double c = (double)cs[m];
            if (c < (double)x && (double)x >= delta2 * c) lo = m + 1; else hi = m;
        }
        const int pre = lo;
        // suffix: first q with cs[q] >= x && cs[q] >= delta2 * x
        lo = pre; hi = kv;
        while (lo < hi) {
            const int m = (lo + hi) >> 1;
            const double c = (double)cs[m];
            if (c >= (double)x && c >= delta2 * (double)x) hi = m; else lo = m + 1;
        }
        cnt += (unsigned long long)pre + (unsigned long long)(kv - lo);
    }
    cnt = warp_sum(cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_low, cnt);
}

// Per row: the Alg 4 distance of its label (SSE_t's term max(0, xn + v)) and whether the label
// changed; one warp per row (lanes over the features).
template <typename LT>
__global__ void mixed_label_eval_kernel(const LT* __restrict__ Xl, const float* __restrict__ Xw,
                                        const LT* __restrict__ Cl, const float* __restrict__ Cw,
                                        const float* __restrict__ xn, const float* __restrict__ sx,
                                        const float* __restrict__ cn, const float* __restrict__ sc,
                                        int64_t n, int d, int d_pad, double delta2,
                                        const int32_t* __restrict__ labels,
                                        const int32_t* __restrict__ prev, double* acc_sse,
                                        double* acc_changed) {
    const int lane = threadIdx.x & 31;
    double sse = 0.0, changed = 0.0;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int j = labels[i];
        const bool trig = mixed_trigger(xn[i], cn[j], delta2);
        float dot = 0.0f;
        if (trig) {
            for (int q = lane; q < d; q += 32)
                dot = fmaf((float)widen(Xl[i * d_pad + q]), (float)widen(Cl[(int64_t)j * d_pad + q]), dot);
        } else {
            for (int q = lane; q < d; q += 32) dot = fmaf(Xw[i * d + q], Cw[(int64_t)j * d + q], dot);
        }
        dot = warp_sum(dot);
        if (lane == 0) {
            const float v = trig ? fmaf(-2.0f * (sx[i] * sc[j]), dot, cn[j]) : fmaf(-2.0f, dot, cn[j]);
            const double md = (double)xn[i] + (double)v;
            sse += md > 0.0 ? md : 0.0;
            if (prev && prev[i] != j) changed += 1.0;
        }
    }
    if (lane == 0) {
        if (acc_sse && sse != 0.0) atomicAdd(acc_sse, sse);
        if (acc_changed && changed != 0.0) atomicAdd(acc_changed, changed);
    }
}

// Gather rows of a float matrix (any width) and of per-row float vectors.
__global__ void gather_float_rows_kernel(const float* __restrict__ src, int d,
                                         const int* __restrict__ rows, int nr,
                                         float* __restrict__ dst) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nr * d) return;
    const int r = (int)(t / d), q = (int)(t - (int64_t)r * d);
    dst[t] = src[(int64_t)rows[r] * d + q];
}
__global__ void scatter_labels_kernel(const int32_t* __restrict__ src, const int* __restrict__ rows,
                                      int nr, int32_t* __restrict__ labels) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nr) labels[rows[r]] = src[r];
}

}  // namespace

#define MPK_LT_SWITCH(dist, CALL)                                                  \
    switch (dist) {                                                                \
        case KMEANS_FP16: { using LT = __half; CALL; } break;                      \
        case KMEANS_BF16: { using LT = __nv_bfloat16; CALL; } break;               \
        case KMEANS_E5M2: { using LT = e5m2_t; CALL; } break;                      \
        default: return cudaErrorInvalidValue;                                     \
    }

cudaError_t launch_cand_exact_mixed(int dist, const void* Xl, const float* Xw, const void* Cl,
                                    const float* Cw, const float* xn, const float* sx,
                                    const float* cn, const float* sc, int d, int d_pad,
                                    double delta2, const int* rows, int nr, const int* cand_cnt,
                                    const int* cand, int cand_q, int32_t* labels, int* left_count,
                                    int* left_rows, unsigned long long* keys, cudaStream_t s) {
    if (nr <= 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(keys, 0xff, (size_t)nr * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    const int threads = 256;
    const int64_t total = (int64_t)nr * cand_q;
    launches_add(2);
    MPK_LT_SWITCH(dist, (cand_exact_mixed_kernel<LT><<<(unsigned)((total + threads - 1) / threads), threads, 0, s>>>(
        (const LT*)Xl, Xw, (const LT*)Cl, Cw, xn, sx, cn, sc, d, d_pad, delta2, rows, nr, cand_cnt,
        cand, cand_q, keys)));
    cand_finalize_kernel<<<(unsigned)((nr + threads - 1) / threads), threads, 0, s>>>(
        rows, nr, cand_cnt, cand_q, keys, labels, left_count, left_rows);
    return cudaGetLastError();
}

cudaError_t launch_mixed_count(const float* xn, int64_t n, const float* cn, int k, double delta2,
                               float* sorted_cn, unsigned long long* n_low, cudaStream_t s) {
    int kp = 1;
    while (kp < k) kp <<= 1;
    if (kp > 16384) return cudaErrorInvalidValue;
    launches_add(2);
    if (kp * sizeof(float) > 48 * 1024)
        cudaFuncSetAttribute(sort_norms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kp * sizeof(float)));
    sort_norms_kernel<<<1, 1024, kp * sizeof(float), s>>>(cn, k, kp, sorted_cn);
    const int64_t want = (n + 255) / 256;
    const int g = (int)(want < 1 ? 1 : (want > kNumSMs * 8 ? kNumSMs * 8 : want));
    mixed_count_kernel<<<g, 256, 0, s>>>(xn, n, sorted_cn, k, delta2, n_low);
    return cudaGetLastError();
}

cudaError_t launch_mixed_label_eval(int dist, const void* Xl, const float* Xw, const void* Cl,
                                    const float* Cw, const float* xn, const float* sx,
                                    const float* cn, const float* sc, int64_t n, int d, int d_pad,
                                    double delta2, const int32_t* labels, const int32_t* prev,
                                    double* acc_sse, double* acc_changed, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    launches_add(1);
    const int64_t want = (n * 32 + 255) / 256;
    const int g = (int)(want < 1 ? 1 : (want > kNumSMs * 16 ? kNumSMs * 16 : want));
    MPK_LT_SWITCH(dist, (mixed_label_eval_kernel<LT><<<g, 256, 0, s>>>(
        (const LT*)Xl, Xw, (const LT*)Cl, Cw, xn, sx, cn, sc, n, d, d_pad, delta2, labels, prev,
        acc_sse, acc_changed)));
    return cudaGetLastError();
}

cudaError_t launch_gather_float_rows(const float* src, int d, const int* rows, int nr, float* dst,
                                     cudaStream_t s) {
    if (nr <= 0) return cudaSuccess;
    launches_add(1);
    const int64_t total = (int64_t)nr * d;
    gather_float_rows_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(src, d, rows, nr, dst);
    return cudaGetLastError();
}

cudaError_t launch_scatter_labels(const int32_t* src, const int* rows, int nr, int32_t* labels,
                                  cudaStream_t s) {
    if (nr <= 0) return cudaSuccess;
    launches_add(1);
    scatter_labels_kernel<<<(unsigned)((nr + 255) / 256), 256, 0, s>>>(src, rows, nr, labels);
    return cudaGetLastError();
}
#undef MPK_LT_SWITCH

}  // namespace mpk
