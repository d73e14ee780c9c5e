// k_seed.cu — D^2 seeding (Alg 1) with Alg 3 step 1's low precision
// (PAPER.md:544), as DESIGN.md reading R6 defines the draw:
//   * D^2(p_i, c) = xn_i - 2 (s_i s_c) (x~_i . x~_c) + xn_c, the dot of the stored low-precision
//     operands accumulated sequentially (t = 0..d-1) in fp64 and every operation in that order
//     rounded in fp64 (no contraction), floored at 0; the centre's own weight is 0;
//   * weights D2[i] = min over the chosen centres; the total and the running sums follow the
//     fixed blocked order (sequential fp64 sums over kSeedBlock consecutive indices, then the
//     block sums sequentially); the next centre is the first index whose running sum exceeds
//     u_j * total; a total of 0 or +inf/NaN falls back to the uniform index (warning).
// The draw is therefore a deterministic function of (X, u) that the oracle (O10) reproduces bit
// for bit. Per round: one pass over X~ (HBM) in CTAs of one seeding block each, which also form
// the block sums, then one sequential pick (block totals, then the chosen block from smem).
#include "common.cuh"
#include "internal.h"

#include <string.h>

namespace mpk {
namespace {

constexpr int kSeedBlock = 4096;

// Widen one 16-byte chunk of a low-precision row (8 fp16/bf16, 16 e5m2, 4 fp32, 2 fp64) to
// doubles; returns the element count.
template <typename LT>
MPK_DEV int widen16(uint4 q, double (&o)[16]) {
    // q is a register copy: taking the chunk by reference made ptxas re-read every element from
    // global memory with 16-bit loads
    constexpr int m = 16 / (int)sizeof(LT);
    LT e[m];
    memcpy(e, &q, 16);
#pragma unroll
    for (int i = 0; i < m; ++i) o[i] = (double)widen(e[i]);
    return m;
}

// One CTA per seeding block of kSeedBlock rows: D2 update for the block's rows (one row per
// thread at a time; 16-byte loads when rows are 16-byte aligned) and the block's sequential sum
// from shared memory (reading R6's order) -> ps[b].
template <typename LT, typename W>
__global__ void __launch_bounds__(256)
seed_update_kernel(const LT* __restrict__ Xl, int64_t n, int d, int d_pad,
                   const W* __restrict__ xn, const W* __restrict__ sx, int guard,
                   const int64_t* __restrict__ idx, int j, double* __restrict__ D2,
                   double* __restrict__ ps) {
    extern __shared__ double smem[];
    double* cs = smem;                          // the newest centre's operands, widened (d)
    double* d2s = smem + d;                     // this block's weights (kSeedBlock)
    const int64_t c = idx[j];
    for (int t = threadIdx.x; t < d; t += blockDim.x) cs[t] = (double)widen(Xl[c * d_pad + t]);
    __syncthreads();
    const double xnc = (double)xn[c];
    const double scc = guard ? (double)sx[c] : 1.0;
    const int64_t b0 = (int64_t)blockIdx.x * kSeedBlock;
    const int64_t b1 = (b0 + kSeedBlock < n) ? b0 + kSeedBlock : n;
    const bool vec = ((d_pad * (int)sizeof(LT)) % 16 == 0) &&
                     ((reinterpret_cast<uintptr_t>(Xl) & 15) == 0);
    // two rows per thread at a time (rows i and i + blockDim.x): two independent fp64 chains
    auto finish = [&](int64_t i, double dot) {
        const double si = guard ? (double)sx[i] : 1.0;
        const double mm = __dmul_rn(__dmul_rn(2.0, __dmul_rn(si, scc)), dot);
        double D = __dadd_rn(__dsub_rn((double)xn[i], mm), xnc);
        D = D > 0.0 ? D : 0.0;                  // NaN -> 0
        if (i == c) D = 0.0;                    // the centre's own weight
        const double old = D2[i];
        const double nw = D < old ? D : old;
        D2[i] = nw;
        d2s[i - b0] = nw;
    };
    const int64_t step = 2 * (int64_t)blockDim.x;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += step) {
        const int64_t i2 = i + blockDim.x;
        const bool two = i2 < b1;
        double dot = 0.0, dot2 = 0.0;
        if (vec) {
            const uint4* xa = reinterpret_cast<const uint4*>(Xl + i * d_pad);
            const uint4* xb = reinterpret_cast<const uint4*>(Xl + (two ? i2 : i) * d_pad);
            constexpr int m = 16 / (int)sizeof(LT);
            int t = 0;
            for (int q = 0; t < d; ++q) {
                double oa[16], ob[16];
                widen16<LT>(__ldg(xa + q), oa);
                widen16<LT>(__ldg(xb + q), ob);
#pragma unroll
                for (int e = 0; e < m; ++e) {
                    if (t + e < d) {
                        dot = __dadd_rn(dot, __dmul_rn(oa[e], cs[t + e]));
                        dot2 = __dadd_rn(dot2, __dmul_rn(ob[e], cs[t + e]));
                    }
                }
                t += m;
            }
        } else {
            const LT* xa = Xl + i * d_pad;
            const LT* xb = Xl + (two ? i2 : i) * d_pad;
            for (int t = 0; t < d; ++t) {
                dot = __dadd_rn(dot, __dmul_rn((double)widen(xa[t]), cs[t]));
                dot2 = __dadd_rn(dot2, __dmul_rn((double)widen(xb[t]), cs[t]));
            }
        }
        finish(i, dot);
        if (two) finish(i2, dot2);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int64_t i = 0; i < b1 - b0; ++i) a = __dadd_rn(a, d2s[i]);
        ps[blockIdx.x] = a;
    }
}

// Sequential pick (reading R6): block totals in order, then the chosen block staged into shared
// memory and scanned in order by one thread.
__global__ void seed_pick_kernel(const double* __restrict__ D2, const double* __restrict__ ps,
                                 int64_t n, int64_t nb, const double* __restrict__ u, int j,
                                 int64_t* __restrict__ idx, int* __restrict__ warn,
                                 int staged) {
    extern __shared__ double pss_smem[];        // the block totals (nb), staged when they fit
    const double* pss = staged ? pss_smem : ps;
    __shared__ double blk[kSeedBlock];
    __shared__ double sh_run, sh_target;
    __shared__ int64_t sh_b;
    __shared__ int sh_mode;                     // 0: scan block sh_b, 1: fallback done
    if (staged)
        for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) pss_smem[b] = ps[b];
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int64_t b = 0; b < nb; ++b) tot = __dadd_rn(tot, pss[b]);
        if (!(tot > 0.0) || isinf(tot)) {
            int64_t c = (int64_t)__dmul_rn(u[j], (double)n);
            if (c > n - 1) c = n - 1;
            *warn |= 1;
            idx[j] = c;
            sh_mode = 1;
        } else {
            const double target = __dmul_rn(u[j], tot);
            double run = 0.0;
            int64_t b = 0;
            for (; b < nb - 1; ++b) {
                if (__dadd_rn(run, pss[b]) > target) break;
                run = __dadd_rn(run, pss[b]);
            }
            sh_run = run;
            sh_target = target;
            sh_b = b;
            sh_mode = 0;
        }
    }
    __syncthreads();
    if (sh_mode) return;
    const int64_t b0 = sh_b * kSeedBlock;
    const int64_t e = (b0 + kSeedBlock < n) ? b0 + kSeedBlock : n;
    for (int64_t i = b0 + threadIdx.x; i < e; i += blockDim.x) blk[i - b0] = D2[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        const double run = sh_run, target = sh_target;
        double loc = 0.0;
        int64_t c = e - 1;
        for (int64_t i = 0; i < e - b0; ++i) {
            loc = __dadd_rn(loc, blk[i]);
            if (__dadd_rn(run, loc) > target) { c = b0 + i; break; }
        }
        idx[j] = c;
    }
}

__global__ void seed_init_kernel(double* D2, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) D2[i] = INFINITY;
}

template <typename LT, typename W>
cudaError_t seed_rounds(const void* Xl, int64_t n, int d, int d_pad, const void* xn,
                        const void* sx, int guard, int k, const double* u, int64_t* idx,
                        double* D2, double* ps, int* warn, cudaStream_t s) {
    const int64_t nb = (n + kSeedBlock - 1) / kSeedBlock;
    const unsigned pb = (unsigned)((n + 255) / 256);
    seed_init_kernel<<<pb, 256, 0, s>>>(D2, n);
    const size_t sm = ((size_t)d + kSeedBlock) * sizeof(double);
    static PerDeviceOnce attr;
    if (attr.need()) {
        cudaFuncSetAttribute(seed_update_kernel<LT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        cudaFuncSetAttribute(seed_pick_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             180 * 1024);
        attr.done();
    }
    // the pick stages the nb block totals in shared memory when they fit (n <= ~73M rows)
    const int staged = (size_t)nb * sizeof(double) <= 140 * 1024 ? 1 : 0;
    for (int j = 1; j < k; ++j) {
        seed_update_kernel<LT, W><<<(unsigned)nb, 256, sm, s>>>(
            (const LT*)Xl, n, d, d_pad, (const W*)xn, (const W*)sx, guard, idx, j - 1, D2, ps);
        seed_pick_kernel<<<1, 256, staged ? (size_t)nb * sizeof(double) : 0, s>>>(D2, ps, n, nb,
                                                                                  u, j, idx, warn,
                                                                                  staged);
    }
    launches_add(1 + 2 * (int64_t)(k - 1));
    return cudaGetLastError();
}

}  // namespace

int64_t seed_blocks(int64_t n) { return (n + kSeedBlock - 1) / kSeedBlock; }

cudaError_t launch_seed_d2(int work, int dist, const void* Xl, int64_t n, int d, int d_pad,
                           const void* xn, const void* sx, int guard, int k, const double* u,
                           int64_t* idx, double* D2, double* ps, int* warn, cudaStream_t s) {
#define SEED(LT, W) return seed_rounds<LT, W>(Xl, n, d, d_pad, xn, sx, guard, k, u, idx, D2, ps, warn, s)
    if (work == KMEANS_FP64) {
        switch (dist) {
            case KMEANS_FP64: SEED(double, double);
            case KMEANS_FP32: SEED(float, double);
            case KMEANS_FP16: SEED(__half, double);
            case KMEANS_BF16: SEED(__nv_bfloat16, double);
            case KMEANS_E5M2: SEED(e5m2_t, double);
        }
    } else {
        switch (dist) {
            case KMEANS_FP32: SEED(float, float);
            case KMEANS_FP16: SEED(__half, float);
            case KMEANS_BF16: SEED(__nv_bfloat16, float);
            case KMEANS_E5M2: SEED(e5m2_t, float);
        }
    }
#undef SEED
    return cudaErrorInvalidValue;
}

}  // namespace mpk
