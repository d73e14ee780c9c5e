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
// for bit. Per round: one pass over X~ (HBM), a block-sum pass over D2, one sequential pick.
#include "common.cuh"
#include "internal.h"

namespace mpk {
namespace {

constexpr int kSeedBlock = 4096;

template <typename LT, typename W>
__global__ void __launch_bounds__(256)
seed_update_kernel(const LT* __restrict__ Xl, int64_t n, int d, int d_pad,
                   const W* __restrict__ xn, const W* __restrict__ sx, int guard,
                   const int64_t* __restrict__ idx, int j, double* __restrict__ D2) {
    extern __shared__ double cs[];             // the newest centre's operands, widened
    const int64_t c = idx[j];
    for (int t = threadIdx.x; t < d; t += blockDim.x) cs[t] = (double)widen(Xl[c * d_pad + t]);
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double D = 0.0;
    if (i != c) {
        const LT* x = Xl + i * d_pad;
        double dot = 0.0;
        for (int t = 0; t < d; ++t) dot = __dadd_rn(dot, __dmul_rn((double)widen(x[t]), cs[t]));
        const double si = guard ? (double)sx[i] : 1.0;
        const double sc = guard ? (double)sx[c] : 1.0;
        const double m = __dmul_rn(__dmul_rn(2.0, __dmul_rn(si, sc)), dot);
        D = __dadd_rn(__dsub_rn((double)xn[i], m), (double)xn[c]);
        D = D > 0.0 ? D : 0.0;                 // NaN -> 0
    }
    if (D < D2[i]) D2[i] = D;
}

__global__ void seed_bsum_kernel(const double* __restrict__ D2, int64_t n, int64_t nb,
                                 double* __restrict__ ps) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const int64_t e = (b + 1) * kSeedBlock < n ? (b + 1) * kSeedBlock : n;
    double a = 0.0;
    int64_t i = b * kSeedBlock;
    for (; i + 8 <= e; i += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = D2[i + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) a = __dadd_rn(a, v[u]);
    }
    for (; i < e; ++i) a = __dadd_rn(a, D2[i]);
    ps[b] = a;
}

__global__ void seed_pick_kernel(const double* __restrict__ D2, const double* __restrict__ ps,
                                 int64_t n, int64_t nb, const double* __restrict__ u, int j,
                                 int64_t* __restrict__ idx, int* __restrict__ warn) {
    if (threadIdx.x != 0) return;
    double tot = 0.0;
    for (int64_t b = 0; b < nb; ++b) tot = __dadd_rn(tot, ps[b]);
    int64_t c;
    if (!(tot > 0.0) || isinf(tot)) {
        c = (int64_t)__dmul_rn(u[j], (double)n);
        if (c > n - 1) c = n - 1;
        *warn |= 1;
    } else {
        const double target = __dmul_rn(u[j], tot);
        double run = 0.0;
        int64_t b = 0;
        for (; b < nb - 1; ++b) {
            if (__dadd_rn(run, ps[b]) > target) break;
            run = __dadd_rn(run, ps[b]);
        }
        const int64_t e = (b + 1) * kSeedBlock < n ? (b + 1) * kSeedBlock : n;
        double loc = 0.0;
        c = e - 1;
        for (int64_t i = b * kSeedBlock; i < e; ++i) {
            loc = __dadd_rn(loc, D2[i]);
            if (__dadd_rn(run, loc) > target) { c = i; break; }
        }
    }
    idx[j] = c;
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
    for (int j = 1; j < k; ++j) {
        seed_update_kernel<LT, W><<<pb, 256, (size_t)d * sizeof(double), s>>>(
            (const LT*)Xl, n, d, d_pad, (const W*)xn, (const W*)sx, guard, idx, j - 1, D2);
        seed_bsum_kernel<<<(unsigned)((nb + 127) / 128), 128, 0, s>>>(D2, n, nb, ps);
        seed_pick_kernel<<<1, 32, 0, s>>>(D2, ps, n, nb, u, j, idx, warn);
    }
    launches_add(1 + 3 * (int64_t)(k - 1));
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
