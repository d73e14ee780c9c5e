// k_prep.cu — K2 normalisation, K1/K3 operand preparation, and the standalone cast kernel.
//
// K2 (one-time): per-feature statistics in fp64 with compensated (Neumaier) partial sums, then
//   x <- round_u((x - shift) / scale) in place. ZSCORE: eq:z-norm, population
//   sigma, sigma = 0 -> 1. MINMAX: (x - min) / (max - min), range 0 -> 1; on 0..255-spanning
//   images this is the paper's "divided by 255".
// K1/K3: per row, ||x||^2 summed in fp64 and stored in precision u; with the
//   guard, s = ||x||_inf and x~ = round_l(round_u(x / s)) (Alg 4 lines 1-5);
//   without, x~ = round_l(x). Rows are padded with zeros to the kernel's row stride (exact:
//   zero columns add nothing to a dot product). Overflowed (+-inf/NaN) and underflowed
//   (nonzero -> zero/subnormal) operands are counted (readings Z7, Z8).
// HBM-bound: one warp per row, lanes over columns (coalesced), grid = a multiple of 148 SMs.
#include "common.cuh"
#include "internal.h"

namespace mpk {

namespace {

constexpr int kStatThreads = 256;
constexpr int kApplySmemD = 2048;
#ifndef MPK_PREP_NO_VEC
#define MPK_PREP_NO_VEC 0               // 1: always the scalar prep_fast_kernel (A/B)
#endif        // norm_apply caches shift / scale / 1/scale up to this d

// One kernel for the three column statistics: mode 0 = sum x, mode 1 = sum (x - mu)^2,
// mode 2 = (min, max). Thread layout: column c = tid % d, row lane = tid / d (d <= 256), else a
// loop over column blocks. Rows are read in batches of kUnroll per thread (all loads issued
// before the compensated accumulation, in the same order), so the pass is HBM-bound instead of
// load-latency-bound; the per-thread summation order is unchanged (deterministic).
constexpr int kUnroll = 8;

template <typename W>
__global__ void __launch_bounds__(kStatThreads)
norm_col_stats_kernel(int mode, const W* __restrict__ X, int64_t n, int d,
                      const double* __restrict__ mu, double* __restrict__ partials) {
    const int tid = threadIdx.x;
    const int lanes = d <= kStatThreads ? kStatThreads / d : 1;
    const int64_t rows_per_block = (n + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
    const int64_t r1 = min(n, r0 + rows_per_block);
    __shared__ double sh_s[kStatThreads], sh_c[kStatThreads];
    for (int cbase = 0; cbase < d; cbase += (d <= kStatThreads ? d : kStatThreads)) {
        int c, lane;
        bool active;
        if (d <= kStatThreads) {
            c = tid % d; lane = tid / d; active = lane < lanes;
        } else {
            c = cbase + tid; lane = 0; active = c < d;
        }
        double s = 0.0, comp = 0.0;   // sums: Neumaier (s, comp); minmax: s = min, comp = max
        if (mode == 2) { s = INFINITY; comp = -INFINITY; }
        if (active) {
            const double m = (mode == 1) ? mu[c] : 0.0;
            for (int64_t i0 = r0 + lane; i0 < r1; i0 += (int64_t)lanes * kUnroll) {
                double xv[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const int64_t i = i0 + (int64_t)u * lanes;
                    xv[u] = i < r1 ? (double)X[i * d + c] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const int64_t i = i0 + (int64_t)u * lanes;
                    if (i >= r1) break;
                    double x = xv[u];
                    if (mode == 2) {
                        s = fmin(s, x);
                        comp = fmax(comp, x);
                    } else {
                        if (mode == 1) { const double z = x - m; x = z * z; }
                        const double t = s + x;
                        comp += (fabs(s) >= fabs(x)) ? ((s - t) + x) : ((x - t) + s);
                        s = t;
                    }
                }
            }
        }
        sh_s[tid] = s;
        sh_c[tid] = comp;
        __syncthreads();
        // combine row lanes of the same column in fixed order (lane 0..lanes-1)
        if (active && lane == 0) {
            double S = s, Cc = comp;
            for (int l = 1; l < lanes; ++l) {
                const double s2 = sh_s[l * d + c], c2 = sh_c[l * d + c];
                if (mode == 2) {
                    S = fmin(S, s2);
                    Cc = fmax(Cc, c2);
                } else {
                    const double t = S + s2;
                    Cc += ((fabs(S) >= fabs(s2)) ? ((S - t) + s2) : ((s2 - t) + S)) + c2;
                    S = t;
                }
            }
            partials[((int64_t)blockIdx.x * d + c) * 2 + 0] = S;
            partials[((int64_t)blockIdx.x * d + c) * 2 + 1] = Cc;
        }
        __syncthreads();
        if (d <= kStatThreads) break;
    }
}

// Vectorised norm_col_stats_kernel for fp32 rows with d % 4 == 0 (d <= 1024): a thread owns
// four adjacent columns (one 16-byte load per row, four independent compensated sums) and
// keeps the next batch of rows in flight while it accumulates the current one. Same per-column
// arithmetic (Neumaier in fp64 over the thread's rows in increasing order, then the row lanes
// combined in lane order), with a different split of rows over lanes than the scalar kernel.
constexpr int kVecBatch = 4;
__global__ void __launch_bounds__(kStatThreads)
norm_col_stats_vec_kernel(int mode, const float* __restrict__ X, int64_t n, int d,
                          const double* __restrict__ mu, double* __restrict__ partials) {
    const int tid = threadIdx.x;
    const int cg = d >> 2;                          // column groups (<= 256)
    const int lanes = kStatThreads / cg;
    const int g = tid % cg, lane = tid / cg;
    const bool active = lane < lanes;
    const int64_t rows_per_block = (n + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
    const int64_t r1 = min(n, r0 + rows_per_block);
    __shared__ double sh_s[kStatThreads * 4], sh_c[kStatThreads * 4];
    double s[4], comp[4], m[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        s[e] = mode == 2 ? INFINITY : 0.0;
        comp[e] = mode == 2 ? -INFINITY : 0.0;
        m[e] = (mode == 1 && active) ? mu[4 * g + e] : 0.0;
    }
    if (active) {
        const float4* X4 = reinterpret_cast<const float4*>(X) + g;
        const int64_t step = (int64_t)lanes;
        float4 nxt[kVecBatch];
        int64_t i0 = r0 + lane;
#pragma unroll
        for (int u = 0; u < kVecBatch; ++u) {
            const int64_t i = i0 + u * step;
            nxt[u] = i < r1 ? __ldg(X4 + i * cg) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (; i0 < r1; i0 += step * kVecBatch) {
            float4 cur[kVecBatch];
#pragma unroll
            for (int u = 0; u < kVecBatch; ++u) cur[u] = nxt[u];
            const int64_t j0 = i0 + step * kVecBatch;
#pragma unroll
            for (int u = 0; u < kVecBatch; ++u) {
                const int64_t i = j0 + u * step;
                nxt[u] = i < r1 ? __ldg(X4 + i * cg) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < kVecBatch; ++u) {
                if (i0 + u * step >= r1) break;
                const float xv[4] = {cur[u].x, cur[u].y, cur[u].z, cur[u].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    double x = (double)xv[e];
                    if (mode == 2) {
                        s[e] = fmin(s[e], x);
                        comp[e] = fmax(comp[e], x);
                    } else {
                        if (mode == 1) { const double z = x - m[e]; x = z * z; }
                        const double t = s[e] + x;
                        comp[e] += (fabs(s[e]) >= fabs(x)) ? ((s[e] - t) + x) : ((x - t) + s[e]);
                        s[e] = t;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        sh_s[tid * 4 + e] = s[e];
        sh_c[tid * 4 + e] = comp[e];
    }
    __syncthreads();
    // combine row lanes of the same column in fixed order (lane 0..lanes-1)
    if (active && lane == 0) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            double S = s[e], Cc = comp[e];
            for (int l = 1; l < lanes; ++l) {
                const double s2 = sh_s[(l * cg + g) * 4 + e], c2 = sh_c[(l * cg + g) * 4 + e];
                if (mode == 2) {
                    S = fmin(S, s2);
                    Cc = fmax(Cc, c2);
                } else {
                    const double t = S + s2;
                    Cc += ((fabs(S) >= fabs(s2)) ? ((S - t) + s2) : ((s2 - t) + S)) + c2;
                    S = t;
                }
            }
            const int c = 4 * g + e;
            partials[((int64_t)blockIdx.x * d + c) * 2 + 0] = S;
            partials[((int64_t)blockIdx.x * d + c) * 2 + 1] = Cc;
        }
    }
}

// One-pass z-score moments (fp32 rows, d % 4 == 0, one rank): per column the compensated sums
// S1 = sum (x - K) and S2 = sum (x - K)^2 about K = the column's value in row 0, so that
// mu = K + S1 / n and sigma^2 = S2 / n - (S1 / n)^2 come from ONE read of X. Shifting by a data
// value keeps the cancellation in sigma^2 at u64 (1 + ((mu - K) / sigma)^2) relative (DESIGN.md
// R4); block 0 also stores K. Partials: S1 in part1, S2 in part2 (same layout as the scalar
// kernel's).
__global__ void __launch_bounds__(kStatThreads)
norm_moments_vec_kernel(const float* __restrict__ X, int64_t n, int d, double* __restrict__ part1,
                        double* __restrict__ part2, double* __restrict__ kbuf) {
    const int tid = threadIdx.x;
    const int cg = d >> 2;
    const int lanes = kStatThreads / cg;
    const int g = tid % cg, lane = tid / cg;
    const bool active = lane < lanes;
    const int64_t rows_per_block = (n + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
    const int64_t r1 = min(n, r0 + rows_per_block);
    __shared__ double sh[4][kStatThreads * 4];
    double s1[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0}, c2[4] = {0, 0, 0, 0};
    double K[4] = {0, 0, 0, 0};
    if (active) {
        const float4 k4 = __ldg(reinterpret_cast<const float4*>(X) + g);
        K[0] = k4.x; K[1] = k4.y; K[2] = k4.z; K[3] = k4.w;
        if (blockIdx.x == 0 && lane == 0)
            for (int e = 0; e < 4; ++e) kbuf[4 * g + e] = K[e];
        const float4* X4 = reinterpret_cast<const float4*>(X) + g;
        const int64_t step = (int64_t)lanes;
        float4 nxt[kVecBatch];
        int64_t i0 = r0 + lane;
#pragma unroll
        for (int u = 0; u < kVecBatch; ++u) {
            const int64_t i = i0 + u * step;
            nxt[u] = i < r1 ? __ldg(X4 + i * cg) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (; i0 < r1; i0 += step * kVecBatch) {
            float4 cur[kVecBatch];
#pragma unroll
            for (int u = 0; u < kVecBatch; ++u) cur[u] = nxt[u];
            const int64_t j0 = i0 + step * kVecBatch;
#pragma unroll
            for (int u = 0; u < kVecBatch; ++u) {
                const int64_t i = j0 + u * step;
                nxt[u] = i < r1 ? __ldg(X4 + i * cg) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < kVecBatch; ++u) {
                if (i0 + u * step >= r1) break;
                const float xv[4] = {cur[u].x, cur[u].y, cur[u].z, cur[u].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const double z = (double)xv[e] - K[e];
                    double t = s1[e] + z;
                    c1[e] += (fabs(s1[e]) >= fabs(z)) ? ((s1[e] - t) + z) : ((z - t) + s1[e]);
                    s1[e] = t;
                    const double z2 = z * z;
                    t = s2[e] + z2;
                    c2[e] += (s2[e] >= z2) ? ((s2[e] - t) + z2) : ((z2 - t) + s2[e]);
                    s2[e] = t;
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        sh[0][tid * 4 + e] = s1[e];
        sh[1][tid * 4 + e] = c1[e];
        sh[2][tid * 4 + e] = s2[e];
        sh[3][tid * 4 + e] = c2[e];
    }
    __syncthreads();
    if (active && lane == 0) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            double S = s1[e], C = c1[e], T = s2[e], D = c2[e];
            for (int l = 1; l < lanes; ++l) {
                const int ix = (l * cg + g) * 4 + e;
                double a = sh[0][ix], t = S + a;
                C += ((fabs(S) >= fabs(a)) ? ((S - t) + a) : ((a - t) + S)) + sh[1][ix];
                S = t;
                a = sh[2][ix];
                t = T + a;
                D += ((T >= a) ? ((T - t) + a) : ((a - t) + T)) + sh[3][ix];
                T = t;
            }
            const int c = 4 * g + e;
            part1[((int64_t)blockIdx.x * d + c) * 2 + 0] = S;
            part1[((int64_t)blockIdx.x * d + c) * 2 + 1] = C;
            part2[((int64_t)blockIdx.x * d + c) * 2 + 0] = T;
            part2[((int64_t)blockIdx.x * d + c) * 2 + 1] = D;
        }
    }
}
// shift = K + S1 / n, scale = sqrt(max(S2 / n - (S1 / n)^2, 0)) (0 -> 1); on entry shift = S1,
// scale = S2 (combined over the blocks)
__global__ void norm_post_moments_kernel(int d, double n_total, const double* __restrict__ kbuf,
                                         double* shift, double* scale) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= d) return;
    const double m1 = shift[c] / n_total;
    const double var = fmax(scale[c] / n_total - m1 * m1, 0.0);
    const double sigma = sqrt(var);
    shift[c] = kbuf[c] + m1;
    scale[c] = (sigma == 0.0) ? 1.0 : sigma;
}

// Combine the per-block partials of one column in block order.
// mode 0: compensated sum (-> a), mode 2: min (-> a) and max (-> b).
__global__ void norm_combine_kernel(int mode, const double* __restrict__ partials, int nblocks,
                                    int d, double* a, double* b) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= d) return;
    if (mode == 2) {
        // min / max are exact in any order: 16 independent loads in flight per batch
        double mn = INFINITY, mx = -INFINITY;
        for (int q0 = 0; q0 < nblocks; q0 += 16) {
            double lo[16], hi[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int q = q0 + u;
                lo[u] = q < nblocks ? partials[((int64_t)q * d + c) * 2 + 0] : INFINITY;
                hi[u] = q < nblocks ? partials[((int64_t)q * d + c) * 2 + 1] : -INFINITY;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                mn = fmin(mn, lo[u]);
                mx = fmax(mx, hi[u]);
            }
        }
        a[c] = mn;
        b[c] = mx;
        return;
    }
    // block order, partials loaded in batches of 16 (independent loads in flight; the serial
    // dependent loads of one thread were ~0.3 ms of pure L2 latency)
    double S = 0.0, Cc = 0.0;
    for (int q0 = 0; q0 < nblocks; q0 += 16) {
        double s2[16], c2[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int q = q0 + u;
            s2[u] = q < nblocks ? partials[((int64_t)q * d + c) * 2 + 0] : 0.0;
            c2[u] = q < nblocks ? partials[((int64_t)q * d + c) * 2 + 1] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (q0 + u >= nblocks) break;
            const double t = S + s2[u];
            Cc += ((fabs(S) >= fabs(s2[u])) ? ((S - t) + s2[u]) : ((s2[u] - t) + S)) + c2[u];
            S = t;
        }
    }
    a[c] = S + Cc;
}

// norm_combine_kernel with one warp per column: the warp stages the column's partials in shared
// memory (all loads in flight at once; the per-thread batches of 16 were one L2 round trip per
// batch: ~74 us for 592 partials at d = 64), then lane 0 combines them in block order with the
// same arithmetic as norm_combine_kernel — the same bits.
__global__ void __launch_bounds__(32)
norm_combine_warp_kernel(int mode, const double* __restrict__ partials, int nblocks, int d,
                         double* a, double* b) {
    extern __shared__ double stage[];                 // [nblocks][2]
    const int c = blockIdx.x, lane = threadIdx.x;
    for (int q = lane; q < nblocks; q += 32) {
        stage[2 * q + 0] = partials[((int64_t)q * d + c) * 2 + 0];
        stage[2 * q + 1] = partials[((int64_t)q * d + c) * 2 + 1];
    }
    __syncwarp();
    if (lane != 0) return;
    if (mode == 2) {
        double mn = INFINITY, mx = -INFINITY;
        for (int q = 0; q < nblocks; ++q) {
            mn = fmin(mn, stage[2 * q + 0]);
            mx = fmax(mx, stage[2 * q + 1]);
        }
        a[c] = mn;
        b[c] = mx;
        return;
    }
    double S = 0.0, Cc = 0.0;
    for (int q = 0; q < nblocks; ++q) {
        const double s2 = stage[2 * q + 0], c2 = stage[2 * q + 1];
        const double t = S + s2;
        Cc += ((fabs(S) >= fabs(s2)) ? ((S - t) + s2) : ((s2 - t) + S)) + c2;
        S = t;
    }
    a[c] = S + Cc;
}

static void launch_combine(int mode, const double* partials, int nblocks, int d, double* a,
                           double* b, cudaStream_t s) {
    const size_t sm = (size_t)nblocks * 2 * sizeof(double);
    if (sm <= 48 * 1024 && !getenv("MPK_COMBINE_THREAD"))
        norm_combine_warp_kernel<<<d, 32, sm, s>>>(mode, partials, nblocks, d, a, b);
    else
        norm_combine_kernel<<<(d + 127) / 128, 128, 0, s>>>(mode, partials, nblocks, d, a, b);
}

// Turn (global) aggregates into the map: 0: shift = sum / n; 1: scale = sqrt(ssq / n), 0 -> 1;
// 2: scale = max - min, 0 -> 1 (shift already holds min).
__global__ void norm_post_kernel(int mode, int d, double n_total, double* shift, double* scale) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= d) return;
    if (mode == 0) {
        shift[c] = shift[c] / n_total;
    } else if (mode == 1) {
        double sigma = sqrt(scale[c] / n_total);
        scale[c] = (sigma == 0.0) ? 1.0 : sigma;
    } else {
        double r = scale[c] - shift[c];
        scale[c] = (r == 0.0) ? 1.0 : r;
    }
}

// Correctly rounded a / b from r = RN(1/b) (Markstein: r within 1/2 ulp of 1/b, a r within
// 1 ulp of a/b  =>  q + r (a - b q) rounds to RN(a/b); the residual is exact by FMA). Checked
// on B200 against division for 2^28 random operand pairs of both the generic and the
// normalisation shapes (tools/div_check.cu). Non-finite or extreme quotients take the division.
MPK_DEV double div_rn(double a, double b, double r) {
    const double q0 = a * r;
    const double aq = fabs(q0);
    if (!(aq > 0x1p-960 && aq < 0x1p960)) return a / b;
    return fma(fma(-q0, b, a), r, q0);
}

template <typename W>
__global__ void norm_apply_kernel(const W* __restrict__ Xin, W* __restrict__ X, int64_t total,
                                  int d, const double* __restrict__ shift,
                                  const double* __restrict__ scale) {
    // x <- round_u((x - shift_c) / scale_c), fp64 arithmetic with a correctly rounded quotient
    // (as the oracle's O1); the column index is tracked incrementally (no 64-bit modulo). The
    // block caches the map and the reciprocals 1 / scale_c in shared memory (d <= kApplySmemD).
    constexpr int WORK = sizeof(W) == 8 ? KMEANS_FP64 : KMEANS_FP32;
    extern __shared__ double tsm[];
    const bool cached = d <= kApplySmemD;
    if (cached) {
        for (int c = threadIdx.x; c < d; c += blockDim.x) {
            tsm[c] = shift[c];
            tsm[d + c] = scale[c];
            tsm[2 * d + c] = 1.0 / scale[c];
        }
        __syncthreads();
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    int c = (int)(i % d);
    const int cstep = (int)(stride % d);
    // 4 elements per thread per step, loads first (memory-level parallelism)
    for (; i < total; i += 4 * stride) {
        W xv[4];
        int cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t iu = i + (int64_t)u * stride;
            xv[u] = iu < total ? Xin[iu] : (W)0;
            cc[u] = c;
            c += cstep;
            if (c >= d) c -= d;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t iu = i + (int64_t)u * stride;
            if (iu >= total) continue;
            const int cu = cc[u];
            double q;
            if (cached) q = div_rn((double)xv[u] - tsm[cu], tsm[d + cu], tsm[2 * d + cu]);
            else q = ((double)xv[u] - shift[cu]) / scale[cu];
            X[iu] = rounder<WORK>::from(q);
        }
    }
}

// ||x||^2 of one row's lane-local values, returned as an fp64 warp total. fp32 rows: each
// product x*x is split exactly (p + e, e = fma(x, x, -p)) and summed with a compensated fp32
// TwoSum, then converted once per lane: as accurate as an fp64 sum without one fp32->fp64
// conversion per element (the conversion unit bounded the per-element form).
MPK_DEV double lane_sumsq(const float* v, int cnt) {
    float s = 0.0f, c = 0.0f;
    for (int q = 0; q < cnt; ++q) {
        const float p = v[q] * v[q];
        const float e = fmaf(v[q], v[q], -p);
        const float t = s + p;
        const float z = t - s;
        c += (s - (t - z)) + (p - z) + e;
        s = t;
    }
    return warp_sum((double)s + (double)c);
}
MPK_DEV double lane_sumsq(const double* v, int cnt) {
    double s = 0.0;
    for (int q = 0; q < cnt; ++q) s = __dadd_rn(s, __dmul_rn(v[q], v[q]));
    return warp_sum(s);
}

// ------------------------------------------------------------------------------------------
// K1 / K3 prep: one warp per row, the row held in registers (up to 32 * kPrepVPL columns per
// pass), all loads of a row issued before use.
// ------------------------------------------------------------------------------------------
constexpr int kPrepVPL = 8;

template <typename W, int DIST>
__global__ void prep_kernel(const W* __restrict__ X, int64_t rows, int d, int d_pad, int guard,
                            W* __restrict__ norms, W* __restrict__ scales,
                            typename low_type<DIST>::T* __restrict__ Xl,
                            unsigned long long* __restrict__ census) {
    griddep_wait();                                   // launched with launch_pdl
    using L = typename low_type<DIST>::T;
    constexpr int WORK = sizeof(W) == 8 ? KMEANS_FP64 : KMEANS_FP32;
    constexpr bool same = (DIST == WORK);
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long n_nonfinite = 0, n_under = 0;
    for (int64_t i = warp; i < rows; i += nwarps) {
        const W* x = X + i * d;
        double acc = 0.0;
        W amax = (W)0;
        W v[kPrepVPL];
        const bool one_pass = d <= 32 * kPrepVPL;
        // pass 1: norm and infinity norm
        for (int c0 = 0; c0 < d; c0 += 32 * kPrepVPL) {
            int cnt = 0;
#pragma unroll
            for (int q = 0; q < kPrepVPL; ++q) {
                const int c = c0 + lane + 32 * q;
                v[q] = c < d ? x[c] : (W)0;
                if (c < d) cnt = q + 1;
            }
#pragma unroll
            for (int q = 0; q < kPrepVPL; ++q) amax = fmax(amax, fabs(v[q]));
            acc += lane_sumsq(v, cnt);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        W s = (W)1;
        if (guard && !same) s = guard_scale(amax, guard);
        if (lane == 0) {
            norms[i] = rounder<WORK>::from(acc);
            if (scales) scales[i] = s;
        }
        // pass 2: low-precision operands (from registers when the row fit in one pass)
        for (int c0 = 0; c0 < d_pad; c0 += 32 * kPrepVPL) {
            if (!one_pass || c0 > 0) {
#pragma unroll
                for (int q = 0; q < kPrepVPL; ++q) {
                    const int c = c0 + lane + 32 * q;
                    v[q] = c < d ? x[c] : (W)0;
                }
            }
#pragma unroll
            for (int q = 0; q < kPrepVPL; ++q) {
                const int c = c0 + lane + 32 * q;
                if (c >= d_pad) break;
                L o;
                if (c < d) {
                    const W vv = v[q];
                    const W qv = (s == (W)1) ? vv : vv / s;     // precision-u division (IEEE, RN)
                    o = rounder<DIST>::from(qv);
                    if (!same) {
                        if (is_nonfinite_low(o)) n_nonfinite++;
                        else if (qv != (W)0 && is_zero_or_subnormal_low(o)) n_under++;
                    }
                } else {
                    o = rounder<DIST>::from((W)0);
                }
                Xl[i * d_pad + c] = o;
            }
        }
    }
    if (census) {
        n_nonfinite = warp_sum(n_nonfinite);
        n_under = warp_sum(n_under);
        if (lane == 0 && (n_nonfinite | n_under)) {
            atomicAdd(&census[0], n_nonfinite);
            atomicAdd(&census[1], n_under);
        }
    }
}

template <typename S, int DST>
__global__ void cast_kernel(const S* __restrict__ in, int64_t count,
                            typename low_type<DST>::T* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = rounder<DST>::from(in[i]);
}

inline int grid_for(int64_t work_items, int threads, int per_sm = 8) {
    int64_t b = (work_items + threads - 1) / threads;
    int64_t cap = (int64_t)kNumSMs * per_sm;
    return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

static bool stats_vec_ok(const void* X, int d) {
    return !MPK_PREP_NO_VEC && d % 4 == 0 && d <= 4 * kStatThreads && ((uintptr_t)X & 15) == 0;
}

int norm_stats_blocks(int64_t n, int d) {
    int64_t b = (n * d + 8191) / 8192;
    if (b < 1) b = 1;
    if (b > kNumSMs * 4) b = kNumSMs * 4;
    return (int)b;
}

cudaError_t launch_norm_stats(int work, int norm, const void* X, int64_t n, int d,
                              double* partials, int nblocks, double* a, double* b,
                              cudaStream_t s) {
    launches_add(2);
    const int mode = norm == KMEANS_NORM_MINMAX ? 2 : 0;
    if (work == KMEANS_FP64)
        norm_col_stats_kernel<double><<<nblocks, kStatThreads, 0, s>>>(mode, (const double*)X, n,
                                                                       d, nullptr, partials);
    else if (stats_vec_ok(X, d))
        norm_col_stats_vec_kernel<<<nblocks, kStatThreads, 0, s>>>(mode, (const float*)X, n, d,
                                                                   nullptr, partials);
    else
        norm_col_stats_kernel<float><<<nblocks, kStatThreads, 0, s>>>(mode, (const float*)X, n,
                                                                      d, nullptr, partials);
    launch_combine(mode, partials, nblocks, d, a, b, s);
    return cudaGetLastError();
}

bool norm_moments_ok(int work, const void* X, int d) {
    return work == KMEANS_FP32 && stats_vec_ok(X, d);
}
cudaError_t launch_norm_moments(const void* X, int64_t n, int d, double* part1, double* part2,
                                int nblocks, double* kbuf, double* shift, double* scale,
                                double n_total, cudaStream_t s) {
    launches_add(4);
    norm_moments_vec_kernel<<<nblocks, kStatThreads, 0, s>>>((const float*)X, n, d, part1, part2,
                                                             kbuf);
    launch_combine(0, part1, nblocks, d, shift, nullptr, s);
    launch_combine(0, part2, nblocks, d, scale, nullptr, s);
    norm_post_moments_kernel<<<(d + 127) / 128, 128, 0, s>>>(d, n_total, kbuf, shift, scale);
    return cudaGetLastError();
}

cudaError_t launch_norm_ssq(int work, const void* X, int64_t n, int d, double* partials,
                            int nblocks, const double* mean, double* ssq, cudaStream_t s) {
    launches_add(2);
    if (work == KMEANS_FP64)
        norm_col_stats_kernel<double><<<nblocks, kStatThreads, 0, s>>>(1, (const double*)X, n, d,
                                                                       mean, partials);
    else if (stats_vec_ok(X, d))
        norm_col_stats_vec_kernel<<<nblocks, kStatThreads, 0, s>>>(1, (const float*)X, n, d,
                                                                   mean, partials);
    else
        norm_col_stats_kernel<float><<<nblocks, kStatThreads, 0, s>>>(1, (const float*)X, n, d,
                                                                      mean, partials);
    launch_combine(0, partials, nblocks, d, ssq, nullptr, s);
    return cudaGetLastError();
}

cudaError_t launch_norm_post(int mode, int d, double n_total, double* shift, double* scale,
                             cudaStream_t s) {
    launches_add(1);
    norm_post_kernel<<<(d + 127) / 128, 128, 0, s>>>(mode, d, n_total, shift, scale);
    return cudaGetLastError();
}

cudaError_t launch_norm_apply(int work, void* X, int64_t rows, int d, const double* shift,
                              const double* scale, cudaStream_t s, const void* Xin) {
    launches_add(1);
    int64_t total = rows * d;
    int g = grid_for(total, 256, 16);
    if (!Xin) Xin = X;   // in place
    const size_t sm = d <= kApplySmemD ? (size_t)3 * d * sizeof(double) : 0;
    if (work == KMEANS_FP64)
        norm_apply_kernel<double><<<g, 256, sm, s>>>((const double*)Xin, (double*)X, total, d,
                                                     shift, scale);
    else
        norm_apply_kernel<float><<<g, 256, sm, s>>>((const float*)Xin, (float*)X, total, d, shift,
                                                    scale);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K1 fast path (fp32 work, d <= 256): the same per-row arithmetic as prep_kernel, optionally
// fused with the normalisation O1 (x <- round_u((x - shift_c) / scale_c), correctly rounded
// quotient via div_rn) so that X is read once: each lane owns the columns lane + 32 q for every
// row (its transform values live in registers) and a warp takes two rows per step with all
// their loads issued first. Writes the normalised rows (NORM), ||x||^2, the guard scale and the
// low-precision operands.
// ------------------------------------------------------------------------------------------
template <int DIST, bool NORM, int Q>
MPK_DEV void prep_row_fast(float (&v)[Q], int64_t i, int lane, int d, int d_pad, int guard,
                           const double (&sh)[Q], const double (&sc)[Q], const double (&rc)[Q],
                           float* __restrict__ Xout, float* __restrict__ norms,
                           float* __restrict__ scales, typename low_type<DIST>::T* __restrict__ Xl,
                           unsigned& n_nonfinite, unsigned& n_under) {
    using L = typename low_type<DIST>::T;
    constexpr bool same = DIST == KMEANS_FP32;
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int c = lane + 32 * q;
        if (c < d) {
            cnt = q + 1;
            if (NORM) {
                v[q] = __double2float_rn(div_rn((double)v[q] - sh[q], sc[q], rc[q]));
                Xout[i * d + c] = v[q];
            }
        }
    }
    // lane_sumsq's arithmetic (exact fp32 products + TwoSum, q = 0..cnt-1), unrolled in
    // registers (the pointer/count form put the row array on the stack)
    float ss = 0.0f, cs = 0.0f;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (q < cnt) {
            const float p = v[q] * v[q];
            const float e = fmaf(v[q], v[q], -p);
            const float t = ss + p;
            const float z = t - ss;
            cs += (ss - (t - z)) + (p - z) + e;
            ss = t;
        }
    }
    const double acc = warp_sum((double)ss + (double)cs);
    float s = 1.0f;
    if (guard && !same) {
        float amax = 0.0f;
#pragma unroll
        for (int q = 0; q < Q; ++q) amax = fmaxf(amax, fabsf(v[q]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        s = guard_scale(amax, guard);
    }
    if (lane == 0) {
        norms[i] = __double2float_rn(acc);
        if (scales) scales[i] = s;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int c = lane + 32 * q;
        if (c >= d_pad) break;
        L o;
        if (c < d) {
            const float qv = (s == 1.0f) ? v[q] : v[q] / s;      // precision-u division (IEEE, RN)
            o = rounder<DIST>::from(qv);
            if (!same) {
                if (is_nonfinite_low(o)) n_nonfinite++;
                else if (qv != 0.0f && is_zero_or_subnormal_low(o)) n_under++;
            }
        } else {
            o = rounder<DIST>::from(0.0f);
        }
        Xl[i * d_pad + c] = o;
    }
}

template <int DIST, bool NORM, int Q, int RPS>
__global__ void __launch_bounds__(256)
prep_fast_kernel(const float* __restrict__ Xin, int64_t rows, int d, int d_pad, int guard,
                 float* __restrict__ norms, float* __restrict__ scales,
                 typename low_type<DIST>::T* __restrict__ Xl,
                 unsigned long long* __restrict__ census, float* __restrict__ Xout,
                 const double* __restrict__ shift, const double* __restrict__ scale) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double sh[Q], sc[Q], rc[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int c = lane + 32 * q;
        sh[q] = (NORM && c < d) ? shift[c] : 0.0;
        sc[q] = (NORM && c < d) ? scale[c] : 1.0;
        rc[q] = 1.0 / sc[q];
    }
    unsigned n_nonfinite = 0, n_under = 0;
    // RPS rows per warp per step (rows i + r * nwarps), all loads first
    for (int64_t i = warp; i < rows; i += RPS * nwarps) {
        float v[RPS][Q];
#pragma unroll
        for (int r = 0; r < RPS; ++r) {
            const int64_t ir = i + r * nwarps;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int c = lane + 32 * q;
                v[r][q] = (c < d && ir < rows) ? Xin[ir * d + c] : 0.0f;
            }
        }
#pragma unroll
        for (int r = 0; r < RPS; ++r) {
            const int64_t ir = i + r * nwarps;
            if (ir < rows)
                prep_row_fast<DIST, NORM, Q>(v[r], ir, lane, d, d_pad, guard, sh, sc, rc, Xout,
                                             norms, scales, Xl, n_nonfinite, n_under);
        }
    }
    if (census) {
        const unsigned long long a = warp_sum((unsigned long long)n_nonfinite);
        const unsigned long long b = warp_sum((unsigned long long)n_under);
        if (lane == 0 && (a | b)) {
            atomicAdd(&census[0], a);
            atomicAdd(&census[1], b);
        }
    }
}

// prep_fast_kernel for d <= 4 (the small-d path: images): one row per thread instead of one per
// warp (a warp per row left 29 of 32 lanes idle at d = 3). The same arithmetic per element as
// prep_row_fast, and ||x||^2 combined in the order prep_row_fast's warp sum gives when column c
// sits in lane c: ((x0^2 + x2^2) + (x1^2 + x3^2)), each square exact in fp64.
template <int DIST, bool NORM, int D>
__global__ void __launch_bounds__(256)
prep_small_kernel(const float* __restrict__ Xin, int64_t rows, int d_pad, int guard,
                  float* __restrict__ norms, float* __restrict__ scales,
                  typename low_type<DIST>::T* __restrict__ Xl,
                  unsigned long long* __restrict__ census, float* __restrict__ Xout,
                  const double* __restrict__ shift, const double* __restrict__ scale) {
    using L = typename low_type<DIST>::T;
    constexpr bool same = DIST == KMEANS_FP32;
    double sh[D], sc[D], rc[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
        sh[c] = NORM ? shift[c] : 0.0;
        sc[c] = NORM ? scale[c] : 1.0;
        rc[c] = 1.0 / sc[c];
    }
    unsigned n_nonfinite = 0, n_under = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += stride) {
        float v[D];
#pragma unroll
        for (int c = 0; c < D; ++c) v[c] = Xin[i * D + c];
        if (NORM) {
#pragma unroll
            for (int c = 0; c < D; ++c) {
                v[c] = __double2float_rn(div_rn((double)v[c] - sh[c], sc[c], rc[c]));
                Xout[i * D + c] = v[c];
            }
        }
        double sq[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int c = 0; c < D; ++c) {
            // prep_row_fast's per-lane TwoSum over one column: (double)p + (double)e = v^2 exactly
            const float p = v[c] * v[c];
            const float e = fmaf(v[c], v[c], -p);
            const float t = 0.0f + p;
            const float z = t - 0.0f;
            const float cs = 0.0f + ((0.0f - (t - z)) + (p - z) + e);
            sq[c] = (double)t + (double)cs;
        }
        const double acc = (sq[0] + sq[2]) + (sq[1] + sq[3]);
        float s = 1.0f;
        if (guard && !same) {
            float amax = 0.0f;
#pragma unroll
            for (int c = 0; c < D; ++c) amax = fmaxf(amax, fabsf(v[c]));
            s = guard_scale(amax, guard);
        }
        norms[i] = __double2float_rn(acc);
        if (scales) scales[i] = s;
        for (int c = 0; c < d_pad; ++c) {
            L o;
            if (c < D) {
                const float vc = c == 0 ? v[0] : c == 1 ? v[D > 1 ? 1 : 0] : c == 2 ? v[D > 2 ? 2 : 0] : v[D > 3 ? 3 : 0];
                const float qv = (s == 1.0f) ? vc : vc / s;     // precision-u division (IEEE, RN)
                o = rounder<DIST>::from(qv);
                if (!same) {
                    if (is_nonfinite_low(o)) n_nonfinite++;
                    else if (qv != 0.0f && is_zero_or_subnormal_low(o)) n_under++;
                }
            } else {
                o = rounder<DIST>::from(0.0f);
            }
            Xl[i * d_pad + c] = o;
        }
    }
    if (census) {
        const unsigned long long a = warp_sum((unsigned long long)n_nonfinite);
        const unsigned long long b = warp_sum((unsigned long long)n_under);
        if ((threadIdx.x & 31) == 0 && (a | b)) {
            atomicAdd(&census[0], a);
            atomicAdd(&census[1], b);
        }
    }
}

// Vectorised form of prep_fast_kernel for rows whose width is a multiple of 128 (d = d_pad,
// d <= 256): a lane owns V float4 column groups (columns 128 w + 4 lane + e), so each row costs
// one 16-byte load, one 16-byte store of the normalised row and one 4-element store of the
// operands per group, and the guard's division runs only for rows with s != 1 (a warp-uniform
// branch). Same arithmetic per element as prep_row_fast: the fp64 correctly rounded quotient
// rounded once to fp32, exact-product TwoSum partials of ||x||^2 summed in fp64 across lanes,
// x~ = round_l(x / s).
template <typename L> struct vec4_of;
template <> struct vec4_of<float> { using T = float4; };
template <> struct vec4_of<__half> { using T = uint2; };
template <> struct vec4_of<__nv_bfloat16> { using T = uint2; };
template <> struct vec4_of<e5m2_t> { using T = uint32_t; };
template <typename L>
MPK_DEV void store_low4(L* dst, const L (&o)[4]) {
    using T = typename vec4_of<L>::T;
    union { L l[4]; T t; } u;
#pragma unroll
    for (int e = 0; e < 4; ++e) u.l[e] = o[e];
    *reinterpret_cast<T*>(dst) = u.t;
}

template <int DIST, bool NORM, int V, int RPS>
__global__ void __launch_bounds__(256)
prep_vec_kernel(const float* __restrict__ Xin, int64_t rows, int d, int guard,
                float* __restrict__ norms, float* __restrict__ scales,
                typename low_type<DIST>::T* __restrict__ Xl,
                unsigned long long* __restrict__ census, float* __restrict__ Xout,
                const double* __restrict__ shift, const double* __restrict__ scale,
                unsigned* __restrict__ amax, int* __restrict__ flags) {
    using L = typename low_type<DIST>::T;
    constexpr bool same = DIST == KMEANS_FP32;
    const int lane = threadIdx.x & 31;
    // amax != nullptr: also the per-column max |x| of the (normalised) rows and flags[2] |= 1 on
    // a non-finite value, for the fixed-point update (k_update.cu FX) — saves it a pass over X
    unsigned mx[V][4] = {};
    unsigned bad = 0;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double sh[V][4], sc[V][4], rc[V][4];
#pragma unroll
    for (int w = 0; w < V; ++w)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = 128 * w + 4 * lane + e;
            sh[w][e] = NORM ? shift[c] : 0.0;
            sc[w][e] = NORM ? scale[c] : 1.0;
            rc[w][e] = 1.0 / sc[w][e];
        }
    unsigned n_nonfinite = 0, n_under = 0;
    for (int64_t i = warp; i < rows; i += RPS * nwarps) {
        float4 xv[RPS][V];
#pragma unroll
        for (int r = 0; r < RPS; ++r) {
            const int64_t ir = i + r * nwarps;
#pragma unroll
            for (int w = 0; w < V; ++w)
                xv[r][w] = ir < rows ? __ldg(reinterpret_cast<const float4*>(Xin + ir * d + 128 * w) + lane)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int r = 0; r < RPS; ++r) {
            const int64_t ir = i + r * nwarps;
            if (ir >= rows) break;
            float v[V][4];
#pragma unroll
            for (int w = 0; w < V; ++w) {
                v[w][0] = xv[r][w].x; v[w][1] = xv[r][w].y; v[w][2] = xv[r][w].z; v[w][3] = xv[r][w].w;
                if (NORM) {
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        v[w][e] = __double2float_rn(div_rn((double)v[w][e] - sh[w][e], sc[w][e], rc[w][e]));
                    reinterpret_cast<float4*>(Xout + ir * d + 128 * w)[lane] =
                        make_float4(v[w][0], v[w][1], v[w][2], v[w][3]);
                }
            }
            if (amax) {
#pragma unroll
                for (int w = 0; w < V; ++w)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float a = fabsf(v[w][e]);
                        if (!(a <= 3.402823466e38f)) bad = 1;
                        else mx[w][e] = max(mx[w][e], __float_as_uint(a));
                    }
            }
            float ss = 0.0f, cs = 0.0f;
#pragma unroll
            for (int w = 0; w < V; ++w)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float x = v[w][e];
                    const float p = x * x;
                    const float ep = fmaf(x, x, -p);
                    const float t = ss + p;
                    const float z = t - ss;
                    cs += (ss - (t - z)) + (p - z) + ep;
                    ss = t;
                }
            const double acc = warp_sum((double)ss + (double)cs);
            float s = 1.0f;
            if (guard && !same) {
                float amax = 0.0f;
#pragma unroll
                for (int w = 0; w < V; ++w)
#pragma unroll
                    for (int e = 0; e < 4; ++e) amax = fmaxf(amax, fabsf(v[w][e]));
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
                s = guard_scale(amax, guard);
                if (s != 1.0f) {          // warp-uniform: s is the row's
#pragma unroll
                    for (int w = 0; w < V; ++w)
#pragma unroll
                        for (int e = 0; e < 4; ++e) v[w][e] = v[w][e] / s;   // precision-u division
                }
            }
            if (lane == 0) {
                norms[ir] = __double2float_rn(acc);
                if (scales) scales[ir] = s;
            }
#pragma unroll
            for (int w = 0; w < V; ++w) {
                L o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    o[e] = rounder<DIST>::from(v[w][e]);
                    if (!same) {
                        if (is_nonfinite_low(o[e])) n_nonfinite++;
                        else if (v[w][e] != 0.0f && is_zero_or_subnormal_low(o[e])) n_under++;
                    }
                }
                store_low4<L>(Xl + ir * d + 128 * w + 4 * lane, o);
            }
        }
    }
    if (amax) {
        __shared__ unsigned smx[256];
        for (int t = threadIdx.x; t < d; t += blockDim.x) smx[t] = 0u;
        __syncthreads();
#pragma unroll
        for (int w = 0; w < V; ++w)
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (mx[w][e]) atomicMax(&smx[128 * w + 4 * lane + e], mx[w][e]);
        __syncthreads();
        for (int t = threadIdx.x; t < d; t += blockDim.x)
            if (smx[t]) atomicMax(&amax[t], smx[t]);
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&flags[2], 1);
    }
    if (census) {
        const unsigned long long a = warp_sum((unsigned long long)n_nonfinite);
        const unsigned long long b = warp_sum((unsigned long long)n_under);
        if (lane == 0 && (a | b)) {
            atomicAdd(&census[0], a);
            atomicAdd(&census[1], b);
        }
    }
}

// prep_vec_kernel for d = 4G (G = 8, 16: d = 32, 64): a group of G lanes per row, 32/G rows per
// warp side by side (a warp per row left the per-row work — shuffles, the fp64 division setup,
// the stores — amortised over one or two columns per lane: issue-bound, ~150 us per million rows).
// Same per-element arithmetic; ||x||^2 and the guard max reduced over the G lanes of the row.
template <int DIST, bool NORM, int RPS, int G>
__global__ void __launch_bounds__(256)
prep_vecg_kernel(const float* __restrict__ Xin, int64_t rows, int d, int guard,
                float* __restrict__ norms, float* __restrict__ scales,
                typename low_type<DIST>::T* __restrict__ Xl,
                unsigned long long* __restrict__ census, float* __restrict__ Xout,
                const double* __restrict__ shift, const double* __restrict__ scale,
                unsigned* __restrict__ amax, int* __restrict__ flags) {
    using L = typename low_type<DIST>::T;
    constexpr bool same = DIST == KMEANS_FP32;
    constexpr int V = 1, PW = 32 / G;
    const int wl = threadIdx.x & 31;
    const int lane = wl % G, sub = wl / G;
    // amax != nullptr: also the per-column max |x| of the (normalised) rows and flags[2] |= 1 on
    // a non-finite value, for the fixed-point update (k_update.cu FX) — saves it a pass over X
    unsigned mx[V][4] = {};
    unsigned bad = 0;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double sh[V][4], sc[V][4], rc[V][4];
#pragma unroll
    for (int w = 0; w < V; ++w)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = 128 * w + 4 * lane + e;
            sh[w][e] = NORM ? shift[c] : 0.0;
            sc[w][e] = NORM ? scale[c] : 1.0;
            rc[w][e] = 1.0 / sc[w][e];
        }
    unsigned n_nonfinite = 0, n_under = 0;
    const int64_t nrb = (rows + PW - 1) / PW;         // row-blocks of PW rows, one per warp step
    for (int64_t i = warp; i < nrb; i += RPS * nwarps) {
        float4 xv[RPS][V];
#pragma unroll
        for (int r = 0; r < RPS; ++r) {
            const int64_t ir = (i + r * nwarps) * PW + sub;
#pragma unroll
            for (int w = 0; w < V; ++w)
                xv[r][w] = ir < rows ? __ldg(reinterpret_cast<const float4*>(Xin + ir * d + 128 * w) + lane)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int r = 0; r < RPS; ++r) {
            if (i + r * nwarps >= nrb) break;         // warp-uniform
            const int64_t ir = (i + r * nwarps) * PW + sub;
            const bool ok = ir < rows;
            float v[V][4];
#pragma unroll
            for (int w = 0; w < V; ++w) {
                v[w][0] = xv[r][w].x; v[w][1] = xv[r][w].y; v[w][2] = xv[r][w].z; v[w][3] = xv[r][w].w;
                if (NORM) {
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        v[w][e] = __double2float_rn(div_rn((double)v[w][e] - sh[w][e], sc[w][e], rc[w][e]));
                    if (ok) reinterpret_cast<float4*>(Xout + ir * d + 128 * w)[lane] =
                        make_float4(v[w][0], v[w][1], v[w][2], v[w][3]);
                }
            }
            if (amax && ok) {
#pragma unroll
                for (int w = 0; w < V; ++w)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float a = fabsf(v[w][e]);
                        if (!(a <= 3.402823466e38f)) bad = 1;
                        else mx[w][e] = max(mx[w][e], __float_as_uint(a));
                    }
            }
            float ss = 0.0f, cs = 0.0f;
#pragma unroll
            for (int w = 0; w < V; ++w)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float x = v[w][e];
                    const float p = x * x;
                    const float ep = fmaf(x, x, -p);
                    const float t = ss + p;
                    const float z = t - ss;
                    cs += (ss - (t - z)) + (p - z) + ep;
                    ss = t;
                }
            double acc = (double)ss + (double)cs;
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            float s = 1.0f;
            if (guard && !same) {
                float amax = 0.0f;
#pragma unroll
                for (int w = 0; w < V; ++w)
#pragma unroll
                    for (int e = 0; e < 4; ++e) amax = fmaxf(amax, fabsf(v[w][e]));
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
                s = guard_scale(amax, guard);
                if (s != 1.0f) {          // group-uniform: s is the row's
#pragma unroll
                    for (int w = 0; w < V; ++w)
#pragma unroll
                        for (int e = 0; e < 4; ++e) v[w][e] = v[w][e] / s;   // precision-u division
                }
            }
            if (!ok) continue;
            if (lane == 0) {
                norms[ir] = __double2float_rn(acc);
                if (scales) scales[ir] = s;
            }
#pragma unroll
            for (int w = 0; w < V; ++w) {
                L o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    o[e] = rounder<DIST>::from(v[w][e]);
                    if (!same) {
                        if (is_nonfinite_low(o[e])) n_nonfinite++;
                        else if (v[w][e] != 0.0f && is_zero_or_subnormal_low(o[e])) n_under++;
                    }
                }
                store_low4<L>(Xl + ir * d + 128 * w + 4 * lane, o);
            }
        }
    }
    if (amax) {
        __shared__ unsigned smx[256];
        for (int t = threadIdx.x; t < d; t += blockDim.x) smx[t] = 0u;
        __syncthreads();
#pragma unroll
        for (int w = 0; w < V; ++w)
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (mx[w][e]) atomicMax(&smx[128 * w + 4 * lane + e], mx[w][e]);
        __syncthreads();
        for (int t = threadIdx.x; t < d; t += blockDim.x)
            if (smx[t]) atomicMax(&amax[t], smx[t]);
        if (__any_sync(0xffffffffu, bad) && wl == 0) atomicOr(&flags[2], 1);
    }
    if (census) {
        const unsigned long long a = warp_sum((unsigned long long)n_nonfinite);
        const unsigned long long b = warp_sum((unsigned long long)n_under);
        if (wl == 0 && (a | b)) {
            atomicAdd(&census[0], a);
            atomicAdd(&census[1], b);
        }
    }
}

template <int DIST>
static void prep_fast_launch(const float* Xin, int64_t rows, int d, int d_pad, int guard,
                             float* norms, float* scales, void* Xl, unsigned long long* census,
                             float* Xout, const double* shift, const double* scale,
                             cudaStream_t s, unsigned* amax, int* flags, bool* amax_done) {
    using L = typename low_type<DIST>::T;
    if (d <= 4 && d_pad <= 8 && !getenv("MPK_PREP_NO_SMALL")) {
        // one row per thread (small d); MPK_PREP_NO_SMALL=1: prep_fast_kernel (A/B, tests)
        const int gs = grid_for(rows, 256, 8);
#define PREP_SMALL(DV)                                                                              \
        if (shift) prep_small_kernel<DIST, true, DV><<<gs, 256, 0, s>>>(Xin, rows, d_pad, guard, norms, \
                                     scales, (L*)Xl, census, Xout, shift, scale);                   \
        else prep_small_kernel<DIST, false, DV><<<gs, 256, 0, s>>>(Xin, rows, d_pad, guard, norms,     \
                                     scales, (L*)Xl, census, Xout, shift, scale);
        switch (d) {
            case 1: PREP_SMALL(1) break;
            case 2: PREP_SMALL(2) break;
            case 3: PREP_SMALL(3) break;
            default: PREP_SMALL(4) break;
        }
#undef PREP_SMALL
        return;
    }
    const int g = grid_for(rows * 8, 256, 8);
    const bool aligned = (((uintptr_t)Xin | (uintptr_t)Xout | (uintptr_t)Xl) & 15) == 0;
    if (d == d_pad && (d == 128 || d == 256) && aligned && !MPK_PREP_NO_VEC) {
        if (d == 128) {
            if (shift)
                prep_vec_kernel<DIST, true, 1, 4><<<g, 256, 0, s>>>(Xin, rows, d, guard, norms, scales,
                                                                    (L*)Xl, census, Xout, shift, scale, amax, flags);
            else
                prep_vec_kernel<DIST, false, 1, 4><<<g, 256, 0, s>>>(Xin, rows, d, guard, norms, scales,
                                                                     (L*)Xl, census, Xout, shift, scale, amax, flags);
        } else {
            if (shift)
                prep_vec_kernel<DIST, true, 2, 2><<<g, 256, 0, s>>>(Xin, rows, d, guard, norms, scales,
                                                                    (L*)Xl, census, Xout, shift, scale, amax, flags);
            else
                prep_vec_kernel<DIST, false, 2, 2><<<g, 256, 0, s>>>(Xin, rows, d, guard, norms, scales,
                                                                     (L*)Xl, census, Xout, shift, scale, amax, flags);
        }
        if (amax_done) *amax_done = amax != nullptr;
        return;
    }
    if (d == d_pad && (d == 32 || d == 64) && aligned && !getenv("MPK_PREP_NO_VECG")) {
        // MPK_PREP_NO_VECG=1: prep_fast_kernel (A/B)
        if (d == 32) {
            if (shift) prep_vecg_kernel<DIST, true, 4, 8><<<g, 256, 0, s>>>(Xin, rows, d, guard, norms, scales, (L*)Xl, census, Xout, shift, scale, amax, flags);
            else prep_vecg_kernel<DIST, false, 4, 8><<<g, 256, 0, s>>>(Xin, rows, d, guard, norms, scales, (L*)Xl, census, Xout, shift, scale, amax, flags);
        } else {
            if (shift) prep_vecg_kernel<DIST, true, 4, 16><<<g, 256, 0, s>>>(Xin, rows, d, guard, norms, scales, (L*)Xl, census, Xout, shift, scale, amax, flags);
            else prep_vecg_kernel<DIST, false, 4, 16><<<g, 256, 0, s>>>(Xin, rows, d, guard, norms, scales, (L*)Xl, census, Xout, shift, scale, amax, flags);
        }
        if (amax_done) *amax_done = amax != nullptr;
        return;
    }
    // d_pad columns of Xl must be covered by the lane's Q slots too
    const int w = d_pad > d ? d_pad : d;
    if (w <= 128) {
        if (shift)
            prep_fast_kernel<DIST, true, 4, 4><<<g, 256, 0, s>>>(Xin, rows, d, d_pad, guard, norms,
                                                                 scales, (L*)Xl, census, Xout, shift, scale);
        else
            prep_fast_kernel<DIST, false, 4, 4><<<g, 256, 0, s>>>(Xin, rows, d, d_pad, guard, norms,
                                                                  scales, (L*)Xl, census, Xout, shift, scale);
    } else {
        if (shift)
            prep_fast_kernel<DIST, true, 8, 2><<<g, 256, 0, s>>>(Xin, rows, d, d_pad, guard, norms,
                                                                 scales, (L*)Xl, census, Xout, shift, scale);
        else
            prep_fast_kernel<DIST, false, 8, 2><<<g, 256, 0, s>>>(Xin, rows, d, d_pad, guard, norms,
                                                                  scales, (L*)Xl, census, Xout, shift, scale);
    }
}

template <typename W>
static cudaError_t prep_dispatch(int dist, const W* X, int64_t rows, int d, int d_pad, int guard,
                                 W* norms, W* scales, void* Xl, unsigned long long* census,
                                 cudaStream_t s) {
    int g = grid_for(rows * 32, 256, 16);
    switch (dist) {
        case KMEANS_FP64:
            launch_pdl(prep_kernel<W, KMEANS_FP64>, dim3(g), dim3(256), 0, s, X, rows, d, d_pad, guard, norms, scales,
                                                         (double*)Xl, census);
            break;
        case KMEANS_FP32:
            launch_pdl(prep_kernel<W, KMEANS_FP32>, dim3(g), dim3(256), 0, s, X, rows, d, d_pad, guard, norms, scales,
                                                         (float*)Xl, census);
            break;
        case KMEANS_FP16:
            launch_pdl(prep_kernel<W, KMEANS_FP16>, dim3(g), dim3(256), 0, s, X, rows, d, d_pad, guard, norms, scales,
                                                         (__half*)Xl, census);
            break;
        case KMEANS_BF16:
            launch_pdl(prep_kernel<W, KMEANS_BF16>, dim3(g), dim3(256), 0, s, X, rows, d, d_pad, guard, norms, scales,
                                                         (__nv_bfloat16*)Xl, census);
            break;
        case KMEANS_E5M2:
            launch_pdl(prep_kernel<W, KMEANS_E5M2>, dim3(g), dim3(256), 0, s, X, rows, d, d_pad, guard, norms, scales,
                                                         (e5m2_t*)Xl, census);
            break;
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

bool prep_fast_ok(int work, int d) { return work == KMEANS_FP32 && d <= 256; }
// (d_pad <= 256 as well: tc_dpad / the SIMT paddings never exceed 256 when d <= 256)

cudaError_t launch_prep_fast(int dist, const void* Xin, int64_t rows, int d, int d_pad, int guard,
                             void* norms, void* scales, void* Xl, unsigned long long* census,
                             void* Xout, const double* shift, const double* scale,
                             cudaStream_t s, unsigned* amax, int* flags, bool* amax_done) {
    launches_add(1);
    if (amax_done) *amax_done = false;
    if (rows <= 0) return cudaSuccess;
    const float* xi = (const float*)Xin;
    float* xo = (float*)Xout;
    float* nr = (float*)norms;
    float* sc = (float*)scales;
    switch (dist) {
        case KMEANS_FP32: prep_fast_launch<KMEANS_FP32>(xi, rows, d, d_pad, guard, nr, sc, Xl, census, xo, shift, scale, s, amax, flags, amax_done); break;
        case KMEANS_FP16: prep_fast_launch<KMEANS_FP16>(xi, rows, d, d_pad, guard, nr, sc, Xl, census, xo, shift, scale, s, amax, flags, amax_done); break;
        case KMEANS_BF16: prep_fast_launch<KMEANS_BF16>(xi, rows, d, d_pad, guard, nr, sc, Xl, census, xo, shift, scale, s, amax, flags, amax_done); break;
        case KMEANS_E5M2: prep_fast_launch<KMEANS_E5M2>(xi, rows, d, d_pad, guard, nr, sc, Xl, census, xo, shift, scale, s, amax, flags, amax_done); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_prep(int work, int dist, const void* Xw, int64_t rows, int d, int d_pad,
                        int guard, void* norms, void* scales, void* Xl,
                        unsigned long long* census, cudaStream_t s) {
    launches_add(1);
    if (rows <= 0) return cudaSuccess;
    if (work == KMEANS_FP64)
        return prep_dispatch<double>(dist, (const double*)Xw, rows, d, d_pad, guard,
                                     (double*)norms, (double*)scales, Xl, census, s);
    // point rows of fp32 work with d = 32 / 64 / 128 / 256 (the final pass's fp16 operands, the
    // rows of kmeans_assign): the lane-group / float4 kernels instead of a warp per row (E5M2 at
    // C5 prepares its final-pass operands here). Centroid rows (k of them, every iteration)
    // stay on prep_kernel. MPK_PREP_GENERIC=1: prep_kernel for all (A/B).
    if (rows >= 65536 && d == d_pad && (d == 32 || d == 64 || d == 128 || d == 256) &&
        (((uintptr_t)Xw | (uintptr_t)Xl) & 15) == 0 && !getenv("MPK_PREP_GENERIC")) {
        const float* xi = (const float*)Xw;
        float* nr = (float*)norms;
        float* sc = (float*)scales;
        switch (dist) {
            case KMEANS_FP32: prep_fast_launch<KMEANS_FP32>(xi, rows, d, d_pad, guard, nr, sc, Xl, census, nullptr, nullptr, nullptr, s, nullptr, nullptr, nullptr); break;
            case KMEANS_FP16: prep_fast_launch<KMEANS_FP16>(xi, rows, d, d_pad, guard, nr, sc, Xl, census, nullptr, nullptr, nullptr, s, nullptr, nullptr, nullptr); break;
            case KMEANS_BF16: prep_fast_launch<KMEANS_BF16>(xi, rows, d, d_pad, guard, nr, sc, Xl, census, nullptr, nullptr, nullptr, s, nullptr, nullptr, nullptr); break;
            case KMEANS_E5M2: prep_fast_launch<KMEANS_E5M2>(xi, rows, d, d_pad, guard, nr, sc, Xl, census, nullptr, nullptr, nullptr, s, nullptr, nullptr, nullptr); break;
            default: return cudaErrorInvalidValue;
        }
        return cudaGetLastError();
    }
    return prep_dispatch<float>(dist, (const float*)Xw, rows, d, d_pad, guard, (float*)norms,
                                (float*)scales, Xl, census, s);
}

template <typename S>
static cudaError_t cast_dispatch(int dst, const S* in, int64_t count, void* out, cudaStream_t s) {
    int g = grid_for(count, 256, 16);
    switch (dst) {
        case KMEANS_FP32: cast_kernel<S, KMEANS_FP32><<<g, 256, 0, s>>>(in, count, (float*)out); break;
        case KMEANS_FP16: cast_kernel<S, KMEANS_FP16><<<g, 256, 0, s>>>(in, count, (__half*)out); break;
        case KMEANS_BF16:
            cast_kernel<S, KMEANS_BF16><<<g, 256, 0, s>>>(in, count, (__nv_bfloat16*)out);
            break;
        case KMEANS_E5M2: cast_kernel<S, KMEANS_E5M2><<<g, 256, 0, s>>>(in, count, (e5m2_t*)out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_cast(int src, int dst, const void* in, int64_t count, void* out,
                        cudaStream_t s) {
    launches_add(1);
    if (count <= 0) return cudaSuccess;
    if (src == KMEANS_FP64) return cast_dispatch<double>(dst, (const double*)in, count, out, s);
    if (src == KMEANS_FP32) return cast_dispatch<float>(dst, (const float*)in, count, out, s);
    return cudaErrorInvalidValue;
}

}  // namespace mpk
