// k_smalld_loop.cu — K5g: a whole Lloyd iteration of the small-d path (d <= 4, k <= 8: the
// image-segmentation workload; configs C1, C2) in ONE kernel launch, for
// one rank:
//   A3  centroid prep (||c||^2, Alg 4 scale, c~ = round_l(c / s)) — every
//       block derives it from the k x d centres in shared memory (<= 32 values);
//   A4  expanded distance + argmin (eq:dist-eval PAPER.md:193-196, Alg 3 step 3 PAPER.md:546);
//   A5  per-cluster sums and counts (eq:center PAPER.md:421-427) in fp64, per block, written as
//       block partials (no floating-point atomics: deterministic);
//   A7  the LAST block to finish (threadfence + ticket) reduces the partials in a fixed order,
//       forms c_j = round_u(sum_j / count_j) (empty clusters keep c_j), the shift, Thm 5.3's
//       terms, the trace record, and the stopping rule of Alg 3 step 6
//       (no label changed, or ||C_t+1 - C_t|| <= tol).
// A launch that finds the stop flag set returns at once, so the host can enqueue (or replay as
// a CUDA graph) a chunk of iterations and poll the flag once per chunk: the iteration costs one
// launch instead of three launches, a memset and a host round trip.
// Rows are staged through shared memory in tiles of kTileRows rows with 16-byte loads.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace mpk {

namespace {

constexpr int LD = 4, LK = 8, LT = 256, kTileRows = 1024;
constexpr int NV = LK * LD + LK + 2;   // sums, counts, sse, changed

template <typename W, int DIST>
__global__ void __launch_bounds__(LT)
smalld_iter_kernel(Problem p, const W* __restrict__ X, W* __restrict__ C,
                   int32_t* __restrict__ labels, double* __restrict__ part,
                   LoopState* __restrict__ st, IterRec* __restrict__ trace,
                   unsigned long long* __restrict__ census) {
    using AT = typename std::conditional<DIST == KMEANS_FP64, double, float>::type;
    using LowT = typename low_type<DIST>::T;
    constexpr int WORK = sizeof(W) == 8 ? KMEANS_FP64 : KMEANS_FP32;
    constexpr bool same = (DIST == WORK);
    if (*(volatile int*)&st->stop) return;            // converged: this launch is a no-op
    __shared__ AT cl_s[LK][LD];
    __shared__ W cn_s[LK], sc_s[LK];
    __shared__ __align__(16) W xs[kTileRows * LD];
    __shared__ double red[LT / 32][NV];
    __shared__ int is_last;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int d = p.d, k = p.k;

    // ---- A3: centroid prep (the arithmetic of prep_kernel: exact squares summed in the warp
    // reduction's order, infinity-norm scale, one rounding of c / s) -------------------------
    if (w < k) {
        const W v = lane < d ? C[w * d + lane] : (W)0;
        const double sq = (double)v * (double)v;       // exact for fp32; fp64: one rounding
        double acc = lane < d ? sq : 0.0;
        W amax = fabs(v);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            acc += __shfl_xor_sync(0xffffffffu, acc, o);
            amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        }
        W s = (W)1;
        if (p.guard && !same) s = (amax == (W)0 || isnan(amax)) ? (W)1 : amax;
        unsigned long long nf = 0, nu = 0;
        if (lane < LD) {
            AT o = (AT)0;
            if (lane < d) {
                const W q = (s == (W)1) ? v : v / s;
                const LowT r = rounder<DIST>::from(q);
                o = (AT)widen(r);
                if (!same) {
                    if (is_nonfinite_low(r)) nf = 1;
                    else if (q != (W)0 && is_zero_or_subnormal_low(r)) nu = 1;
                }
            }
            cl_s[w][lane] = o;
        }
        if (lane == 0) {
            cn_s[w] = rounder<WORK>::from(acc);
            sc_s[w] = s;
        }
        if (blockIdx.x == 0 && census) {
            nf = warp_sum(nf);
            nu = warp_sum(nu);
            if (lane == 0 && (nf | nu)) { atomicAdd(&census[0], nf); atomicAdd(&census[1], nu); }
        }
    }
    __syncthreads();

    double sums[LK][LD];
    double cnts[LK];
#pragma unroll
    for (int j = 0; j < LK; ++j) {
        cnts[j] = 0.0;
#pragma unroll
        for (int t = 0; t < LD; ++t) sums[j][t] = 0.0;
    }
    double my_sse = 0.0, my_changed = 0.0;

    // ---- A4 + A5 over this block's tiles -----------------------------------------------------
    const int64_t ntiles = (p.n + kTileRows - 1) / kTileRows;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t r0 = tile * kTileRows;
        const int rows = (int)std::min<int64_t>(kTileRows, p.n - r0);
        const int64_t e0 = r0 * d;
        const int ne = rows * d;
        __syncthreads();                               // xs reuse
        constexpr int VW = 16 / sizeof(W);             // elements per 16-byte load
        const W* src = X + e0;
        if ((((uintptr_t)src) & 15) == 0) {
            const int nv = ne / VW;
            for (int q = tid; q < nv; q += LT)
                reinterpret_cast<int4*>(xs)[q] = __ldg(reinterpret_cast<const int4*>(src) + q);
            for (int q = nv * VW + tid; q < ne; q += LT) xs[q] = src[q];
        } else {
            for (int q = tid; q < ne; q += LT) xs[q] = src[q];
        }
        __syncthreads();
        for (int r = tid; r < rows; r += LT) {
            const int64_t i = r0 + r;
            W x[LD];
            double nrm = 0.0, amax = 0.0;
#pragma unroll
            for (int t = 0; t < LD; ++t) {
                x[t] = t < d ? xs[r * d + t] : (W)0;
                const double v = (double)x[t];
                nrm = __dadd_rn(nrm, __dmul_rn(v, v));
                amax = fmax(amax, fabs(v));
            }
            const W xn = rounder<WORK>::from(nrm);
            W s = (W)1;
            if (p.guard && !same) s = (amax == 0.0 || isnan(amax)) ? (W)1 : (W)amax;
            AT xl[LD];
#pragma unroll
            for (int t = 0; t < LD; ++t) {
                const W q = (s == (W)1) ? x[t] : x[t] / s;
                xl[t] = (AT)widen(rounder<DIST>::from(q));
            }
            W best = (W)INFINITY;
            int bj = 0;
#pragma unroll
            for (int j = 0; j < LK; ++j) {
                if (j < k) {
                    AT dot = (AT)0;
#pragma unroll
                    for (int t = 0; t < LD; ++t) dot = fma(xl[t], cl_s[j][t], dot);
                    const W v = fma((W)-2 * (s * sc_s[j]), (W)dot, cn_s[j]);
                    if (v < best) { best = v; bj = j; }
                }
            }
            if (labels[i] != bj) my_changed += 1.0;
            labels[i] = bj;
            const double md = (double)xn + (double)best;
            my_sse += md > 0.0 ? md : 0.0;
#pragma unroll
            for (int j = 0; j < LK; ++j) {
                const bool hit = (bj == j);
                cnts[j] += hit ? 1.0 : 0.0;
#pragma unroll
                for (int t = 0; t < LD; ++t) sums[j][t] += hit ? (double)x[t] : 0.0;
            }
        }
    }
    // ---- block partial (warp shuffles, then warps in order) ---------------------------------
#pragma unroll
    for (int j = 0; j < LK; ++j) {
#pragma unroll
        for (int t = 0; t < LD; ++t) {
            const double v = warp_sum(sums[j][t]);
            if (lane == 0) red[w][j * LD + t] = v;
        }
        const double c = warp_sum(cnts[j]);
        if (lane == 0) red[w][LK * LD + j] = c;
    }
    my_sse = warp_sum(my_sse);
    my_changed = warp_sum(my_changed);
    if (lane == 0) { red[w][NV - 2] = my_sse; red[w][NV - 1] = my_changed; }
    __syncthreads();
    if (tid < NV) {
        double a = 0.0;
#pragma unroll
        for (int q = 0; q < LT / 32; ++q) a += red[q][tid];
        part[(size_t)blockIdx.x * NV + tid] = a;
    }
    // ---- the last block finalises -------------------------------------------------------------
    __threadfence();
    __syncthreads();
    if (tid == 0) is_last = atomicAdd(&st->counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    // partials of all blocks, summed in block order (thread per value; at most a few hundred
    // blocks), into red[0][.]
    if (tid < NV) {
        double a = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) a += __ldcg(part + (size_t)b * NV + tid);
        red[0][tid] = a;
    }
    __syncthreads();
    if (w == 0) {
        // one lane per (cluster, feature): new centre, shift and Thm 5.3 terms
        double num = 0.0, den = 0.0, sh = 0.0, empty = 0.0, rmax = 0.0;
        for (int j = 0; j < k; ++j) {
            const double c = red[0][LK * LD + j];
            double nm = 0.0, dn = 0.0;
            if (lane < d) {
                const int idx = j * d + lane;
                const W old = C[idx];
                W nw = old;
                if (c > 0.0) nw = rounder<WORK>::from(red[0][j * LD + lane] / c);
                const double df = (double)nw - (double)old;
                nm = df * df;
                dn = fabs(df) * fabs((double)nw);
                C[idx] = nw;
            }
            nm = warp_sum(nm);
            dn = warp_sum(dn);
            sh += nm;
            if (c == 0.0) empty += 1.0;
            if (nm > 0.0 && dn > 0.0) rmax = fmax(rmax, 2.0 * dn / nm);
        }
        (void)num; (void)den;
        if (lane == 0) {
            const int it = st->iter;
            IterRec* rec = trace + (it < KMEANS_MAX_TRACE - 1 ? it : KMEANS_MAX_TRACE - 1);
            rec->sse = red[0][NV - 2];
            rec->shift2 = sh;
            rec->changed = red[0][NV - 1];
            rec->empty = empty;
            rec->ub_inv = rmax;
            st->iter = it + 1;
            if (st->tol >= 0.0 && (red[0][NV - 1] == 0.0 || sqrt(sh) <= st->tol)) {
                st->stop = 1;
                st->converged = 1;
            }
            st->counter = 0;
            __threadfence();
        }
    }
}

template <typename W, int DIST>
cudaError_t launch_t(const Problem& p, const void* X, void* C, int32_t* labels, double* part,
                     int grid, LoopState* st, IterRec* trace, unsigned long long* census,
                     cudaStream_t s) {
    smalld_iter_kernel<W, DIST><<<grid, LT, 0, s>>>(p, (const W*)X, (W*)C, labels, part, st, trace,
                                                    census);
    return cudaGetLastError();
}

}  // namespace

bool smalld_loop_supported(int d, int k) { return d <= LD && k <= LK; }

int smalld_loop_grid(int64_t n) {
    const int64_t tiles = (n + kTileRows - 1) / kTileRows;
    return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, kNumSMs));
}

size_t smalld_loop_part_bytes(int64_t n) { return (size_t)smalld_loop_grid(n) * NV * sizeof(double); }

cudaError_t launch_smalld_iter(int work, int dist, const Problem& p, const void* Xw, void* Cw,
                               int32_t* labels, double* part, LoopState* st, IterRec* trace,
                               unsigned long long* census, cudaStream_t s) {
    launches_add(1);
    const int g = smalld_loop_grid(p.n);
#define MPK_SL(W)                                                                                  \
    switch (dist) {                                                                                \
        case KMEANS_FP64: return launch_t<W, KMEANS_FP64>(p, Xw, Cw, labels, part, g, st, trace, census, s); \
        case KMEANS_FP32: return launch_t<W, KMEANS_FP32>(p, Xw, Cw, labels, part, g, st, trace, census, s); \
        case KMEANS_FP16: return launch_t<W, KMEANS_FP16>(p, Xw, Cw, labels, part, g, st, trace, census, s); \
        case KMEANS_BF16: return launch_t<W, KMEANS_BF16>(p, Xw, Cw, labels, part, g, st, trace, census, s); \
        case KMEANS_E5M2: return launch_t<W, KMEANS_E5M2>(p, Xw, Cw, labels, part, g, st, trace, census, s); \
    }
    if (work == KMEANS_FP64) {
        MPK_SL(double)
    } else {
        if (dist == KMEANS_FP64) return cudaErrorInvalidValue;
        MPK_SL(float)
    }
#undef MPK_SL
    return cudaErrorInvalidValue;
}

}  // namespace mpk
