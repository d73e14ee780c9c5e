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
// K5p (PERSIST = true, the default when the rows fit): the same iteration, all max_iter of them
// in ONE cooperative launch. Each block keeps its tiles resident in shared memory (loaded once)
// with the loop-invariant operands of Alg 3 step 2 (x~, s, ||x||^2; formed in the first
// iteration); per iteration one grid barrier (a monotone arrival counter), after which EVERY
// block reduces the double-buffered partials in the same fixed order and forms the same new
// centres (no last-block tail); block 0 publishes C and the trace record. Measured at C2 (512^2
// image): 12.1 -> 8.5 us per iteration; the remaining time is the tile's row loop at 8 warps per
// SM (~7k cycles) and the barrier / reduction / finalize latency chain (~7k cycles).
// Rows (and the previous labels) stream through shared memory in a ring of kStages tiles of
// kTileRows rows filled by 1-D bulk copies (the TMA engine), so the next tiles' HBM reads overlap
// this tile's arithmetic; each thread's rows of up to 4 tiles (<= 32 rows) are summed in fp32, then
// converted to fp64 and reduced by a warp tree into the warp's fp64 totals (DESIGN.md reading
// R1 / R11): a fixed order.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace mpk {

namespace {

constexpr int LD = 4, LK = 8, LT = 256;
static_assert(LK * LD == 32, "the finalize maps (cluster, feature) onto the 32 lanes of a warp");
#ifndef MPK_SL_TILE
#define MPK_SL_TILE 2048
#endif
// K5g blocks per SM (registers capped at 128 per thread): the streaming kernel is latency-bound
// on its row loop, so a second block per SM hides it (4096^2 image: 186 -> 129 us per iteration).
// fp64 work keeps one (its 3-stage ring of fp64 rows fills the shared memory; no register cap).
constexpr int kK5gBlocksPerSM = 2;
constexpr int kTileRows = MPK_SL_TILE;   // rows per pipeline stage (8 per thread)
constexpr int kStages = 3;           // tiles in flight per block (bulk copies)
constexpr int kMaxResident = 8;
#ifndef MPK_K5P_TRACE
#define MPK_K5P_TRACE 0                  // debug: per-phase clock64 of blocks 0 and last (printf)
#endif      // K5p: tiles per block kept in shared memory
constexpr int kFlushTiles = 4;       // tiles per per-thread partial (<= 32 rows)
constexpr int NV = LK * LD + LK + 2;   // sums, counts, sse, changed
constexpr int kRedGroups = LT / NV;    // the last block reduces the partials in this many groups

MPK_DEV uint32_t sm_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
MPK_DEV void bar_init(uint32_t b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c) : "memory");
}
MPK_DEV void bar_expect(uint32_t b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                 : "memory");
}
MPK_DEV void bar_wait(uint32_t b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra W_%=;\n\t}" ::"r"(b),
        "r"(parity)
        : "memory");
}
// GPU-scope loads of the loop state (a volatile load is system scope: LDG.STRONG.SYS, slow)
MPK_DEV int ld_relaxed_gpu(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
MPK_DEV unsigned ld_relaxed_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on the mbarrier
MPK_DEV void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// D: the feature count (exact, 1..4); KT: the centroid loop bound (4 or 8, >= k).
// PERSIST (K5p): all max_iter iterations in one cooperative launch; every tile of the block stays
// in shared memory (stage m = tile m, loaded once), and the iterations are separated by a grid
// barrier that the last block releases after its finalize (same arithmetic, same order as K5g).
template <typename W, int DIST, int D, int KT, bool PERSIST>
__global__ void __launch_bounds__(LT, (PERSIST || sizeof(W) == 8 || DIST == KMEANS_FP64) ? 1 : kK5gBlocksPerSM)
smalld_iter_kernel(Problem p, const W* __restrict__ X, W* __restrict__ C,
                   int32_t* __restrict__ labels, double* __restrict__ part,
                   LoopState* __restrict__ st, IterRec* __restrict__ trace,
                   unsigned long long* __restrict__ census, int max_iter) {
    using AT = typename std::conditional<DIST == KMEANS_FP64, double, float>::type;
    using LowT = typename low_type<DIST>::T;
    constexpr int WORK = sizeof(W) == 8 ? KMEANS_FP64 : KMEANS_FP32;
    constexpr bool same = (DIST == WORK);
    if (!PERSIST && ld_relaxed_gpu(&st->stop)) return;   // converged: this launch is a no-op
    const double tol = st->tol;
    extern __shared__ __align__(128) unsigned char dsm[];
    const int d = p.d, k = p.k;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t ntiles = (p.n + kTileRows - 1) / kTileRows;
    const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int nst = PERSIST ? (int)my_tiles : kStages;   // stages (K5p: one per tile, resident)
    const size_t xbytes = (size_t)kTileRows * d * sizeof(W);
    W* xs0 = reinterpret_cast<W*>(dsm);                                   // [nst][rows*d]
    // K5p: the loop-invariant point operands (Alg 3 step 2: x~ = round_l(x / s), s, ||x||^2),
    // formed in the first iteration and kept next to the rows
    AT* xl0 = reinterpret_cast<AT*>(dsm + nst * xbytes);                 // [nst][rows*D]
    W* xn0 = reinterpret_cast<W*>(xl0 + (PERSIST ? (size_t)nst * kTileRows * D : 0));
    W* sx0 = xn0 + (PERSIST ? (size_t)nst * kTileRows : 0);
    int32_t* ls0 = reinterpret_cast<int32_t*>(sx0 + (PERSIST ? (size_t)nst * kTileRows : 0));
    __shared__ AT cl_s[LK][LD];
    __shared__ W cn_s[LK], sc_s[LK], m2_s[LK];
    __shared__ double red[LT / 32][NV];
    __shared__ __align__(8) uint64_t full[kStages > kMaxResident ? kStages : kMaxResident];
    __shared__ int is_last, leave;
    __shared__ W C_s[LK * LD];                       // K5p: the centres, kept by every block
    auto tile_rows = [&](int64_t m) {
        const int64_t r0 = ((int64_t)blockIdx.x + m * gridDim.x) * kTileRows;
        return (int)std::min<int64_t>(kTileRows, p.n - r0);
    };
    // a tile whose X bytes are not a multiple of 16 (only the ragged last one) is read with
    // plain loads; the others stream through the bulk-copy ring
    auto bulk_ok = [&](int rows) { return ((size_t)rows * d * sizeof(W)) % 16 == 0 && (rows * 4) % 16 == 0; };
    auto issue = [&](int64_t m) {
        const int stg = PERSIST ? (int)m : (int)(m % kStages);
        const int rows = tile_rows(m);
        if (!bulk_ok(rows)) return;
        const int64_t r0 = ((int64_t)blockIdx.x + m * gridDim.x) * kTileRows;
        const uint32_t xb = (uint32_t)((size_t)rows * d * sizeof(W));
        const uint32_t fb = sm_u32(&full[stg]);
        bar_expect(fb, xb + (uint32_t)rows * 4u);
        bulk_g2s(sm_u32(xs0 + (size_t)stg * kTileRows * d), X + r0 * d, xb, fb);
        bulk_g2s(sm_u32(ls0 + (size_t)stg * kTileRows), labels + r0, (uint32_t)rows * 4u, fb);
    };
    if (tid == 0) {
        for (int q = 0; q < nst; ++q) bar_init(sm_u32(&full[q]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int64_t m = 0; m < my_tiles && m < nst; ++m) issue(m);

    if (PERSIST) {
        if (tid < k * d) C_s[tid] = C[tid];
        __syncthreads();
    }
#if MPK_K5P_TRACE
    long long ts[10];
#define K5P_STAMP(i) do { if (PERSIST && tid == 0) ts[i] = clock64(); } while (0)
#else
#define K5P_STAMP(i) do { } while (0)
#endif
    for (int itx = 0; itx < (PERSIST ? max_iter : 1); ++itx) {
    K5P_STAMP(0);
    // ---- A3: centroid prep (the arithmetic of prep_kernel: exact squares summed in the warp
    // reduction's order, infinity-norm scale, one rounding of c / s) -------------------------
    if (w < k) {
        const W v = lane < d ? (PERSIST ? C_s[w * d + lane] : C[w * d + lane]) : (W)0;
        const double sq = (double)v * (double)v;       // exact for fp32; fp64: one rounding
        double acc = lane < d ? sq : 0.0;
        W amax = fabs(v);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            acc += __shfl_xor_sync(0xffffffffu, acc, o);
            amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        }
        W s = (W)1;
        if (p.guard && !same) s = guard_scale(amax, p.guard);
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
            m2_s[w] = (W)-2 * s;
        }
        if (blockIdx.x == 0 && census) {
            nf = warp_sum(nf);
            nu = warp_sum(nu);
            if (lane == 0 && (nf | nu)) { atomicAdd(&census[0], nf); atomicAdd(&census[1], nu); }
        }
    }
    __syncthreads();

    K5P_STAMP(1);
    // the block's running totals per warp (fp64, in shared memory: red[w][.]); each tile's
    // per-thread partials are converted to fp64 and reduced by a warp tree into them
    for (int q = lane; q < NV; q += 32) red[w][q] = 0.0;
    double my_sse = 0.0, my_changed = 0.0;

    // ---- A4 + A5 over this block's tiles -----------------------------------------------------
    // per-thread partials of up to kFlushTiles tiles (<= 32 rows) in the working precision, then
    // fp64 (reading R1; fp64 work: fp64 throughout)
    W ps[KT][D], pc[KT];
    for (int64_t m = 0; m < my_tiles; ++m) {
        const int stg = PERSIST ? (int)m : (int)(m % kStages);
        const int rows = tile_rows(m);
        const int64_t r0 = ((int64_t)blockIdx.x + m * gridDim.x) * kTileRows;
        W* xs = xs0 + (size_t)stg * kTileRows * d;
        int32_t* ls = ls0 + (size_t)stg * kTileRows;
        if (PERSIST && itx > 0) {
            // resident since the first iteration
        } else if (bulk_ok(rows)) {
            bar_wait(sm_u32(&full[stg]), PERSIST ? 0u : (uint32_t)((m / kStages) & 1));
        } else {
            for (int q = tid; q < rows * d; q += LT) xs[q] = X[r0 * d + q];
            for (int q = tid; q < rows; q += LT) ls[q] = labels[r0 + q];
            __syncthreads();
        }
        if (m % kFlushTiles == 0) {
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                pc[j] = (W)0;
#pragma unroll
                for (int t = 0; t < D; ++t) ps[j][t] = (W)0;
            }
        }
        AT* xlc = xl0 + (size_t)stg * kTileRows * D;
        W* xnc = xn0 + (size_t)stg * kTileRows;
        W* sxc = sx0 + (size_t)stg * kTileRows;
        for (int r = tid; r < rows; r += LT) {
            const int64_t i = r0 + r;
            W x[D];
#pragma unroll
            for (int t = 0; t < D; ++t) x[t] = xs[r * D + t];
            W xn, s = (W)1;
            AT xl[D];
            if (PERSIST && itx > 0) {
                xn = xnc[r];
                s = sxc[r];
#pragma unroll
                for (int t = 0; t < D; ++t) xl[t] = xlc[r * D + t];
            } else {
                double nrm = 0.0;
#pragma unroll
                for (int t = 0; t < D; ++t) {
                    const double v = (double)x[t];
                    nrm = __dadd_rn(nrm, __dmul_rn(v, v));
                }
                xn = rounder<WORK>::from(nrm);
                if (p.guard && !same) {
                    W amax = (W)0;
#pragma unroll
                    for (int t = 0; t < D; ++t) amax = fmax(amax, fabs(x[t]));
                    s = guard_scale(amax, p.guard);
                }
                if (s == (W)1) {                       // no scaling: no division issued
#pragma unroll
                    for (int t = 0; t < D; ++t) xl[t] = (AT)widen(rounder<DIST>::from(x[t]));
                } else {
#pragma unroll
                    for (int t = 0; t < D; ++t) xl[t] = (AT)widen(rounder<DIST>::from(x[t] / s));
                }
                if (PERSIST) {
                    xnc[r] = xn;
                    sxc[r] = s;
#pragma unroll
                    for (int t = 0; t < D; ++t) xlc[r * D + t] = xl[t];
                }
            }
            W best = (W)INFINITY;
            int bj = 0;
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                if (j >= k) break;                     // uniform: no predicated columns
                AT dot = (AT)0;
#pragma unroll
                for (int t = 0; t < D; ++t) dot = fma(xl[t], cl_s[j][t], dot);
                // -2 (s s_j) = s (-2 s_j) exactly (a power-of-two factor)
                const W v = fma(s * m2_s[j], (W)dot, cn_s[j]);
                if (v < best) { best = v; bj = j; }
            }
            if (ls[r] != bj) my_changed += 1.0;
            labels[i] = bj;
            if (PERSIST) ls[r] = bj;                   // this thread's row, next iteration
            const double md = (double)xn + (double)best;
            my_sse += md > 0.0 ? md : 0.0;
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                if (j >= k) break;
                const W hit = (bj == j) ? (W)1 : (W)0;
                pc[j] += hit;
#pragma unroll
                for (int t = 0; t < D; ++t) ps[j][t] = fma(hit, x[t], ps[j][t]);
            }
        }
        if (m % kFlushTiles == kFlushTiles - 1 || m == my_tiles - 1) {
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                if (j >= k) break;                     // uniform
                const double c = warp_sum((double)pc[j]);
                if (lane == 0) red[w][LK * LD + j] += c;
#pragma unroll
                for (int t = 0; t < D; ++t) {
                    const double v = warp_sum((double)ps[j][t]);
                    if (lane == 0) red[w][j * LD + t] += v;
                }
            }
        }
        __syncthreads();                               // every thread is done with this stage
        if (!PERSIST && tid == 0 && m + kStages < my_tiles) issue(m + kStages);
    }
    K5P_STAMP(2);
    // ---- block partial (the warps' totals in order) ------------------------------------------
    my_sse = warp_sum(my_sse);
    my_changed = warp_sum(my_changed);
    if (lane == 0) { red[w][NV - 2] = my_sse; red[w][NV - 1] = my_changed; }
    __syncthreads();
    // K5p: partials double-buffered by iteration parity (a block can write iteration t + 1's
    // partial only after every block has arrived at t + 1, i.e. has read iteration t's)
    double* partb = part + (PERSIST ? (size_t)(itx & 1) * gridDim.x * NV : 0);
    if (tid < NV) {
        double a = 0.0;
#pragma unroll
        for (int q = 0; q < LT / 32; ++q) a += red[q][tid];
        partb[(size_t)blockIdx.x * NV + tid] = a;
        if (PERSIST) __threadfence();
    }
    K5P_STAMP(3);
    if (PERSIST) {
        // grid barrier: every block arrives (a monotone counter), then EVERY block reduces the
        // partials and forms the same new centres itself — no last-block tail, no release round
        // trip. A block that waits ~30 s gives up (fault) instead of hanging the device.
        __syncthreads();
        if (tid == 0) {
            atomicAdd(&st->counter, 1u);
            const unsigned target = gridDim.x * ((unsigned)itx + 1u);
            const long long t0 = clock64();
            int f = 0;
            // relaxed polls (an acquire load per poll would invalidate L1 each time), then one
            // acquire fence
            while (ld_relaxed_gpu(&st->counter) < target) {
                if (clock64() - t0 > (1LL << 36)) { atomicExch(&st->fault, 1); f = 1; break; }
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            leave = f;
        }
        __syncthreads();
        K5P_STAMP(4);
        if (leave) break;
    } else {
        // ---- the last block finalises ---------------------------------------------------------
        __threadfence();
        __syncthreads();
        if (tid == 0) is_last = atomicAdd(&st->counter, 1u) == gridDim.x - 1;
        __syncthreads();
        if (!is_last) return;
        __threadfence();
    }
    // partials of all blocks in a fixed order: group g sums the blocks b = g (mod kRedGroups)
    // in increasing b (independent loads in flight), then the groups are added in order
    if (tid < NV * kRedGroups) {
        const int c = tid % NV, g = tid / NV;
        // at most ceil(grid / 6) blocks per group: every load is issued before the adds
        constexpr int kMaxPer = (kNumSMs * kK5gBlocksPerSM + kRedGroups - 1) / kRedGroups;
        double v[kMaxPer];
#pragma unroll
        for (int q = 0; q < kMaxPer; ++q) {
            const unsigned b = g + q * kRedGroups;
            v[q] = b < gridDim.x ? __ldcg(partb + (size_t)b * NV + c) : 0.0;
        }
        double a = 0.0;
#pragma unroll
        for (int q = 0; q < kMaxPer; ++q) a += v[q];
        red[g][c] = a;
    }
    __syncthreads();
    if (tid < NV) {
        double a = 0.0;
        for (int g = 0; g < kRedGroups; ++g) a += red[g][tid];
        red[LT / 32 - 1][tid] = a;
    }
    __syncthreads();
    K5P_STAMP(5);
    const double* tot = red[LT / 32 - 1];
    // K5p: every block holds the same centres (C_s); block 0 publishes them and the trace
    const bool writer = !PERSIST || blockIdx.x == 0;
    if (w == 0) {
        // one lane per (cluster, feature) — lane = LD j + t, LK LD = 32 — all clusters at once:
        // new centre, then the per-cluster shift and Thm 5.3 terms summed over the cluster's LD
        // lanes by the xor-2, xor-1 tree (the order of a warp sum over d <= 4 lanes), and the
        // clusters' terms added in increasing j by lane 0
        const int j = lane / LD, t = lane % LD;
        double nm = 0.0, dn = 0.0;
        if (j < k && t < d) {
            const double c = tot[LK * LD + j];
            const int idx = j * d + t;
            const W old = PERSIST ? C_s[idx] : C[idx];
            W nw = old;
            if (c > 0.0) nw = rounder<WORK>::from(tot[j * LD + t] / c);
            const double df = (double)nw - (double)old;
            nm = df * df;
            dn = fabs(df) * fabs((double)nw);
            if (PERSIST) C_s[idx] = nw;
            if (writer) C[idx] = nw;
        }
        nm += __shfl_xor_sync(0xffffffffu, nm, 2);
        dn += __shfl_xor_sync(0xffffffffu, dn, 2);
        nm += __shfl_xor_sync(0xffffffffu, nm, 1);
        dn += __shfl_xor_sync(0xffffffffu, dn, 1);
        double sh = 0.0, empty = 0.0, rmax = 0.0;
        for (int jj = 0; jj < k; ++jj) {
            const double nmj = __shfl_sync(0xffffffffu, nm, jj * LD);
            const double dnj = __shfl_sync(0xffffffffu, dn, jj * LD);
            sh += nmj;
            if (tot[LK * LD + jj] == 0.0) empty += 1.0;
            if (nmj > 0.0 && dnj > 0.0) rmax = fmax(rmax, 2.0 * dnj / nmj);
        }
        if (lane == 0) {
            // Alg 3 step 6: no label changed, or ||C_t+1 - C_t|| <= tol
            const bool stop = tol >= 0.0 && (tot[NV - 1] == 0.0 || sqrt(sh) <= tol);
            if (writer) {
                const int it = PERSIST ? itx : st->iter;
                IterRec* rec = trace + (it < KMEANS_MAX_TRACE - 1 ? it : KMEANS_MAX_TRACE - 1);
                rec->sse = tot[NV - 2];
                rec->shift2 = sh;
                rec->changed = tot[NV - 1];
                rec->empty = empty;
                rec->ub_inv = rmax;
                st->iter = it + 1;
                if (stop) {
                    st->stop = 1;
                    st->converged = 1;
                }
                if (!PERSIST) st->counter = 0;
            }
            if (PERSIST) leave = stop;
        }
    }
    if (PERSIST) {
        __syncthreads();                               // C_s, leave
        K5P_STAMP(6);
#if MPK_K5P_TRACE
        if (tid == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && itx >= 2 && itx < 5)
            printf("K5P b%d it%d: A3 %lld tiles %lld partial %lld barrier %lld reduce %lld final %lld total %lld\n",
                   blockIdx.x, itx, ts[1] - ts[0], ts[2] - ts[1], ts[3] - ts[2], ts[4] - ts[3],
                   ts[5] - ts[4], ts[6] - ts[5], ts[6] - ts[0]);
#endif
        if (leave) break;
    }
    }   // iterations
}

// Grid: K5p runs one block per SM (cooperative, up to 227 KB of shared memory each); K5g the
// same grid whenever K5p could run this n (so the two partition the rows identically and agree
// bit for bit), else up to kK5gBlocksPerSM blocks per SM.
static int loop_grid(int64_t n, bool one_per_sm) {
    const int64_t tiles = (n + kTileRows - 1) / kTileRows;
    return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, one_per_sm ? kNumSMs : kNumSMs * kK5gBlocksPerSM));
}

template <typename W>
size_t smem_bytes_for(int d, int stages) {
    return (size_t)stages * kTileRows * ((size_t)d * sizeof(W) + sizeof(int32_t));
}
// K5p: rows, labels and the cached operands (x~ in AT, ||x||^2 and s in W) of every tile
template <typename W, typename AT>
size_t smem_bytes_persist(int d, int tiles) {
    return (size_t)tiles * kTileRows *
           ((size_t)d * sizeof(W) + (size_t)d * sizeof(AT) + 2 * sizeof(W) + sizeof(int32_t));
}

// persist < 0: K5g (one iteration per launch); persist = max_iter >= 1: K5p (cooperative)
template <typename W, int DIST, int D, int KT>
cudaError_t launch_dk(const Problem& p, const void* X, void* C, int32_t* labels, double* part,
                      int grid, LoopState* st, IterRec* trace, unsigned long long* census,
                      int persist, cudaStream_t s) {
    using AT = typename std::conditional<DIST == KMEANS_FP64, double, float>::type;
    // could K5p hold this n? (one block per SM, its tiles and cached operands in shared memory)
    const int64_t ntiles = (p.n + kTileRows - 1) / kTileRows;
    const int g1 = loop_grid(p.n, true);
    const int per = (int)((ntiles + g1 - 1) / g1);              // tiles of the busiest block
    const size_t smp = smem_bytes_persist<W, AT>(D, per);
    const bool fits = per <= kMaxResident && smp <= 227 * 1024;
    if (persist < 0) {
        grid = fits ? g1 : loop_grid(p.n, false);
        const size_t sm = smem_bytes_for<W>(D, kStages);
        if (!X) {   // attribute-only call (before a stream capture: not a stream operation)
            return cudaFuncSetAttribute(smalld_iter_kernel<W, DIST, D, KT, false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        }
        smalld_iter_kernel<W, DIST, D, KT, false><<<grid, LT, sm, s>>>(
            p, (const W*)X, (W*)C, labels, part, st, trace, census, 1);
        return cudaGetLastError();
    }
    if (!fits) return cudaErrorNotSupported;
    grid = g1;
    const size_t sm = smp;
    auto kern = smalld_iter_kernel<W, DIST, D, KT, true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) { cudaGetLastError(); return cudaErrorNotSupported; }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(LT);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // every block resident, or the launch fails
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, p, (const W*)X, (W*)C, labels, part, st, trace, census,
                           persist);
    if (e == cudaErrorCooperativeLaunchTooLarge) { cudaGetLastError(); return cudaErrorNotSupported; }
    return e;
}

template <typename W, int DIST>
cudaError_t launch_t(const Problem& p, const void* X, void* C, int32_t* labels, double* part,
                     int grid, LoopState* st, IterRec* trace, unsigned long long* census,
                     int persist, cudaStream_t s) {
#define MPK_DK(Dv) \
    return p.k <= 4 ? launch_dk<W, DIST, Dv, 4>(p, X, C, labels, part, grid, st, trace, census, persist, s) \
                    : launch_dk<W, DIST, Dv, 8>(p, X, C, labels, part, grid, st, trace, census, persist, s)
    switch (p.d) {
        case 1: MPK_DK(1);
        case 2: MPK_DK(2);
        case 3: MPK_DK(3);
        default: MPK_DK(4);
    }
#undef MPK_DK
}

}  // namespace

bool smalld_loop_supported(int d, int k) { return d <= LD && k <= LK; }


// two buffers: K5p alternates them by iteration parity
size_t smalld_loop_part_bytes(int64_t n) {
    return 2 * (size_t)loop_grid(n, false) * NV * sizeof(double);   // the larger grid
}

namespace {
cudaError_t launch_any(int work, int dist, const Problem& p, const void* Xw, void* Cw,
                       int32_t* labels, double* part, LoopState* st, IterRec* trace,
                       unsigned long long* census, int persist, cudaStream_t s) {
    const int g = 0;                                   // launch_dk chooses the grid
#define MPK_SL(W)                                                                                  \
    switch (dist) {                                                                                \
        case KMEANS_FP64: return launch_t<W, KMEANS_FP64>(p, Xw, Cw, labels, part, g, st, trace, census, persist, s); \
        case KMEANS_FP32: return launch_t<W, KMEANS_FP32>(p, Xw, Cw, labels, part, g, st, trace, census, persist, s); \
        case KMEANS_FP16: return launch_t<W, KMEANS_FP16>(p, Xw, Cw, labels, part, g, st, trace, census, persist, s); \
        case KMEANS_BF16: return launch_t<W, KMEANS_BF16>(p, Xw, Cw, labels, part, g, st, trace, census, persist, s); \
        case KMEANS_E5M2: return launch_t<W, KMEANS_E5M2>(p, Xw, Cw, labels, part, g, st, trace, census, persist, s); \
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
}  // namespace

cudaError_t launch_smalld_iter(int work, int dist, const Problem& p, const void* Xw, void* Cw,
                               int32_t* labels, double* part, LoopState* st, IterRec* trace,
                               unsigned long long* census, cudaStream_t s) {
    if (Xw) launches_add(1);
    return launch_any(work, dist, p, Xw, Cw, labels, part, st, trace, census, -1, s);
}

cudaError_t launch_smalld_persist(int work, int dist, const Problem& p, const void* Xw, void* Cw,
                                  int32_t* labels, double* part, LoopState* st, IterRec* trace,
                                  unsigned long long* census, int max_iter, cudaStream_t s) {
    const cudaError_t e = launch_any(work, dist, p, Xw, Cw, labels, part, st, trace, census,
                                     max_iter < 1 ? 1 : max_iter, s);
    if (e == cudaSuccess) launches_add(1);
    return e;
}

}  // namespace mpk
