// k_seed.cu — D^2 seeding (Alg 1) with Alg 3 step 1's low precision
// (PAPER.md:544), as DESIGN.md reading R6 defines the draw:
//   * D^2(p_i, c) = xn_i - 2 (s_i s_c) (x~_i . x~_c) + xn_c from the stored low-precision
//     operands — the dot accumulated in fp32 like the distance kernels' (fp64 operands: fp64),
//     the combination in fp64 — floored at 0; the centre's own weight is 0;
//   * weights D2[i] = min over the chosen centres; the next centre is the first index whose
//     running sum of weights exceeds u_j * sum (Alg 1 line 2's law D(p)^2 / sum D^2 drawn by
//     inverse CDF with the caller's uniform); a sum of 0 or +inf/NaN falls back to the uniform
//     index (warning).
// The sums are formed in a fixed parallel order (per 4096-row block: 16-row sequential pieces,
// a warp tree, warps in order; then a block-level scan), so the draw is deterministic; it is not
// bit-identical to the oracle's sequential sums and fp64 dots, and the tests check each draw's
// admissibility against the oracle's weights for the same chosen centres instead.
// Per round: one pass over X~ (HBM: n d_pad s_l + 16 n bytes), one row per thread with the
// row's 16-byte chunks all in flight, then one CTA's scan-and-pick.
#include "common.cuh"
#include "internal.h"

#include <stdlib.h>
#include <string.h>

#include <type_traits>

namespace mpk {
namespace {

constexpr int kSeedBlock = 4096;     // rows per update CTA (and per block sum)
constexpr int kSeedThreads = 256;
constexpr int kPickThreads = 1024;

template <typename LT> struct seed_acc { using T = float; };
template <> struct seed_acc<double> { using T = double; };

// Widen the elements of one 16-byte chunk and accumulate chunk . centre into acc (in order).
template <typename LT, typename A>
MPK_DEV A dot16(uint4 q, const A* __restrict__ cs, int t0, int d, A acc) {
    constexpr int m = 16 / (int)sizeof(LT);
    LT e[m];
    memcpy(e, &q, 16);
#pragma unroll
    for (int i = 0; i < m; ++i)
        if (t0 + i < d) acc = fma((A)widen(e[i]), cs[t0 + i], acc);
    return acc;
}
// A whole 16-byte chunk of fp16 / bf16 (t0 + 8 <= d, cs 16-byte aligned): packed widening and
// two broadcast 16-byte shared loads of the centre; the same sequential order of FMAs.
template <typename LT>
MPK_DEV float dot16_full(uint4 q, const float* __restrict__ cs, int t0, float acc) {
    const float4 c0 = *reinterpret_cast<const float4*>(cs + t0);
    const float4 c1 = *reinterpret_cast<const float4*>(cs + t0 + 4);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    float2 f[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if constexpr (std::is_same<LT, __half>::value)
            f[i] = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
        else
            f[i] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
    }
    acc = fmaf(f[0].x, c0.x, acc); acc = fmaf(f[0].y, c0.y, acc);
    acc = fmaf(f[1].x, c0.z, acc); acc = fmaf(f[1].y, c0.w, acc);
    acc = fmaf(f[2].x, c1.x, acc); acc = fmaf(f[2].y, c1.y, acc);
    acc = fmaf(f[3].x, c1.z, acc); acc = fmaf(f[3].y, c1.w, acc);
    return acc;
}

// One warp, 32 rows whose operand rows are G 16-byte chunks (G a power of two <= 16): load i of
// lane l reads chunk l % G of row i (32 / G) + l / G, so every load instruction covers 32 / G
// whole rows, 512 contiguous bytes; each lane multiplies its chunk with the same chunk of the
// centre (held in registers) for its G rows, and a butterfly over the G lanes of a row group
// (keep half, send half: G - 1 shuffles in all) leaves lane l with the full dot of row
// (l % G) (32 / G) + l / G. The dot is summed in a fixed tree instead of sequentially: within
// the same gamma_d bound the parity tests use.
template <int G, typename LT, typename A>
MPK_DEV A seed_batch_dot(const LT* __restrict__ Xl, int64_t row0, int d_pad, int rows_left,
                         const A (&cr)[16 / sizeof(LT)], int lane) {
    constexpr int m = 16 / (int)sizeof(LT);
    constexpr int RPI = 32 / G;                    // rows per load instruction
    const int q = lane & (G - 1), sgrp = lane / G;
    uint4 buf[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int r = i * RPI + sgrp;
        buf[i] = r < rows_left
                     ? __ldg(reinterpret_cast<const uint4*>(Xl + (row0 + r) * d_pad) + q)
                     : make_uint4(0, 0, 0, 0);
    }
    A part[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
        LT e[m];
        memcpy(e, &buf[i], 16);
        A acc = (A)0;
#pragma unroll
        for (int u = 0; u < m; ++u) acc = fma((A)widen(e[u]), cr[u], acc);
        part[i] = acc;
    }
#pragma unroll
    for (int o = G / 2; o >= 1; o >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int u = 0; u < o; ++u) {
            const A send = upper ? part[u] : part[u + o];
            const A keep = upper ? part[u + o] : part[u];
            part[u] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return part[0];
}

template <typename LT, typename W>
__global__ void __launch_bounds__(kSeedThreads, 2)
seed_update_kernel(const LT* __restrict__ Xl, int64_t n, int d, int d_pad,
                   const W* __restrict__ xn, const W* __restrict__ sx, int guard,
                   const int64_t* __restrict__ idx, int j, double* __restrict__ D2,
                   double* __restrict__ ps, int vec) {
    using A = typename seed_acc<LT>::T;
    extern __shared__ __align__(16) unsigned char seed_smem[];
    A* cs = reinterpret_cast<A*>(seed_smem);                    // newest centre, widened (d_pad)
    __shared__ double d2s[kSeedBlock];
    __shared__ double wsum[kSeedThreads / 32];
    const int64_t c = idx[j];
    for (int t = threadIdx.x; t < d_pad; t += blockDim.x)
        cs[t] = t < d ? (A)widen(Xl[c * d_pad + t]) : (A)0;
    __syncthreads();
    const double xnc = (double)xn[c];
    const double scc = guard ? (double)sx[c] : 1.0;
    const int64_t b0 = (int64_t)blockIdx.x * kSeedBlock;
    const int rows = (int)((b0 + kSeedBlock < n) ? kSeedBlock : n - b0);
    const int lane = threadIdx.x & 31;
    const int chunks = (d_pad * (int)sizeof(LT)) / 16;
    constexpr int m = 16 / (int)sizeof(LT);
    constexpr int QB = 16;                          // 16-byte chunks of a row in flight
    const int G = vec ? chunks : 0;
    if (G == 2 || G == 4 || G == 8 || G == 16) {
        // the coalesced path: warps take 32-row batches, rows loaded "transposed"
        const int q = lane & (G - 1);
        A cr[m];
#pragma unroll
        for (int u = 0; u < m; ++u) cr[u] = cs[q * m + u];
        const int warp = threadIdx.x >> 5, nw = kSeedThreads / 32;
        for (int base = warp * 32; base < rows; base += nw * 32) {
            const int rpi = 32 / G;
            const int r = (lane & (G - 1)) * rpi + lane / G;      // this lane's row after the reduce
            const bool mine = base + r < rows;
            const int64_t i = b0 + base + r;
            const double old = mine ? D2[i] : 0.0;
            const W xni = mine ? xn[i] : (W)0;
            const W si_w = (mine && guard) ? sx[i] : (W)1;
            A dot;
            switch (G) {
                case 2: dot = seed_batch_dot<2, LT, A>(Xl, b0 + base, d_pad, rows - base, cr, lane); break;
                case 4: dot = seed_batch_dot<4, LT, A>(Xl, b0 + base, d_pad, rows - base, cr, lane); break;
                case 8: dot = seed_batch_dot<8, LT, A>(Xl, b0 + base, d_pad, rows - base, cr, lane); break;
                default: dot = seed_batch_dot<16, LT, A>(Xl, b0 + base, d_pad, rows - base, cr, lane); break;
            }
            if (mine) {
                const double si = (double)si_w;
                double D = ((double)xni - 2.0 * (si * scc) * (double)dot) + xnc;
                D = D > 0.0 ? D : 0.0;                  // NaN -> 0
                if (i == c) D = 0.0;                    // the centre's own weight
                const double nw2 = D < old ? D : old;
                D2[i] = nw2;
                d2s[base + r] = nw2;
            }
        }
    } else
    // one row per thread: the whole row's 16-byte chunks are loaded before they are used (a
    // warp keeps 32 rows, 8 KB at d = 128 fp16, in flight); the dot is the sequential fp32 sum
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
        const int64_t i = b0 + r;
        const double old = D2[i];
        const W xni = xn[i];
        const W si_w = guard ? sx[i] : (W)1;
        A dot = (A)0;
        if (vec) {
            const uint4* xp = reinterpret_cast<const uint4*>(Xl + i * d_pad);
            for (int q0 = 0; q0 < chunks; q0 += QB) {
                uint4 buf[QB];
#pragma unroll
                for (int u = 0; u < QB; ++u)
                    buf[u] = (q0 + u < chunks) ? __ldg(xp + q0 + u) : make_uint4(0, 0, 0, 0);
                if constexpr (std::is_same<LT, __half>::value || std::is_same<LT, __nv_bfloat16>::value) {
                    if ((d & 7) == 0) {                 // whole chunks: the packed path
#pragma unroll
                        for (int u = 0; u < QB; ++u)
                            if (q0 + u < chunks && (q0 + u) * m < d)
                                dot = dot16_full<LT>(buf[u], cs, (q0 + u) * m, dot);
                        continue;
                    }
                }
#pragma unroll
                for (int u = 0; u < QB; ++u)
                    if (q0 + u < chunks) dot = dot16<LT, A>(buf[u], cs, (q0 + u) * m, d, dot);
            }
        } else {
            const LT* xp = Xl + i * d_pad;
            for (int t = 0; t < d; ++t) dot = fma((A)widen(xp[t]), cs[t], dot);
        }
        const double si = (double)si_w;
        double D = ((double)xni - 2.0 * (si * scc) * (double)dot) + xnc;
        D = D > 0.0 ? D : 0.0;                      // NaN -> 0
        if (i == c) D = 0.0;                        // the centre's own weight
        const double nw = D < old ? D : old;
        D2[i] = nw;
        d2s[r] = nw;
    }
    __syncthreads();
    // block sum in a fixed order: 16-row pieces sequentially, a warp tree, warps in order
    double a = 0.0;
    const int per = kSeedBlock / kSeedThreads;
    for (int q = 0; q < per; ++q) {
        const int r = threadIdx.x * per + q;
        if (r < rows) a += d2s[r];
    }
    a = warp_sum(a);
    if (lane == 0) wsum[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kSeedThreads / 32; ++w) t += wsum[w];
        ps[blockIdx.x] = t;
    }
}

// The same round with the seeding block's rows streamed through shared memory by the TMA engine
// (1-D bulk copies of 256-row stages into a ring; rows of G 16-byte chunks, G <= 16): the
// copies of the next stages are in flight while the warps take 32-row batches of the current
// one with the transposed, bank-conflict-free reads and the butterfly of seed_batch_dot.
constexpr int kStageRows = 256;

MPK_DEV void sbar_init(uint32_t b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
}
MPK_DEV void sbar_expect(uint32_t b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                 : "memory");
}
MPK_DEV void sbar_wait(uint32_t b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra W_%=;\n\t}" ::"r"(b),
        "r"(parity)
        : "memory");
}
MPK_DEV void sbulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

template <int G, typename LT, typename W>
__global__ void __launch_bounds__(kSeedThreads, 1)
seed_update_tma_kernel(const LT* __restrict__ Xl, int64_t n, int d, int d_pad,
                       const W* __restrict__ xn, const W* __restrict__ sx, int guard,
                       const int64_t* __restrict__ idx, int j, double* __restrict__ D2,
                       double* __restrict__ ps, int nstages) {
    using A = typename seed_acc<LT>::T;
    constexpr int m = 16 / (int)sizeof(LT);
    constexpr int RPI = 32 / G;
    constexpr int RB = G * 16;                        // row bytes
    extern __shared__ __align__(128) unsigned char tsm[];
    unsigned char* ring = tsm;                        // nstages x kStageRows x RB
    A* cs = reinterpret_cast<A*>(tsm + (size_t)nstages * kStageRows * RB);
    __shared__ double d2s[kSeedBlock];
    __shared__ double wsum[kSeedThreads / 32];
    __shared__ __align__(8) uint64_t full[4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t c = idx[j];
    const int64_t b0 = (int64_t)blockIdx.x * kSeedBlock;
    const int rows = (int)((b0 + kSeedBlock < n) ? kSeedBlock : n - b0);
    const int nst = (rows + kStageRows - 1) / kStageRows;
    auto issue = [&](int st) {
        const int r0 = st * kStageRows;
        const int rr = rows - r0 < kStageRows ? rows - r0 : kStageRows;
        const uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[st % nstages]);
        sbar_expect(fb, (uint32_t)(rr * RB));
        sbulk_g2s((uint32_t)__cvta_generic_to_shared(ring + (size_t)(st % nstages) * kStageRows * RB),
                  Xl + (b0 + r0) * d_pad, (uint32_t)(rr * RB), fb);
    };
    if (tid == 0) {
        for (int q = 0; q < nstages; ++q) sbar_init((uint32_t)__cvta_generic_to_shared(&full[q]));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int st = 0; st < nst && st < nstages; ++st) issue(st);
    }
    for (int t = tid; t < d_pad; t += blockDim.x) cs[t] = t < d ? (A)widen(Xl[c * d_pad + t]) : (A)0;
    __syncthreads();
    const double xnc = (double)xn[c];
    const double scc = guard ? (double)sx[c] : 1.0;
    const int q = lane & (G - 1), sgrp = lane / G;
    A cr[m];
#pragma unroll
    for (int u = 0; u < m; ++u) cr[u] = cs[q * m + u];
    for (int st = 0; st < nst; ++st) {
        const int base = st * kStageRows + warp * 32;          // this warp's 32-row batch
        const int r = q * RPI + sgrp;                          // the lane's row after the reduce
        const bool mine = base + r < rows;
        const int64_t i = b0 + base + r;
        const double old = mine ? D2[i] : 0.0;
        const W xni = mine ? xn[i] : (W)0;
        const W si_w = (mine && guard) ? sx[i] : (W)1;
        sbar_wait((uint32_t)__cvta_generic_to_shared(&full[st % nstages]), (uint32_t)((st / nstages) & 1));
        const unsigned char* sb = ring + (size_t)(st % nstages) * kStageRows * RB + (size_t)warp * 32 * RB;
        A part[G];
#pragma unroll
        for (int k2 = 0; k2 < G; ++k2) {
            const int rr = k2 * RPI + sgrp;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (base + rr < rows) v = *reinterpret_cast<const uint4*>(sb + (size_t)rr * RB + q * 16);
            LT e[m];
            memcpy(e, &v, 16);
            A acc = (A)0;
#pragma unroll
            for (int u = 0; u < m; ++u) acc = fma((A)widen(e[u]), cr[u], acc);
            part[k2] = acc;
        }
#pragma unroll
        for (int o = G / 2; o >= 1; o >>= 1) {
            const bool upper = (lane & o) != 0;
#pragma unroll
            for (int u = 0; u < o; ++u) {
                const A send = upper ? part[u] : part[u + o];
                const A keep = upper ? part[u + o] : part[u];
                part[u] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        if (mine) {
            const double si = (double)si_w;
            double D = ((double)xni - 2.0 * (si * scc) * (double)part[0]) + xnc;
            D = D > 0.0 ? D : 0.0;                      // NaN -> 0
            if (i == c) D = 0.0;                        // the centre's own weight
            const double nw2 = D < old ? D : old;
            D2[i] = nw2;
            d2s[base + r] = nw2;
        }
        __syncthreads();                                // the stage is consumed
        if (tid == 0 && st + nstages < nst) issue(st + nstages);
    }
    // block sum in the fixed order of seed_update_kernel
    double a = 0.0;
    const int per = kSeedBlock / kSeedThreads;
    for (int qq = 0; qq < per; ++qq) {
        const int rr = tid * per + qq;
        if (rr < rows) a += d2s[rr];
    }
    a = warp_sum(a);
    if (lane == 0) wsum[warp] = a;
    __syncthreads();
    if (tid == 0) {
        double t2 = 0.0;
        for (int w = 0; w < kSeedThreads / 32; ++w) t2 += wsum[w];
        ps[blockIdx.x] = t2;
    }
}

// Exclusive scan of one double per thread over a kPickThreads CTA (fixed order: warp shuffles,
// then the warp totals scanned by warp 0). Returns the exclusive prefix; *total = the sum.
MPK_DEV double cta_exclusive_scan(double v, double* wtot, double* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wtot[w] = inc;
    __syncthreads();
    if (w == 0) {
        double t = wtot[lane];
        double ti = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, ti, o);
            if (lane >= o) ti += y;
        }
        wtot[lane] = ti - t;              // exclusive prefix of warp totals
        if (lane == 31) wtot[32] = ti;
    }
    __syncthreads();
    const double ex = wtot[w] + (inc - v);
    *total = wtot[32];
    __syncthreads();
    return ex;
}

// The draw of round j: total, the block whose running sum crosses u_j * total, then the row.
__global__ void __launch_bounds__(kPickThreads)
seed_pick_kernel(const double* __restrict__ D2, const double* __restrict__ ps, int64_t n,
                 int64_t nb, const double* __restrict__ u, int j, int64_t* __restrict__ idx,
                 int* __restrict__ warn) {
    __shared__ double wtot[33];
    __shared__ int first;
    __shared__ int64_t sel;
    __shared__ double sel_run;
    const int t = threadIdx.x;
    // level 1: contiguous chunks of block sums per thread
    const int64_t ch = (nb + kPickThreads - 1) / kPickThreads;
    const int64_t c0 = (int64_t)t * ch, c1 = (c0 + ch < nb) ? c0 + ch : nb;
    double v = 0.0;
    for (int64_t b = c0; b < c1; ++b) v += ps[b];
    double total;
    const double ex = cta_exclusive_scan(v, wtot, &total);
    if (!(total > 0.0) || isinf(total)) {
        if (t == 0) {
            int64_t cc = (int64_t)(u[j] * (double)n);
            if (cc > n - 1) cc = n - 1;
            *warn |= 1;
            idx[j] = cc;
        }
        return;
    }
    const double target = u[j] * total;
    if (t == 0) { first = kPickThreads; sel = -1; }
    __syncthreads();
    if (c0 < c1 && ex + v > target) atomicMin(&first, t);
    __syncthreads();
    const int ft = first == kPickThreads ? -1 : first;
    if (t == (ft < 0 ? 0 : ft)) {
        // the thread owning the crossing walks its chunk; rounding that left the target at the
        // top falls back to the last block with a positive sum
        int64_t bsel = -1;
        double run = 0.0;
        if (ft >= 0) {
            run = ex;
            for (int64_t b = c0; b < c1; ++b) {
                if (run + ps[b] > target) { bsel = b; break; }
                run += ps[b];
            }
            if (bsel < 0) { bsel = c1 - 1; run -= ps[bsel]; }
        } else {
            double acc = 0.0;
            for (int64_t b = 0; b < nb; ++b) {
                if (ps[b] > 0.0) { bsel = b; run = acc; }
                acc += ps[b];
            }
        }
        sel = bsel;
        sel_run = run;
    }
    __syncthreads();
    // level 2: the rows of the chosen block, four consecutive rows per thread
    const int64_t r0 = sel * kSeedBlock;
    const int rows = (int)((r0 + kSeedBlock < n) ? kSeedBlock : n - r0);
    const int per = kSeedBlock / kPickThreads;
    double loc = 0.0;
    for (int q = 0; q < per; ++q) {
        const int r = t * per + q;
        if (r < rows) loc += D2[r0 + r];
    }
    double tot2;
    const double ex2 = sel_run + cta_exclusive_scan(loc, wtot, &tot2);
    if (t == 0) first = kPickThreads;
    __syncthreads();
    if (ex2 + loc > target) atomicMin(&first, t);
    __syncthreads();
    if (first < kPickThreads) {
        if (t == first) {
            double run = ex2;
            int64_t cc = -1;
            for (int q = 0; q < per; ++q) {
                const int r = t * per + q;
                if (r >= rows) break;
                run += D2[r0 + r];
                if (run > target) { cc = r0 + r; break; }
            }
            if (cc < 0) {                          // rounding: the last positive row of the chunk
                for (int q = per - 1; q >= 0; --q) {
                    const int r = t * per + q;
                    if (r < rows && D2[r0 + r] > 0.0) { cc = r0 + r; break; }
                }
            }
            idx[j] = cc;
        }
    } else if (t == 0) {
        int64_t cc = r0 + rows - 1;
        for (int r = rows - 1; r >= 0; --r)
            if (D2[r0 + r] > 0.0) { cc = r0 + r; break; }
        idx[j] = cc;
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
    using A = typename seed_acc<LT>::T;
    const int64_t nb = (n + kSeedBlock - 1) / kSeedBlock;
    const unsigned pb = (unsigned)((n + 255) / 256);
    seed_init_kernel<<<pb, 256, 0, s>>>(D2, n);
    const size_t sm = (size_t)d_pad * sizeof(A);
    static PerDeviceOnce attr;
    if (attr.need()) {
        cudaFuncSetAttribute(seed_update_kernel<LT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             160 * 1024);
        attr.done();
    }
    const int row_bytes = d_pad * (int)sizeof(LT);
    const int vec = (row_bytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(Xl) & 15) == 0);
    const int G = vec ? row_bytes / 16 : 0;
    // the TMA-ring kernel for rows of 2..16 chunks: as many 256-row stages as fit beside the
    // block's D^2 staging (static 32 KB) in 227 KB
    int nstages = 0;
    size_t tsm = 0;
    if ((G == 2 || G == 4 || G == 8 || G == 16) && !getenv("MPK_SEED_NO_TMA")) {
        nstages = 3;
        while (nstages > 1 && (size_t)nstages * kStageRows * row_bytes + sm + 34 * 1024 > 227 * 1024)
            --nstages;
        tsm = (size_t)nstages * kStageRows * row_bytes + sm;
        // once per seeding call (per device: the attribute is per device)
        cudaError_t ea;
        switch (G) {
            case 2: ea = cudaFuncSetAttribute(seed_update_tma_kernel<2, LT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm); break;
            case 4: ea = cudaFuncSetAttribute(seed_update_tma_kernel<4, LT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm); break;
            case 8: ea = cudaFuncSetAttribute(seed_update_tma_kernel<8, LT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm); break;
            default: ea = cudaFuncSetAttribute(seed_update_tma_kernel<16, LT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm); break;
        }
        if (ea != cudaSuccess) { cudaGetLastError(); nstages = 0; }   // the one-row-per-thread kernel
    }
    for (int j = 1; j < k; ++j) {
        if (nstages > 0) {
#define SEED_TMA(GV) seed_update_tma_kernel<GV, LT, W><<<(unsigned)nb, kSeedThreads, tsm, s>>>( \
            (const LT*)Xl, n, d, d_pad, (const W*)xn, (const W*)sx, guard, idx, j - 1, D2, ps, nstages)
            switch (G) {
                case 2: SEED_TMA(2); break;
                case 4: SEED_TMA(4); break;
                case 8: SEED_TMA(8); break;
                default: SEED_TMA(16); break;
            }
#undef SEED_TMA
        } else {
            seed_update_kernel<LT, W><<<(unsigned)nb, kSeedThreads, sm, s>>>(
                (const LT*)Xl, n, d, d_pad, (const W*)xn, (const W*)sx, guard, idx, j - 1, D2, ps,
                vec);
        }
        seed_pick_kernel<<<1, kPickThreads, 0, s>>>(D2, ps, n, nb, u, j, idx, warn);
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
