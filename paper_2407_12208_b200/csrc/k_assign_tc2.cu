// k_assign_tc2.cu — K4 fast path: CTA-pair (cta_group::2), centroid-stationary distance + argmin.
//
// Same arithmetic as k_assign_tc.cu (x~_i . c~_j on tcgen05 with fp32 accumulation in TMEM,
// epilogue v_ij = fma(-2 s_i s_j, acc, ||c_j||^2) and a per-point running argmin; eq:dist-eval
// PAPER.md:193-196, Alg 3 step 3 PAPER.md:546, Alg 4 line 6 PAPER.md:624-625), organised for
// B200's CTA pairs:
//   * a cluster of two CTAs on one TPC issues M = 256 (128 points per CTA) x N = NB (<= 256)
//     MMAs with cta_group::2; each CTA holds half of every centroid tile (NB/2 rows) RESIDENT in
//     shared memory for the whole kernel, so C~ (up to 256 KB) crosses L2 -> SM once per CTA and
//     only X~ streams (TMA, ring of SA slots per CTA, both CTAs' bytes complete on the leader's
//     barrier);
//   * the leader CTA's single MMA thread issues, tcgen05.commit multicasts "accumulator full" /
//     "slot free" to both CTAs; each CTA's two epilogue warpgroups split the NB columns of an
//     accumulator, merge per row-block through shared memory, and arrive remotely on the leader's
//     "accumulator empty" barrier.
// FINAL mode: certified top-2 filter for Alg 3 step 7, as in k_assign_tc.cu.
#include "common.cuh"
#include "internal.h"
#include "tc_common.cuh"
#include "tc_pair.h"

#include <stdlib.h>

namespace mpk {
namespace tcdev {

constexpr int P_BM = 128;
constexpr int P_NON_EPI = 4;
constexpr int P_EWG = 4;                 // epilogue warpgroups
constexpr int P_EPI = 4 * P_EWG;
constexpr int P_THREADS = (P_NON_EPI + P_EPI) * 32;
constexpr int P_MAX_ACC = 4;
constexpr size_t P_BUDGET = 227 * 1024;

MPK_DEV void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
MPK_DEV void named_bar_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <bool FINAL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(P_THREADS, 1)
assign_pair_kernel(const __grid_constant__ CUtensorMap tmap_x,
                   const __grid_constant__ CUtensorMap tmap_c, PairParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* b_base = smem;                                             // resident centroid halves
    uint8_t* a_base = b_base + (size_t)p.NT * p.b_half_bytes;           // X~ ring
    float* cn_s = (float*)(a_base + (size_t)p.SA * p.a_tile_bytes);
    float* sc_s = cn_s + p.k_pad;
    float* mg_v = sc_s + p.k_pad;              // [2][P_EWG-1][128] partial minima
    float* mg_v2 = mg_v + 2 * (P_EWG - 1) * P_BM;   // second minima (FINAL)
    int* mg_j = (int*)(mg_v2 + 2 * (P_EWG - 1) * P_BM);
    uint64_t* bars = (uint64_t*)(((uintptr_t)(mg_j + 2 * (P_EWG - 1) * P_BM) + 7) & ~(uintptr_t)7);
    uint64_t* a_full = bars;
    uint64_t* a_empty = a_full + p.SA;
    uint64_t* b_full = a_empty + p.SA;
    uint64_t* t_full = b_full + 1;
    uint64_t* t_empty = t_full + P_MAX_ACC;
    uint32_t* tmem_slot = (uint32_t*)(t_empty + P_MAX_ACC);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;

    for (int j = threadIdx.x; j < p.k_pad; j += blockDim.x) {
        cn_s[j] = j < p.k ? p.cn[j] : INFINITY;       // padded centroids never win
        sc_s[j] = (p.guard && j < p.k) ? p.sc[j] : 1.0f;
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < p.SA; ++i) { mbar_init(smem_u32(&a_full[i]), 1); mbar_init(smem_u32(&a_empty[i]), 1); }
        mbar_init(smem_u32(b_full), 1);
        for (int i = 0; i < p.nacc; ++i) {
            mbar_init(smem_u32(&t_full[i]), 1);
            mbar_init(smem_u32(&t_empty[i]), 2 * P_EPI);   // every epilogue warp of both CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_c)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(p.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int64_t rows_per_rb = 2 * P_BM;
    const int64_t num_rb = (p.n + rows_per_rb - 1) / rows_per_rb;
    const int64_t pair = blockIdx.x >> 1;
    const int64_t npairs = gridDim.x >> 1;
    const int eps = p.SWZ / (p.is_f8 ? 1 : 2);      // elements per swizzle row
    const int half = p.NB / 2;

    if (warp == 2) {
        // ------------------------------------------------ resident centroid halves (once)
        if (lane == 0) {
            const uint32_t fb = smem_u32(b_full);
            if (leader) mbar_expect_tx(fb, 2u * p.NT * p.b_half_bytes);
            for (int t = 0; t < p.NT; ++t) {
                const uint32_t dst = smem_u32(b_base + (size_t)t * p.b_half_bytes);
                for (int kb = 0; kb < p.KB; ++kb)
                    tma_load_2d_pair(dst + kb * p.kb_b_bytes, &tmap_c, kb * eps,
                                     t * p.NB + (int)rank * half, fb);
            }
        }
    } else if (warp == 0) {
        // ------------------------------------------------ X~ producer (this CTA's 128 rows)
        if (lane == 0) {
            uint32_t u = 0;
            for (int64_t rb = pair; rb < num_rb; rb += npairs, ++u) {
                const int slot = u % p.SA;
                mbar_wait(smem_u32(&a_empty[slot]), ((u / p.SA) & 1) ^ 1);
                const uint32_t fb = smem_u32(&a_full[slot]);
                if (leader) mbar_expect_tx(fb, 2u * p.a_tile_bytes);
                const uint32_t dst = smem_u32(a_base + (size_t)slot * p.a_tile_bytes);
                const int row0 = (int)(rb * rows_per_rb + rank * P_BM);
                for (int kb = 0; kb < p.KB; ++kb)
                    tma_load_2d_pair(dst + kb * p.kb_a_bytes, &tmap_x, kb * eps, row0, fb);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA only)
        if (leader && lane == 0) {
            mbar_wait(smem_u32(b_full), 0);
            tc_fence_after();
            const int ksteps = p.SWZ / 32;
            const uint32_t b0 = smem_u32(b_base);
            uint32_t u = 0, ai = 0;
            for (int64_t rb = pair; rb < num_rb; rb += npairs, ++u) {
                const int slot = u % p.SA;
                mbar_wait(smem_u32(&a_full[slot]), (u / p.SA) & 1);
                tc_fence_after();
                const uint32_t a_addr = smem_u32(a_base + (size_t)slot * p.a_tile_bytes);
                for (int t = 0; t < p.NT; ++t, ++ai) {
                    const int buf = ai % p.nacc;
                    mbar_wait(smem_u32(&t_empty[buf]), ((ai / p.nacc) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + buf * p.NB;
                    const uint32_t b_addr = b0 + t * p.b_half_bytes;
                    for (int kb = 0; kb < p.KB; ++kb) {
                        for (int ks = 0; ks < ksteps; ++ks) {
                            const uint64_t ad = umma_desc(a_addr + kb * p.kb_a_bytes + ks * 32, p.SWZ);
                            const uint64_t bd = umma_desc(b_addr + kb * p.kb_b_bytes + ks * 32, p.SWZ);
                            const uint32_t accum = (kb | ks) ? 1u : 0u;
                            if (p.dbg & 2) continue;
                            if (p.is_f8) mma2_f8(d_tmem, ad, bd, p.idesc, accum);
                            else mma2_f16(d_tmem, ad, bd, p.idesc, accum);
                        }
                    }
                    tc_commit_pair(smem_u32(&t_full[buf]));
                }
                tc_commit_pair(smem_u32(&a_empty[slot]));
            }
        }
    } else if (warp >= P_NON_EPI) {
        // ------------------------------------------------ epilogue: P_EWG warpgroups split the
        // NB columns of every accumulator (4 warps per SM sub-partition hide TMEM/smem latency)
        const int wg = (warp - P_NON_EPI) >> 2;
        const int quarter = warp & 3;
        const int q = quarter * 32 + lane;                 // row within this CTA's 128
        const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
        const int wcols = p.NB / P_EWG;                    // multiple of 16
        const int col_off = wg * wcols;
        float cn_max = 0.0f, s_max = 1.0f;
        if (FINAL) {
            for (int j = 0; j < p.k; ++j) {
                cn_max = fmaxf(cn_max, cn_s[j]);
                s_max = fmaxf(s_max, sc_s[j]);
            }
        }
        double my_sse = 0.0, my_changed = 0.0;
        uint32_t ai = 0, rbi = 0;
        for (int64_t rb = pair; rb < num_rb; rb += npairs, ++rbi) {
            const int64_t row = rb * rows_per_rb + rank * P_BM + q;
            const bool valid = row < p.n;
            const float m2 = (p.guard && valid) ? -2.0f * p.sx[row] : -2.0f;
            // prefetch what the row-block epilogue needs (hidden behind the tile loop)
            int old_label = 0;
            float xn_row = 0.0f;
            if (wg == 0 && valid) {
                xn_row = p.xn[row];
                if (!FINAL) old_label = p.labels[row];
            }
            float cv[NCH], c2[NCH];
            int cj[NCH];
#pragma unroll
            for (int c = 0; c < NCH; ++c) { cv[c] = INFINITY; c2[c] = INFINITY; cj[c] = 0; }
            for (int t = 0; t < p.NT; ++t, ++ai) {
                const int buf = ai % p.nacc;
                mbar_wait(smem_u32(&t_full[buf]), (ai / p.nacc) & 1);
                tc_fence_after();
                const uint32_t col0 = tmem_base + lane_addr + buf * p.NB + col_off;
                const int jbase = t * p.NB + col_off;
                if (!(p.dbg & 1)) {
                    if ((wcols & 31) == 0) {
                        for (int c = 0; c < wcols; c += 32) {
                            uint32_t va[32];
                            tmem_ld32(col0 + c, va);
                            tmem_wait_ld();
                            if (p.guard) fold32<true, FINAL>(va, cn_s, sc_s, m2, jbase + c, cv, cj, c2);
                            else fold32<false, FINAL>(va, cn_s, sc_s, m2, jbase + c, cv, cj, c2);
                        }
                    } else {   // wcols == 16
                        uint32_t va[32];
                        tmem_ld16(col0, va);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const int j = jbase + e;
                            const float s = p.guard ? m2 * sc_s[j] : -2.0f;
                            const float x = fmaf(__uint_as_float(va[e]), s, cn_s[j]);
                            const int c = e & 7, grp = j >> 3;
                            if (FINAL) {
                                const bool pr = x < cv[c];
                                const float t2 = fminf(c2[c], x);
                                c2[c] = pr ? cv[c] : t2;
                                cv[c] = pr ? x : cv[c];
                                cj[c] = pr ? grp : cj[c];
                            } else if (x < cv[c]) {
                                cv[c] = x;
                                cj[c] = grp;
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(mapa(smem_u32(&t_empty[buf]), 0));
            }
            // merge the 8 chains: lowest value, then lowest index (sequential-scan semantics)
            int w = 0;
            float b1;
            int j1;
            merge_chains(cv, cj, b1, j1, &w);
            float b2 = INFINITY;
            if (FINAL) {
#pragma unroll
                for (int c = 0; c < NCH; ++c) b2 = fminf(b2, c == w ? c2[c] : cv[c]);
            }
            // warpgroups 1..P_EWG-1 hand their partial to warpgroup 0 through smem
            const int ms = rbi & 1;
            if (wg != 0) {
                const int slot = (ms * (P_EWG - 1) + (wg - 1)) * P_BM + q;
                mg_v[slot] = b1;
                mg_j[slot] = j1;
                if (FINAL) mg_v2[slot] = b2;
                named_bar_arrive(1, P_EPI * 32);
                continue;
            }
            named_bar_sync(1, P_EPI * 32);
#pragma unroll
            for (int o = 0; o < P_EWG - 1; ++o) {
                const int slot = (ms * (P_EWG - 1) + o) * P_BM + q;
                const float ob1 = mg_v[slot];
                const int oj1 = mg_j[slot];
                const float ob2 = FINAL ? mg_v2[slot] : INFINITY;
                if (ob1 < b1 || (ob1 == b1 && oj1 < j1)) {
                    b2 = fminf(ob2, b1);
                    b1 = ob1;
                    j1 = oj1;
                } else {
                    b2 = fminf(b2, ob1);
                }
            }
            if (!valid) continue;
            if (!FINAL) {
                if (old_label != j1) my_changed += 1.0;
                p.labels[row] = j1;
                const float md = xn_row + b1;
                my_sse += md > 0.0f ? (double)md : 0.0;
            } else {
                p.labels[row] = j1;
                const double xn = (double)xn_row;
                const double si = p.guard ? (double)p.sx[row] : 1.0;
                const double cmax = (double)cn_max, smax = (double)s_max;
                const double S = sqrt(fmax(xn, 0.0) * fmax(cmax, 0.0)) * (1.0 + 1e-6);
                const double u32 = 5.9604644775390625e-08;
                const double ul = p.u_low;
                const double gacc = (double)(p.d_pad + 2) * 2.384185791015625e-07;
                const double gd = (double)p.d * u32 / (1.0 - (double)p.d * u32);
                const double E = 2.0 * (2.0 * ul + ul * ul + gacc + 2.0 * u32) * S +
                                 2.0 * p.eta_low * sqrt((double)p.d) *
                                     (si * sqrt(fmax(cmax, 0.0)) + smax * sqrt(fmax(xn, 0.0))) +
                                 u32 * (cmax + 2.0 * S);
                const double B32 = gd * 2.0 * S + u32 * (cmax + 2.0 * S);
                const double thr = 2.0 * (E + B32) * 1.001;
                const bool ok = isfinite(b1) && isfinite(xn) && isfinite(cmax) &&
                                ((double)b2 - (double)b1 > thr);
                if (!ok) {
                    const int slot = atomicAdd(p.fb_count, 1);
                    p.fb_rows[slot] = (int)row;
                }
            }
        }
        if (!FINAL && wg == 0) {
            my_sse = warp_sum(my_sse);
            my_changed = warp_sum(my_changed);
            if (lane == 0) {
                if (p.acc_sse) atomicAdd(p.acc_sse, my_sse);
                if (p.acc_changed && my_changed != 0.0) atomicAdd(p.acc_changed, my_changed);
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(p.tmem_cols)
                     : "memory");
    }
}

bool pair_plan(int dist, int d, int d_pad, int k, PairParams* pp, size_t* smem_bytes) {
    const int es = dist == KMEANS_E5M2 ? 1 : 2;
    const int RB = d_pad * es;
    const int SWZ = RB >= 128 ? 128 : RB;
    const int KB = RB / SWZ;
    // Centroid tile width: 256 (M = 256 x N = 256 MMAs; measured fastest: the per-tile handshake
    // cost dominates narrower tiles); MPK_PAIR_NB overrides (64/128/256) for experiments.
    int nb_cap = 256;
    if (const char* e = getenv("MPK_PAIR_NB")) nb_cap = atoi(e);
    if (nb_cap != 64 && nb_cap != 128 && nb_cap != 256) nb_cap = 256;
    int NB = k >= nb_cap ? nb_cap : ((k + 63) / 64) * 64;
    const int NT = (k + NB - 1) / NB;
    const int k_pad = NT * NB;
    const size_t b_half = (size_t)(NB / 2) * RB;
    const size_t a_tile = (size_t)P_BM * RB;
    const size_t fixed = 1024 + (size_t)k_pad * 8 + 3 * 2 * (P_EWG - 1) * P_BM * 4 + 8 +
                         (size_t)(2 * 8 + 1 + 2 * P_MAX_ACC) * 8 + 16;
    const size_t bres = (size_t)NT * b_half;
    if (fixed + bres + 2 * a_tile > P_BUDGET) return false;
    int SA = (int)std::min<size_t>(4, (P_BUDGET - fixed - bres) / a_tile);
    PairParams& p = *pp;
    p = PairParams{};
    p.k = k; p.k_pad = k_pad; p.d = d; p.d_pad = d_pad; p.NB = NB; p.NT = NT; p.KB = KB;
    p.SWZ = SWZ; p.SA = SA;
    p.nacc = std::min(P_MAX_ACC, 512 / NB);
    int cols = p.nacc * NB, pw = 32;
    while (pw < cols) pw <<= 1;
    p.tmem_cols = pw;
    p.a_tile_bytes = (uint32_t)a_tile;
    p.b_half_bytes = (uint32_t)b_half;
    p.kb_a_bytes = (uint32_t)P_BM * SWZ;
    p.kb_b_bytes = (uint32_t)(NB / 2) * SWZ;
    p.is_f8 = dist == KMEANS_E5M2;
    if (const char* e = getenv("MPK_PAIR_DBG")) p.dbg = atoi(e);
    p.u_low = dist == KMEANS_FP16 ? 0x1p-11 : (dist == KMEANS_BF16 ? 0x1p-8 : 0x1p-3);
    p.eta_low = dist == KMEANS_FP16 ? 0x1p-25 : (dist == KMEANS_BF16 ? 0x1p-134 : 0x1p-17);
    const uint32_t fmt = dist == KMEANS_BF16 ? 1u : (dist == KMEANS_E5M2 ? 1u : 0u);
    p.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(NB >> 3) << 17) |
              ((uint32_t)(256 >> 4) << 24);
    *smem_bytes = fixed + bres + (size_t)SA * a_tile;
    return true;
}

int pair_box_rows(const PairParams& p) { return p.NB / 2; }

cudaError_t pair_set_smem(size_t bytes) {
    cudaError_t e = cudaFuncSetAttribute(assign_pair_kernel<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(assign_pair_kernel<true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

cudaError_t pair_launch(const CUtensorMap& tmap_x, const CUtensorMap& tmap_c, const PairParams& p,
                        bool final_mode, size_t smem_bytes, cudaStream_t s) {
    const int64_t num_rb = (p.n + 2 * P_BM - 1) / (2 * P_BM);
    int64_t grid = std::min<int64_t>(kNumSMs, 2 * num_rb);
    grid &= ~int64_t(1);
    if (grid < 2) grid = 2;
    launches_add(1);
    if (final_mode)
        assign_pair_kernel<true><<<(unsigned)grid, P_THREADS, smem_bytes, s>>>(tmap_x, tmap_c, p);
    else
        assign_pair_kernel<false><<<(unsigned)grid, P_THREADS, smem_bytes, s>>>(tmap_x, tmap_c, p);
    return cudaGetLastError();
}

}  // namespace tcdev
}  // namespace mpk
