// k_assign_tc.cu — K4: the hot kernel. Distance + argmin on the 5th-generation tensor cores.
//
// For a block of 128 points and a tile of BN centroids the contraction x~_i . c~_j
// (the -2 P^T C term of eq:dist-eval, "level-3 BLAS" PAPER.md:208) runs as
// tcgen05.mma (kind::f16 for fp16/bf16, kind::f8f6f4 for E5M2 = the paper's q52) from
// TMA-loaded, 128B/64B/32B-swizzled shared-memory tiles into an fp32 accumulator in TMEM
// (fp32 accumulation: reading Z2/Z3). The epilogue warps read the accumulator with tcgen05.ld
// (one thread = one TMEM lane = one point) and fold
//     v_ij = fma(-2 s_i s_j, acc_ij, ||c_j||^2)          (Alg 4 line 6)
// into per-point (min, argmin) chains in registers, merged with lowest-j-on-ties (reading
// Z12): the n x k distance matrix never leaves the SM. Only labels, the changed-label count and
// the SSE_t partial (sum_i max(0, ||x_i||^2 + min_j v_ij)) are written.
//
// FINAL mode (Alg 3 step 7, "computed in precision u") runs the same contraction
// as a certified filter: the epilogue also keeps the second-smallest v, and a row whose gap
// v_(2) - v_(1) exceeds twice a rigorous bound on |v^ - v| (operand rounding, fp32
// accumulation, and the working-precision evaluation's own error) gets the
// low-precision argmin, which then provably equals the working-precision argmin. Other rows are
// appended to a list that the CUDA-core working-precision kernel re-evaluates.
//
// Structure (persistent, one CTA per SM, 384 threads):
//   warp 0      A producer (TMA): R row-blocks of X~ per group, ring of 2R slots (the next group
//               prefetches while the current one computes).
//   warp 2      B producer (TMA): centroid tiles, ring of SB stages (runs ahead independently).
//   warp 1      MMA issuer (one elected thread): per centroid tile, R MMAs (one per row-block)
//               into rotating TMEM accumulators; tcgen05.commit frees smem and signals TMEM.
//   warps 4-11  epilogue, two warpgroups: warpgroup w handles the row-blocks r = w (mod 2),
//               so one warpgroup computes while the other waits on TMEM.
// C~ is at most 256 KB (L2-resident) and is re-streamed once per group of R*128 points.
#include <cuda.h>

#include <string>

#include "common.cuh"
#include "internal.h"
#include "tc_common.cuh"
#include "tc_pair.h"

#include <stdlib.h>

namespace mpk {

namespace tcdev {

constexpr int BM = 128;
constexpr int kNonEpiWarps = 4;
constexpr int kEpiWarps = 8;
constexpr int kThreads = (kNonEpiWarps + kEpiWarps) * 32;
constexpr int MAX_ACC = 8;

struct Params {
    int64_t n;
    int k, k_pad, d, d_pad, BN, NT, KB, SWZ, R, SB, nacc, acc_cols, tmem_cols;
    uint32_t a_tile_bytes, b_tile_bytes, kb_a_bytes, kb_b_bytes;
    uint32_t idesc;
    int guard, is_f8;
    const float* xn;
    const float* sx;
    const float* cn;
    const float* sc;
    int32_t* labels;
    double* acc_sse;
    double* acc_changed;
    // FINAL mode: uncertified rows are appended here
    int* fb_count;
    int* fb_rows;
    double u_low;     // unit roundoff of the filter operands
    double eta_low;   // half the smallest subnormal of the filter format (absolute underflow)
};

template <int R, bool FINAL>
__global__ void __launch_bounds__(kThreads, 1)
assign_tc_kernel(const __grid_constant__ CUtensorMap tmap_x,
                 const __grid_constant__ CUtensorMap tmap_c, Params p) {
    static_assert(R % 2 == 0, "two epilogue warpgroups split the row-blocks by parity");
    constexpr int RH = R / 2;   // row-blocks per warpgroup
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int NA = 2 * R;
    uint8_t* a_base = smem;
    uint8_t* b_base = a_base + (size_t)NA * p.a_tile_bytes;
    float* cn_s = (float*)(b_base + (size_t)p.SB * p.b_tile_bytes);
    float* sc_s = cn_s + p.k_pad;
    uint64_t* bars = (uint64_t*)(sc_s + p.k_pad);
    uint64_t* a_full = bars;
    uint64_t* a_empty = a_full + NA;
    uint64_t* b_full = a_empty + NA;
    uint64_t* b_empty = b_full + p.SB;
    uint64_t* t_full = b_empty + p.SB;
    uint64_t* t_empty = t_full + MAX_ACC;
    uint32_t* tmem_slot = (uint32_t*)(t_empty + MAX_ACC);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    for (int j = threadIdx.x; j < p.k_pad; j += blockDim.x) {
        cn_s[j] = j < p.k ? p.cn[j] : INFINITY;       // padded centroids never win
        sc_s[j] = (p.guard && j < p.k) ? p.sc[j] : 1.0f;
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < NA; ++i) { mbar_init(smem_u32(&a_full[i]), 1); mbar_init(smem_u32(&a_empty[i]), 1); }
        for (int i = 0; i < p.SB; ++i) { mbar_init(smem_u32(&b_full[i]), 1); mbar_init(smem_u32(&b_empty[i]), 1); }
        for (int i = 0; i < p.nacc; ++i) { mbar_init(smem_u32(&t_full[i]), 1); mbar_init(smem_u32(&t_empty[i]), 4); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_c)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(p.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int64_t rows_per_group = (int64_t)R * BM;
    const int64_t num_groups = (p.n + rows_per_group - 1) / rows_per_group;
    const int elem_per_swz = p.SWZ / (p.is_f8 ? 1 : 2);

    if (warp == 0) {
        // ------------------------------------------------ A producer
        if (lane == 0) {
            uint32_t u = 0;
            for (int64_t g = blockIdx.x; g < num_groups; g += gridDim.x) {
                for (int r = 0; r < R; ++r, ++u) {
                    const int slot = u % NA;
                    mbar_wait(smem_u32(&a_empty[slot]), ((u / NA) & 1) ^ 1);
                    const uint32_t fb = smem_u32(&a_full[slot]);
                    mbar_expect_tx(fb, p.a_tile_bytes);
                    const uint32_t dst = smem_u32(a_base + (size_t)slot * p.a_tile_bytes);
                    const int row0 = (int)(g * rows_per_group + r * BM);
                    for (int kb = 0; kb < p.KB; ++kb)
                        tma_load_2d(dst + kb * p.kb_a_bytes, &tmap_x, kb * elem_per_swz, row0, fb);
                }
            }
        }
    } else if (warp == 2) {
        // ------------------------------------------------ B producer
        if (lane == 0) {
            uint32_t bi = 0;
            for (int64_t g = blockIdx.x; g < num_groups; g += gridDim.x) {
                for (int t = 0; t < p.NT; ++t, ++bi) {
                    const int st = bi % p.SB;
                    mbar_wait(smem_u32(&b_empty[st]), ((bi / p.SB) & 1) ^ 1);
                    const uint32_t fb = smem_u32(&b_full[st]);
                    mbar_expect_tx(fb, p.b_tile_bytes);
                    const uint32_t dst = smem_u32(b_base + (size_t)st * p.b_tile_bytes);
                    for (int kb = 0; kb < p.KB; ++kb)
                        tma_load_2d(dst + kb * p.kb_b_bytes, &tmap_c, kb * elem_per_swz, t * p.BN,
                                    fb);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            uint32_t gi = 0, bi = 0, ai = 0;
            const int ksteps = p.SWZ / 32;   // 32-byte K per MMA: 16 fp16/bf16 or 32 e5m2
            for (int64_t g = blockIdx.x; g < num_groups; g += gridDim.x, ++gi) {
                for (int t = 0; t < p.NT; ++t, ++bi) {
                    const int st = bi % p.SB;
                    mbar_wait(smem_u32(&b_full[st]), (bi / p.SB) & 1);
                    const uint32_t b_addr = smem_u32(b_base + (size_t)st * p.b_tile_bytes);
                    for (int r = 0; r < R; ++r, ++ai) {
                        const uint32_t u = gi * R + r;
                        const int slot = u % NA;
                        if (t == 0) mbar_wait(smem_u32(&a_full[slot]), (u / NA) & 1);
                        const int buf = ai % p.nacc;
                        mbar_wait(smem_u32(&t_empty[buf]), ((ai / p.nacc) & 1) ^ 1);
                        tc_fence_after();
                        const uint32_t a_addr = smem_u32(a_base + (size_t)slot * p.a_tile_bytes);
                        const uint32_t d_tmem = tmem_base + buf * p.acc_cols;
                        for (int kb = 0; kb < p.KB; ++kb) {
                            for (int ks = 0; ks < ksteps; ++ks) {
                                const uint64_t ad =
                                    umma_desc(a_addr + kb * p.kb_a_bytes + ks * 32, p.SWZ);
                                const uint64_t bd =
                                    umma_desc(b_addr + kb * p.kb_b_bytes + ks * 32, p.SWZ);
                                const uint32_t accum = (kb | ks) ? 1u : 0u;
                                if (p.is_f8) mma_f8(d_tmem, ad, bd, p.idesc, accum);
                                else mma_f16(d_tmem, ad, bd, p.idesc, accum);
                            }
                        }
                        tc_commit(smem_u32(&t_full[buf]));
                        if (t == p.NT - 1) tc_commit(smem_u32(&a_empty[slot]));
                    }
                    tc_commit(smem_u32(&b_empty[st]));
                }
            }
        }
    } else if (warp >= kNonEpiWarps) {
        // ------------------------------------------------ epilogue (2 warpgroups)
        const int wg = (warp - kNonEpiWarps) >> 2;      // row-blocks r = wg (mod 2)
        const int quarter = warp & 3;                   // TMEM lanes 32*quarter .. +31
        const int q = quarter * 32 + lane;              // row within the row-block
        const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
        float cn_max = 0.0f, s_max = 1.0f;
        if (FINAL) {
            for (int j = 0; j < p.k; ++j) {
                cn_max = fmaxf(cn_max, cn_s[j]);
                s_max = fmaxf(s_max, sc_s[j]);
            }
        }
        double my_sse = 0.0, my_changed = 0.0;
        uint32_t gi = 0;
        for (int64_t g = blockIdx.x; g < num_groups; g += gridDim.x, ++gi) {
            float cv[RH][NCH], c2[RH][NCH], cs[RH][NCH];
            float m2[RH];
#pragma unroll
            for (int h = 0; h < RH; ++h) {
                chains_init(cv[h], cs[h], c2[h]);
                const int64_t row = g * rows_per_group + (2 * h + wg) * BM + q;
                m2[h] = (p.guard && row < p.n) ? -2.0f * p.sx[row] : -2.0f;
            }
            for (int t = 0; t < p.NT; ++t) {
#pragma unroll
                for (int h = 0; h < RH; ++h) {
                    const int r = 2 * h + wg;
                    const uint32_t ai = (gi * p.NT + t) * R + r;
                    const int buf = ai % p.nacc;
                    mbar_wait(smem_u32(&t_full[buf]), (ai / p.nacc) & 1);
                    tc_fence_after();
                    const uint32_t col0 = tmem_base + lane_addr + buf * p.acc_cols;
                    if ((p.BN & 63) == 0) {
                        for (int c = 0; c < p.BN; c += 64) {
                            uint32_t v0[32], v1[32];
                            tmem_ld32(col0 + c, v0);
                            tmem_ld32(col0 + c + 32, v1);
                            tmem_wait_ld();
                            const int j0 = t * p.BN + c;
                            if (p.guard) {
                                fold32<true, FINAL>(v0, cn_s, sc_s, m2[h], j0, cv[h], cs[h], c2[h]);
                                fold32<true, FINAL>(v1, cn_s, sc_s, m2[h], j0 + 32, cv[h], cs[h], c2[h]);
                            } else {
                                fold32<false, FINAL>(v0, cn_s, sc_s, m2[h], j0, cv[h], cs[h], c2[h]);
                                fold32<false, FINAL>(v1, cn_s, sc_s, m2[h], j0 + 32, cv[h], cs[h], c2[h]);
                            }
                        }
                    } else if ((p.BN & 31) == 0) {   // BN = 32, 96: 32-column chunks
                        for (int c = 0; c < p.BN; c += 32) {
                            uint32_t v0[32];
                            tmem_ld32(col0 + c, v0);
                            tmem_wait_ld();
                            const int j0 = t * p.BN + c;
                            if (p.guard) fold32<true, FINAL>(v0, cn_s, sc_s, m2[h], j0, cv[h], cs[h], c2[h]);
                            else fold32<false, FINAL>(v0, cn_s, sc_s, m2[h], j0, cv[h], cs[h], c2[h]);
                        }
                    } else {   // BN == 16
                        uint32_t v[32];
                        tmem_ld16(col0, v);
                        tmem_wait_ld();
                        const int j0 = t * p.BN;
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const float s = p.guard ? m2[h] * sc_s[j0 + e] : -2.0f;
                            const float x = fmaf(__uint_as_float(v[e]), s, cn_s[j0 + e]);
                            const int c = e & 7;                 // chain c = (j0 + e) & 7
                            if (FINAL) chain_step2(x, cv[h][c], c2[h][c], cs[h][c]);
                            else chain_step(x, cv[h][c], cs[h][c]);
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(smem_u32(&t_empty[buf]));
                }
            }
#pragma unroll
            for (int h = 0; h < RH; ++h) {
                // every thread visits all groups of all tiles in order: ordinal = group
                int jj[NCH];
#pragma unroll
                for (int c = 0; c < NCH; ++c) jj[c] = 8 * chain_ordinal(cs[h][c], p.NT * (p.BN >> 3)) + c;
                int w = 0;
                float b1;
                int j1;
                merge_chains(cv[h], jj, b1, j1, &w);
                const int64_t row = g * rows_per_group + (2 * h + wg) * BM + q;
                if (row >= p.n) continue;
                if (!FINAL) {
                    const int old = p.labels[row];
                    if (old != j1) my_changed += 1.0;
                    p.labels[row] = j1;
                    const double md = (double)p.xn[row] + (double)b1;
                    my_sse += md > 0.0 ? md : 0.0;
                } else {
                    float b2 = INFINITY;
#pragma unroll
                    for (int c = 0; c < NCH; ++c) b2 = fminf(b2, c == w ? c2[h][c] : cv[h][c]);
                    p.labels[row] = j1;
                    // certification: |v^ - v| <= E, |fl32(v) - v| <= B32
                    const double xn = (double)p.xn[row];
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
        }
        if (!FINAL) {
            my_sse = warp_sum(my_sse);
            my_changed = warp_sum(my_changed);
            if (lane == 0) {
                if (p.acc_sse) atomicAdd(p.acc_sse, my_sse);
                if (p.acc_changed && my_changed != 0.0) atomicAdd(p.acc_changed, my_changed);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(p.tmem_cols)
                     : "memory");
    }
}

}  // namespace tcdev

// ----------------------------------------------------------------------------------------------
// Host side: plan (tile shapes, smem budget, TMA descriptors) and launch.
// ----------------------------------------------------------------------------------------------
struct TcPlan {
    int dist, d, d_pad, k, R, esize;
    int kind;                      // 2 = CTA-pair centroid-stationary, 1 = streaming
    int64_t n;
    CUtensorMap tmap_x, tmap_c;
    tcdev::Params prm;             // kind 1
    tcdev::PairParams pp;          // kind 2
    size_t smem_bytes;
    const void* Xl;                // the operand rows tmap_x covers (for gathers)
};

static int esize_of(int dist) { return dist == KMEANS_E5M2 ? 1 : 2; }

int tc_dpad(int dist, int d) {
    int es = esize_of(dist);
    int rb = ((d * es + 31) / 32) * 32;           // at least one 32-byte MMA K step
    if (rb > 64) rb = ((rb + 127) / 128) * 128;   // 96 -> 128; multiples of 128 otherwise
    return rb / es;
}

// The streaming kernel keeps 2R (R >= 2) row-block slots of 128 rows: 4 x 128 x RB bytes must
// leave room for at least two centroid stages, which holds for rows of at most 256 bytes.
static bool stream_plan_fits(int rb) { return rb <= 256; }

bool tc_supported(int dist, int d_pad, int k) {
    if (dist != KMEANS_FP16 && dist != KMEANS_BF16 && dist != KMEANS_E5M2) return false;
    int rb = d_pad * esize_of(dist);
    if (rb > 512) return false;    // A tile <= 64 KB
    if (k < 16) return false;      // tiny k: the CUDA-core kernels are the right tool
    if (!stream_plan_fits(rb)) {
        // 512-byte rows (fp16/bf16, 192 < d <= 256): only the CTA-pair kernel, and only while
        // its resident centroid halves fit; beyond that the CUDA-core kernel serves
        tcdev::PairParams pp;
        size_t smem = 0;
        return tcdev::pair_plan(dist, d_pad, d_pad, k, &pp, &smem);
    }
    return true;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

static bool encode(CUtensorMap* m, int dist, const void* base, int64_t rows, int d_pad, int swz,
                   int box_rows, std::string* err) {
    EncodeTiledFn fn = get_encode();
    if (!fn) { if (err) *err = "cuTensorMapEncodeTiled unavailable"; return false; }
    int es = esize_of(dist);
    CUtensorMapDataType dt = dist == KMEANS_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                             : dist == KMEANS_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                   : CU_TENSOR_MAP_DATA_TYPE_UINT8;
    cuuint64_t gdim[2] = {(cuuint64_t)d_pad, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)d_pad * es};
    cuuint32_t box[2] = {(cuuint32_t)(swz / es), (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUtensorMapSwizzle sw = swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                        : CU_TENSOR_MAP_SWIZZLE_32B;
    CUresult r = fn(m, dt, 2, const_cast<void*>(base), gdim, gstride, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        if (err) *err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
        return false;
    }
    return true;
}

template <int R, bool FINAL>
static cudaError_t set_smem(size_t bytes) {
    return cudaFuncSetAttribute(tcdev::assign_tc_kernel<R, FINAL>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

TcPlan* tc_plan_create(int dist, int64_t n, int d, int d_pad, int k, const void* Xl,
                       const void* Cl, std::string* err) {
    TcPlan* pl = new TcPlan();
    pl->dist = dist; pl->n = n; pl->d = d; pl->d_pad = d_pad; pl->k = k;
    pl->Xl = Xl;
    const int es = esize_of(dist);
    pl->esize = es;
    // Preferred: CTA pairs with the centroid tiles resident in shared memory (k_assign_tc2.cu).
    const char* force = getenv("MPK_TC_KIND");
    // MPK_TC_KIND=1 (tests, experiments) forces the streaming kernel where its plan fits
    if (!(force && force[0] == '1' && stream_plan_fits(d_pad * es))) {
        size_t smem = 0;
        if (tcdev::pair_plan(dist, d, d_pad, k, &pl->pp, &smem)) {
            const int swz = pl->pp.SWZ;
            if (encode(&pl->tmap_x, dist, Xl, n, d_pad, swz, 128, err) &&
                encode(&pl->tmap_c, dist, Cl, k, d_pad, swz, tcdev::pair_box_rows(pl->pp), err) &&
                tcdev::pair_set_smem(smem) == cudaSuccess) {
                pl->kind = 2;
                pl->smem_bytes = smem;
                pl->R = 2;
                return pl;
            }
            cudaGetLastError();
        }
    }
    pl->kind = 1;
    const int RB = d_pad * es;
    const int SWZ = RB >= 128 ? 128 : RB;   // 32, 64 or 128
    const int KB = RB / SWZ;
    const double rate = dist == KMEANS_E5M2 ? 8192.0 : 4096.0;   // dense MAC / clk / SM
    const size_t budget = 227 * 1024;
    // Choose (BN, R, SB): enough B stages in flight to cover the L2 -> smem latency
    // (>= ~4096 MMA cycles), then the largest R*BN (less re-streaming), then more stages.
    int bestBN = 0, bestR = 0, bestSB = 0;
    double best_key[3] = {-1, -1, -1};
    for (int bn_cap : {128, 64, 32}) {
        int bn = k >= bn_cap ? bn_cap : ((k + 15) / 16) * 16;
        if (bn > 32 && (bn & 31)) bn = ((bn + 31) / 32) * 32;
        const int nt = (k + bn - 1) / bn;
        const size_t fixed = 1024 + (size_t)nt * bn * 8 + 64 * 8 + 64;
        for (int r : {4, 2}) {
            const size_t a = (size_t)2 * r * tcdev::BM * RB;
            const size_t b = (size_t)bn * RB;
            if (fixed + a + 2 * b > budget) continue;
            int sb = (int)std::min<size_t>(8, (budget - fixed - a) / b);
            const double stage = (double)r * tcdev::BM * bn * d_pad / rate;
            const double key[3] = {std::min(stage * sb, 4096.0), (double)r * bn, (double)sb};
            bool better = false;
            for (int q = 0; q < 3; ++q) {
                if (key[q] != best_key[q]) { better = key[q] > best_key[q]; break; }
            }
            if (better) {
                for (int q = 0; q < 3; ++q) best_key[q] = key[q];
                bestBN = bn; bestR = r; bestSB = sb;
            }
        }
    }
    if (!bestR) { if (err) *err = "tile does not fit in shared memory"; delete pl; return nullptr; }
    const int BN = bestBN, R = bestR, SB = bestSB;
    const int NT = (k + BN - 1) / BN;
    const int k_pad = NT * BN;
    pl->R = R;
    tcdev::Params& p = pl->prm;
    p = tcdev::Params{};
    p.k = k; p.k_pad = k_pad; p.d = d; p.d_pad = d_pad; p.BN = BN; p.NT = NT; p.KB = KB;
    p.SWZ = SWZ; p.R = R; p.SB = SB;
    p.acc_cols = BN < 32 ? 32 : BN;
    p.nacc = std::min(tcdev::MAX_ACC, 512 / p.acc_cols);
    int cols = p.nacc * p.acc_cols;
    int pw = 32;
    while (pw < cols) pw <<= 1;
    p.tmem_cols = pw;
    p.a_tile_bytes = (uint32_t)tcdev::BM * RB;
    p.b_tile_bytes = (uint32_t)BN * RB;
    p.kb_a_bytes = (uint32_t)tcdev::BM * SWZ;
    p.kb_b_bytes = (uint32_t)BN * SWZ;
    p.is_f8 = dist == KMEANS_E5M2;
    // filter constants for FINAL mode (unit roundoff, half smallest subnormal)
    p.u_low = dist == KMEANS_FP16 ? 0x1p-11 : (dist == KMEANS_BF16 ? 0x1p-8 : 0x1p-3);
    p.eta_low = dist == KMEANS_FP16 ? 0x1p-25 : (dist == KMEANS_BF16 ? 0x1p-134 : 0x1p-17);
    // instruction descriptor: fp32 accumulate, K-major A/B, M = 128, N = BN
    const uint32_t fmt = dist == KMEANS_BF16 ? 1u : (dist == KMEANS_E5M2 ? 1u : 0u);
    p.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(BN >> 3) << 17) |
              ((uint32_t)(tcdev::BM >> 4) << 24);
    pl->smem_bytes = 1024 + (size_t)2 * R * p.a_tile_bytes + (size_t)SB * p.b_tile_bytes +
                     (size_t)k_pad * 8 + 2 * tcdev::MAX_ACC * 8 + (size_t)(4 * R + 2 * SB) * 8 +
                     64;
    if (pl->smem_bytes > budget + 1024) {
        if (err) *err = "smem plan overflow";
        delete pl;
        return nullptr;
    }
    if (!encode(&pl->tmap_x, dist, Xl, n, d_pad, SWZ, tcdev::BM, err) ||
        !encode(&pl->tmap_c, dist, Cl, k, d_pad, SWZ, BN, err)) {
        delete pl;
        return nullptr;
    }
    cudaError_t e = R == 4 ? set_smem<4, false>(pl->smem_bytes) : set_smem<2, false>(pl->smem_bytes);
    if (e == cudaSuccess)
        e = R == 4 ? set_smem<4, true>(pl->smem_bytes) : set_smem<2, true>(pl->smem_bytes);
    if (e != cudaSuccess) {
        if (err) *err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
        delete pl;
        return nullptr;
    }
    return pl;
}

void tc_plan_destroy(TcPlan* p) { delete p; }

static cudaError_t launch_impl(TcPlan* pl, const tcdev::Params& p, bool final_mode,
                               cudaStream_t s) {
    const int64_t groups = (p.n + (int64_t)pl->R * tcdev::BM - 1) / ((int64_t)pl->R * tcdev::BM);
    const int grid = (int)(groups < kNumSMs ? groups : kNumSMs);
    if (grid < 1) return cudaSuccess;
    launches_add(1);
    const size_t smem = pl->smem_bytes;
    if (pl->R == 4) {
        if (final_mode)
            tcdev::assign_tc_kernel<4, true><<<grid, tcdev::kThreads, smem, s>>>(pl->tmap_x, pl->tmap_c, p);
        else
            tcdev::assign_tc_kernel<4, false><<<grid, tcdev::kThreads, smem, s>>>(pl->tmap_x, pl->tmap_c, p);
    } else {
        if (final_mode)
            tcdev::assign_tc_kernel<2, true><<<grid, tcdev::kThreads, smem, s>>>(pl->tmap_x, pl->tmap_c, p);
        else
            tcdev::assign_tc_kernel<2, false><<<grid, tcdev::kThreads, smem, s>>>(pl->tmap_x, pl->tmap_c, p);
    }
    return cudaGetLastError();
}

cudaError_t launch_assign_tc(TcPlan* pl, const Problem& pb, const float* xn, const float* sx,
                             const float* cn, const float* sc, int32_t* labels, double* acc_sse,
                             double* acc_changed, cudaStream_t s, FxState* fx, bool* fx_listed) {
    if (fx_listed) *fx_listed = false;
    tcdev::Params p = pl->prm;
    p.n = pb.n;
    p.guard = pb.guard;
    p.xn = xn; p.sx = sx; p.cn = cn; p.sc = sc;
    p.labels = labels;
    p.acc_sse = acc_sse;
    p.acc_changed = acc_changed;
    if (pl->kind == 2) {
        tcdev::PairParams q = pl->pp;
        q.n = pb.n; q.guard = pb.guard; q.xn = xn; q.sx = sx; q.cn = cn; q.sc = sc;
        q.labels = labels; q.acc_sse = acc_sse; q.acc_changed = acc_changed;
        if (fx && !getenv("MPK_NO_FX_LIST")) {
            // gate[0] (the count) is zero here: zeroed before the first iteration, then by
            // finalize_fx after each update
            q.fx_list = fx->list; q.fx_seg_cnt = fx->seg_cnt; q.fx_gate = fx->gate;
            if (fx_listed) *fx_listed = true;
        }
        return tcdev::pair_launch(pl->tmap_x, pl->tmap_c, q, tcdev::PAIR_ASSIGN, pl->smem_bytes, s);
    }
    return launch_impl(pl, p, false, s);
}

cudaError_t launch_final_tc(TcPlan* pl, const Problem& pb, const float* xn, const float* sx,
                            const float* cn, const float* sc, int32_t* labels, int* fb_count,
                            int* fb_rows, float* fb_thr, cudaStream_t s) {
    tcdev::Params p = pl->prm;
    p.n = pb.n;
    p.guard = pb.guard;
    p.xn = xn; p.sx = sx; p.cn = cn; p.sc = sc;
    p.labels = labels;
    p.fb_count = fb_count;
    p.fb_rows = fb_rows;
    if (pl->kind == 2) {
        tcdev::PairParams q = pl->pp;
        q.n = pb.n; q.guard = pb.guard; q.xn = xn; q.sx = sx; q.cn = cn; q.sc = sc;
        q.labels = labels; q.fb_count = fb_count; q.fb_rows = fb_rows; q.fb_thr = fb_thr;
        return tcdev::pair_launch(pl->tmap_x, pl->tmap_c, q, tcdev::PAIR_FINAL, pl->smem_bytes, s);
    }
    return launch_impl(pl, p, true, s);
}

bool tc_plan_has_cand(const TcPlan* pl) { return pl && pl->kind == 2; }
int tc_plan_kind(const TcPlan* pl) { return pl ? pl->kind : 0; }
const void* tc_plan_operands(const TcPlan* pl, int* row_bytes) {
    *row_bytes = pl->d_pad * pl->esize;
    return pl->Xl;
}

cudaError_t launch_cand_tc(TcPlan* pl, const void* Xc, int64_t nc, int guard, const float* sxc,
                           const float* cn, const float* sc, const float* thr, int* cand_cnt,
                           int* cand, int cand_q, cudaStream_t s) {
    if (pl->kind != 2) return cudaErrorNotSupported;
    if (nc <= 0) return cudaSuccess;
    CUtensorMap tmx;
    std::string err;
    if (!encode(&tmx, pl->dist, Xc, nc, pl->d_pad, pl->pp.SWZ, 128, &err))
        return cudaErrorInvalidValue;
    tcdev::PairParams q = pl->pp;
    q.n = nc; q.guard = guard; q.sx = sxc; q.cn = cn; q.sc = sc;
    q.thr = thr; q.cand_cnt = cand_cnt; q.cand = cand; q.cand_q = cand_q;
    return tcdev::pair_launch(tmx, pl->tmap_c, q, tcdev::PAIR_CAND, pl->smem_bytes, s);
}

}  // namespace mpk
