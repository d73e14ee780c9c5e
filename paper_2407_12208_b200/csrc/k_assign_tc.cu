// k_assign_tc.cu — K4: the hot kernel. Distance + argmin on the 5th-generation tensor cores.
//
// For a block of 128 points and a tile of BN centroids the contraction x~_i . c~_j
// (the -2 P^T C term of eq:dist-eval, "level-3 BLAS" PAPER.md:208) runs as
// tcgen05.mma (kind::f16 for fp16/bf16, kind::f8f6f4 for E5M2 = the paper's q52) from
// TMA-loaded, 128B/64B/32B-swizzled shared-memory tiles into an fp32 accumulator in TMEM
// (fp32 accumulation: reading Z2/Z3). The epilogue warps read the accumulator with tcgen05.ld
// (one thread = one TMEM lane = one point) and fold
//     v_ij = fma(-2 s_i s_j, acc_ij, ||c_j||^2)          (Alg 4 line 6)
// into a running per-point (min, argmin) in registers, lowest j on ties (reading Z12): the
// n x k distance matrix never leaves the SM. Only labels, the changed-label count and the SSE_t
// partial (sum_i max(0, ||x_i||^2 + min_j v_ij)) are written.
//
// Structure (persistent, one CTA per SM, 192 threads):
//   warp 0      TMA producer: A = R row-blocks of X~ per group (ring of 2R slots, so the next
//               group prefetches while this one computes), B = centroid tiles (ring of S_B).
//   warp 1      MMA issuer (one elected thread): for each centroid tile, R MMAs (one per
//               row-block) into 4 rotating TMEM accumulators of 128 columns; tcgen05.commit
//               signals "accumulator full" and "smem slot free".
//   warps 2..5  epilogue: TMEM -> registers -> fma + argmin; arrive "accumulator empty".
// B tiles are re-streamed from L2 once per group of R*128 points (C~ is at most 256 KB).
#include <cuda.h>

#include <string>

#include "common.cuh"
#include "internal.h"

namespace mpk {

namespace tcdev {

constexpr int BM = 128;
constexpr int NUM_ACC = 4;
constexpr int ACC_COLS = 128;
constexpr int kThreads = 192;

struct Params {
    int64_t n;
    int k, k_pad, BN, NT, KB, SWZ, R, SB;
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
};

MPK_DEV uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
MPK_DEV void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
MPK_DEV void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
MPK_DEV void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
MPK_DEV void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
MPK_DEV void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
MPK_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
MPK_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
MPK_DEV void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     bar)
                 : "memory");
}
MPK_DEV void mma_f16(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accum)
        : "memory");
}
MPK_DEV void mma_f8(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accum)
        : "memory");
}
// K-major operand, canonical swizzled layout: rows of SWZ bytes, 8-row atoms (SBO = 8*SWZ).
MPK_DEV uint64_t umma_desc(uint32_t saddr, int swz) {
    uint64_t layout = swz == 128 ? 2ull : (swz == 64 ? 4ull : 6ull);
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;                              // LBO (unused for swizzled K-major)
    d |= (uint64_t)(((8u * (uint32_t)swz) >> 4) & 0x3FFFu) << 32;   // SBO
    d |= (uint64_t)1u << 46;                              // descriptor version (sm_100)
    d |= layout << 61;
    return d;
}
MPK_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}
MPK_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
MPK_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <int R>
__global__ void __launch_bounds__(kThreads, 1)
assign_tc_kernel(const __grid_constant__ CUtensorMap tmap_x,
                 const __grid_constant__ CUtensorMap tmap_c, Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-align the dynamic smem base (SW128 atoms)
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int NA = 2 * R;
    uint8_t* a_base = smem;
    uint8_t* b_base = a_base + (size_t)NA * p.a_tile_bytes;
    float* cn_s = (float*)(b_base + (size_t)p.SB * p.b_tile_bytes);
    float* sc_s = cn_s + p.k_pad;
    uint64_t* bars = (uint64_t*)(sc_s + (p.guard ? p.k_pad : 0));
    uint64_t* a_full = bars;
    uint64_t* a_empty = a_full + NA;
    uint64_t* b_full = a_empty + NA;
    uint64_t* b_empty = b_full + p.SB;
    uint64_t* t_full = b_empty + p.SB;
    uint64_t* t_empty = t_full + NUM_ACC;
    uint32_t* tmem_slot = (uint32_t*)(t_empty + NUM_ACC);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    for (int j = threadIdx.x; j < p.k_pad; j += blockDim.x) {
        cn_s[j] = j < p.k ? p.cn[j] : INFINITY;       // padded centroids never win
        if (p.guard) sc_s[j] = j < p.k ? p.sc[j] : 1.0f;
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < NA; ++i) { mbar_init(smem_u32(&a_full[i]), 1); mbar_init(smem_u32(&a_empty[i]), 1); }
        for (int i = 0; i < p.SB; ++i) { mbar_init(smem_u32(&b_full[i]), 1); mbar_init(smem_u32(&b_empty[i]), 1); }
        for (int i = 0; i < NUM_ACC; ++i) { mbar_init(smem_u32(&t_full[i]), 1); mbar_init(smem_u32(&t_empty[i]), 4); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_c)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(NUM_ACC * ACC_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int64_t rows_per_group = (int64_t)R * BM;
    const int64_t num_groups = (p.n + rows_per_group - 1) / rows_per_group;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            uint32_t gi = 0, bi = 0;
            for (int64_t g = blockIdx.x; g < num_groups; g += gridDim.x, ++gi) {
                for (int r = 0; r < R; ++r) {
                    uint32_t u = gi * R + r;
                    int slot = u % NA;
                    mbar_wait(smem_u32(&a_empty[slot]), ((u / NA) & 1) ^ 1);
                    uint32_t fb = smem_u32(&a_full[slot]);
                    mbar_expect_tx(fb, p.a_tile_bytes);
                    uint32_t dst = smem_u32(a_base + (size_t)slot * p.a_tile_bytes);
                    int row0 = (int)(g * rows_per_group + r * BM);
                    for (int kb = 0; kb < p.KB; ++kb)
                        tma_load_2d(dst + kb * p.kb_a_bytes, &tmap_x, kb * p.SWZ / (p.is_f8 ? 1 : 2),
                                    row0, fb);
                }
                for (int t = 0; t < p.NT; ++t, ++bi) {
                    int st = bi % p.SB;
                    mbar_wait(smem_u32(&b_empty[st]), ((bi / p.SB) & 1) ^ 1);
                    uint32_t fb = smem_u32(&b_full[st]);
                    mbar_expect_tx(fb, p.b_tile_bytes);
                    uint32_t dst = smem_u32(b_base + (size_t)st * p.b_tile_bytes);
                    for (int kb = 0; kb < p.KB; ++kb)
                        tma_load_2d(dst + kb * p.kb_b_bytes, &tmap_c, kb * p.SWZ / (p.is_f8 ? 1 : 2),
                                    t * p.BN, fb);
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
                    int st = bi % p.SB;
                    mbar_wait(smem_u32(&b_full[st]), (bi / p.SB) & 1);
                    const uint32_t b_addr = smem_u32(b_base + (size_t)st * p.b_tile_bytes);
                    for (int r = 0; r < R; ++r, ++ai) {
                        uint32_t u = gi * R + r;
                        int slot = u % NA;
                        if (t == 0) mbar_wait(smem_u32(&a_full[slot]), (u / NA) & 1);
                        int buf = ai % NUM_ACC;
                        mbar_wait(smem_u32(&t_empty[buf]), ((ai / NUM_ACC) & 1) ^ 1);
                        tc_fence_after();
                        const uint32_t a_addr = smem_u32(a_base + (size_t)slot * p.a_tile_bytes);
                        const uint32_t d_tmem = tmem_base + buf * ACC_COLS;
                        for (int kb = 0; kb < p.KB; ++kb) {
                            for (int ks = 0; ks < ksteps; ++ks) {
                                uint64_t ad = umma_desc(a_addr + kb * p.kb_a_bytes + ks * 32, p.SWZ);
                                uint64_t bd = umma_desc(b_addr + kb * p.kb_b_bytes + ks * 32, p.SWZ);
                                uint32_t accum = (kb | ks) ? 1u : 0u;
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
    } else {
        // ------------------------------------------------ epilogue (warps 2..5)
        const int quarter = warp & 3;                 // TMEM lanes 32*quarter .. +31
        const int q = quarter * 32 + lane;            // row within the row-block
        const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
        double my_sse = 0.0, my_changed = 0.0;
        uint32_t ai = 0;
        for (int64_t g = blockIdx.x; g < num_groups; g += gridDim.x) {
            float best[R];
            int bidx[R];
            float m2[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                best[r] = INFINITY;
                bidx[r] = 0;
                int64_t row = g * rows_per_group + r * BM + q;
                m2[r] = (p.guard && row < p.n) ? -2.0f * p.sx[row] : -2.0f;
            }
            for (int t = 0; t < p.NT; ++t) {
#pragma unroll
                for (int r = 0; r < R; ++r, ++ai) {
                    int buf = ai % NUM_ACC;
                    mbar_wait(smem_u32(&t_full[buf]), (ai / NUM_ACC) & 1);
                    tc_fence_after();
                    const uint32_t col0 = tmem_base + lane_addr + buf * ACC_COLS;
                    float bv = best[r];
                    int bj = bidx[r];
                    if ((p.BN & 31) == 0) {
                        for (int c = 0; c < p.BN; c += 32) {
                            uint32_t v[32];
                            tmem_ld32(col0 + c, v);
                            tmem_wait_ld();
                            const int j0 = t * p.BN + c;
                            const float4* cn4 = reinterpret_cast<const float4*>(cn_s + j0);
                            if (!p.guard) {
#pragma unroll
                                for (int e = 0; e < 8; ++e) {
                                    float4 cc = cn4[e];
                                    float x0 = fmaf(__uint_as_float(v[4 * e + 0]), -2.0f, cc.x);
                                    float x1 = fmaf(__uint_as_float(v[4 * e + 1]), -2.0f, cc.y);
                                    float x2 = fmaf(__uint_as_float(v[4 * e + 2]), -2.0f, cc.z);
                                    float x3 = fmaf(__uint_as_float(v[4 * e + 3]), -2.0f, cc.w);
                                    if (x0 < bv) { bv = x0; bj = j0 + 4 * e + 0; }
                                    if (x1 < bv) { bv = x1; bj = j0 + 4 * e + 1; }
                                    if (x2 < bv) { bv = x2; bj = j0 + 4 * e + 2; }
                                    if (x3 < bv) { bv = x3; bj = j0 + 4 * e + 3; }
                                }
                            } else {
                                const float4* sc4 = reinterpret_cast<const float4*>(sc_s + j0);
#pragma unroll
                                for (int e = 0; e < 8; ++e) {
                                    float4 cc = cn4[e];
                                    float4 ss = sc4[e];
                                    float x0 = fmaf(__uint_as_float(v[4 * e + 0]), m2[r] * ss.x, cc.x);
                                    float x1 = fmaf(__uint_as_float(v[4 * e + 1]), m2[r] * ss.y, cc.y);
                                    float x2 = fmaf(__uint_as_float(v[4 * e + 2]), m2[r] * ss.z, cc.z);
                                    float x3 = fmaf(__uint_as_float(v[4 * e + 3]), m2[r] * ss.w, cc.w);
                                    if (x0 < bv) { bv = x0; bj = j0 + 4 * e + 0; }
                                    if (x1 < bv) { bv = x1; bj = j0 + 4 * e + 1; }
                                    if (x2 < bv) { bv = x2; bj = j0 + 4 * e + 2; }
                                    if (x3 < bv) { bv = x3; bj = j0 + 4 * e + 3; }
                                }
                            }
                        }
                    } else {
                        for (int c = 0; c < p.BN; c += 16) {
                            uint32_t v[32];
                            tmem_ld16(col0 + c, v);
                            tmem_wait_ld();
                            const int j0 = t * p.BN + c;
#pragma unroll
                            for (int e = 0; e < 16; ++e) {
                                float s = p.guard ? m2[r] * sc_s[j0 + e] : -2.0f;
                                float x = fmaf(__uint_as_float(v[e]), s, cn_s[j0 + e]);
                                if (x < bv) { bv = x; bj = j0 + e; }
                            }
                        }
                    }
                    best[r] = bv;
                    bidx[r] = bj;
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(smem_u32(&t_empty[buf]));
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                int64_t row = g * rows_per_group + r * BM + q;
                if (row < p.n) {
                    int old = p.labels[row];
                    if (old != bidx[r]) my_changed += 1.0;
                    p.labels[row] = bidx[r];
                    double md = (double)p.xn[row] + (double)best[r];
                    my_sse += md > 0.0 ? md : 0.0;
                }
            }
        }
        my_sse = warp_sum(my_sse);
        my_changed = warp_sum(my_changed);
        if (lane == 0) {
            if (p.acc_sse) atomicAdd(p.acc_sse, my_sse);
            if (p.acc_changed && my_changed != 0.0) atomicAdd(p.acc_changed, my_changed);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(NUM_ACC * ACC_COLS)
                     : "memory");
    }
}

}  // namespace tcdev

// ----------------------------------------------------------------------------------------------
// Host side: plan (tile shapes, smem budget, TMA descriptors) and launch.
// ----------------------------------------------------------------------------------------------
struct TcPlan {
    int dist, d, d_pad, k, R, esize;
    int64_t n;
    CUtensorMap tmap_x, tmap_c;
    tcdev::Params prm;
    size_t smem_bytes;
};

static int esize_of(int dist) { return dist == KMEANS_E5M2 ? 1 : 2; }

int tc_dpad(int dist, int d) {
    int es = esize_of(dist);
    int rb = ((d * es + 31) / 32) * 32;           // at least one 32-byte MMA K step
    if (rb > 64) rb = ((rb + 127) / 128) * 128;   // 96 -> 128; multiples of 128 otherwise
    return rb / es;
}

bool tc_supported(int dist, int d_pad, int k) {
    if (dist != KMEANS_FP16 && dist != KMEANS_BF16 && dist != KMEANS_E5M2) return false;
    int rb = d_pad * esize_of(dist);
    if (rb > 512) return false;    // d <= 256 (fp16/bf16) / 512 (e5m2): A tile <= 64 KB
    if (k < 16) return false;      // tiny k: the SIMT kernels are the right tool
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

TcPlan* tc_plan_create(int dist, int64_t n, int d, int d_pad, int k, const void* Xl,
                       const void* Cl, std::string* err) {
    TcPlan* pl = new TcPlan();
    pl->dist = dist; pl->n = n; pl->d = d; pl->d_pad = d_pad; pl->k = k;
    const int es = esize_of(dist);
    pl->esize = es;
    const int RB = d_pad * es;
    const int SWZ = RB >= 128 ? 128 : RB;   // 32, 64 or 128
    const int KB = RB / SWZ;
    int BN = k >= 128 ? 128 : ((k + 15) / 16) * 16;
    if (BN > 32 && (BN & 31)) BN = ((BN + 31) / 32) * 32;
    const int NT = (k + BN - 1) / BN;
    const int k_pad = NT * BN;
    const uint32_t a_tile = (uint32_t)tcdev::BM * RB;
    const uint32_t b_tile = (uint32_t)BN * RB;
    const size_t budget = 227 * 1024;
    int R = 0, SB = 0;
    for (int r : {4, 2, 1}) {
        for (int sb : {4, 3, 2}) {
            size_t bytes = 1024 + (size_t)2 * r * a_tile + (size_t)sb * b_tile +
                           (size_t)k_pad * 8 + 64 * 8 + 16;
            if (bytes <= budget) { R = r; SB = sb; break; }
        }
        if (R) break;
    }
    if (!R) { if (err) *err = "tile does not fit in shared memory"; delete pl; return nullptr; }
    pl->R = R;
    tcdev::Params& p = pl->prm;
    p = tcdev::Params{};
    p.k = k; p.k_pad = k_pad; p.BN = BN; p.NT = NT; p.KB = KB; p.SWZ = SWZ; p.R = R; p.SB = SB;
    p.a_tile_bytes = a_tile; p.b_tile_bytes = b_tile;
    p.kb_a_bytes = (uint32_t)tcdev::BM * SWZ;
    p.kb_b_bytes = (uint32_t)BN * SWZ;
    p.is_f8 = dist == KMEANS_E5M2;
    // instruction descriptor: fp32 accumulate, K-major A/B, M = 128, N = BN
    uint32_t fmt = dist == KMEANS_BF16 ? 1u : (dist == KMEANS_E5M2 ? 1u : 0u);
    p.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(BN >> 3) << 17) |
              ((uint32_t)(tcdev::BM >> 4) << 24);
    pl->smem_bytes = 1024 + (size_t)2 * R * a_tile + (size_t)SB * b_tile + (size_t)k_pad * 8 +
                     64 * 8 + 16;
    if (!encode(&pl->tmap_x, dist, Xl, n, d_pad, SWZ, tcdev::BM, err) ||
        !encode(&pl->tmap_c, dist, Cl, k, d_pad, SWZ, BN, err)) {
        delete pl;
        return nullptr;
    }
    cudaError_t e = cudaSuccess;
    if (R == 4)
        e = cudaFuncSetAttribute(tcdev::assign_tc_kernel<4>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl->smem_bytes);
    else if (R == 2)
        e = cudaFuncSetAttribute(tcdev::assign_tc_kernel<2>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl->smem_bytes);
    else
        e = cudaFuncSetAttribute(tcdev::assign_tc_kernel<1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl->smem_bytes);
    if (e != cudaSuccess) {
        if (err) *err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
        delete pl;
        return nullptr;
    }
    return pl;
}

void tc_plan_destroy(TcPlan* p) { delete p; }

cudaError_t launch_assign_tc(TcPlan* pl, const Problem& pb, const float* xn, const float* sx,
                             const float* cn, const float* sc, int32_t* labels, double* acc_sse,
                             double* acc_changed, cudaStream_t s) {
    launches_add(1);
    tcdev::Params p = pl->prm;
    p.n = pb.n;
    p.guard = pb.guard;
    p.xn = xn; p.sx = sx; p.cn = cn; p.sc = sc;
    p.labels = labels;
    p.acc_sse = acc_sse;
    p.acc_changed = acc_changed;
    size_t smem = pl->smem_bytes;
    int64_t groups = (pb.n + (int64_t)pl->R * tcdev::BM - 1) / ((int64_t)pl->R * tcdev::BM);
    int grid = (int)(groups < kNumSMs ? groups : kNumSMs);
    if (grid < 1) return cudaSuccess;
    if (pl->R == 4)
        tcdev::assign_tc_kernel<4><<<grid, tcdev::kThreads, smem, s>>>(pl->tmap_x, pl->tmap_c, p);
    else if (pl->R == 2)
        tcdev::assign_tc_kernel<2><<<grid, tcdev::kThreads, smem, s>>>(pl->tmap_x, pl->tmap_c, p);
    else
        tcdev::assign_tc_kernel<1><<<grid, tcdev::kThreads, smem, s>>>(pl->tmap_x, pl->tmap_c, p);
    return cudaGetLastError();
}

}  // namespace mpk
