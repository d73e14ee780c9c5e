// tc_common.cuh — device helpers shared by the tcgen05 kernels (inline PTX for sm_100a):
// mbarriers, TMA, tcgen05 MMA / commit / TMEM loads, UMMA shared-memory descriptors, and the
// argmin fold of the epilogue.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace mpk {
namespace tcdev {

constexpr int NCH = 8;   // independent argmin chains per point

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


MPK_DEV float4 lds_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}

// Fold 32 accumulator columns j0..j0+31 (j0 a multiple of 8) into the chains:
//   v = fma(acc, -2 s_i s_j, ||c_j||^2).
// Chain c takes the columns j = 8g + c; it records the GROUP g of its minimum (one add per 8
// columns instead of per column); the column is recovered as 8 g + c when chains merge.
// TOP2 also tracks the second-smallest value of each chain.
template <bool GUARD, bool TOP2>
MPK_DEV void fold32(const uint32_t (&v)[32], const float* cn_s, const float* sc_s, float m2,
                    int j0, float (&cv)[NCH], int (&cg)[NCH], float (&c2)[NCH]) {
    const uint32_t cn_a = smem_u32(cn_s + j0);
    const uint32_t sc_a = smem_u32(sc_s + j0);
    const int g0 = j0 >> 3;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const float4 cc = lds_f4(cn_a + 16 * e);
        float s[4] = {-2.0f, -2.0f, -2.0f, -2.0f};
        if (GUARD) {
            const float4 ss = lds_f4(sc_a + 16 * e);
            s[0] = m2 * ss.x; s[1] = m2 * ss.y; s[2] = m2 * ss.z; s[3] = m2 * ss.w;
        }
        const float cnv[4] = {cc.x, cc.y, cc.z, cc.w};
        const int g = g0 + (e >> 1);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float x = fmaf(__uint_as_float(v[4 * e + u]), s[u], cnv[u]);
            const int c = (e & 1) * 4 + u;
            if (TOP2) {
                const bool p = x < cv[c];
                const float t2 = fminf(c2[c], x);
                c2[c] = p ? cv[c] : t2;
                cv[c] = p ? x : cv[c];
                cg[c] = p ? g : cg[c];
            } else {
                if (x < cv[c]) { cv[c] = x; cg[c] = g; }
            }
        }
    }
}

// Merge the chains of one point: smallest value, then smallest column (the sequential scan's
// result). Returns the winning chain in *w (for the TOP2 second minimum).
MPK_DEV void merge_chains(const float (&cv)[NCH], const int (&cg)[NCH], float& b1, int& j1,
                          int* w) {
    b1 = cv[0];
    j1 = cg[0] * 8;
    int wc = 0;
#pragma unroll
    for (int c = 1; c < NCH; ++c) {
        const int j = cg[c] * 8 + c;
        if (cv[c] < b1 || (cv[c] == b1 && j < j1)) { b1 = cv[c]; j1 = j; wc = c; }
    }
    if (w) *w = wc;
}

// ---------------------------------------------------------------- CTA-pair (cta_group::2) helpers
MPK_DEV uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
MPK_DEV void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
MPK_DEV uint32_t mapa(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
MPK_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
// TMA load issued by either CTA of the pair; bytes complete on the LEADER's barrier (peer bit
// cleared, as CUTLASS SM100_TMA_2SM_LOAD does).
MPK_DEV void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar & 0xFEFFFFFFu)
        : "memory");
}
MPK_DEV void mma2_f16(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accum)
        : "memory");
}
MPK_DEV void mma2_f8(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accum)
        : "memory");
}
// commit arriving on the barrier at this smem offset in both CTAs of the pair
MPK_DEV void tc_commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar),
        "h"((uint16_t)0x3)
        : "memory");
}

}  // namespace tcdev
}  // namespace mpk
