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
// try_wait with a suspend-time hint: the waiting warp is parked until the phase flips (or the
// hint expires) instead of re-polling; bare try_wait loops of the idle role warps measurably
// slowed the epilogue's memory instructions on the same SM.
MPK_DEV void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity), "r"(0x989680)
        : "memory");
}
// Non-suspending wait for the epilogue's "accumulator full": test_wait first (the phase has
// usually flipped long before the fold of the previous tile ends), then a bare try_wait loop.
// The suspend-hinted try_wait of mbar_wait() measured ~170 cycles per tile even when the phase
// was already complete.
MPK_DEV void mbar_wait_hot(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// Five phases at once (the grouped MMA issue: one accumulator and up to four X~ slots): all
// test_waits are issued back to back so their latencies (~150 cycles each) overlap, then a
// spinning try_wait on each one not yet complete. Repeating a barrier is allowed.
MPK_DEV void mbar_wait5_hot(uint32_t b0, uint32_t p0, const uint32_t (&b)[4], const uint32_t (&p)[4]) {
    asm volatile(
        "{\n\t.reg .pred Q0, Q1, Q2, Q3, Q4;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 Q0, [%0], %1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 Q1, [%2], %3;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 Q2, [%4], %5;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 Q3, [%6], %7;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 Q4, [%8], %9;\n\t"
        "@Q0 bra C1_%=;\n\t"
        "W0_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 Q0, [%0], %1;\n\t@!Q0 bra W0_%=;\n\t"
        "C1_%=:\n\t@Q1 bra C2_%=;\n\t"
        "W1_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 Q1, [%2], %3;\n\t@!Q1 bra W1_%=;\n\t"
        "C2_%=:\n\t@Q2 bra C3_%=;\n\t"
        "W2_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 Q2, [%4], %5;\n\t@!Q2 bra W2_%=;\n\t"
        "C3_%=:\n\t@Q3 bra C4_%=;\n\t"
        "W3_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 Q3, [%6], %7;\n\t@!Q3 bra W3_%=;\n\t"
        "C4_%=:\n\t@Q4 bra DONE_%=;\n\t"
        "W4_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 Q4, [%8], %9;\n\t@!Q4 bra W4_%=;\n\t"
        "DONE_%=:\n\t}" ::"r"(b0),
        "r"(p0), "r"(b[0]), "r"(p[0]), "r"(b[1]), "r"(p[1]), "r"(b[2]), "r"(p[2]), "r"(b[3]),
        "r"(p[3])
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
MPK_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31, %32};"
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
          "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),
          "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]),
          "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
          "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
MPK_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// wait::ld that also "defines" r, so the compiler cannot schedule reads of a prefetched
// tcgen05.ld destination above the wait (needed when loads are double-buffered)
MPK_DEV void tmem_wait_ld_dep(uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.wait::ld.sync.aligned;"
        : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
          "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]),
          "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]),
          "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]),
          "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]),
          "+r"(r[31])
        :
        : "memory");
}


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
// Argmin chains. Chain c of a point takes the columns j = 8 g + c; its state is
//   v : the running minimum of its values,
//   s : the position of its last STRICT improvement, as an offset (-1, -2, ...) from the next
//       group the chain will visit (a float; exact, |s| << 2^24),
// so that one column costs two alu-pipe ops and one fma-pipe op:
//   nf = !(x < v) ? 1 : 0   (set.geu: alu; NaN -> 1, no improvement)
//   v  = min(v, x)          (FMNMX: alu; keeps v for NaN x, equal values stay equal)
//   s  = s * nf - 1         (FFMA: fma pipe; 0 * s - 1 = -1 after an improvement)
// instead of FSETP + FSEL + SEL (three alu ops at rt 2, which bounded the fold at 6 cycles per
// warp-column). Ties keep the earlier group, the sequential scan's rule; merge_chains() then
// breaks ties across chains by the smaller column.
MPK_DEV void chain_step(float x, float& v, float& s) {
    float nf;
    asm("set.geu.f32.f32 %0, %1, %2;" : "=f"(nf) : "f"(x), "f"(v));
    v = fminf(v, x);
    s = fmaf(s, nf, -1.0f);
}
// Same with the chain's second minimum: new second = min(second, max(x, v)) (x < v: the old v,
// which is <= second; otherwise min(second, x)).
MPK_DEV void chain_step2(float x, float& v, float& v2, float& s) {
    v2 = fminf(v2, fmaxf(x, v));
    chain_step(x, v, s);
}
MPK_DEV void chains_init(float (&cv)[NCH], float (&cs)[NCH], float (&c2)[NCH]) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) { cv[c] = INFINITY; c2[c] = INFINITY; cs[c] = -1.0f; }
}
// Visited-group ordinal of chain c's last improvement after V groups (0 if it never improved,
// i.e. all its values were +inf or NaN — the scan's default label).
MPK_DEV int chain_ordinal(float s, int V) {
    const int v = V + (int)s;
    return v < 0 ? 0 : v;
}

// Warp-uniform 16-byte read of a small, hot, read-only global array (||c||^2, guard scales),
// kept in L1 (evict_last): the pair kernel spends its shared memory on the resident centroids
// and the X~ ring instead.
MPK_DEV float4 ldg_f4_keep(const float* p) {
    float4 r;
    asm("ld.global.nc.L1::evict_last.v4.f32 {%0, %1, %2, %3}, [%4];"
        : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
        : "l"(p));
    return r;
}
MPK_DEV float ldg_keep(const float* p) {
    float r;
    asm("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(r) : "l"(p));
    return r;
}

// Fold 32 TMEM accumulator columns (j0 .. j0+31, four groups) of one point into its 8 chains.
// GCN: cn / sc are global arrays (padded, see ldg_f4_keep) instead of shared memory.
template <bool GUARD, bool TOP2, bool GCN = false>
MPK_DEV void fold32(const uint32_t (&v)[32], const float* cn_s, const float* sc_s, float m2,
                    int j0, float (&cv)[NCH], float (&cs)[NCH], float (&c2)[NCH]) {
    const uint32_t cn_a = GCN ? 0u : smem_u32(cn_s + j0);
    const uint32_t sc_a = GCN ? 0u : smem_u32(sc_s + j0);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const float4 cc = GCN ? ldg_f4_keep(cn_s + j0 + 4 * e) : lds_f4(cn_a + 16 * e);
        float s[4] = {-2.0f, -2.0f, -2.0f, -2.0f};
        if (GUARD) {
            const float4 ss = GCN ? ldg_f4_keep(sc_s + j0 + 4 * e) : lds_f4(sc_a + 16 * e);
            s[0] = m2 * ss.x; s[1] = m2 * ss.y; s[2] = m2 * ss.z; s[3] = m2 * ss.w;
        }
        const float cnv[4] = {cc.x, cc.y, cc.z, cc.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float x = fmaf(__uint_as_float(v[4 * e + u]), s[u], cnv[u]);
            const int c = (e & 1) * 4 + u;
            if (TOP2) chain_step2(x, cv[c], c2[c], cs[c]);
            else chain_step(x, cv[c], cs[c]);
        }
    }
}

// Packed form of chain_step for two adjacent chains (c, c+1) and the two columns of one group
// that feed them: the two values x = acc * m + cn and the two offset updates s = s * nf - 1 are
// single FFMA2 (fp32x2) instructions, so a column costs 2 alu-pipe ops (set.geu, min) plus half
// of two fma-pipe ops, and the alu pipe — not instruction issue — bounds the fold.
// acc2 / cn2 / m2 hold (column c, column c+1) as the low / high words; s2 likewise.
MPK_DEV void chain_step_x2(uint64_t acc2, uint64_t cn2, uint64_t m2, float& va, float& vb,
                           uint64_t& s2, uint64_t m1) {
    asm("{\n\t"
        ".reg .b64 x2, nf2;\n\t"
        ".reg .f32 xa, xb, na, nb;\n\t"
        "fma.rn.f32x2 x2, %3, %4, %5;\n\t"
        "mov.b64 {xa, xb}, x2;\n\t"
        "set.geu.f32.f32 na, xa, %0;\n\t"
        "set.geu.f32.f32 nb, xb, %1;\n\t"
        "min.f32 %0, %0, xa;\n\t"
        "min.f32 %1, %1, xb;\n\t"
        "mov.b64 nf2, {na, nb};\n\t"
        "fma.rn.f32x2 %2, %2, nf2, %6;\n\t"
        "}"
        : "+f"(va), "+f"(vb), "+l"(s2)
        : "l"(acc2), "l"(m2), "l"(cn2), "l"(m1));
}
MPK_DEV uint64_t pack2(float lo, float hi) {
    return ((uint64_t)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
MPK_DEV uint64_t pack2u(uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | lo; }
MPK_DEV void unpack2(uint64_t v, float& lo, float& hi) {
    lo = __uint_as_float((uint32_t)v);
    hi = __uint_as_float((uint32_t)(v >> 32));
}
// fold32 without the second minimum, chain offsets kept packed in pairs (s2[m] = chains 2m,
// 2m+1). Same results as fold32<GUARD, false>: x is the same single-rounding fma per column and
// the chain update is the same three operations.
template <bool GUARD, bool GCN = false>
MPK_DEV void fold32_x2(const uint32_t (&v)[32], const float* cn_s, const float* sc_s, float m2,
                       int j0, float (&cv)[NCH], uint64_t (&s2)[NCH / 2]) {
    const uint32_t cn_a = GCN ? 0u : smem_u32(cn_s + j0);
    const uint32_t sc_a = GCN ? 0u : smem_u32(sc_s + j0);
    const uint64_t m1 = pack2(-1.0f, -1.0f);
    const uint64_t mm = pack2(-2.0f, -2.0f);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const float4 cc = GCN ? ldg_f4_keep(cn_s + j0 + 4 * e) : lds_f4(cn_a + 16 * e);
        uint64_t s01 = mm, s23 = mm;
        if (GUARD) {
            const float4 ss = GCN ? ldg_f4_keep(sc_s + j0 + 4 * e) : lds_f4(sc_a + 16 * e);
            s01 = pack2(m2 * ss.x, m2 * ss.y);
            s23 = pack2(m2 * ss.z, m2 * ss.w);
        }
        const int c0 = (e & 1) * 4;          // chains c0 .. c0+3 take columns 4e .. 4e+3
        chain_step_x2(pack2u(v[4 * e + 0], v[4 * e + 1]), pack2(cc.x, cc.y), s01, cv[c0 + 0],
                      cv[c0 + 1], s2[c0 / 2 + 0], m1);
        chain_step_x2(pack2u(v[4 * e + 2], v[4 * e + 3]), pack2(cc.z, cc.w), s23, cv[c0 + 2],
                      cv[c0 + 3], s2[c0 / 2 + 1], m1);
    }
}

// ---------------------------------------------------------------- reverse scan, 3-input minima
// ASSIGN mode of the pair kernel visits the columns in DECREASING order (tiles, chunks and
// groups reversed), so the sequential scan's "first column among equal minima" becomes "the
// LAST visit among equal minima": a non-strict improvement. That lets one chain take two
// columns per step with a single FMNMX3:
//   v' = min(v, xa, xb)            (xa visited first = the larger column; FMNMX3: alu)
//   na = (xa > v)  ? 1 : 0         (set.gtu: alu; NaN -> 1)
//   nb = (xb > v') ? 1 : 0         (set.gtu: alu; xb <= min(v, xa) <=> xb == v', NaN -> 1)
//   s  = (s * na - 1) * nb - 1     (two FFMA: fma pipe; packed over chains c, c+1)
// i.e. 1.5 alu ops per distance instead of 2. s is minus the number of visits since (and
// including) the chain's last improvement, so the forward ordinal of that visit is -1 - s
// (== V, out of range, if the chain never improved: all its values NaN). min ignores a NaN
// operand, so v never becomes NaN; NaN never improves. A chain whose minimum is +inf reports
// some +inf column; the caller maps a +inf row minimum to column 0, the forward scan's
// default, so results equal fold32_x2's.
// xa2 / xb2: the (chain c, chain c+1) values of the first / second visited group.
MPK_DEV void chain_pair_x2(uint64_t xa2, uint64_t xb2, float& va, float& vb, uint64_t& s2,
                           uint64_t m1) {
    asm("{\n\t"
        ".reg .b64 na2, nb2;\n\t"
        ".reg .f32 a0, a1, b0, b1, n0, n1, p0, p1, w0, w1;\n\t"
        "mov.b64 {a0, a1}, %3;\n\t"
        "mov.b64 {b0, b1}, %4;\n\t"
        "min.f32 w0, %0, a0, b0;\n\t"
        "min.f32 w1, %1, a1, b1;\n\t"
        "set.gtu.f32.f32 n0, a0, %0;\n\t"
        "set.gtu.f32.f32 n1, a1, %1;\n\t"
        "set.gtu.f32.f32 p0, b0, w0;\n\t"
        "set.gtu.f32.f32 p1, b1, w1;\n\t"
        "mov.f32 %0, w0;\n\t"
        "mov.f32 %1, w1;\n\t"
        "mov.b64 na2, {n0, n1};\n\t"
        "mov.b64 nb2, {p0, p1};\n\t"
        "fma.rn.f32x2 %2, %2, na2, %5;\n\t"
        "fma.rn.f32x2 %2, %2, nb2, %5;\n\t"
        "}"
        : "+f"(va), "+f"(vb), "+l"(s2)
        : "l"(xa2), "l"(xb2), "l"(m1));
}
MPK_DEV uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
// ||c_j||^2 (and the guard scales s_j) of G groups of 8 columns, loaded into registers ahead of
// the chunk's TMEM load so that the shared-memory latency overlaps the tcgen05.ld.
template <int G, bool GUARD>
struct ChunkCn {
    float4 cc[2 * G];
    float4 ss[GUARD ? 2 * G : 1];
};
template <int G, bool GUARD>
MPK_DEV void load_chunk_cn(const float* cn_s, const float* sc_s, int j0, ChunkCn<G, GUARD>& q) {
    const uint32_t cn_a = smem_u32(cn_s + j0);
    const uint32_t sc_a = smem_u32(sc_s + j0);
#pragma unroll
    for (int e = 0; e < 2 * G; ++e) {
        q.cc[e] = lds_f4(cn_a + 16 * e);
        if (GUARD) q.ss[e] = lds_f4(sc_a + 16 * e);
    }
}
// Fold G groups of 8 columns (j0 .. j0 + 8G - 1; G even) in reverse: group pairs (G-1, G-2),
// ..., (1, 0). Each value is the same single-rounding fma(acc, -2 s_i s_j, ||c_j||^2) as in
// fold32 / fold32_x2.
template <int G, bool GUARD>
MPK_DEV void fold_rev_m3(const uint32_t (&v)[32], const ChunkCn<G, GUARD>& q, float m2,
                         float (&cv)[NCH], uint64_t (&s2)[NCH / 2]) {
    static_assert(G % 2 == 0 && G <= 4, "group pairs");
    const uint64_t m1 = pack2(-1.0f, -1.0f);
    const uint64_t mm = pack2(-2.0f, -2.0f);
#pragma unroll
    for (int gp = G / 2 - 1; gp >= 0; --gp) {
        uint64_t x2[2][4];                   // [a = group 2gp+1, b = group 2gp][chain pair]
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int g = 2 * gp + 1 - h;
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
                const int col = 8 * g + 4 * qq;      // columns col .. col+3 = chains 4qq .. 4qq+3
                const float4 cc = q.cc[col / 4];
                uint64_t s01 = mm, s23 = mm;
                if (GUARD) {
                    const float4 ss = q.ss[col / 4];
                    s01 = pack2(m2 * ss.x, m2 * ss.y);
                    s23 = pack2(m2 * ss.z, m2 * ss.w);
                }
                x2[h][2 * qq + 0] = fma2(pack2u(v[col + 0], v[col + 1]), s01, pack2(cc.x, cc.y));
                x2[h][2 * qq + 1] = fma2(pack2u(v[col + 2], v[col + 3]), s23, pack2(cc.z, cc.w));
            }
        }
#pragma unroll
        for (int m = 0; m < NCH / 2; ++m)
            chain_pair_x2(x2[0][m], x2[1][m], cv[2 * m], cv[2 * m + 1], s2[m], m1);
    }
}
// Fold of an accumulator that already holds the (halved) distance ||c_j||^2 / 2 - x~.c~_j (the
// pair kernel's pre-loaded mode, k_assign_tc2.cu "cn init"): the values enter the chains as they
// are, no fma with ||c||^2 per column.
template <int G>
MPK_DEV void fold_rev_m3_direct(const uint32_t (&v)[32], float (&cv)[NCH], uint64_t (&s2)[NCH / 2]) {
    const uint64_t m1 = pack2(-1.0f, -1.0f);
#pragma unroll
    for (int gp = G / 2 - 1; gp >= 0; --gp) {
        uint64_t x2[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int g = 2 * gp + 1 - h;
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
                const int col = 8 * g + 4 * qq;
                x2[h][2 * qq + 0] = pack2u(v[col + 0], v[col + 1]);
                x2[h][2 * qq + 1] = pack2u(v[col + 2], v[col + 3]);
            }
        }
#pragma unroll
        for (int m = 0; m < NCH / 2; ++m)
            chain_pair_x2(x2[0][m], x2[1][m], cv[2 * m], cv[2 * m + 1], s2[m], m1);
    }
}
template <int G, bool GUARD>
MPK_DEV void fold_rev_m3(const uint32_t (&v)[32], const float* cn_s, const float* sc_s, float m2,
                         int j0, float (&cv)[NCH], uint64_t (&s2)[NCH / 2]) {
    ChunkCn<G, GUARD> q;
    load_chunk_cn<G, GUARD>(cn_s, sc_s, j0, q);
    fold_rev_m3<G, GUARD>(v, q, m2, cv, s2);
}

// Scalar-offset form of fold_rev_m3 (same values, same chain rule; two scalar FFMAs per chain
// step instead of two packed FFMA2 per chain pair): with 4 warps per SM sub-partition it issued
// faster than the packed form in tools/fold_bench.cu (112 vs 143 cycles per chunk per SMSP).
MPK_DEV void chain_pair(float xa, float xb, float& v, float& s) {
    float w, na, nb;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(w) : "f"(v), "f"(xa), "f"(xb));
    asm("set.gtu.f32.f32 %0, %1, %2;" : "=f"(na) : "f"(xa), "f"(v));
    asm("set.gtu.f32.f32 %0, %1, %2;" : "=f"(nb) : "f"(xb), "f"(w));
    v = w;
    s = fmaf(fmaf(s, na, -1.0f), nb, -1.0f);
}
template <int G, bool GUARD>
MPK_DEV void fold_rev_m3s(const uint32_t (&v)[32], const ChunkCn<G, GUARD>& q, float m2,
                          float (&cv)[NCH], float (&cs)[NCH]) {
    static_assert(G % 2 == 0 && G <= 4, "group pairs");
#pragma unroll
    for (int gp = G / 2 - 1; gp >= 0; --gp) {
        float x[2][NCH];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int g = 2 * gp + 1 - h;
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
                const int col = 8 * g + 4 * qq;
                const float4 cc = q.cc[col / 4];
                float sc[4] = {-2.0f, -2.0f, -2.0f, -2.0f};
                if (GUARD) {
                    const float4 ss = q.ss[col / 4];
                    sc[0] = m2 * ss.x; sc[1] = m2 * ss.y; sc[2] = m2 * ss.z; sc[3] = m2 * ss.w;
                }
                x[h][4 * qq + 0] = fmaf(__uint_as_float(v[col + 0]), sc[0], cc.x);
                x[h][4 * qq + 1] = fmaf(__uint_as_float(v[col + 1]), sc[1], cc.y);
                x[h][4 * qq + 2] = fmaf(__uint_as_float(v[col + 2]), sc[2], cc.z);
                x[h][4 * qq + 3] = fmaf(__uint_as_float(v[col + 3]), sc[3], cc.w);
            }
        }
#pragma unroll
        for (int c = 0; c < NCH; ++c) chain_pair(x[0][c], x[1][c], cv[c], cs[c]);
    }
}

// Reverse-scan chain step that also keeps the chain's second smallest value v2 (FINAL mode's
// certified filter): with m = min(xa, xb) (NaN ignored) and M = max.NaN(xa, xb) (NaN kept, so a
// NaN column contributes nothing),
//   v2' = min(v2, max(v, m), M)     (the second smallest of {v <= v2, xa, xb})
//   v'  = min(v, m);  n_a = [xa > v];  n_b = [xb > v'];  s = (s n_a - 1) n_b - 1
// 7 ALU ops per two columns instead of 4 per column (chain_step2).
MPK_DEV void chain_pair_t2(float xa, float xb, float& v, float& v2, float& s) {
    float m, M, t, w, na, nb;
    asm("min.f32 %0, %1, %2;" : "=f"(m) : "f"(xa), "f"(xb));
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(M) : "f"(xa), "f"(xb));
    asm("max.f32 %0, %1, %2;" : "=f"(t) : "f"(v), "f"(m));
    asm("min.f32 %0, %1, %2, %3;" : "=f"(v2) : "f"(v2), "f"(t), "f"(M));
    asm("min.f32 %0, %1, %2;" : "=f"(w) : "f"(v), "f"(m));
    asm("set.gtu.f32.f32 %0, %1, %2;" : "=f"(na) : "f"(xa), "f"(v));
    asm("set.gtu.f32.f32 %0, %1, %2;" : "=f"(nb) : "f"(xb), "f"(w));
    v = w;
    s = fmaf(fmaf(s, na, -1.0f), nb, -1.0f);
}
template <int G, bool GUARD>
MPK_DEV void fold_rev_t2(const uint32_t (&v)[32], const ChunkCn<G, GUARD>& q, float m2,
                         float (&cv)[NCH], float (&c2)[NCH], float (&cs)[NCH]) {
    static_assert(G % 2 == 0 && G <= 4, "group pairs");
#pragma unroll
    for (int gp = G / 2 - 1; gp >= 0; --gp) {
        float x[2][NCH];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int g = 2 * gp + 1 - h;
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
                const int col = 8 * g + 4 * qq;
                const float4 cc = q.cc[col / 4];
                float sc[4] = {-2.0f, -2.0f, -2.0f, -2.0f};
                if (GUARD) {
                    const float4 ss = q.ss[col / 4];
                    sc[0] = m2 * ss.x; sc[1] = m2 * ss.y; sc[2] = m2 * ss.z; sc[3] = m2 * ss.w;
                }
                x[h][4 * qq + 0] = fmaf(__uint_as_float(v[col + 0]), sc[0], cc.x);
                x[h][4 * qq + 1] = fmaf(__uint_as_float(v[col + 1]), sc[1], cc.y);
                x[h][4 * qq + 2] = fmaf(__uint_as_float(v[col + 2]), sc[2], cc.z);
                x[h][4 * qq + 3] = fmaf(__uint_as_float(v[col + 3]), sc[3], cc.w);
            }
        }
#pragma unroll
        for (int c = 0; c < NCH; ++c) chain_pair_t2(x[0][c], x[1][c], cv[c], c2[c], cs[c]);
    }
}

// Merge the chains of one point given each chain's column jj[c]: smallest value, then smallest
// column (the sequential scan's result). Returns the winning chain in *w (for TOP2).
MPK_DEV void merge_chains(const float (&cv)[NCH], const int (&jj)[NCH], float& b1, int& j1,
                          int* w) {
    b1 = cv[0];
    j1 = jj[0];
    int wc = 0;
#pragma unroll
    for (int c = 1; c < NCH; ++c) {
        if (cv[c] < b1 || (cv[c] == b1 && jj[c] < j1)) { b1 = cv[c]; j1 = jj[c]; wc = c; }
    }
    if (w) *w = wc;
}

// Opaque register copy of a kernel parameter: ptxas otherwise rematerialises parameters from
// the constant bank inside hot loops (LDC/LDCU on every iteration), which measured as hundreds of
// cycles per row-block in the pair kernel. The empty asm makes the value unknown, so it stays in
// a register.
MPK_DEV int pin(int v) { asm volatile("" : "+r"(v)); return v; }
MPK_DEV uint32_t pin(uint32_t v) { asm volatile("" : "+r"(v)); return v; }
MPK_DEV int64_t pin(int64_t v) { asm volatile("" : "+l"(v)); return v; }
MPK_DEV float pin(float v) { asm volatile("" : "+f"(v)); return v; }
template <typename T>
MPK_DEV T* pin(T* v) {
    asm volatile("" : "+l"(v));
    return v;
}

// One lane of a converged warp (elect.sync). Role loops run on the whole warp so that their
// barrier/descriptor arithmetic stays in uniform registers, and only the issue is elected:
// branching on `lane == 0` first makes every tcgen05/TMA operand divergent and ptxas wraps each
// issue in an R2UR.BROADCAST waterfall loop (~120 dependent cycles per MMA, measured).
MPK_DEV bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}
// Upper / lower words of umma_desc(): the K-advance inside a tile only touches the start
// address (bits 0-13, in 16-byte units), so a loop adds (bytes >> 4) to a precomputed low word.
MPK_DEV uint32_t umma_desc_lo(uint32_t saddr) { return ((saddr >> 4) & 0x3FFFu) | (1u << 16); }
MPK_DEV uint32_t umma_desc_hi(int swz) {
    const uint32_t layout = swz == 128 ? 2u : (swz == 64 ? 4u : 6u);
    return ((8u * (uint32_t)swz) >> 4) | (1u << 14) | (layout << 29);
}
MPK_DEV uint64_t desc_join(uint32_t hi, uint32_t lo) { return ((uint64_t)hi << 32) | lo; }

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
