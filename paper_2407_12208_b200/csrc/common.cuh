// common.cuh — shared device helpers of the B200 mixed-precision k-means library.
// Formats: Table 1. Rounding: one round-to-nearest-even step from the working
// value, gradual underflow, IEEE overflow to +-inf (readings Z5-Z8 in DESIGN.md).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <stdint.h>

#include "../../include/kmeans.h"

#define MPK_DEV __device__ __forceinline__

namespace mpk {

constexpr int kNumSMs = 148;

// ------------------------------------------------------------------------------------------
// Low-precision storage types and single-step RNE conversions.
// ------------------------------------------------------------------------------------------
struct e5m2_t { uint8_t bits; };

template <int P> struct low_type;
template <> struct low_type<KMEANS_FP64> { using T = double; };
template <> struct low_type<KMEANS_FP32> { using T = float; };
template <> struct low_type<KMEANS_FP16> { using T = __half; };
template <> struct low_type<KMEANS_BF16> { using T = __nv_bfloat16; };
template <> struct low_type<KMEANS_E5M2> { using T = e5m2_t; };

template <int P> constexpr int low_size() { return (int)sizeof(typename low_type<P>::T); }

// E5M2 overflow threshold 2^15 (2 - 2^-3) = 61440 (midpoint of x_max = 57344 and 2^16).
constexpr float kE5M2Overflow = 61440.0f;

MPK_DEV uint8_t e5m2_from_float(float v) {
    // cvt.rn.satfinite.e5m2x2.f32 rounds once (RNE, subnormals) but saturates at 57344;
    // values at/above the midpoint 61440 must become +-inf (IEEE, reading Z7).
    __nv_fp8x2_storage_t s = __nv_cvt_float2_to_fp8x2(make_float2(v, 0.0f), __NV_SATFINITE,
                                                      __NV_E5M2);
    uint8_t b = (uint8_t)(s & 0xff);
    if (fabsf(v) >= kE5M2Overflow) b = (uint8_t)(signbit(v) ? 0xFC : 0x7C);
    return b;
}
MPK_DEV uint8_t e5m2_from_double(double v) {
    return (uint8_t)__nv_cvt_double_to_fp8(v, __NV_NOSAT, __NV_E5M2);   // one rounding
}
MPK_DEV float e5m2_to_float(uint8_t b) {
    // E5M2 is the top byte of an IEEE half: widening is exact.
    return __half2float(__ushort_as_half((unsigned short)b << 8));
}

// Round a working value to the storage type of precision P (one RNE step).
template <int P> struct rounder;
template <> struct rounder<KMEANS_FP64> {
    MPK_DEV static double from(double v) { return v; }
    MPK_DEV static double from(float v) { return (double)v; }
};
template <> struct rounder<KMEANS_FP32> {
    MPK_DEV static float from(double v) { return __double2float_rn(v); }
    MPK_DEV static float from(float v) { return v; }
};
template <> struct rounder<KMEANS_FP16> {
    MPK_DEV static __half from(double v) { return __double2half(v); }     // cvt.rn.f16.f64
    MPK_DEV static __half from(float v) { return __float2half_rn(v); }    // cvt.rn.f16.f32
};
template <> struct rounder<KMEANS_BF16> {
    MPK_DEV static __nv_bfloat16 from(double v) { return __double2bfloat16(v); }  // cvt.rn.bf16.f64
    MPK_DEV static __nv_bfloat16 from(float v) { return __float2bfloat16_rn(v); }
};
template <> struct rounder<KMEANS_E5M2> {
    MPK_DEV static e5m2_t from(double v) { return e5m2_t{e5m2_from_double(v)}; }
    MPK_DEV static e5m2_t from(float v) { return e5m2_t{e5m2_from_float(v)}; }
};

// Widen a stored low-precision value to float (exact for fp16/bf16/e5m2) or keep double.
MPK_DEV float widen(__half v) { return __half2float(v); }
MPK_DEV float widen(__nv_bfloat16 v) { return __bfloat162float(v); }
MPK_DEV float widen(e5m2_t v) { return e5m2_to_float(v.bits); }
MPK_DEV float widen(float v) { return v; }
MPK_DEV double widen(double v) { return v; }

MPK_DEV bool is_nonfinite_low(__half v) { return !isfinite(__half2float(v)); }
MPK_DEV bool is_nonfinite_low(__nv_bfloat16 v) { return !isfinite(__bfloat162float(v)); }
MPK_DEV bool is_nonfinite_low(e5m2_t v) { return (v.bits & 0x7C) == 0x7C; }
MPK_DEV bool is_nonfinite_low(float v) { return !isfinite(v); }
MPK_DEV bool is_nonfinite_low(double v) { return !isfinite(v); }

// "underflow": a nonzero source value whose rounded value is zero or subnormal (reading Z8).
MPK_DEV bool is_zero_or_subnormal_low(__half v) {
    unsigned short b = __half_as_ushort(v);
    return (b & 0x7C00) == 0;
}
MPK_DEV bool is_zero_or_subnormal_low(__nv_bfloat16 v) {
    unsigned short b = __bfloat16_as_ushort(v);
    return (b & 0x7F80) == 0;
}
MPK_DEV bool is_zero_or_subnormal_low(e5m2_t v) { return (v.bits & 0x7C) == 0; }
MPK_DEV bool is_zero_or_subnormal_low(float v) { return fabsf(v) < 1.17549435e-38f; }
MPK_DEV bool is_zero_or_subnormal_low(double v) { return fabs(v) < 2.2250738585072014e-308; }

// Alg 4's operand scale from a vector's infinity norm: guard 1 (reading Z9
// A) s = ||x||_inf; guard 2 (reading Z9 B, KMEANS_GUARD_POW2) s = 2^ceil(log2 ||x||_inf), the
// smallest power of two >= the norm, so x / s is exact (an MX / UE8M0 block scale with the row
// as one block). Zero or NaN norm -> 1 (reading Z10); a power of two that would overflow -> the
// norm itself.
MPK_DEV float guard_scale(float amax, int guard) {
    if (amax == 0.0f || isnan(amax)) return 1.0f;
    if (guard != 2) return amax;
    const uint32_t b = __float_as_uint(amax);
    if ((b & 0x007fffffu) == 0u && (b & 0x7f800000u) != 0u) return amax;   // already 2^e
    int e;
    (void)frexpf(amax, &e);                   // amax = m 2^e, m in [0.5, 1)
    const float s = ldexpf(1.0f, e);
    return isinf(s) ? amax : s;
}
MPK_DEV double guard_scale(double amax, int guard) {
    if (amax == 0.0 || isnan(amax)) return 1.0;
    if (guard != 2) return amax;
    int e;
    const double m = frexp(amax, &e);
    if (m == 0.5) return amax;
    const double s = ldexp(1.0, e);
    return isinf(s) ? amax : s;
}

// ------------------------------------------------------------------------------------------
// Reductions.
// ------------------------------------------------------------------------------------------
// Programmatic dependent launch: a kernel launched with launch_pdl may start while its
// predecessor in the stream drains; it waits here (first statement) for that predecessor's
// completion and memory. A no-op for an ordinary launch.
MPK_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename T> MPK_DEV T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// (value, index) argmin merge: smaller value wins; equal values -> lower index (reading Z12).
MPK_DEV void argmin_merge(float& v, int& j, float v2, int j2) {
    if (v2 < v || (v2 == v && j2 < j)) { v = v2; j = j2; }
}
MPK_DEV void argmin_merge(double& v, int& j, double v2, int j2) {
    if (v2 < v || (v2 == v && j2 < j)) { v = v2; j = j2; }
}

MPK_DEV double atomic_add_f64(double* p, double v) { return atomicAdd(p, v); }

}  // namespace mpk
