// qgroup.cuh -- one 32-element MXFP4 group per call, scalar fp32 (the v3 quantizer pipeline).
//
// Bit-exact restatement of the reference transforms and quantizers (mx4train/_backend/_native.pyx):
//   FWHT-32  fwht                 _native.pyx:353-379  stages h = 1..16, (a+b)*c / (a-b)*c, c = fp32(1/sqrt 2)
//   RTN      quantize_rtn         _native.pyx:104-131
//   SR       quantize_sr          _native.pyx:134-168  (sr_code in quant.cuh)
//   QuEST    quantize_quest       _native.pyx:171-245  (fp32 search, exact f64 near-tie fallback)
//
// Why scalar: on B200 a packed FFMA2/FADD2 costs two issue cycles (measured, tools/ubench), so it moves
// no more elements per clock than FFMA/FADD, while scalar code lets each thread hold ONE group (32
// registers) and ptxas cannot contract __fmul_rn/__fadd_rn (it does contract mul.rn.f32x2 ->
// add.rn.f32x2, see quant.cuh).  Every quantizer here is issue-bound, so the design counts issue slots:
//   * bf16 inputs enter the first butterfly stage through FHADD.BF16 (add.rn.f32.bf16: one operand
//     converted exactly inside the add), so the conversion of half the elements is free;
//   * randomized-Hadamard signs are XORed onto whole bf16 words (one LOP3 per two elements) or folded
//     into the dequantization scale (requantization of an MXFP4 operand);
//   * the backward pre-scale 0.75 is folded into the power-of-two quantization scale when that is
//     provably exact (e >= 4, see rtn_scale);
//   * e2m1 bytes are packed with PRMT, -0 canonicalised with three LOP3/IADD per 8 nibbles.
#pragma once
#include "common.cuh"
#include "launch.h"
#include "quant.cuh"  // sr_code, quest_exact_cold (f64 reference search)

namespace qt {

constexpr float kHc = 0.70710678118654752440f;  // 0x3F3504F3 == (float)(1.0 / sqrt(2.0))

// ------------------------------------------------------------------------- bf16 halves
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(__byte_perm(w, 0u, 0x1044)); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
// fp32 a +/- c where a is the low / high bf16 half of w (exact widening inside the add, one rounding).
__device__ __forceinline__ float fh_add_lo(uint32_t w, float c) {
    float d;
    asm("{\n .reg .b16 l, h;\n mov.b32 {l, h}, %1;\n add.rn.f32.bf16 %0, l, %2;\n}" : "=f"(d) : "r"(w), "f"(c));
    return d;
}
__device__ __forceinline__ float fh_sub_lo(uint32_t w, float c) {
    float d;
    asm("{\n .reg .b16 l, h;\n mov.b32 {l, h}, %1;\n sub.rn.f32.bf16 %0, l, %2;\n}" : "=f"(d) : "r"(w), "f"(c));
    return d;
}
__device__ __forceinline__ float fh_add_hi(uint32_t w, float c) {
    float d;
    asm("{\n .reg .b16 l, h;\n mov.b32 {l, h}, %1;\n add.rn.f32.bf16 %0, h, %2;\n}" : "=f"(d) : "r"(w), "f"(c));
    return d;
}
__device__ __forceinline__ float fh_sub_hi(uint32_t w, float c) {
    float d;
    asm("{\n .reg .b16 l, h;\n mov.b32 {l, h}, %1;\n sub.rn.f32.bf16 %0, h, %2;\n}" : "=f"(d) : "r"(w), "f"(c));
    return d;
}

// ------------------------------------------------------------------------------- FWHT-32
__device__ __forceinline__ void bfly(float& a, float& b) {
    const float s = __fadd_rn(a, b), d = __fsub_rn(a, b);
    a = __fmul_rn(s, kHc);
    b = __fmul_rn(d, kHc);
}
template <int H>
__device__ __forceinline__ void fwht_stage1(float (&v)[32]) {
#pragma unroll
    for (int t = 0; t < 32; ++t)
        if (!(t & H)) bfly(v[t], v[t + H]);
}
// Stages h = H0 .. 16 with packed f32x2 arithmetic: lanes (v[i], v[i + 16]) carry two independent butterflies
// of every stage h < 16 (pairs (t, t + h) and (t + 16, t + 16 + h)), so one FADD2 / FFMA2 does the work of two
// scalar ops; stage 16 pairs the two lanes and stays scalar.  Same operations and order as the reference
// (lower index as minuend, (a + b) * c and (a - b) * c rounded separately: the product is an FFMA2 with an
// opaque -0 addend, which ptxas can neither drop nor fuse with the next add -- see opaque_nz2).
template <int H0>
__device__ __forceinline__ void fwht_from(float (&v)[32]) {
    const float2 c2 = f2(kHc), nz = opaque_nz2();
    float2 p[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) p[i] = make_float2(v[i], v[i + 16]);
#pragma unroll
    for (int h = H0; h < 16; h <<= 1) {
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            if (t & h) continue;
            const float2 a = p[t], b = p[t + h];
            p[t] = fma2(add2(a, b), c2, nz);
            p[t + h] = fma2(sub2(a, b), c2, nz);
        }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        v[i] = p[i].x;
        v[i + 16] = p[i].y;
        bfly(v[i], v[i + 16]);
    }
}
// stages h = 2..16 (stage 1 is done while loading)
__device__ __forceinline__ void fwht_tail(float (&v)[32]) { fwht_from<2>(v); }
__device__ __forceinline__ void fwht_full(float (&v)[32]) { fwht_from<1>(v); }

// ------------------------------------------------------------------------------ absmax
__device__ __forceinline__ float max3_nan(float a, float b, float c) {
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// NaN-propagating max |v| (a NaN or Inf input shows up as a non-finite result)
__device__ __forceinline__ float absmax32(const float (&v)[32]) {
    float m0 = fabsf(v[0]), m1 = fabsf(v[1]);
#pragma unroll
    for (int j = 2; j < 30; j += 4) {
        m0 = max3_nan(m0, fabsf(v[j]), fabsf(v[j + 1]));
        m1 = max3_nan(m1, fabsf(v[j + 2]), fabsf(v[j + 3]));
    }
    return max3_nan(m0, fabsf(v[30]), max3_nan(m1, fabsf(v[31]), 0.0f));
}

// --------------------------------------------------------------------------- e2m1 pack
__device__ __forceinline__ uint32_t e2m1b(float lo, float hi) {  // byte in bits 0..7, rest unspecified
    uint32_t r;
    asm("{\n .reg .b8 t;\n cvt.rn.satfinite.e2m1x2.f32 t, %2, %1;\n cvt.u32.u8 %0, t;\n}" : "=r"(r) : "f"(lo), "f"(hi));
    return r;
}
// 8 values -> 4 E2M1 bytes in one register (element 2k in the low nibble of byte k): ptxas merges the
// four conversions with F2FP.PACK_AB_MERGE_C, no byte packing instructions.
__device__ __forceinline__ uint32_t e2m1x8(float a0, float a1, float a2, float a3, float a4, float a5, float a6,
                                           float a7) {
    uint32_t r;
    asm("{\n .reg .b8 b0, b1, b2, b3;\n .reg .b16 h0, h1;\n"
        " cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n"
        " cvt.rn.satfinite.e2m1x2.f32 b2, %6, %5;\n cvt.rn.satfinite.e2m1x2.f32 b3, %8, %7;\n"
        " mov.b16 h0, {b0, b1};\n mov.b16 h1, {b2, b3};\n mov.b32 %0, {h0, h1};\n}"
        : "=r"(r)
        : "f"(a0), "f"(a1), "f"(a2), "f"(a3), "f"(a4), "f"(a5), "f"(a6), "f"(a7));
    return r;
}
// E2M1 round trip of (a, b) as f16x2 grid values (exact), a in the low half
__device__ __forceinline__ uint32_t e2m1_rt_h2(float a, float b) {
    uint32_t h2;
    asm("{\n .reg .b8 t;\n cvt.rn.satfinite.e2m1x2.f32 t, %2, %1;\n cvt.rn.f16x2.e2m1x2 %0, t;\n}"
        : "=r"(h2)
        : "f"(a), "f"(b));
    return h2;
}
__device__ __forceinline__ uint32_t pack4(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) {
    return __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
}
// -0 (code 8) -> +0 on 8 nibbles: keep the sign only where the magnitude bits are non-zero
__device__ __forceinline__ uint32_t canon8(uint32_t c) {
    const uint32_t u = (c & 0x77777777u) + 0x77777777u;
    return c & (u | 0x77777777u);
}

// RTN codes of v * sc (v * sc exact or rounded as the caller arranged), element 2k in the low nibble.
__device__ __forceinline__ uint4 encode32(const float (&v)[32], float sc) {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        float a[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __fmul_rn(v[8 * q + k], sc);
        w[q] = canon8(e2m1x8(a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7]));
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}
// Same plus the QuEST trust mask: bit j = |v_j * sc| <= 6 (6 - |a| is negative exactly when clipped,
// and a funnel shift collects the sign bits).
__device__ __forceinline__ uint4 encode32_mask(const float (&v)[32], float sc, uint32_t& keep) {
    uint32_t w[4], clip = 0;
#pragma unroll
    for (int q = 3; q >= 0; --q) {
        float a[8];
#pragma unroll
        for (int k = 7; k >= 0; --k) {
            a[k] = __fmul_rn(v[8 * q + k], sc);
            clip = __funnelshift_l(__float_as_uint(__fsub_rn(6.0f, fabsf(a[k]))), clip, 1);
        }
        w[q] = canon8(e2m1x8(a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7]));
    }
    keep = ~clip;
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// ------------------------------------------------------------------------------- QuEST
// q - a for a = fp32, q = the low / high f16 half of h (exact widening inside the subtraction)
__device__ __forceinline__ float fh16_sub_lo(uint32_t h, float a) {
    float d;
    asm("{\n .reg .b16 l, u;\n mov.b32 {l, u}, %1;\n sub.rn.f32.f16 %0, l, %2;\n}" : "=f"(d) : "r"(h), "f"(a));
    return d;
}
__device__ __forceinline__ float fh16_sub_hi(uint32_t h, float a) {
    float d;
    asm("{\n .reg .b16 l, u;\n mov.b32 {l, u}, %1;\n sub.rn.f32.f16 %0, u, %2;\n}" : "=f"(d) : "r"(h), "f"(a));
    return d;
}
// E2M1 byte -> f16x2 grid values (exact), low nibble in the low half
__device__ __forceinline__ uint32_t e2m1x2_to_h2(uint32_t byte) {
    uint32_t h2;
    asm("{\n .reg .b8 t;\n cvt.u8.u32 t, %1;\n cvt.rn.f16x2.e2m1x2 %0, t;\n}" : "=r"(h2) : "r"(byte));
    return h2;
}
// Squared FP4 rounding error of v * sc (the error is sign-symmetric, so signed values round directly):
// per element one FMUL, half an F2FP pack + unpack, one FHADD.F16 (q - a with q widened inside) and one FFMA.
__device__ __forceinline__ float quest_err32(const float (&v)[32], float sc) {
    float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
        const float a = __fmul_rn(v[j], sc), b = __fmul_rn(v[j + 1], sc);
        const uint32_t q = e2m1_rt_h2(a, b);
        const float ta = fh16_sub_lo(q, a), tb = fh16_sub_hi(q, b);
        acc0 = __fmaf_rn(ta, ta, acc0);
        acc1 = __fmaf_rn(tb, tb, acc1);
    }
    return __fadd_rn(acc0, acc1);
}

constexpr float kQTol = 6.103515625e-05f;        // 2^-14 relative near-tie guard
constexpr float kQAtol = 7.52316384526264e-37f;  // 2^-120 absolute guard

// QuEST scale exponent of one group with absmax `amax` (> 0, finite).  Candidates e_hi .. e_lo
// (k = e_hi - e).  E_0 and E_1 always; k >= 2 only while the single-element clipping lower bound
// (amax*sc_k - 6)^2 / sc_k^2, monotone in k, does not clear the best error by the guard -- so a
// skipped candidate can never be the reference's choice.  Near-ties go to the exact f64 search.
__device__ __forceinline__ int quest_search32(const float (&v)[32], float amax, int* fallback_counter) {
    const int e_hi = ceil_scale_exp(amax), e_lo = quest_low_exp(amax);
    if (e_hi <= e_lo) return e_hi;
    const float sc0 = exp2i(127 - e_hi);
    const float a0 = __fmul_rn(amax, sc0);
    float best = __int_as_float(0x7f800000), second = best;
    int bk = 0;
    // one inlined copy of the error loop (instruction-cache footprint): k = 0, 1 always, then pruned
    for (int k = 0; k <= e_hi - e_lo; ++k) {
        const float sk = exp2i(k), ik = exp2i(-2 * k);
        if (k >= 2) {
            const float d = __fsub_rn(__fmul_rn(a0, sk), 6.0f);
            const float lb = __fmul_rn(__fmul_rn(d, d), ik);
            if (__fmul_rn(lb, 0.99999905f) > __fadd_rn(__fmul_rn(best, 1.0f + kQTol), kQAtol)) break;
        }
        const float ek = __fmul_rn(quest_err32(v, __fmul_rn(sc0, sk)), ik);
        if (ek < best) {
            second = best;
            best = ek;
            bk = k;
        } else if (ek < second) {
            second = ek;
        }
    }
    if (!(__fsub_rn(second, best) > __fadd_rn(__fmul_rn(second, kQTol), kQAtol))) {
        if (fallback_counter) atomicAdd(fallback_counter, 1);
        float xs[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) xs[j] = v[j];
        return quest_exact_cold(xs, e_hi, e_lo);
    }
    return e_hi - bk;
}

// ---------------------------------------------------------------------- RTN scale rule
// Quantization scale of a group whose values are y (FWHT output) and whose reference input is
// fl(y * prescale): E8M0 e from fl(amax * prescale) (rounding is monotone, so that IS the absmax of the
// pre-scaled values) and the multiplier prescale * 2^(127-e).  fl(y * (p * 2^k)) == fl(fl(y * p) * 2^k)
// whenever neither product is subnormal; values whose scaled magnitude could reach a rounding
// threshold (>= 0.25) are normal once e >= 4.  Below that the caller pre-scales explicitly.
__device__ __forceinline__ bool rtn_scale(float amax, float prescale, int& e, float& sc) {
    const float amp = prescale == 1.0f ? amax : __fmul_rn(amax, prescale);
    e = ceil_scale_exp(amp);
    if (prescale == 1.0f || e >= 4) {
        sc = __fmul_rn(prescale, exp2i(127 - e));
        return true;
    }
    sc = exp2i(127 - e);
    return false;
}

// ------------------------------------------------------------------------ group quantizer
// Quantize one transformed group v (pre-scale NOT yet applied).  Returns the E8M0 byte.
// SR_REF: exact SR by the reference form inline (sr_code_ref_body) instead of sr_code -- same codes, faster in the
// register-heavy fused forward kernels.
template <int ROUND, bool SR_REF = false>
__device__ __forceinline__ int quant_group(float (&v)[32], const QuantCfg& cf, uint64_t sr_idx, int* err,
                                           int* fallbacks, uint4& codes, uint32_t& mask) {
    const float am = absmax32(v);
    if (!(am <= 3.4028234663852886e38f) && err) atomicOr(err, 1);
    mask = 0xFFFFFFFFu;
    int e;
    if (ROUND == kQuest) {
        if (cf.prescale != 1.0f) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __fmul_rn(v[j], cf.prescale);
        }
        const float amp = cf.prescale != 1.0f ? __fmul_rn(am, cf.prescale) : am;
        if (amp > 0.0f && amp <= 3.4028234663852886e38f) {
            e = quest_search32(v, amp, fallbacks);
            codes = encode32_mask(v, exp2i(127 - e), mask);
        } else {
            e = 0;  // zero group: e = 0, codes 0, all kept (_native.pyx:228-233)
            codes = make_uint4(0, 0, 0, 0);
        }
    } else if (ROUND == kRtn) {
        float sc;
        if (!rtn_scale(am, cf.prescale, e, sc)) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __fmul_rn(v[j], cf.prescale);
        }
        codes = encode32(v, sc);
    } else {
        if (cf.prescale != 1.0f) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __fmul_rn(v[j], cf.prescale);
        }
        e = ceil_scale_exp(cf.prescale != 1.0f ? __fmul_rn(am, cf.prescale) : am);
        const float sc_f = exp2i(127 - e);
        const double sc_d = (double)sc_f;
        uint32_t w[4];
        if (cf.sr_fast) {   // QT_ROUND_SR_FAST: statistically unbiased, not the reference's stream
            const uint32_t base = srf_base((uint32_t)cf.sr_base, (uint32_t)(cf.sr_base >> 32), sr_idx);
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const int j = qq * 8;
                w[qq] = srf_quad(__fmul_rn(v[j], sc_f), __fmul_rn(v[j + 1], sc_f), __fmul_rn(v[j + 2], sc_f),
                                 __fmul_rn(v[j + 3], sc_f), srf_rbits(base, 2 * qq)) |
                        srf_quad(__fmul_rn(v[j + 4], sc_f), __fmul_rn(v[j + 5], sc_f), __fmul_rn(v[j + 6], sc_f),
                                 __fmul_rn(v[j + 7], sc_f), srf_rbits(base, 2 * qq + 1)) << 16;
            }
        } else {
            const uint64_t z0 = cf.sr_base + (sr_idx + 1) * kGolden;   // splitmix64 counter of element 0
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                uint32_t acc = 0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int j = qq * 8 + k;
                    const uint64_t z = z0 + (uint64_t)j * kGolden;
                    acc |= (SR_REF ? sr_code_ref_body(v[j], sc_f, sc_d, z) : sr_code(v[j], sc_f, sc_d, z)) << (4 * k);
                }
                w[qq] = acc;
            }
        }
        codes = make_uint4(w[0], w[1], w[2], w[3]);
    }
    return e;
}

}  // namespace qt
