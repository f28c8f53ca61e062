// quant.cuh -- pieces of the CUDA-core quantizers shared by quant.cu, qgroup.cuh and gemm.cu:
//   * the two-group ("Pair") FWHT-32 used by the transform-only seam kernel and the GEMM epilogue
//     (reference fwht, _native.pyx:353-379);
//   * the exact f64 QuEST scale search, the cold path of qgroup.cuh's pruned fp32 search
//     (_native.pyx:171-203);
//   * one stochastic-rounding decision (_native.pyx:134-168).
#pragma once
#include "common.cuh"

namespace qt {

enum Rounding : int { kQuest = 0, kRtn = 1, kSr = 2 };

struct Pair {
    float2 p[32];
};

// ------------------------------------------------------------------ packed f32x2 helpers
// CUDA 12.9 float2 builtins (sm_100): the compiler allocates the register pairs itself.
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// ptxas contracts packed mul.rn.f32x2 -> add.rn.f32x2 into FFMA2 even with --fmad=false, which
// would skip the reference's intermediate rounding.  Multiplies that feed an add are therefore
// issued as fma(a, c, z) with z = -0.0 read from memory: the result is bit-identical to a*c
// (x + (-0) == x, including signed zeros) and ptxas cannot fold z away or fuse the following add.
static __device__ float g_opaque_neg_zero = -0.0f;
__device__ __forceinline__ float2 opaque_nz2() {
    const float z = *const_cast<volatile float*>(&g_opaque_neg_zero);
    return make_float2(z, z);
}

// One butterfly stage of span H over both groups (pairs (t, t + H) with bit H of t clear).
template <int H>
__device__ __forceinline__ void fwht_stage(Pair& g, float2 c2, float2 nz) {
#pragma unroll
    for (int t = 0; t < 32; ++t) {
        if (t & H) continue;
        const float2 a = g.p[t], b = g.p[t + H];
        g.p[t] = fma2(add2(a, b), c2, nz);
        g.p[t + H] = fma2(sub2(a, b), c2, nz);
    }
}

// Reference FWHT-32 (_native.pyx:366-378) on both groups: stages h = 1, 2, 4, 8, 16, lower index
// as minuend, (a + b) * c and (a - b) * c each rounded separately, c = fp32(1/sqrt(2)).
__device__ __forceinline__ void fwht_pair(Pair& g, float2 nz) {
    const float2 c2 = f2(0.70710678118654752440f);  // 0x3F3504F3 == (float)(1.0 / sqrt(2.0))
    fwht_stage<1>(g, c2, nz);
    fwht_stage<2>(g, c2, nz);
    fwht_stage<4>(g, c2, nz);
    fwht_stage<8>(g, c2, nz);
    fwht_stage<16>(g, c2, nz);
}

// Randomized-Hadamard sign flips: bit i of sA / sB flips element i of group A / B.
__device__ __forceinline__ void flip_pair(Pair& g, uint32_t sA, uint32_t sB) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        // funnel shift (SHF, ALU pipe) + LOP3: bit i of s -> bit 31
        g.p[i].x = __uint_as_float(__float_as_uint(g.p[i].x) ^ (__funnelshift_l(0u, sA, 31 - i) & 0x80000000u));
        g.p[i].y = __uint_as_float(__float_as_uint(g.p[i].y) ^ (__funnelshift_l(0u, sB, 31 - i) & 0x80000000u));
    }
}

__device__ __forceinline__ void scale_pair(Pair& g, float f) {
#pragma unroll
    for (int i = 0; i < 32; ++i) g.p[i] = mul2(g.p[i], f2(f));
}

// grid_index ladder (_native.pyx:46-63) on an exact double magnitude -> grid value.
__device__ __forceinline__ double grid_round_d(double a) {
    int idx = (a > 0.25) + (a >= 0.75) + (a > 1.25) + (a >= 1.75) + (a > 2.5) + (a >= 3.5) + (a > 5.0);
    return idx <= 4 ? 0.5 * idx : (idx == 5 ? 3.0 : (idx == 6 ? 4.0 : 6.0));
}

// Exact reference scale search (_native.pyx:171-203), cold path for near-ties of the fast search:
// ascending-j f64 accumulation, strict '<' (ties keep the larger scale).  vbuf[j] * 2^k of the
// reference equals |x_j| * 2^(127 - e) exactly, so it is recomputed per candidate.
static __device__ __noinline__ int quest_exact_cold(const float* xs, int e_hi, int e_lo) {
    int best_e = e_hi;
    double best_err = -1.0;
    for (int e = e_hi; e >= e_lo; --e) {
        const double sc = ldexp(1.0, 127 - e);
        double acc = 0.0;
        for (int j = 0; j < 32; ++j) {
            double a = fabs((double)xs[j] * sc);
            double t = a - grid_round_d(a);
            acc = __dadd_rn(acc, __dmul_rn(t, t));
        }
        double err = ldexp(acc, 2 * (e - 127));
        if (best_err < 0.0 || err < best_err) {
            best_err = err;
            best_e = e;
        }
    }
    return best_e;
}

// Stochastic rounding of one element (_native.pyx:156-167): v = x / s in f64, neighbours on the
// signed grid, p = (v - lo) / (hi - lo) in f64, u = splitmix64 uniform at stream position index, hi when u < p.
// z = base + (index + 1) * kGolden (the pre-mix counter; callers step it by kGolden per element).
// Reference form.  sr_code calls it out of line for zero, tiny or non-finite scaled values only (an inlined copy,
// or no call at all, measured slower: the rare path costs the hot loop registers and scheduling); the fused
// forward kernels use it inline for their X_t / W_t (measured faster there than sr_code).
__device__ __forceinline__ uint32_t sr_code_ref_body(float x, float sc_f, double sc_d, uint64_t z) {
    const float a = fabsf(x) * sc_f;
    int b;
    double lo;
    uint32_t c_lo, c_hi;
    if (x > 0.0f) {
        b = (a > 0.5f) + (a > 1.0f) + (a > 1.5f) + (a > 2.0f) + (a > 3.0f) + (a > 4.0f);
        lo = b <= 4 ? 0.5 * b : (double)(b - 2);                              // grid(b)
        c_lo = (uint32_t)b;
        c_hi = (uint32_t)(b + 1);
    } else {
        b = (a >= 0.5f) + (a >= 1.0f) + (a >= 1.5f) + (a >= 2.0f) + (a >= 3.0f) + (a >= 4.0f);
        lo = -(b + 1 <= 4 ? 0.5 * (b + 1) : (b + 1 == 7 ? 6.0 : (double)(b - 1)));   // -grid(b + 1)
        c_lo = 8u | (uint32_t)(b + 1);
        c_hi = b == 0 ? 0u : (8u | (uint32_t)b);
    }
    const double v = (double)x * sc_d;
    // the span hi - lo is 0.5 (b < 4), 1 (b = 4, 5) or 2 (b = 6): dividing by it equals multiplying by the
    // exact reciprocal (both are the correctly rounded value of the same real), with no double division
    const double inv_span = b < 4 ? 2.0 : (b < 6 ? 1.0 : 0.5);
    const double p = __dmul_rn(__dsub_rn(v, lo), inv_span);
    const double u = (double)(mix64(z) >> 11) * (1.0 / 9007199254740992.0);
    return u < p ? c_hi : c_lo;
}

static __device__ __noinline__ uint32_t sr_code_ref(float x, float sc_f, double sc_d, uint64_t z) {
    return sr_code_ref_body(x, sc_f, sc_d, z);
}

// The same decision, branch-free and in magnitudes.  a = |x| s is exact in fp32 (a normal power-of-two
// multiple of x); with bl = #{grid points 0.5 .. 4 <= a} and on = (a is one of them), the reference's interval
// index is b = bl - on for x > 0 (grid(b) < a <= grid(b+1)) and b = bl for x <= 0 (grid(b) <= a < grid(b+1)),
// read off a's exponent and top mantissa bit.  q = (a - grid(b)) / span(b) is exact in fp32 (grid(b) = 0, or
// grid(b) <= a <= 2 grid(b): Sterbenz; the span is a power of two), and the reference's p is q (x > 0) or
// 1 - q (x <= 0), both exact in f64: so u < p is the same comparison.  x > 0: magnitude b + [u < q];
// x <= 0: magnitude b + [u >= 1 - q], negative sign unless the magnitude is 0.
// 2.2x fewer instructions than the reference form (a divergent sign branch, f64 grid arithmetic).
__device__ __forceinline__ uint32_t sr_code(float x, float sc_f, double sc_d, uint64_t z) {
    const float a = fabsf(x) * sc_f;
    if (!(a >= 1.0e-30f && a <= 6.0f)) return sr_code_ref(x, sc_f, sc_d, z);   // zero, tiny, non-finite
    const uint32_t t = __float_as_uint(a);
    const int idx = a >= 1.0f ? 2 + 2 * ((int)(t >> 23) - 127) + (int)((t >> 22) & 1u) : (a >= 0.5f ? 1 : 0);
    const int bl = idx < 6 ? idx : 6;
    const bool on = (a >= 1.0f && a <= 4.0f && (t & 0x3FFFFFu) == 0) || a == 0.5f;
    const bool pos = x > 0.0f;
    const int b = pos && on ? bl - 1 : bl;
    const uint32_t gbits = b >= 2 ? ((uint32_t)(127 + ((b - 2) >> 1)) << 23) | ((uint32_t)((b - 2) & 1) << 22)
                                  : (b == 1 ? 0x3F000000u : 0u);
    const float isp = b < 4 ? 2.0f : (b < 6 ? 1.0f : 0.5f);
    const float q = __fmul_rn(__fsub_rn(a, __uint_as_float(gbits)), isp);
    const double qd = (double)q;
    const double u = (double)(mix64(z) >> 11) * (1.0 / 9007199254740992.0);
    const bool up = pos ? u < qd : !(u < 1.0 - qd);
    const uint32_t mag = (uint32_t)b + (up ? 1u : 0u);
    return mag == 0 ? 0u : (mag | (pos ? 0u : 8u));
}

// Fast stochastic rounding (B200 extension, QT_ROUND_SR_FAST; SURVEY.md section 7.3 "fast mode"): the same two
// grid neighbours as sr_code, picked by the hardware's stochastic-rounding conversion
// cvt.rs.satfinite.e2m1x4.f32 (F2FP.E2M1.RS: four values, 32 random bits) -- the draws are NOT the reference's.
// Measured exhaustively over all 2^32 random words (tools/ubench/cvt_rs_exh.cu): the upper neighbour is taken with
// probability floor(p * 2^16) / 2^16, p = (|v| - lo) / (hi - lo), in every grid interval -- unbiased up to a
// shrink toward zero below 2^-16 of a grid step; the four decisions of one conversion are uncorrelated to
// |r| <= 3e-4 (tools/ubench/cvt_rs_corr.cu).
// Random words: quad q (elements 4q .. 4q+3) of the group whose first stream position is P takes
// lowbias32(srf_base(P) + q * C), srf_base(P) = lo32(P) * C + k0 + (hi32(P) * C' ^ k1) (groups of every operand lie
// along the stream's contiguous axis, so the words are a function of stream positions alone).
constexpr uint32_t kSrfC = 0x9E3779B1u;
__device__ __forceinline__ uint32_t srf_base(uint32_t k0, uint32_t k1, uint64_t p) {
    return (uint32_t)p * kSrfC + k0 + ((uint32_t)(p >> 32) * 0x85EBCA77u ^ k1);
}
__device__ __forceinline__ uint32_t srf_rbits(uint32_t base, uint32_t q) {
    uint32_t h = base + q * kSrfC;   // lowbias32
    h ^= h >> 16;
    h *= 0x7FEB352Du;
    h ^= h >> 15;
    h *= 0x846CA68Bu;
    h ^= h >> 16;
    return h;
}
// E2M1 codes of four scaled values (|v| <= 6), element k in nibble k; -0 -> +0 (_native.pyx:127-130)
__device__ __forceinline__ uint32_t srf_quad(float e0, float e1, float e2, float e3, uint32_t rbits) {
    uint16_t o;
    asm("cvt.rs.satfinite.e2m1x4.f32 %0, {%1, %2, %3, %4}, %5;" : "=h"(o) : "f"(e3), "f"(e2), "f"(e1), "f"(e0), "r"(rbits));
    const uint32_t w = o, mag = w & 0x7777u;
    return mag | (w & ((mag + 0x7777u) & 0x8888u));
}
}  // namespace qt
