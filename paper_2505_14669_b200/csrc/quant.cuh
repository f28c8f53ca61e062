// quant.cuh -- per-group MXFP4 quantizers on one 32-element group held in registers.
//
// Bit-exact restatements of the reference quantizers (mx4train/_backend/_native.pyx):
//   QUEST  quantize_quest   _native.pyx:171-245  (pruned fp32 search + exact f64 fallback)
//   RTN    quantize_rtn     _native.pyx:104-131
//   SR     quantize_sr      _native.pyx:134-168  (same splitmix64 stream, f64 p)
//
// Register layout of a group ("Grp"): p[i] = (v[i], v[i + 16]) as packed f32x2, i = 0..15.
// Butterfly stages h = 1..8 of the FWHT then pair lanes with identical op sequences, so they run
// as packed add/sub/mul.rn.f32x2 (half the FMA-pipe issue slots); stage 16 is scalar.
#pragma once
#include "common.cuh"

namespace qt {

enum Rounding : int { kQuest = 0, kRtn = 1, kSr = 2 };

struct Grp {
    float2 p[16];
    __device__ __forceinline__ float& v(int j) { return j < 16 ? p[j].x : p[j - 16].y; }
    __device__ __forceinline__ float v(int j) const { return j < 16 ? p[j].x : p[j - 16].y; }
};

struct GroupOut {
    uint4 codes;    // 32 nibbles, element 2k in the low nibble of byte k
    uint32_t sf;    // E8M0 exponent
    uint32_t mask;  // bit j: |x_j / s| <= 6
};

// ------------------------------------------------------------------ packed f32x2 helpers
__device__ __forceinline__ uint64_t f2u(float2 a) { return *reinterpret_cast<uint64_t*>(&a); }
__device__ __forceinline__ float2 u2f(uint64_t a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(r);
}
__device__ __forceinline__ float max_nan(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

// ptxas contracts packed mul.rn.f32x2 -> add.rn.f32x2 into FFMA2 even with --fmad=false, which
// would skip the reference's intermediate rounding.  Multiplies that feed an add are therefore
// issued as fma(a, c, z) with z = -0.0 read from memory: the result is bit-identical to a*c
// (x + (-0) == x, including signed zeros) and ptxas cannot fold z away or fuse the following add.
__device__ float g_opaque_neg_zero = -0.0f;

__device__ __forceinline__ float2 opaque_nz2() {
    const float z = *const_cast<volatile float*>(&g_opaque_neg_zero);
    return make_float2(z, z);
}

// Reference FWHT-32 (_native.pyx:366-378) on the packed layout: every op rounded separately.
__device__ __forceinline__ void fwht32(Grp& g) {
    const float c = 0.70710678118654752440f;  // 0x3F3504F3 == (float)(1.0 / sqrt(2.0))
    const float2 c2 = make_float2(c, c);
    const float2 nz = opaque_nz2();
#pragma unroll
    for (int h = 1; h < 16; h *= 2) {
#pragma unroll
        for (int s = 0; s < 16; s += 2 * h) {
#pragma unroll
            for (int t = s; t < s + h; ++t) {
                float2 a = g.p[t], b = g.p[t + h];
                g.p[t] = fma2(add2(a, b), c2, nz);
                g.p[t + h] = fma2(sub2(a, b), c2, nz);
            }
        }
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) {
        float a = g.p[t].x, b = g.p[t].y;
        g.p[t].x = __fmul_rn(__fadd_rn(a, b), c);
        g.p[t].y = __fmul_rn(__fsub_rn(a, b), c);
    }
}

__device__ __forceinline__ void flip_signs(Grp& g, uint32_t s) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        g.p[i].x = __uint_as_float(__float_as_uint(g.p[i].x) ^ (((s >> i) & 1u) << 31));
        g.p[i].y = __uint_as_float(__float_as_uint(g.p[i].y) ^ (((s >> (i + 16)) & 1u) << 31));
    }
}

__device__ __forceinline__ void scale_grp(Grp& g, float f) {
    const float2 f2 = make_float2(f, f);
#pragma unroll
    for (int i = 0; i < 16; ++i) g.p[i] = mul2(g.p[i], f2);
}

// grid_index ladder (_native.pyx:46-63) on an exact double magnitude -> grid value.
__device__ __forceinline__ double grid_round_d(double a) {
    int idx = (a > 0.25) + (a >= 0.75) + (a > 1.25) + (a >= 1.75) + (a > 2.5) + (a >= 3.5) + (a > 5.0);
    return idx <= 4 ? 0.5 * idx : (idx == 5 ? 3.0 : (idx == 6 ? 4.0 : 6.0));
}

// Exact reference scale search (_native.pyx:171-203), cold path for near-ties of the fast search:
// ascending-j f64 accumulation, strict '<' (ties keep the larger scale).  vbuf[j] * 2^k of the
// reference equals |x_j| * 2^(127 - e) exactly, so it is recomputed per candidate.
__device__ __noinline__ int quest_exact_cold(const float* xs, int e_hi, int e_lo) {
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

// Squared FP4 rounding error of the group at scale multiplier `sc` (fp32; |x| * sc exact).
__device__ __forceinline__ float quest_err(const Grp& g, float sc) {
    float2 acc0 = make_float2(0.f, 0.f), acc1 = acc0;
    const float2 sc2 = make_float2(sc, sc);
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
        // elements (i, i+1) and (i+16, i+17)
        float2 a = mul2(make_float2(fabsf(g.p[i].x), fabsf(g.p[i + 1].x)), sc2);
        float2 b = mul2(make_float2(fabsf(g.p[i].y), fabsf(g.p[i + 1].y)), sc2);
        float2 qa = e2m1x2_to_f32(e2m1x2(a.x, a.y));
        float2 qb = e2m1x2_to_f32(e2m1x2(b.x, b.y));
        float2 ta = sub2(a, qa), tb = sub2(b, qb);
        acc0 = fma2(ta, ta, acc0);
        acc1 = fma2(tb, tb, acc1);
    }
    return (acc0.x + acc0.y) + (acc1.x + acc1.y);
}

// Clipping-only lower bound of the candidate with clip level c (u-domain): sum max(u - c, 0)^2.
__device__ __forceinline__ float quest_clip_lb(const Grp& g, float sc0, float c) {
    float2 acc = make_float2(0.f, 0.f);
    const float2 sc2 = make_float2(sc0, sc0), nc2 = make_float2(-c, -c);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        float2 d = fma2(make_float2(fabsf(g.p[i].x), fabsf(g.p[i].y)), sc2, nc2);
        d.x = fmaxf(d.x, 0.f);
        d.y = fmaxf(d.y, 0.f);
        acc = fma2(d, d, acc);
    }
    return acc.x + acc.y;
}

// QuEST scale search.  Candidates e_hi, e_hi-1, ..., e_lo (k = e_hi - e).  E_0 and E_1 are always
// evaluated; a candidate k >= 2 is skipped once its clipping-only lower bound LB_k (monotone in k)
// exceeds the best error with a 2^-14 guard, which the exact search can never contradict.  Groups
// whose best and runner-up errors lie within the guard go to the exact f64 search.
__device__ __forceinline__ int quest_search(const Grp& g, float amax, int* fallback_counter) {
    const int e_hi = ceil_scale_exp(amax);
    const int e_lo = quest_low_exp(amax);
    const int ncand = e_hi - e_lo + 1;
    if (ncand <= 1) return e_hi;
    const float sc0 = exp2i(127 - e_hi);
    const float tol = 6.103515625e-05f, atol = 7.52316384526264e-37f;
    float best = quest_err(g, sc0), second;
    int best_k = 0;
    {
        float e1 = quest_err(g, sc0 * 2.0f) * 0.25f;
        if (e1 < best) {
            second = best;
            best = e1;
            best_k = 1;
        } else {
            second = e1;
        }
    }
    int k = 2;
    bool more = ncand > 2 && !(quest_clip_lb(g, sc0, 1.5f) > best * (1.0f + tol) + atol);
    while (more) {
        {
            float ek = quest_err(g, sc0 * (float)(1 << k)) * exp2i(-2 * k);
            if (ek < best) {
                second = best;
                best = ek;
                best_k = k;
            } else if (ek < second) {
                second = ek;
            }
            ++k;
            more = k < ncand && !(quest_clip_lb(g, sc0, 6.0f * exp2i(-k)) > best * (1.0f + tol) + atol);
        }
    }
    if (!(second - best > second * tol + atol)) {
        if (fallback_counter) atomicAdd(fallback_counter, 1);
        float xs[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) xs[j] = g.v(j);
        return quest_exact_cold(xs, e_hi, e_lo);
    }
    return e_hi - best_k;
}

// Pack the 32 E2M1 codes of x * 2^(127 - e) (RNE, satfinite, -0 -> +0).
__device__ __forceinline__ uint4 encode_grp(const Grp& g, int e) {
    const float sc = exp2i(127 - e);
    const float2 sc2 = make_float2(sc, sc);
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t acc = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int j = q * 8 + b * 2;  // elements j, j+1 (same half of the packed layout)
            float2 s = j < 16 ? mul2(make_float2(g.p[j].x, g.p[j + 1].x), sc2)
                              : mul2(make_float2(g.p[j - 16].y, g.p[j - 15].y), sc2);
            acc |= e2m1x2(s.x, s.y) << (8 * b);
        }
        w[q] = canon_nz(acc);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// Stochastic rounding of one element (_native.pyx:156-167).
__device__ __forceinline__ uint32_t sr_code(float x, float sc_f, double sc_d, uint64_t base, uint64_t index) {
    float a = fabsf(x) * sc_f;
    int b;
    double lo, hi;
    uint32_t c_lo, c_hi;
    if (x > 0.0f) {
        b = (a > 0.5f) + (a > 1.0f) + (a > 1.5f) + (a > 2.0f) + (a > 3.0f) + (a > 4.0f);
        lo = b <= 4 ? 0.5 * b : (double)(b - 2);
        hi = b + 1 <= 4 ? 0.5 * (b + 1) : (b + 1 == 7 ? 6.0 : (double)(b - 1));
        c_lo = (uint32_t)b;
        c_hi = (uint32_t)(b + 1);
    } else {
        b = (a >= 0.5f) + (a >= 1.0f) + (a >= 1.5f) + (a >= 2.0f) + (a >= 3.0f) + (a >= 4.0f);
        double plo = b <= 4 ? 0.5 * b : (double)(b - 2);
        double phi = b + 1 <= 4 ? 0.5 * (b + 1) : (b + 1 == 7 ? 6.0 : (double)(b - 1));
        lo = -phi;
        hi = -plo;
        c_lo = 8u | (uint32_t)(b + 1);
        c_hi = b == 0 ? 0u : (8u | (uint32_t)b);
    }
    double v = (double)x * sc_d;
    double p = __dmul_rn(__dsub_rn(v, lo), 1.0 / (hi - lo));  // span is a power of two: exact
    uint64_t h = mix64(base + (index + 1) * kGolden);
    double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
    return u < p ? c_hi : c_lo;
}

__device__ __forceinline__ uint4 encode_grp_sr(const Grp& g, int e, uint64_t base, uint64_t idx0) {
    const float sc_f = exp2i(127 - e);
    const double sc_d = (double)sc_f;
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t acc = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int j = q * 8 + b;
            acc |= sr_code(g.v(j), sc_f, sc_d, base, idx0 + (uint64_t)j) << (4 * b);
        }
        w[q] = acc;
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ float grp_absmax(const Grp& g) {
    float m0 = 0.f, m1 = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        m0 = max_nan(m0, fabsf(g.p[i].x));
        m1 = max_nan(m1, fabsf(g.p[i].y));
    }
    return max_nan(m0, m1);
}

// Quantize one group already in its final (transformed, pre-scaled) fp32 form.
template <int ROUND>
__device__ __forceinline__ GroupOut quantize_grp(const Grp& g, uint64_t sr_base, uint64_t idx0, int* err_flag,
                                                 int* fallback_counter) {
    GroupOut o;
    const float amax = grp_absmax(g);  // NaN-propagating
    if (!(amax <= 3.4028234663852886e38f)) {
        if (err_flag) atomicOr(err_flag, 1);
    }
    if (ROUND == kQuest) {
        if (!(amax > 0.0f)) {  // zero group: e = 0, codes 0, all kept (_native.pyx:228-233)
            o.codes = make_uint4(0, 0, 0, 0);
            o.sf = 0;
            o.mask = 0xFFFFFFFFu;
            return o;
        }
        const int e = quest_search(g, amax, fallback_counter);
        o.codes = encode_grp(g, e);
        o.sf = (uint32_t)e;
        const float lim = 6.0f * exp2i(e - 127);  // |x| <= 6 s  <=>  |x / s| <= 6 (exact)
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            lo |= (fabsf(g.p[i].x) <= lim ? 1u : 0u) << i;
            hi |= (fabsf(g.p[i].y) <= lim ? 1u : 0u) << i;
        }
        o.mask = lo | (hi << 16);
        return o;
    }
    const int e = ceil_scale_exp(amax);
    o.sf = (uint32_t)e;
    o.mask = 0xFFFFFFFFu;
    if (ROUND == kRtn)
        o.codes = encode_grp(g, e);
    else
        o.codes = encode_grp_sr(g, e, sr_base, idx0);
    return o;
}

}  // namespace qt
