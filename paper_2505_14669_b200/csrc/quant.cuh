// quant.cuh -- MXFP4 group quantizers on TWO 32-element groups held in registers.
//
// Bit-exact restatements of the reference quantizers (mx4train/_backend/_native.pyx):
//   QUEST  quantize_quest   _native.pyx:171-245  (pruned fp32 search + exact f64 fallback)
//   RTN    quantize_rtn     _native.pyx:104-131
//   SR     quantize_sr      _native.pyx:134-168  (same splitmix64 stream, f64 p)
//
// Register layout ("Pair"): p[i] = (A[i], B[i]) as packed f32x2 for two independent groups A, B.
// Every step of the pipeline applies the same op sequence to A and B, so the FWHT, the scale
// multiplies and the QuEST error sums all run as packed add/sub/mul/fma.rn.f32x2 with no register
// re-pairing: one issue slot per two elements on the FMA pipe.
#pragma once
#include "common.cuh"

namespace qt {

enum Rounding : int { kQuest = 0, kRtn = 1, kSr = 2 };

struct Pair {
    float2 p[32];
};

struct PairOut {
    uint4 codes[2];   // 32 nibbles per group, element 2k in the low nibble of byte k
    uint32_t sf[2];   // E8M0 exponents
    uint32_t mask[2]; // bit j: |x_j / s| <= 6
};

// ------------------------------------------------------------------ packed f32x2 helpers
// CUDA 12.9 float2 builtins (sm_100): the compiler allocates the register pairs itself.
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float max_nan(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
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

// E2M1 round trip of (a, b): the two grid values as fp32 (exact).
__device__ __forceinline__ float2 e2m1_round2(float2 v) { return e2m1x2_to_f32(e2m1x2(v.x, v.y)); }

// Squared FP4 rounding errors of both groups at per-group scale multipliers sc = (scA, scB).
// x * sc is exact and the rounding error is sign-symmetric, so signed values are rounded directly.
__device__ __forceinline__ float2 quest_err(const Pair& g, float2 sc) {
    float2 acc0 = f2(0.f), acc1 = acc0;
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
        float2 a = mul2(g.p[i], sc), b = mul2(g.p[i + 1], sc);
        float2 ta = sub2(a, e2m1_round2(a)), tb = sub2(b, e2m1_round2(b));
        acc0 = fma2(ta, ta, acc0);
        acc1 = fma2(tb, tb, acc1);
    }
    return add2(acc0, acc1);
}

// Clipping-only lower bound sum max(|x| sc0 - c, 0)^2 for both groups (nc = -c).
__device__ __forceinline__ float2 quest_clip_lb(const Pair& g, float2 sc0, float2 nc) {
    float2 acc = f2(0.f);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        float2 d = fma2(make_float2(fabsf(g.p[i].x), fabsf(g.p[i].y)), sc0, nc);
        d.x = fmaxf(d.x, 0.f);
        d.y = fmaxf(d.y, 0.f);
        acc = fma2(d, d, acc);
    }
    return acc;
}

struct QuestState {
    int e_hi, e_lo, best_k, k;
    float best, second;
    bool more;
};

__device__ __forceinline__ void quest_update(QuestState& s, float ek, int k) {
    if (ek < s.best) {
        s.second = s.best;
        s.best = ek;
        s.best_k = k;
    } else if (ek < s.second) {
        s.second = ek;
    }
}

constexpr float kQuestTol = 6.103515625e-05f;        // 2^-14 relative guard
constexpr float kQuestAtol = 7.52316384526264e-37f;  // 2^-120 absolute guard

// QuEST scale search for both groups.  Candidates e_hi, e_hi-1, ..., e_lo (k = e_hi - e).  E_0
// and E_1 are always evaluated; candidate k >= 2 is evaluated only while its clipping-only lower
// bound (monotone in k) does not exceed the best error by the guard, so a skipped candidate can
// never be the reference's choice.  Near-ties go to the exact f64 search.
__device__ __forceinline__ void quest_search_pair(const Pair& g, float amaxA, float amaxB, int* e_out,
                                                  int* fallback_counter) {
    QuestState st[2];
    const float amax[2] = {amaxA, amaxB};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        st[h].e_hi = ceil_scale_exp(amax[h]);
        st[h].e_lo = quest_low_exp(amax[h]);
        st[h].best_k = 0;
        st[h].k = 2;
    }
    const float2 sc0 = make_float2(exp2i(127 - st[0].e_hi), exp2i(127 - st[1].e_hi));
    const float2 e0 = quest_err(g, sc0);
    const float2 e1 = mul2(quest_err(g, mul2(sc0, f2(2.0f))), f2(0.25f));
    const float e0v[2] = {e0.x, e0.y}, e1v[2] = {e1.x, e1.y};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        st[h].best = e0v[h];
        st[h].second = __int_as_float(0x7f800000);
        if (st[h].e_hi - st[h].e_lo >= 1) quest_update(st[h], e1v[h], 1);
    }
    {
        const float2 lb = quest_clip_lb(g, sc0, f2(-1.5f));
        const float lbv[2] = {lb.x, lb.y};
#pragma unroll
        for (int h = 0; h < 2; ++h)
            st[h].more = st[h].e_hi - st[h].e_lo >= 2 && !(lbv[h] > st[h].best * (1.0f + kQuestTol) + kQuestAtol);
    }
    while (st[0].more || st[1].more) {
        const int k = st[0].more ? st[0].k : st[1].k;
        // evaluate candidate k for both lanes (a lane that is done just ignores the result)
        const float2 sck = mul2(sc0, f2((float)(1 << k)));
        const float2 ek = mul2(quest_err(g, sck), f2(exp2i(-2 * k)));
        const float2 lb = quest_clip_lb(g, sc0, f2(-6.0f * exp2i(-(k + 1))));
        const float ekv[2] = {ek.x, ek.y}, lbv[2] = {lb.x, lb.y};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (st[h].more && st[h].k == k) {
                quest_update(st[h], ekv[h], k);
                st[h].k = k + 1;
                st[h].more = st[h].k <= st[h].e_hi - st[h].e_lo &&
                             !(lbv[h] > st[h].best * (1.0f + kQuestTol) + kQuestAtol);
            }
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        int e = st[h].e_hi - st[h].best_k;
        if (st[h].e_hi > st[h].e_lo && !(st[h].second - st[h].best > st[h].second * kQuestTol + kQuestAtol)) {
            if (fallback_counter) atomicAdd(fallback_counter, 1);
            float xs[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) xs[j] = h == 0 ? g.p[j].x : g.p[j].y;
            e = quest_exact_cold(xs, st[h].e_hi, st[h].e_lo);
        }
        e_out[h] = e;
    }
}

// Pack the E2M1 codes of both groups at exponents (eA, eB) (RNE, satfinite, -0 -> +0).
__device__ __forceinline__ void encode_pair(const Pair& g, int eA, int eB, uint4* out) {
    const float2 sc = make_float2(exp2i(127 - eA), exp2i(127 - eB));
    uint32_t wa[4], wb[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t accA = 0, accB = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int j = q * 8 + b * 2;
            const float2 lo = mul2(g.p[j], sc), hi = mul2(g.p[j + 1], sc);
            accA |= e2m1x2(lo.x, hi.x) << (8 * b);
            accB |= e2m1x2(lo.y, hi.y) << (8 * b);
        }
        wa[q] = canon_nz(accA);
        wb[q] = canon_nz(accB);
    }
    out[0] = make_uint4(wa[0], wa[1], wa[2], wa[3]);
    out[1] = make_uint4(wb[0], wb[1], wb[2], wb[3]);
}

// Stochastic rounding of one element (_native.pyx:156-167): v = x / s in f64, neighbours on the
// signed grid, p = (v - lo) / (hi - lo) in f64, u = splitmix64 uniform at `index`, hi when u < p.
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

__device__ __forceinline__ uint4 encode_sr(const Pair& g, int half, int e, uint64_t base, uint64_t idx0) {
    const float sc_f = exp2i(127 - e);
    const double sc_d = (double)sc_f;
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t acc = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int j = q * 8 + b;
            acc |= sr_code(half ? g.p[j].y : g.p[j].x, sc_f, sc_d, base, idx0 + (uint64_t)j) << (4 * b);
        }
        w[q] = acc;
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// NaN-propagating absmax of both groups.
__device__ __forceinline__ float2 pair_absmax(const Pair& g) {
    float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
        a0 = max_nan(a0, fabsf(g.p[i].x));
        a1 = max_nan(a1, fabsf(g.p[i + 1].x));
        b0 = max_nan(b0, fabsf(g.p[i].y));
        b1 = max_nan(b1, fabsf(g.p[i + 1].y));
    }
    return make_float2(max_nan(a0, a1), max_nan(b0, b1));
}

// Quantize both groups (already transformed and pre-scaled).  idxA / idxB: SR stream positions of
// element 0 of each group.
template <int ROUND>
__device__ __forceinline__ PairOut quantize_pair(const Pair& g, uint64_t sr_base, uint64_t idxA, uint64_t idxB,
                                                 int* err_flag, int* fallback_counter) {
    PairOut o;
    const float2 am = pair_absmax(g);
    if (!(am.x <= 3.4028234663852886e38f) || !(am.y <= 3.4028234663852886e38f)) {
        if (err_flag) atomicOr(err_flag, 1);
    }
    int e[2];
    if (ROUND == kQuest) {
        quest_search_pair(g, am.x, am.y, e, fallback_counter);
        // zero group: e = 0, codes 0, all kept (_native.pyx:228-233)
        if (!(am.x > 0.0f)) e[0] = 0;
        if (!(am.y > 0.0f)) e[1] = 0;
        encode_pair(g, e[0], e[1], o.codes);
        const float2 lim = make_float2(6.0f * exp2i(e[0] - 127), 6.0f * exp2i(e[1] - 127));
        uint32_t ma = 0, mb = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            ma |= (fabsf(g.p[i].x) <= lim.x ? 1u : 0u) << i;
            mb |= (fabsf(g.p[i].y) <= lim.y ? 1u : 0u) << i;
        }
        o.mask[0] = ma;
        o.mask[1] = mb;
    } else {
        e[0] = ceil_scale_exp(am.x);
        e[1] = ceil_scale_exp(am.y);
        o.mask[0] = o.mask[1] = 0xFFFFFFFFu;
        if (ROUND == kRtn) {
            encode_pair(g, e[0], e[1], o.codes);
        } else {
            o.codes[0] = encode_sr(g, 0, e[0], sr_base, idxA);
            o.codes[1] = encode_sr(g, 1, e[1], sr_base, idxB);
        }
    }
    o.sf[0] = (uint32_t)e[0];
    o.sf[1] = (uint32_t)e[1];
    return o;
}

}  // namespace qt
