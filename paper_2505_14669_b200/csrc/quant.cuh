// quant.cuh -- per-group MXFP4 quantizers (one group of 32 values held in registers).
//
// Bit-exact restatements of the reference quantizers (mx4train/_backend/_native.pyx):
//   QUEST  quantize_quest          _native.pyx:171-245  (fast fp32 search + exact f64 fallback)
//   RTN    quantize_rtn            _native.pyx:104-131
//   SR     quantize_sr             _native.pyx:134-168  (same splitmix64 stream, f64 p)
#pragma once
#include "common.cuh"

namespace qt {

enum Rounding : int { kQuest = 0, kRtn = 1, kSr = 2 };

struct GroupOut {
    uint4 codes;    // 32 nibbles, element 2k in the low nibble of byte k
    uint32_t sf;    // E8M0 exponent (low byte)
    uint32_t mask;  // bit j: |x_j / s| <= 6
};

// grid_index ladder (_native.pyx:46-63) on an exact double magnitude.
__device__ __forceinline__ double grid_round_d(double a) {
    int idx = (a > 0.25) + (a >= 0.75) + (a > 1.25) + (a >= 1.75) + (a > 2.5) + (a >= 3.5) + (a > 5.0);
    // GRID = {0, .5, 1, 1.5, 2, 3, 4, 6}
    double g = idx <= 4 ? 0.5 * idx : (idx == 5 ? 3.0 : (idx == 6 ? 4.0 : 6.0));
    return g;
}

// Exact reference scale search (_native.pyx:171-203) -- cold path for near-ties of the fast
// search.  Sequential ascending-j f64 accumulation, strict '<' (ties keep the larger scale).
// vbuf[j] * 2^k of the reference equals |x_j| * 2^(127-e) exactly, so it is recomputed per
// candidate instead of being carried in a second register array.
__device__ __forceinline__ int quest_exact(const float (&x)[32], int e_hi, int e_lo) {
    int best_e = e_hi;
    double best_err = -1.0;
    for (int e = e_hi; e >= e_lo; --e) {
        const double sc = (double)exp2i(127 - e_hi) * (double)(1 << (e_hi - e));
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            double a = fabs((double)x[j] * sc);
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

// Fast QuEST candidate search: fp32 errors via the hardware E2M1 round trip, with a guard band
// that routes any group whose best and runner-up errors are within the fp32 error bound to the
// exact f64 search above.  Returns the chosen E8M0 exponent.
__device__ __forceinline__ int quest_search(const float (&x)[32], float amax, int* fallback_counter) {
    const int e_hi = ceil_scale_exp(amax);
    const int e_lo = quest_low_exp(amax);
    const float sc = exp2i(127 - e_hi);
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fabsf(x[j]) * sc;
    float best = __int_as_float(0x7f800000), second = best;
    int best_k = 0;
    const int ncand = e_hi - e_lo + 1;
    float wscale = 1.0f;  // 4^-k
    for (int k = 0; k < ncand; ++k) {
        float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            float2 q0 = e2m1x2_to_f32(e2m1x2(v[j], v[j + 1]));
            float2 q1 = e2m1x2_to_f32(e2m1x2(v[j + 2], v[j + 3]));
            float t0 = v[j] - q0.x, t1 = v[j + 1] - q0.y, t2 = v[j + 2] - q1.x, t3 = v[j + 3] - q1.y;
            acc0 = fmaf(t0, t0, acc0);
            acc1 = fmaf(t1, t1, acc1);
            acc2 = fmaf(t2, t2, acc2);
            acc3 = fmaf(t3, t3, acc3);
        }
        float err = ((acc0 + acc1) + (acc2 + acc3)) * wscale;
        if (err < best) {
            second = best;
            best = err;
            best_k = k;
        } else if (err < second) {
            second = err;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = v[j] * 2.0f;
        wscale *= 0.25f;
    }
    // fp32 path: each term exact up to 2^-24 relative, the 32-term sum within ~2^-19; the
    // reference's own f64 sum within 2^-47.  A gap above 2^-14 relative cannot flip the order.
    if (ncand > 1 && !(second - best > second * 6.103515625e-05f + 7.52316384526264e-37f)) {
        if (fallback_counter) atomicAdd(fallback_counter, 1);
        return quest_exact(x, e_hi, e_lo);
    }
    return e_hi - best_k;
}

// Pack the 32 E2M1 codes of x * 2^(127 - e) (RNE, satfinite, -0 -> +0).
__device__ __forceinline__ uint4 encode_group(const float (&x)[32], int e) {
    const float sc = exp2i(127 - e);
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t acc = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            int j = q * 8 + b * 2;
            acc |= e2m1x2(x[j] * sc, x[j + 1] * sc) << (8 * b);
        }
        w[q] = canon_nz(acc);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// Stochastic rounding of one element (_native.pyx:156-167): v = x / s in f64, neighbours on the
// signed grid, p = (v - lo) / (hi - lo) in f64, u = splitmix64 uniform at `index`, code of hi
// when u < p.
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

__device__ __forceinline__ uint4 encode_group_sr(const float (&x)[32], int e, uint64_t base, uint64_t idx0) {
    const float sc_f = exp2i(127 - e);
    const double sc_d = (double)exp2i(127 - e);
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t acc = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            int j = q * 8 + b;
            acc |= sr_code(x[j], sc_f, sc_d, base, idx0 + (uint64_t)j) << (4 * b);
        }
        w[q] = acc;
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// Quantize one 32-element group already in its final (transformed, pre-scaled) fp32 form.
__device__ __forceinline__ GroupOut quantize_group(const float (&x)[32], int rounding, uint64_t sr_base,
                                                   uint64_t idx0, int* err_flag, int* fallback_counter) {
    GroupOut o;
    float amax = 0.0f;
    bool finite = true;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        amax = fmaxf(amax, fabsf(x[j]));
        finite &= isfinite(x[j]);
    }
    if (!finite && err_flag) atomicOr(err_flag, 1);
    if (rounding == kQuest) {
        if (amax <= 0.0f) {  // zero group: e = 0, codes 0, all kept (_native.pyx:228-233)
            o.codes = make_uint4(0, 0, 0, 0);
            o.sf = 0;
            o.mask = 0xFFFFFFFFu;
            return o;
        }
        int e = quest_search(x, amax, fallback_counter);
        o.codes = encode_group(x, e);
        o.sf = (uint32_t)e;
        const float sc = exp2i(127 - e);
        uint32_t m = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) m |= (fabsf(x[j]) * sc <= 6.0f ? 1u : 0u) << j;
        o.mask = m;
        return o;
    }
    int e = ceil_scale_exp(amax);
    o.sf = (uint32_t)e;
    o.mask = 0xFFFFFFFFu;
    o.codes = rounding == kRtn ? encode_group(x, e) : encode_group_sr(x, e, sr_base, idx0);
    return o;
}

}  // namespace qt
