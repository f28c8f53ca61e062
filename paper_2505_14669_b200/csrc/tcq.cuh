// tcq.cuh -- shared pieces of the tensor-core Hadamard quantizers (tcq.cu: backward dy operands,
// tcq_x.cu: forward activation operand + transposed requantization).  See tcq.cu for the error-bound proof.
#pragma once
#include "launch.h"
#include "qgroup.cuh"

#ifndef QT_RTN_L2
#define QT_RTN_L2 0  // build flag: 1 = L2-norm bound in rtn_checked (one FFMA per element more, 1/4 of the exact-path
                     // groups; with the warp-cooperative fallback the cheaper sqrt(32) max|Hx| bound is 3 % faster)
#endif

namespace qt {

// element (r, c) of a 128 x 128 bf16 tile stored as two TMA SWIZZLE_128B boxes of 64 columns
__device__ __forceinline__ int tq_off(int r, int c) {
    return (c >> 6) * 16384 + r * 128 + ((((c & 63) >> 3) ^ (r & 7)) << 4) + ((c & 7) << 1);
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// tcgen05.mma kind::f16 (bf16 x bf16 -> fp32), D[tmem] (+)= A[smem] B[smem]^T
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// instruction descriptor: D f32, A/B bf16, A K-major (a_mn = 0) or MN-major (1), B K-major
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

// Fast stochastic rounding (QT_ROUND_SR_FAST) of one group from tensor-core sums: the E8M0 exponent is checked like
// rtn_checked's (false -> caller takes the exact path); the codes are drawn for the tensor-core values themselves
// (within the bound B of the reference's, ~1e-6 of a grid step: the mode is statistical, not the reference's draws).
// Element j uses stream position idx0 + j.
__device__ __forceinline__ bool srf_checked(const float (&acc)[32], float prescale, uint32_t k0, uint32_t k1,
                                            uint64_t idx0, uint4& codes, int& e_out) {
    constexpr float kC5 = 0.17677669f;
    constexpr float kU = 5.9604645e-08f;
    const float amax = absmax32(acc);
    bool ok = amax <= 1.0e30f && (amax >= 1.0e-25f || amax == 0.0f);
    const float nrm = amax * 5.65685463f;
    const float bnd = 20.0f * kU * kC5 * nrm * 1.001f;
    const float amp = amax * kC5 * prescale;
    const float d = bnd * prescale + 4.0f * kU * amp;
    const uint32_t ab = __float_as_uint(amp);
    const int e = amax == 0.0f ? 0 : (int)(ab >> 23) - 2 + ((ab & 0x7FFFFFu) > 0x400000u ? 1 : 0);
    const float s2 = __uint_as_float((uint32_t)(254 - e) << 23);
    ok = ok && (amax == 0.0f || (__fmul_rd(amp - d, s2) > 3.0f && __fmul_ru(amp + d, s2) < 6.0f));
    const float sc = kC5 * prescale * s2;
    const uint32_t base = srf_base(k0, k1, idx0);
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int j = 8 * q;
        w[q] = srf_quad(__fmul_rn(acc[j], sc), __fmul_rn(acc[j + 1], sc), __fmul_rn(acc[j + 2], sc),
                        __fmul_rn(acc[j + 3], sc), srf_rbits(base, 2 * q)) |
               srf_quad(__fmul_rn(acc[j + 4], sc), __fmul_rn(acc[j + 5], sc), __fmul_rn(acc[j + 6], sc),
                        __fmul_rn(acc[j + 7], sc), srf_rbits(base, 2 * q + 1)) << 16;
    }
    codes = make_uint4(w[0], w[1], w[2], w[3]);
    e_out = e;
    return ok;
}

// Checked RTN of one group from tensor-core sums acc (= H (s.x), exact up to 8u sum|x|).
// Returns false when a decision is within the error bound (caller falls back to the exact path).
__device__ __forceinline__ bool rtn_checked(const float (&acc)[32], float prescale, uint4& codes, int& e_out) {
    constexpr float kC5 = 0.17677669f;          // fl(c^5) ~ 2^-2.5 (the tensor-core sum lacks the c^5)
    constexpr float kU = 5.9604645e-08f;        // 2^-24
    const float amax = absmax32(acc);
    // branch-free so that two groups interleave; acc == 0 only for x == 0 (H is invertible and the error
    // is below |Hx|), which encodes to zero codes with e = 0 like the reference
    // NaN / huge / tiny -> exact.  Below 1e-25 a subnormal bf16 operand the tensor core may flush (<= 32 * 2^-126
    // in all) would no longer sit far below the bound
    bool ok = amax <= 1.0e30f && (amax >= 1.0e-25f || amax == 0.0f);
#if QT_RTN_L2
    // sum|x| <= ||H x||_2: one FFMA per element buys a ~2.5x tighter bound than sqrt(32) max|H x|
    float ss0 = 0.f, ss1 = 0.f;
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
        ss0 = __fmaf_rn(acc[j], acc[j], ss0);
        ss1 = __fmaf_rn(acc[j + 1], acc[j + 1], ss1);
    }
    const float nrm = __fsqrt_ru(__fadd_ru(ss0, ss1));
#else
    // sum|x| <= ||H x||_2 <= sqrt(32) max|H x| (max|H x| <= amax (1 + 3e-6), covered by the 1.001 below):
    // no per-element work; the looser bound sends ~2.5x more groups (still ~0.2 %) to the exact path
    const float nrm = amax * 5.65685463f;                               // sqrt(32), rounded up
#endif
    const float bnd = 20.0f * kU * kC5 * nrm * 1.001f;                 // |y - acc c^5| (y units)
    const float amp = amax * kC5 * prescale;
    const float d = bnd * prescale + 4.0f * kU * amp;
    // E8M0 of the ceil rule (ceil_scale_exp without clamps: 1e-30 <= amax <= 1e30 keeps e in [22, 227]);
    // the reference's exponent is e iff its absmax lies in (3, 6] * 2^(e-127): check with margin d
    const uint32_t ab = __float_as_uint(amp);
    const int e = amax == 0.0f ? 0 : (int)(ab >> 23) - 2 + ((ab & 0x7FFFFFu) > 0x400000u ? 1 : 0);
    const float s2 = __uint_as_float((uint32_t)(254 - e) << 23);       // 2^(127 - e), normal here
    ok = ok && (amax == 0.0f || (__fmul_rd(amp - d, s2) > 3.0f && __fmul_ru(amp + d, s2) < 6.0f));
    const float sc = kC5 * prescale * s2;                               // acc -> scaled value
    const float bv = (bnd * prescale + 2.0f * kU * amp) * s2 + 1.0e-6f;  // + fma rounding at |v| <= 7
    uint32_t diff = 0, w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        float lo[8], hi[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            lo[k] = __fmaf_rn(acc[8 * q + k], sc, -bv);
            hi[k] = __fmaf_rn(acc[8 * q + k], sc, bv);
        }
        // magnitudes must agree; a sign difference with equal magnitudes needs |v| < bv << 0.25, i.e. both
        // codes are +-0, which canonicalise alike -- so only the hi word is canonicalised
        const uint32_t wl = e2m1x8(lo[0], lo[1], lo[2], lo[3], lo[4], lo[5], lo[6], lo[7]);
        const uint32_t wh = e2m1x8(hi[0], hi[1], hi[2], hi[3], hi[4], hi[5], hi[6], hi[7]);
        diff |= (wl ^ wh) & 0x77777777u;
        w[q] = canon8(wh);
    }
    codes = make_uint4(w[0], w[1], w[2], w[3]);
    e_out = e;
    return ok && diff == 0;
}

// Exact path for ONE undecided group of the staged bf16 tile, warp-cooperative (all 32 lanes; lane j holds element
// j): row group (row idx, columns 32g..) or column group (column idx, rows 32g..), signs sw, the reference's FWHT
// and RTN.  The checked epilogues hand their rare undecided groups to it one at a time instead of running a scalar
// exact path in a single diverged lane.  Same operations as the scalar path: the butterfly pairs (t, t + h) meet through a shuffle,
// the lower index stays the minuend; max |v| is order-independent; each lane encodes its own element.
__device__ __forceinline__ float max_nan2(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void exact_group_warp(const uint8_t* tile, bool col, int idx, int g, uint32_t sw,
                                                 float prescale, int* err, uint4& codes, int& e_out,
                                                 bool srf = false, uint32_t k0 = 0, uint32_t k1 = 0,
                                                 uint64_t idx0 = 0) {
    const int j = threadIdx.x & 31;
    const int r = col ? g * 32 + j : idx, c = col ? idx : g * 32 + j;
    const uint16_t h16 = *reinterpret_cast<const uint16_t*>(tile + tq_off(r, c));
    float v = __uint_as_float(((uint32_t)h16 << 16) ^ (((sw >> j) & 1u) << 31));
#pragma unroll
    for (int h = 1; h < 32; h <<= 1) {
        const float o = __shfl_xor_sync(0xffffffffu, v, h);
        v = __fmul_rn((j & h) ? __fsub_rn(o, v) : __fadd_rn(v, o), kHc);
    }
    float am = fabsf(v);
#pragma unroll
    for (int h = 1; h < 32; h <<= 1) am = max_nan2(am, __shfl_xor_sync(0xffffffffu, am, h));
    if (!(am <= 3.4028234663852886e38f) && err && j == 0) atomicOr(err, 1);
    int e;
    float sc;
    uint32_t nib;
    if (srf) {   // QT_ROUND_SR_FAST: quant_group<kSr>'s order -- pre-scale, ceil exponent of the pre-scaled amax
        v = __fmul_rn(v, prescale);
        e = ceil_scale_exp(__fmul_rn(am, prescale));
        const float vs = __fmul_rn(v, exp2i(127 - e));
        const int q0 = j & ~3;
        const float e0 = __shfl_sync(0xffffffffu, vs, q0), e1 = __shfl_sync(0xffffffffu, vs, q0 + 1);
        const float e2 = __shfl_sync(0xffffffffu, vs, q0 + 2), e3 = __shfl_sync(0xffffffffu, vs, q0 + 3);
        nib = (srf_quad(e0, e1, e2, e3, srf_rbits(srf_base(k0, k1, idx0), (uint32_t)(j >> 2))) >> (4 * (j & 3))) & 0xFu;
    } else {
        if (!rtn_scale(am, prescale, e, sc)) v = __fmul_rn(v, prescale);
        nib = e2m1b(__fmul_rn(v, sc), 0.0f) & 0xFu;
        if ((nib & 7u) == 0) nib = 0;   // -0 -> +0 (_native.pyx:127-130)
    }
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = __reduce_or_sync(0xffffffffu, (j >> 3) == q ? nib << (4 * (j & 7)) : 0u);
    codes = make_uint4(w[0], w[1], w[2], w[3]);
    e_out = e;
}

// sign byte -> 8 bf16 +-1.0 (bit i set -> element i negative), 4 KB
__device__ __forceinline__ void build_sign_lut(uint8_t* lut) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            w[k] = 0x3F803F80u | (((i >> (2 * k)) & 1u) << 15) | (((i >> (2 * k + 1)) & 1u) << 31);
        reinterpret_cast<uint4*>(lut)[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// 16-byte chunk (n, k8) of a signed 32 x 32 Hadamard block B[n][k] = s_k H[k][n] (K-major, no swizzle:
// core matrix (n/8, k8) at ((n/8) * 4 + k8) * 128, row n % 8 at 16 B); sgn = the 32 sign bits (bit k).
__device__ __forceinline__ void store_b_chunk(uint32_t blk_base, const uint8_t* lut, int n, int k8, uint32_t sgn) {
    // byte m of P = sign pattern of popc(i & m) & 1 over i = 0..7 (Sylvester row pattern)
    const uint32_t pat = (uint32_t)(0x963C5AF066CCAA00ull >> (8 * (n & 7))) & 0xFFu;
    const uint32_t byte = pat ^ ((__popc(k8 & (n >> 3)) & 1) ? 0xFFu : 0u) ^ ((sgn >> (8 * k8)) & 0xFFu);
    uint32_t v0, v1, v2, v3;  // explicit shared-window load (lut is a generic pointer into smem)
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                 : "r"(smem_u32(lut) + byte * 16));
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(blk_base + ((n >> 3) * 4 + k8) * 128 + (n & 7) * 16),
                 "r"(v0), "r"(v1), "r"(v2), "r"(v3)
                 : "memory");
}

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                      CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t tq_encode() {
    static PFN_encodeTiled_t fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled_t>(p);
    }
    return fn;
}

// [rows, cols] matrix (row stride ld_bytes) as TMA boxes of 128 bytes x 128 rows, 128-byte swizzle
static int tq_map(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int esz, int64_t rows, int64_t cols,
                  int64_t ld_bytes) {
    PFN_encodeTiled_t enc = tq_encode();
    if (!enc) return 1001;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld_bytes};
    cuuint32_t box[2] = {(cuuint32_t)(128 / esz), 128};
    cuuint32_t es[2] = {1, 1};
    return enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                   CUDA_SUCCESS
               ? 0
               : 1002;
}

}  // namespace qt
