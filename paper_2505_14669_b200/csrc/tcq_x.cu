// tcq_x.cu -- forward activation quantizer fully on the tensor cores, bit-exact by proof + fallback.
//
//   X_q, M_x = QuEST(H32(x))                      row transform: tcgen05 (x . H), checked QuEST search
//   X_t      = RTN(H32(deq(X_q)^T (.) s) * 0.75)  col transform: tcgen05 (deq^T . diag(s) H), checked RTN
//   (qlinear.py:139-157, 206-207, 235)
//
// The transforms are bf16 GEMMs with +-1 Hadamard blocks (error bound: tcq.cu header).  The CUDA cores
// only make decisions, each with a rigorous margin:
//   * E8M0 exponents: the reference's absmax must lie in the same (3, 6] * 2^(e-127) interval under +-B;
//   * QuEST candidate errors: R_k = sum d(v_j)^2 with d the (1-Lipschitz) distance to the FP4 grid, so
//     |R_k(approx) - R_k(ref)| <= B_k (2 sqrt(32 R_k) + 32 B_k) + fp32 rounding; the best candidate must
//     beat every other candidate by more than both bounds (pruned candidates by their clipping bound);
//   * E2M1 codes: v - B_k and v + B_k encode identically (RTN is monotone);
//   * trust mask: |v -+ B_k| agree on the side of 6.
// A group failing any check is recomputed on the CUDA cores by the exact v3 path from the bf16 tile
// still in shared memory.
//
// Pipeline (persistent, 1 CTA / SM): warp 0 TMA producer (x tile: two 64-column SW128 boxes, 3 stages),
// warp 1 MMA issuer (per tile 8 row MMAs on the x tile with the plain H block, then -- once the epilogue
// has written deq(X_q) -- 8 col MMAs on that tile read MN-major with the 4 signed blocks), warps 2-17
// epilogue: iteration i does the row phase of tile i and the col phase of tile i-1 (whose MMAs ran
// meanwhile), thread = (TMEM lane quadrant, group).
#include "tcq.cuh"

namespace qt {

constexpr int kXqStages = 3;
constexpr int kXqEpiWarps = 16;
constexpr int kXqThreads = 64 + 32 * kXqEpiWarps;
constexpr int kXqIn = 32768;                     // x tile (bf16 128 x 128)
constexpr int kXqDeqA = 32768, kXqDeq = kXqDeqA + 4 * 2048;
constexpr int kXqOffDeq = kXqStages * kXqIn;
constexpr int kXqOffH = kXqOffDeq + 2 * kXqDeq;  // plain H block (row transform)
constexpr int kXqOffLut = kXqOffH + 2048;
constexpr int kXqOffBar = kXqOffLut + 4096;
constexpr int kXqBytes = kXqOffBar + 256 + 1024;

struct XqArgs {
    int64_t R, C;
    QuantOut row_out;         // X_q [R, C] + mask
    const uint32_t* sign_r;   // RHT signs along R (tokens)
    QuantOut col_out;         // X_t [C, R]
    float col_prescale;
    int* fallbacks;           // re-decided groups (nullable): [0] X_q search, [1] X_t, [2] X_q codes only
    int dbg;                  // experiment knobs (0 in production): 1 skip QuEST decisions, 2 skip RTN decisions,
                              // 4 exact CUDA-core row phase for every group
    int srf;                  // X_t by QT_ROUND_SR_FAST: key, stream start and row stride (c * ld + r)
    uint64_t key, ctr;
    int64_t ld;
};

constexpr float kU24 = 5.9604645e-08f;  // 2^-24
constexpr float kC5f = 0.17677669f;     // fl(c^5)

// |{q - a}| summed squares at scale K (acc * K = the candidate's scaled values)
__device__ __forceinline__ float raw_err(const float (&acc)[32], float K) {
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
        const float a = __fmul_rn(acc[j], K), b = __fmul_rn(acc[j + 1], K);
        const uint32_t q = e2m1_rt_h2(a, b);
        const float ta = fh16_sub_lo(q, a), tb = fh16_sub_hi(q, b);
        s0 = __fmaf_rn(ta, ta, s0);
        s1 = __fmaf_rn(tb, tb, s1);
    }
    return __fadd_rn(s0, s1);
}

// raw_err at K and 2K in one interleaved pass (the two always-evaluated candidates)
__device__ __forceinline__ void raw_err2(const float (&acc)[32], float K, float& r0, float& r1) {
    float s0 = 0.f, s1 = 0.f, u0 = 0.f, u1 = 0.f;
    const float K2 = 2.0f * K;
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
        const float a = __fmul_rn(acc[j], K), b = __fmul_rn(acc[j + 1], K);
        const float c = __fmul_rn(acc[j], K2), d = __fmul_rn(acc[j + 1], K2);
        const uint32_t q = e2m1_rt_h2(a, b), p = e2m1_rt_h2(c, d);
        const float ta = fh16_sub_lo(q, a), tb = fh16_sub_hi(q, b);
        const float tc = fh16_sub_lo(p, c), td = fh16_sub_hi(p, d);
        s0 = __fmaf_rn(ta, ta, s0);
        s1 = __fmaf_rn(tb, tb, s1);
        u0 = __fmaf_rn(tc, tc, u0);
        u1 = __fmaf_rn(td, td, u1);
    }
    r0 = __fadd_rn(s0, s1);
    r1 = __fadd_rn(u0, u1);
}

// Checked QuEST of one group from tensor-core sums acc (= H x).  Returns 0 when every decision is certain,
// 1 when the scale exponent is not (caller re-runs the exact search), 2 when only codes / mask are not
// (e_out is the reference's exponent; caller re-encodes the exact transform at e_out).
__device__ __forceinline__ int quest_checked(const float (&acc)[32], uint4& codes, int& e_out, uint32_t& keep) {
    const float amax = absmax32(acc);
    codes = make_uint4(0, 0, 0, 0);
    keep = 0xFFFFFFFFu;
    e_out = 0;
    if (amax == 0.0f) return 0;                             // x == 0: zero group (e = 0, all kept)
    if (!(amax >= 1.0e-30f && amax <= 1.0e30f)) return 1;
    float ss0 = 0.f, ss1 = 0.f;
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
        ss0 = __fmaf_rn(acc[j], acc[j], ss0);
        ss1 = __fmaf_rn(acc[j + 1], acc[j + 1], ss1);
    }
    const float B = 20.0f * kU24 * kC5f * __fsqrt_ru(__fadd_ru(ss0, ss1)) * 1.001f;  // |y - acc c^5|
    const float amp = amax * kC5f;
    // e_hi (ceil rule) and e_lo (floor rule) share the thresholds 1.5 * 2^m: stable iff amp * 2^(127-e_hi)
    // stays inside (3, 6] under +-(B + rounding)
    const uint32_t ab = __float_as_uint(amp);
    const int e_hi = (int)(ab >> 23) - 2 + ((ab & 0x7FFFFFu) > 0x400000u ? 1 : 0);
    const float S0 = __uint_as_float((uint32_t)(254 - e_hi) << 23);   // 2^(127 - e_hi)
    const float d = B + 4.0f * kU24 * amp;
    if (!(__fmul_rd(amp - d, S0) > 3.0f && __fmul_ru(amp + d, S0) < 6.0f)) return 1;
    const float K0 = kC5f * S0;
    // candidate errors (raw scaled units) with their bounds.  The stability check pins amp * S0 to (3, 6),
    // so e_hi - e_lo == 5: candidates k = 0 .. 5, k = 0 and 1 always evaluated (one interleaved pass)
    const float Bk0 = (B * S0) * 1.001f + 2.0e-6f;
    float R0, R1;
    raw_err2(acc, K0, R0, R1);
    const float D0 = Bk0 * (2.0f * __fsqrt_ru(32.0f * R0) + 32.0f * Bk0) + 4.0e-6f * R0;
    const float Bk1 = 2.0f * Bk0;
    const float D1 = Bk1 * (2.0f * __fsqrt_ru(32.0f * R1) + 32.0f * Bk1) + 4.0e-6f * R1;
    const float E1 = __fmul_rn(R1, 0.25f), F1 = __fmul_ru(D1, 0.25f);
    float best = R0, bestD = D0, second = E1, secondD = F1;
    int bk = 0;
    if (E1 < R0) {
        best = E1;
        bestD = F1;
        second = R0;
        secondD = D0;
        bk = 1;
    }
    for (int k = 2; k <= 5; ++k) {
        const float sk = exp2i(k), ik = exp2i(-2 * k);
        // clipping-only bound of the true largest element, monotone in k
        const float dl = __fsub_rd(__fmul_rd(__fmul_rd(amp - d, S0), sk), 6.0f);
        const float lb = dl > 0.f ? __fmul_rd(__fmul_rd(dl, dl), ik) : 0.f;
        if (__fmul_rd(lb, 0.99999905f) > __fmul_ru(best + bestD, 1.0f + kQTol)) break;
        const float Bk = Bk0 * sk;
        const float R = raw_err(acc, __fmul_rn(K0, sk));
        const float D = Bk * (2.0f * __fsqrt_ru(32.0f * R) + 32.0f * Bk) + 4.0e-6f * R;
        const float Ek = __fmul_rn(R, ik), Dk = __fmul_ru(D, ik);
        if (Ek < best) {
            second = best;
            secondD = bestD;
            best = Ek;
            bestD = Dk;
            bk = k;
        } else if (Ek < second) {
            second = Ek;
            secondD = Dk;
        }
    }
    if (!(__fsub_rd(second - secondD, best + bestD) > __fadd_ru(__fmul_ru(second, kQTol), kQAtol))) return 1;
    const int e = e_hi - bk;
    // final codes and trust mask at e, each decision checked against +-B_k
    const float K = __fmul_rn(K0, exp2i(bk));
    const float Bk = Bk0 * exp2i(bk) + 1.0e-6f * exp2i(bk);
    // mask: sign of 6 - |hi| per element; the reference's |v| is within 2 B_k of |hi|, so the bits are
    // certain when no |6 - |hi|| is below that
    uint32_t diff = 0, w[4], clip = 0;
    float m0 = 3.0e38f, m1 = 3.0e38f;
#pragma unroll
    for (int q = 3; q >= 0; --q) {
        float lo[8], hi[8], t[8];
#pragma unroll
        for (int k = 7; k >= 0; --k) {
            lo[k] = __fmaf_rn(acc[8 * q + k], K, -Bk);
            hi[k] = __fmaf_rn(acc[8 * q + k], K, Bk);
            t[k] = __fsub_rn(6.0f, fabsf(hi[k]));
            clip = __funnelshift_l(__float_as_uint(t[k]), clip, 1);
        }
        m0 = fminf(m0, fminf(fabsf(t[0]), fabsf(t[1])));
        m1 = fminf(m1, fminf(fabsf(t[2]), fabsf(t[3])));
        m0 = fminf(m0, fminf(fabsf(t[4]), fabsf(t[5])));
        m1 = fminf(m1, fminf(fabsf(t[6]), fabsf(t[7])));
        const uint32_t wl = canon8(e2m1x8(lo[0], lo[1], lo[2], lo[3], lo[4], lo[5], lo[6], lo[7]));
        w[q] = canon8(e2m1x8(hi[0], hi[1], hi[2], hi[3], hi[4], hi[5], hi[6], hi[7]));
        diff |= wl ^ w[q];
    }
    codes = make_uint4(w[0], w[1], w[2], w[3]);
    e_out = e;
    keep = ~clip;
    return diff == 0 && fminf(m0, m1) > 2.5f * Bk ? 0 : 2;
}

// exact bf16 of code * 2^(e-127) for the 8 nibbles of a codes word
__device__ __forceinline__ uint4 xq_deq8(uint32_t w, float s) {
    uint32_t o[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const float2 f = e2m1x2_to_f32((w >> (8 * b)) & 0xFFu);
        __nv_bfloat162 h = __floats2bfloat162_rn(__fmul_rn(f.x, s), __fmul_rn(f.y, s));
        o[b] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

struct XqGroup {
    uint4 codes;
    uint32_t keep;
    int e;
};

// Warp-cooperative exact row group (all 32 lanes; lane j holds element j of tile row r, group g): the
// reference's butterfly through shuffles (lower index the minuend), then
//   status 1: the QuEST search of quest_search32 -- per-candidate errors summed by a warp tree (any fp32 order is
//             within 31 u of the exact sum, far inside the 2^-14 near-tie guard), near-ties decided by the exact
//             f64 search (quest_exact_cold) in lane 0;
//   status 2: the exponent e is certain; codes and trust mask at e.
// Every lane returns the group's codes, exponent and mask.
static __device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1) x = __fadd_rn(x, __shfl_xor_sync(0xffffffffu, x, h));
    return x;
}
static __device__ XqGroup xq_exact_row_warp(const uint8_t* tile, int r, int g, int status, int e_known, int* err) {
    const int j = threadIdx.x & 31;
    const uint16_t h16 = *reinterpret_cast<const uint16_t*>(tile + tq_off(r, 32 * g + j));
    float v = __uint_as_float((uint32_t)h16 << 16);
#pragma unroll
    for (int h = 1; h < 32; h <<= 1) {
        const float o = __shfl_xor_sync(0xffffffffu, v, h);
        v = __fmul_rn((j & h) ? __fsub_rn(o, v) : __fadd_rn(v, o), kHc);
    }
    XqGroup o;
    int e = e_known;
    if (status == 1) {
        float am = fabsf(v);
#pragma unroll
        for (int h = 1; h < 32; h <<= 1) am = max_nan2(am, __shfl_xor_sync(0xffffffffu, am, h));
        if (!(am <= 3.4028234663852886e38f) && err && j == 0) atomicOr(err, 1);
        if (!(am > 0.0f && am <= 3.4028234663852886e38f)) {   // zero group (or non-finite): _native.pyx:228-233
            o.codes = make_uint4(0, 0, 0, 0);
            o.keep = 0xFFFFFFFFu;
            o.e = 0;
            return o;
        }
        const int e_hi = ceil_scale_exp(am), e_lo = quest_low_exp(am);
        e = e_hi;
        if (e_hi > e_lo) {
            const float sc0 = exp2i(127 - e_hi), a0 = __fmul_rn(am, sc0);
            float best = __int_as_float(0x7f800000), second = best;
            int bk = 0;
            for (int k = 0; k <= e_hi - e_lo; ++k) {
                const float sk = exp2i(k), ik = exp2i(-2 * k);
                if (k >= 2) {
                    const float d = __fsub_rn(__fmul_rn(a0, sk), 6.0f);
                    const float lb = __fmul_rn(__fmul_rn(d, d), ik);
                    if (__fmul_rn(lb, 0.99999905f) > __fadd_rn(__fmul_rn(best, 1.0f + kQTol), kQAtol)) break;
                }
                const float a = __fmul_rn(v, __fmul_rn(sc0, sk));
                const uint32_t q = e2m1_rt_h2(a, 0.0f);
                const float t = fh16_sub_lo(q, a);
                const float ek = __fmul_rn(warp_sum(__fmul_rn(t, t)), ik);
                if (ek < best) {
                    second = best;
                    best = ek;
                    bk = k;
                } else if (ek < second) {
                    second = ek;
                }
            }
            if (!(__fsub_rn(second, best) > __fadd_rn(__fmul_rn(second, kQTol), kQAtol))) {
                float xs[32];   // near-tie: the exact sequential f64 search of the reference, in lane 0
#pragma unroll
                for (int i = 0; i < 32; ++i) xs[i] = __shfl_sync(0xffffffffu, v, i);
                int ex = 0;
                if (j == 0) ex = quest_exact_cold(xs, e_hi, e_lo);
                e = __shfl_sync(0xffffffffu, ex, 0);
            } else {
                e = e_hi - bk;
            }
        }
    }
    const float a = __fmul_rn(v, exp2i(127 - e));
    uint32_t nib = e2m1b(a, 0.0f) & 0xFu;
    if ((nib & 7u) == 0) nib = 0;
    const bool clip = (__float_as_uint(__fsub_rn(6.0f, fabsf(a))) >> 31) != 0;
    o.keep = ~__ballot_sync(0xffffffffu, clip);
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = __reduce_or_sync(0xffffffffu, (j >> 3) == q ? nib << (4 * (j & 7)) : 0u);
    o.codes = make_uint4(w[0], w[1], w[2], w[3]);
    o.e = e;
    return o;
}

template <bool SRF>   // SRF: X_t by QT_ROUND_SR_FAST instead of checked RTN (its own instantiation)
__global__ void __launch_bounds__(kXqThreads, 1) k_tcq_xq(const __grid_constant__ CUtensorMap tmX, XqArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* lut = smem + kXqOffLut;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kXqOffBar);   // [3] x tile landed
    uint64_t* empty = full + kXqStages;                                // [3] row phase done with it
    uint64_t* rdone = empty + kXqStages;                               // [2] row MMAs committed
    uint64_t* rfree = rdone + 2;                                       // [2] row accumulators read
    uint64_t* dfull = rfree + 2;                                       // [2] deq tile written
    uint64_t* cdone = dfull + 2;                                       // [2] col MMAs committed
    uint64_t* cfree = cdone + 2;                                       // [2] col accumulators read
    uint64_t* dfree = cfree + 2;                                       // [2] col phase done with deq tile
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(dfree + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t nRT = (a.R + 127) / 128, nCT = (a.C + 127) / 128, NT = nRT * nCT;
    const int ntiles = (int)(NT > (int64_t)blockIdx.x ? (NT - 1 - blockIdx.x) / gridDim.x + 1 : 0);

    build_sign_lut(lut);
    __syncthreads();
    if (threadIdx.x >= 64 && threadIdx.x < 64 + 128) {  // the plain H block: 32 n x 4 k8 chunks
        const int c = threadIdx.x - 64;
        store_b_chunk(smem_u32(smem + kXqOffH), lut, c >> 2, c & 3, 0u);
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmX);
        for (int i = 0; i < kXqStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kXqEpiWarps);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&rdone[i], 1);
            mbar_init(&rfree[i], kXqEpiWarps);
            mbar_init(&dfull[i], kXqEpiWarps);
            mbar_init(&cdone[i], 1);
            mbar_init(&cfree[i], kXqEpiWarps);
            mbar_init(&dfree[i], kXqEpiWarps);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_holder, 512);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;  // row accumulators at b * 128, col accumulators at 256 + b * 128

    if (warp == 0) {
        if (lane == 0) {
            for (int it = 0; it < ntiles; ++it) {
                const int64_t t = blockIdx.x + (int64_t)it * gridDim.x;
                const int s = it % kXqStages;
                const int64_t r0 = (t % nRT) * 128, c0 = (t / nRT) * 128;
                mbar_wait_role(&empty[s], ((it / kXqStages) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], kXqIn);
                tma_load_2d(smem + s * kXqIn, &tmX, &full[s], (int)c0, (int)r0);
                tma_load_2d(smem + s * kXqIn + 16384, &tmX, &full[s], (int)c0 + 64, (int)r0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t id_row = idesc_bf16(128, 32, 0), id_col = idesc_bf16(128, 32, 1);
            const uint32_t Hs = smem_u32(smem + kXqOffH);
            // row MMAs of tile it run one step ahead of the col MMAs of tile it - 1
            for (int it = 0; it <= ntiles; ++it) {
                if (it < ntiles) {
                    const int s = it % kXqStages, b = it & 1;
                    mbar_wait_role(&rfree[b], ((it >> 1) & 1) ^ 1);
                    mbar_wait_role(&full[s], (it / kXqStages) & 1);
                    tc_fence_after();
                    const uint32_t As = smem_u32(smem + s * kXqIn);
#pragma unroll
                    for (int g = 0; g < 4; ++g)
#pragma unroll
                        for (int ks = 0; ks < 2; ++ks)
                            mma_bf16(tmem + b * 128 + 32 * g,
                                     make_sdesc(As + (g >> 1) * 16384 + (g & 1) * 64 + ks * 32, 16, 1024, kLayoutSW128),
                                     make_sdesc(Hs + ks * 256, 128, 512, kLayoutNone), id_row, ks);
                    tc_commit(&rdone[b]);
                }
                if (it >= 1) {
                    const int jt = it - 1, d = jt & 1;
                    mbar_wait_role(&cfree[d], ((jt >> 1) & 1) ^ 1);
                    mbar_wait_role(&dfull[d], (jt >> 1) & 1);
                    tc_fence_after();
                    const uint32_t Ds = smem_u32(smem + kXqOffDeq + d * kXqDeq), Bs = Ds + kXqDeqA;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
#pragma unroll
                        for (int ks = 0; ks < 2; ++ks)
                            mma_bf16(tmem + 256 + d * 128 + 32 * q,
                                     make_sdesc(Ds + (q * 32 + ks * 16) * 128, 16384, 1024, kLayoutSW128),
                                     make_sdesc(Bs + q * 2048 + ks * 256, 128, 512, kLayoutNone), id_col, ks);
                    tc_commit(&cdone[d]);
                }
            }
        }
    } else {
        const int ew = warp - 2, quad = warp & 3, g = ew >> 2;  // TMEM lane quadrant, group 0..3
        const int li = quad * 32 + lane;                           // tile row (row phase) / column (col phase)
        const int et = ew * 32 + lane;                             // 0..511
        for (int it = 0; it <= ntiles; ++it) {
            // ------------------------------------------------------------ row phase of tile it
            if (it < ntiles) {
                const int64_t t = blockIdx.x + (int64_t)it * gridDim.x;
                const int s = it % kXqStages, b = it & 1, d = it & 1;
                const int64_t r0 = (t % nRT) * 128, c0 = (t / nRT) * 128;
                const int64_t pos = r0 + 32 * (et >> 7);
                const uint32_t sgn = (a.sign_r && pos < a.R) ? __ldg(a.sign_r + (pos >> 5)) : 0u;
                mbar_wait_hint<1000>(&rdone[b], (it >> 1) & 1);
                tc_fence_after();
                uint32_t raw[32];
                tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + b * 128 + 32 * g, raw);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&rfree[b]);
                float acc[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[j] = __uint_as_float(raw[j]);
                uint4 codes;
                int e;
                uint32_t keep;
                const int64_t row = r0 + li, gg = c0 / 32 + g;
                const bool valid = row < a.R && gg * 32 < a.C;
                const uint8_t* tile = smem + s * kXqIn;
                int st = 0;
                if (a.dbg & 4) {  // experiment: every row group on the exact CUDA-core path (hybrid timing)
                    st = 1;
                } else if (a.dbg & 1) {  // experiment: skip the QuEST decisions (timing only)
                    codes = make_uint4(__float_as_uint(acc[0]), __float_as_uint(acc[9]), __float_as_uint(acc[17]),
                                       __float_as_uint(acc[31]));
                    e = 120;
                    keep = 0u;
                } else {
                    st = quest_checked(acc, codes, e, keep);
                }
                // undecided groups: the whole warp recomputes them exactly, one at a time (no diverged lane)
                for (uint32_t todo = __ballot_sync(0xffffffffu, st && valid); todo; todo &= todo - 1) {
                    const int f = __ffs(todo) - 1;
                    const int stf = __shfl_sync(0xffffffffu, st, f), ef = __shfl_sync(0xffffffffu, e, f);
                    if (a.fallbacks && lane == 0) atomicAdd(a.fallbacks + (stf == 2 ? 2 : 0), 1);
                    const XqGroup o = xq_exact_row_warp(tile, quad * 32 + f, g, stf, ef, a.row_out.err);
                    if (lane == f) {
                        codes = o.codes;
                        e = o.e;
                        keep = o.keep;
                    }
                }
                if (!valid) {
                    codes = make_uint4(0, 0, 0, 0);
                    e = 0;
                } else {
                    *reinterpret_cast<uint4*>(a.row_out.codes + row * a.row_out.ldc + gg * 16) = codes;
                    if (a.row_out.mask) a.row_out.mask[row * (a.C / 32) + gg] = keep;
                    a.row_out.sf[sf_offset(row, gg, a.row_out.katoms)] = (uint8_t)e;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);  // the exact path no longer needs the x tile
                // deq(X_q) into buffer d once the col phase of tile it - 2 (MMAs and exact reads) is done
                mbar_wait_hint<1000>(&dfree[d], ((it >> 1) & 1) ^ 1);
                uint8_t* dq = smem + kXqOffDeq + d * kXqDeq;
                const float sc = exp2i(e - 127);
                uint8_t* dp = dq + (g >> 1) * 16384 + li * 128;
                *reinterpret_cast<uint4*>(dp + ((((g & 1) * 4 + 0) ^ (li & 7)) << 4)) = xq_deq8(codes.x, sc);
                *reinterpret_cast<uint4*>(dp + ((((g & 1) * 4 + 1) ^ (li & 7)) << 4)) = xq_deq8(codes.y, sc);
                *reinterpret_cast<uint4*>(dp + ((((g & 1) * 4 + 2) ^ (li & 7)) << 4)) = xq_deq8(codes.z, sc);
                *reinterpret_cast<uint4*>(dp + ((((g & 1) * 4 + 3) ^ (li & 7)) << 4)) = xq_deq8(codes.w, sc);
                store_b_chunk(smem_u32(dq + kXqDeqA + (et >> 7) * 2048), lut, (et >> 2) & 31, et & 3, sgn);
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(&dfull[d]);
            }
            // ------------------------------------------------------------ col phase of tile it - 1
            if (it >= 1) {
                const int jt = it - 1, d = jt & 1;
                const int64_t t = blockIdx.x + (int64_t)jt * gridDim.x;
                const int64_t r0 = (t % nRT) * 128, c0 = (t / nRT) * 128;
                mbar_wait_hint<1000>(&cdone[d], (jt >> 1) & 1);
                tc_fence_after();
                uint32_t raw[32];
                tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + 256 + d * 128 + 32 * g, raw);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&cfree[d]);
                float acc[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[j] = __uint_as_float(raw[j]);
                uint4 codes;
                int e;
                const int64_t orow = c0 + li, gk = r0 + 32 * g;
                bool ok = true;
                if (a.dbg & 2) {  // experiment: skip the RTN decisions (timing only)
                    codes = make_uint4(__float_as_uint(acc[0]), __float_as_uint(acc[9]), __float_as_uint(acc[17]),
                                       __float_as_uint(acc[31]));
                    e = 120;
                } else if (SRF) {
                    ok = srf_checked(acc, a.col_prescale, (uint32_t)a.key, (uint32_t)(a.key >> 32),
                                     a.ctr + (uint64_t)(orow * a.ld + gk), codes, e);
                } else {
                    ok = rtn_checked(acc, a.col_prescale, codes, e);
                }
                {
                    const uint32_t sw = a.sign_r && gk < a.R ? __ldg(a.sign_r + (gk >> 5)) : 0u;
                    for (uint32_t todo = __ballot_sync(0xffffffffu, !ok && orow < a.C && gk < a.R); todo;
                         todo &= todo - 1) {
                        const int f = __ffs(todo) - 1;
                        if (a.fallbacks && lane == 0) atomicAdd(a.fallbacks + 1, 1);
                        uint4 cx;
                        int ex;
                        const int64_t orf = c0 + quad * 32 + f;
                        exact_group_warp(smem + kXqOffDeq + d * kXqDeq, true, quad * 32 + f, g, sw, a.col_prescale,
                                         a.col_out.err, cx, ex, SRF, (uint32_t)a.key, (uint32_t)(a.key >> 32),
                                         a.ctr + (uint64_t)(orf * a.ld + gk));
                        if (lane == f) {
                            codes = cx;
                            e = ex;
                        }
                    }
                }
                if (orow < a.C && gk < a.R) {
                    *reinterpret_cast<uint4*>(a.col_out.codes + orow * a.col_out.ldc + (gk >> 5) * 16) = codes;
                    a.col_out.sf[sf_offset(orow, gk >> 5, a.col_out.katoms)] = (uint8_t)e;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&dfree[d]);
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// bf16 x [R, C]: X_q (QuEST of H32 rows, + trust mask) and X_t (RTN of the randomized-Hadamard transposed
// requantization, signs along R) in one pass, transforms on the tensor cores.
int launch_tcq_xq(const void* x, int64_t ldx, int64_t R, int64_t C, const QuantOut& row_out,
                  const uint32_t* col_sign_bits, float col_prescale, const QuantOut& col_out, int* fallbacks,
                  cudaStream_t st, const QuantCfg* srf_col) {
    if (R == 0 || C == 0) return 0;
    CUtensorMap m;
    const int rc = tq_map(&m, x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, R, C, ldx * 2);
    if (rc) return rc;
    static int attr_set[kMaxDevices];
    if (first_use_on_device(attr_set)) {
        cudaFuncSetAttribute(k_tcq_xq<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kXqBytes);
        cudaFuncSetAttribute(k_tcq_xq<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kXqBytes);
    }
    const int64_t sms = device_sms();
    XqArgs a{R, C, row_out, col_sign_bits, col_out, col_prescale, fallbacks, g_tcq_dbg, 0, 0, 0, R};
    if (srf_col) {
        a.srf = 1;
        a.key = srf_col->sr_base;
        a.ctr = srf_col->counter_start;
        a.ld = srf_col->counter_ld ? srf_col->counter_ld : R;
    }
    const int64_t tiles = ((R + 127) / 128) * ((C + 127) / 128);
    const unsigned grid = (unsigned)cap_grid(tiles < sms ? tiles : sms);
    if (a.srf)
        k_tcq_xq<true><<<grid, kXqThreads, kXqBytes, st>>>(m, a);
    else
        k_tcq_xq<false><<<grid, kXqThreads, kXqBytes, st>>>(m, a);
    return (int)cudaGetLastError();
}

}  // namespace qt
