// tcq_fwd.cu -- fused forward quantizer with the transposed requantization on the tensor cores.
//
//   X_q, M_x = QuEST(H32(x))                      row pass, CUDA cores (bit-exact butterfly + search)
//   X_t      = RTN(H32(deq(X_q)^T (.) s) * 0.75)  col pass, tensor cores + checked RTN (tcq.cu proof)
//   (qlinear.py:139-157 and 206-207, 215, 235; same for W -> W_q, M_w, W_t)
//
// One read of x per tile: TMA brings the 128 x 128 tile (bf16: two 64-column boxes, fp32: four
// 32-column boxes, 128-byte swizzle); the row warps quantize it (QuEST / RTN / SR of qgroup.cuh),
// store X_q / M_x, and write deq(X_q) as an exact bf16 tile plus the 4 signed Hadamard blocks of the
// tile's token groups into a shared-memory buffer; the MMA warp multiplies deq(X_q)^T by those blocks
// (8 x tcgen05.mma kind::f16 M128 N32 K16, the deq tile read MN-major); the col warps quantize the
// TMEM result with the checked RTN and recompute a group exactly from the deq tile if a decision is
// within the error bound.
//
// Warps: 0-15 row pass (one group per thread: the QuEST row pass is the issue-bound part and gets the
// warps), 16-19 col epilogue (one TMEM lane quadrant each, 4 groups per thread), 20 control: TMEM
// allocator, lane 0 TMA producer, lane 1 MMA issuer (independent-thread-scheduled lanes).
#include "tcq.cuh"

namespace qt {

constexpr int kFwRowWarps = 16, kFwColWarps = 4;
constexpr int kFwCtl = kFwRowWarps + kFwColWarps;     // control warp index
constexpr int kFwThreads = 32 * (kFwCtl + 1);

template <int IN>
struct FwGeom {
    static constexpr int ESZ = IN == kInF32 ? 4 : 2;
    static constexpr int IN_BYTES = 128 * 128 * ESZ;
    static constexpr int NBOX = 128 * ESZ / 128;                 // 128-byte boxes per tile row
    static constexpr int DEQ_A = 32768, DEQ = DEQ_A + 4 * 2048;  // deq tile + 4 signed H blocks
    static constexpr int STAGES = IN == kInF32 ? 2 : 3;
    static constexpr int OFF_DEQ = STAGES * IN_BYTES;
    static constexpr int OFF_LUT = OFF_DEQ + 2 * DEQ;
    static constexpr int OFF_BAR = OFF_LUT + 4096;
    static constexpr int BYTES = OFF_BAR + 256 + 1024;
};

struct FwArgs {
    int64_t R, C;
    QuantCfg rc;              // row pass (transform H, QuEST / RTN / SR)
    QuantOut row_out;         // X_q [R, C] (+ mask)
    const uint32_t* sign_r;   // RHT signs along R (the col operand's contraction axis)
    QuantOut col_out;         // X_t [C, R]
    float col_prescale;
    int* fallbacks;
    int dbg;   // experiment knobs (0 in production): 1 col epilogue skips the quantization
};

// group g of tile row r, transform stage 1 fused into the load (SWIZZLE_128B TMA layout)
template <int IN>
__device__ __forceinline__ void fw_load_row(const uint8_t* tile, int r, int g, int transform, float (&v)[32]) {
    if (IN == kInBF16) {
        const uint8_t* rowp = tile + (g >> 1) * 16384 + r * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 c = *reinterpret_cast<const uint4*>(rowp + ((((g & 1) * 4 + q) ^ (r & 7)) << 4));
            const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int j = q * 8 + 2 * t;
                if (transform != kNone) {
                    const float hi = bf_hi(w[t]);
                    v[j] = __fmul_rn(fh_add_lo(w[t], hi), kHc);
                    v[j + 1] = __fmul_rn(fh_sub_lo(w[t], hi), kHc);
                } else {
                    v[j] = bf_lo(w[t]);
                    v[j + 1] = bf_hi(w[t]);
                }
            }
        }
        if (transform != kNone) fwht_tail(v);
    } else {
        const uint8_t* rowp = tile + g * 16384 + r * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float4 c = *reinterpret_cast<const float4*>(rowp + ((q ^ (r & 7)) << 4));
            v[4 * q] = c.x;
            v[4 * q + 1] = c.y;
            v[4 * q + 2] = c.z;
            v[4 * q + 3] = c.w;
        }
        if (transform != kNone) fwht_full(v);
    }
}

// exact bf16 of code * 2^(e-127) for the 8 nibbles of a codes word (element 2k in the low nibble)
__device__ __forceinline__ uint4 deq8_bf16(uint32_t w, float s) {
    uint32_t o[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const float2 f = e2m1x2_to_f32((w >> (8 * b)) & 0xFFu);
        __nv_bfloat162 h = __floats2bfloat162_rn(__fmul_rn(f.x, s), __fmul_rn(f.y, s));
        o[b] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

template <int IN, int ROW>
__global__ void __launch_bounds__(kFwThreads, 1) k_tcq_fwd(const __grid_constant__ CUtensorMap tmX, FwArgs a) {
    using G = FwGeom<IN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* lut = smem + G::OFF_LUT;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
    uint64_t* empty = full + 3;
    uint64_t* deq_full = empty + 3;
    uint64_t* deq_empty = deq_full + 2;
    uint64_t* tmem_full = deq_empty + 2;
    uint64_t* tmem_empty = tmem_full + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t nRT = (a.R + 127) / 128, nCT = (a.C + 127) / 128, NT = nRT * nCT;

    build_sign_lut(lut);
    if (warp == kFwCtl && lane == 0) {
        tma_prefetch(&tmX);
        for (int i = 0; i < G::STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kFwRowWarps);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&deq_full[i], kFwRowWarps);
            mbar_init(&deq_empty[i], kFwColWarps);
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], kFwColWarps);
        }
        fence_barrier_init();
    }
    if (warp == kFwCtl) tmem_alloc(tmem_holder, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;

    if (warp == kFwCtl) {
        if (lane == 0) {
            // ------------------------------------------------------------ TMA producer
            int it = 0;
            for (int64_t t = blockIdx.x; t < NT; t += gridDim.x, ++it) {
                const int s = it % G::STAGES;
                const int64_t r0 = (t % nRT) * 128, c0 = (t / nRT) * 128;
                mbar_wait_hint<1000>(&empty[s], ((it / G::STAGES) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], G::IN_BYTES);
#pragma unroll
                for (int b = 0; b < G::NBOX; ++b)
                    tma_load_2d(smem + s * G::IN_BYTES + b * 16384, &tmX, &full[s], (int)c0 + b * (128 / G::ESZ),
                                (int)r0);
            }
        } else if (lane == 1) {
            // ------------------------------------------------------------ MMA issuer
            constexpr uint32_t id_col = idesc_bf16(128, 32, 1);
            int it = 0;
            for (int64_t t = blockIdx.x; t < NT; t += gridDim.x, ++it) {
                const int d = it & 1;
                mbar_wait_hint<1000>(&tmem_empty[d], ((it >> 1) & 1) ^ 1);
                mbar_wait_hint<1000>(&deq_full[d], (it >> 1) & 1);
                tc_fence_after();
                const uint32_t As = smem_u32(smem + G::OFF_DEQ + d * G::DEQ), Bs = As + G::DEQ_A;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
#pragma unroll
                    for (int ks = 0; ks < 2; ++ks) {
                        const uint64_t bd = make_sdesc(Bs + q * 2048 + ks * 256, 128, 512, kLayoutNone);
                        const uint64_t ad = make_sdesc(As + (q * 32 + ks * 16) * 128, 16384, 1024, kLayoutSW128);
                        mma_bf16(tmem + d * 128 + 32 * q, ad, bd, id_col, ks);
                    }
                }
                tc_commit(&tmem_full[d]);
            }
        }
    } else if (warp < kFwRowWarps) {
        // ---------------------------------------------------------------- row pass (CUDA cores)
        const int rt = threadIdx.x;                // 0..511
        const int rr = rt >> 2, g = rt & 3;        // tile row, group (4 per row)
        int it = 0;
        for (int64_t t = blockIdx.x; t < NT; t += gridDim.x, ++it) {
            const int s = it % G::STAGES, d = it & 1;
            const int64_t r0 = (t % nRT) * 128, c0 = (t / nRT) * 128;
            const int nr = (int)(a.R - r0 < 128 ? a.R - r0 : 128), nc = (int)(a.C - c0 < 128 ? a.C - c0 : 128);
            mbar_wait_hint<1000>(&deq_empty[d], ((it >> 1) & 1) ^ 1);
            mbar_wait_hint<1000>(&full[s], (it / G::STAGES) & 1);
            const uint8_t* tile = smem + s * G::IN_BYTES;
            uint8_t* dq = smem + G::OFF_DEQ + d * G::DEQ;
            const int64_t row = r0 + rr, gg = c0 / 32 + g;
            uint4 codes = make_uint4(0, 0, 0, 0);
            int e = 0;
            if (rr < nr && g * 32 < nc) {
                float v[32];
                fw_load_row<IN>(tile, rr, g, a.rc.transform, v);
                const int64_t cld = a.rc.counter_ld ? a.rc.counter_ld : a.C;
                uint32_t mask;
                e = quant_group<ROW>(v, a.rc, a.rc.counter_start + (uint64_t)(row * cld + gg * 32), a.row_out.err,
                                     a.row_out.fallbacks, codes, mask);
                *reinterpret_cast<uint4*>(a.row_out.codes + row * a.row_out.ldc + gg * 16) = codes;
                if (a.row_out.mask) a.row_out.mask[row * (a.C / 32) + gg] = mask;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);  // input stage consumed
            // the 4 scale bytes of this tile row form one atom word (lanes 4k .. 4k+3)
            uint32_t sfw = (uint32_t)e << (8 * g);
            sfw |= __shfl_xor_sync(0xffffffffu, sfw, 1);
            sfw |= __shfl_xor_sync(0xffffffffu, sfw, 2);
            if (g == 0 && rr < nr) {
                uint8_t* sp = a.row_out.sf + sf_offset(row, c0 / 32, a.row_out.katoms);
                if (nc == 128)
                    *reinterpret_cast<uint32_t*>(sp) = sfw;
                else
                    for (int j = 0; j * 32 < nc; ++j) sp[j] = (uint8_t)(sfw >> (8 * j));
            }
            // deq(X_q) tile (bf16, the MMA's MN-major A operand) + the 4 signed Hadamard blocks
            const float sc = exp2i(e - 127);
            uint8_t* dp = dq + (g >> 1) * 16384 + rr * 128;
            *reinterpret_cast<uint4*>(dp + ((((g & 1) * 4 + 0) ^ (rr & 7)) << 4)) = deq8_bf16(codes.x, sc);
            *reinterpret_cast<uint4*>(dp + ((((g & 1) * 4 + 1) ^ (rr & 7)) << 4)) = deq8_bf16(codes.y, sc);
            *reinterpret_cast<uint4*>(dp + ((((g & 1) * 4 + 2) ^ (rr & 7)) << 4)) = deq8_bf16(codes.z, sc);
            *reinterpret_cast<uint4*>(dp + ((((g & 1) * 4 + 3) ^ (rr & 7)) << 4)) = deq8_bf16(codes.w, sc);
            {
                const int blk = rt >> 7, n = (rt >> 2) & 31, k8 = rt & 3;
                const int64_t pos = r0 + 32 * blk;
                const uint32_t sgn = (a.sign_r && pos < a.R) ? __ldg(a.sign_r + (pos >> 5)) : 0u;
                store_b_chunk(smem_u32(dq + G::DEQ_A + blk * 2048), lut, n, k8, sgn);
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&deq_full[d]);
        }
    } else {
        // ---------------------------------------------------------------- col epilogue
        const int quad = warp & 3;
        const int lc = quad * 32 + lane;  // tile column = output row of X_t
        int it = 0;
        for (int64_t t = blockIdx.x; t < NT; t += gridDim.x, ++it) {
            const int d = it & 1;
            const int64_t r0 = (t % nRT) * 128, c0 = (t / nRT) * 128;
            mbar_wait_hint<1000>(&tmem_full[d], (it >> 1) & 1);
            tc_fence_after();
            const uint8_t* dq = smem + G::OFF_DEQ + d * G::DEQ;
            const int64_t orow = c0 + lc;
            uint32_t sfw = 0;
#pragma unroll 1
            for (int hp = 0; hp < 2; ++hp) {
                uint32_t r0w[32], r1w[32];
                const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + d * 128 + 64 * hp;
                tmem_ld32(ta, r0w);
                tmem_ld32(ta + 32, r1w);
                tmem_ld_wait();
                if (hp == 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tmem_empty[d]);
                }
                if (a.dbg & 1) {
                    if (r0w[5] == 0x7fc00001u && r1w[9] == 0x7fc00001u) a.col_out.codes[0] = 1;
                    continue;
                }
                float v0[32], v1[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    v0[j] = __uint_as_float(r0w[j]);
                    v1[j] = __uint_as_float(r1w[j]);
                }
                uint4 cA, cB;
                int eA, eB;
                const bool okA = rtn_checked(v0, a.col_prescale, cA, eA);
                const bool okB = rtn_checked(v1, a.col_prescale, cB, eB);
                if (orow < a.C) {
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int q = 2 * hp + u;
                        const int64_t gk = r0 + 32 * q;
                        if (gk >= a.R) continue;
                        uint4& cc = u ? cB : cA;
                        int& ee = u ? eB : eA;
                        if (!(u ? okB : okA)) {
                            if (a.fallbacks) atomicAdd(a.fallbacks, 1);
                            exact_group(dq, true, lc, q, a.sign_r ? __ldg(a.sign_r + (gk >> 5)) : 0u, a.col_prescale,
                                        a.col_out.err, cc, ee);
                        }
                        *reinterpret_cast<uint4*>(a.col_out.codes + orow * a.col_out.ldc + (gk >> 5) * 16) = cc;
                        sfw |= (uint32_t)ee << (8 * q);
                    }
                }
            }
            if (orow < a.C) {
                uint8_t* sp = a.col_out.sf + sf_offset(orow, r0 / 32, a.col_out.katoms);
                const int ng = (int)((a.R - r0) >= 128 ? 4 : (a.R - r0 + 31) / 32);
                if (ng == 4)
                    *reinterpret_cast<uint32_t*>(sp) = sfw;
                else
                    for (int j = 0; j < ng; ++j) sp[j] = (uint8_t)(sfw >> (8 * j));
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&deq_empty[d]);
        }
    }
    __syncthreads();
    if (warp == kFwCtl) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

template <int IN, int ROW>
static int fw_launch(const CUtensorMap& m, const FwArgs& a, cudaStream_t st) {
    using G = FwGeom<IN>;
    auto fn = k_tcq_fwd<IN, ROW>;
    static int sms = 0;
    if (!sms) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, G::BYTES);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t tiles = ((a.R + 127) / 128) * ((a.C + 127) / 128);
    fn<<<(unsigned)(tiles < sms ? tiles : sms), kFwThreads, G::BYTES, st>>>(m, a);
    return (int)cudaGetLastError();
}

// Fused forward on the tensor-core path: row pass (QuEST / RTN / SR, transform H or none) of x [R, C] and
// the RTN, randomized-Hadamard transposed requantization of its result.
int launch_tcq_fwd(const void* x, int in_type, int64_t ldx, int64_t R, int64_t C, const QuantCfg& rc,
                   const QuantOut& row_out, const uint32_t* col_sign_bits, float col_prescale, const QuantOut& col_out,
                   int* fallbacks, cudaStream_t st) {
    if (R == 0 || C == 0) return 0;
    CUtensorMap m;
    const int esz = in_type == kInF32 ? 4 : 2;
    int r = tq_map(&m, x, in_type == kInF32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, esz,
                   R, C, ldx * esz);
    if (r) return r;
    FwArgs a{R, C, rc, row_out, col_sign_bits, col_out, col_prescale, fallbacks, g_tcq_dbg};
    if (in_type == kInF32) {
        if (rc.rounding == kQuest) return fw_launch<kInF32, kQuest>(m, a, st);
        if (rc.rounding == kRtn) return fw_launch<kInF32, kRtn>(m, a, st);
        return fw_launch<kInF32, kSr>(m, a, st);
    }
    if (rc.rounding == kQuest) return fw_launch<kInBF16, kQuest>(m, a, st);
    if (rc.rounding == kRtn) return fw_launch<kInBF16, kRtn>(m, a, st);
    return fw_launch<kInBF16, kSr>(m, a, st);
}

}  // namespace qt
