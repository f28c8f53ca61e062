// tcq.cu -- tensor-core Hadamard quantizer: the backward dy operands G and G_t on tcgen05.
//
//   G   = RTN(H32(dy (.) s_dout) * 0.75)  groups along d_out   (qlinear.py:214, 219, 225)
//   G_t = RTN(H32(dy^T (.) s_tok) * 0.75) groups along tokens  (qlinear.py:234, 239, 245)
//
// The reference's FWHT is an fp32 butterfly with a rounding after every add and multiply
// (_native.pyx:353-379); 10 roundings per element make it the dominant cost of a CUDA-core quantizer
// (5 FADD + 5 FMUL per element and pass).  Here the transform runs on the tensor cores as a GEMM with a
// +-1 Hadamard block whose rows carry the randomized-Hadamard signs (B = diag(s) H, bf16 exact), and the
// CUDA cores only quantize -- with a proof obligation:
//
//   |y_ref - y_tc| <= B = 20 u c^5 ||H (s.x)||_2        u = 2^-24, c = fp32(1/sqrt 2)
//     * reference butterfly vs exact real transform: <= gamma_10 c^5 sum|x| (10 u, induction over the
//       5 stages, every value bounded by the stage's absolute transform c^k sum|x|),
//     * tensor-core sum of 32 exact +-x products vs exact: measured <= 5.7 u sum|x| on adversarial inputs
//       (tools/ubench/tc_acc.py), budgeted at 8 u,
//     * the fp32 multiply by fl(c^5) and fl(0.75): 2 u,
//     * sum|x| <= sqrt(32) ||x||_2 = ||H x||_2 (H^T H = 32 I).
//   Each group's E8M0 exponent and every element's E2M1 code are decisions against fixed thresholds; the
//   epilogue encodes v - B_v and v + B_v and keeps the codes only if both agree (and the exponent is
//   stable under +-B).  Otherwise that one group is recomputed exactly on the CUDA cores from the bf16
//   tile still in shared memory (the v3 bit-exact path).  The result is bit-identical to the reference.
//
// Layout: persistent, one CTA per SM, 18 warps:
//   warp 0      TMA producer: dy tile (128 x 128 bf16, two 128B-swizzled boxes)
//   warp 1      TMEM allocator + MMA issuer (16 x tcgen05.mma kind::f16 M128 N32 K16 per tile)
//   warps 2-17  epilogue, two teams of 8 warps taking alternate tiles (TMEM buffer = team): TMEM ->
//               registers -> checked RTN -> codes / scales; 2 row groups + 2 column groups per thread and
//               tile.  Before releasing a stage a team writes the 8 signed Hadamard B blocks (row pass:
//               column signs, col pass: row signs) of the tile that will reuse it (4 x 16 B per thread)
#include "tcq.cuh"

namespace qt {

constexpr int kTqStages = 4;
constexpr int kTqEpiWarps = 16;           // two teams of 8, alternating tiles
constexpr int kTqTeam = 8;
constexpr int kTqThreads = 64 + 32 * kTqEpiWarps;
constexpr int kTqA = 32768;                  // two 64-column boxes of 128 rows
constexpr int kTqB = 8 * 2048;               // 8 Hadamard blocks, 32 x 32 bf16 each
constexpr int kTqStage = kTqA + kTqB;
constexpr int kTqLut = 256 * 16;             // sign byte -> 8 x bf16 (+-1)
constexpr int kTqBytes = kTqStages * kTqStage + kTqLut + 1024 /*align*/ + 256 /*barriers*/;

struct TqArgs {
    int64_t R, C;
    const uint32_t* sign_c;      // RHT signs along C (row operand G), bit c
    const uint32_t* sign_r;      // RHT signs along R (col operand G_t), bit r
    QuantOut row_out, col_out;   // G [R, C], G_t [C, R]
    float prescale;
    int* fallbacks;              // nullable: groups recomputed exactly
    int dbg;                     // experiment knobs (0 in production): 1 skip quantize, 2 skip B build, 4 skip TMEM ld, 8 skip stores
    // QT_ROUND_SR_FAST (srf != 0): keys and stream layout of the two operands (qt_quant_dual's positions:
    // G r*ld_r + c from ctr_r, G_t c*ld_c + r from ctr_c)
    int srf;
    uint64_t key_r, key_c, ctr_r, ctr_c;
    int64_t ld_r, ld_c;
};

// Four of the 1024 16-byte chunks of a tile's 8 signed Hadamard blocks (4 row-pass blocks from the column
// signs, 4 col-pass blocks from the row signs), built by team thread et (0..255):
//   chunk (blk, n, k8) = B_blk[n][8 k8 + i] = s_k H[k][n], i < 8, H[k][n] = (-1)^popc(k & n)
// stored K-major without swizzle: core matrix (n/8, k8) at ((n/8) * 4 + k8) * 128, row n % 8 at 16 B.
// blk = 2u + (et >> 7): the sign words are fetched by tq_sign_words ahead of use.
__device__ __forceinline__ void tq_sign_words(const TqArgs& a, int64_t t, int64_t nRT, int et, uint32_t (&sw)[4]) {
    const int64_t r0 = (t % nRT) * 128, c0 = (t / nRT) * 128;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int blk = 2 * u + (et >> 7);
        const int64_t pos = blk < 4 ? c0 + 32 * blk : r0 + 32 * (blk - 4);
        const int64_t lim = blk < 4 ? a.C : a.R;
        const uint32_t* sb = blk < 4 ? a.sign_c : a.sign_r;
        sw[u] = pos < lim ? __ldg(sb + (pos >> 5)) : 0u;
    }
}
__device__ __forceinline__ void build_b_chunks(uint32_t Bs, const uint8_t* lut, int et, const uint32_t (&sw)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int ch = et + 256 * u, blk = ch >> 7, n = (ch >> 2) & 31, k8 = ch & 3;
        store_b_chunk(Bs + blk * 2048, lut, n, k8, sw[u]);
    }
}

template <bool SRF>   // SRF: QT_ROUND_SR_FAST codes instead of checked RTN (its own instantiation: no cost for RTN)
__global__ void __launch_bounds__(kTqThreads, 1)
    k_tcq_dual(const __grid_constant__ CUtensorMap tmX, TqArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* lut = smem + kTqStages * kTqStage;
    uint64_t* full = reinterpret_cast<uint64_t*>(lut + kTqLut);
    uint64_t* empty = full + kTqStages;
    uint64_t* tmem_full = empty + kTqStages;
    uint64_t* tmem_empty = tmem_full + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t nRT = (a.R + 127) / 128, nCT = (a.C + 127) / 128, NT = nRT * nCT;

    build_sign_lut(lut);
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmX);
        for (int s = 0; s < kTqStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTqTeam);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tmem_full[b], 1);
            mbar_init(&tmem_empty[b], kTqTeam);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_holder, 512);
    __syncthreads();  // LUT ready
    if (warp >= 2) {  // B blocks of the first tiles: team (k & 1) owns stage k
        const int team = (warp - 2) >> 3, et = threadIdx.x - 64 - team * 256;
        for (int k = team; k < kTqStages; k += 2) {
            const int64_t t = blockIdx.x + (int64_t)k * gridDim.x;
            if (t < NT) {
                uint32_t sw[4];
                tq_sign_words(a, t, nRT, et, sw);
                build_b_chunks(smem_u32(smem + k * kTqStage + kTqA), lut, et, sw);
            }
        }
        fence_proxy_async();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;

    if (warp == 0) {
        // ------------------------------------------------------------------ producer
        int it = 0;
        for (int64_t t = blockIdx.x; t < NT; t += gridDim.x, ++it) {
            const int s = it % kTqStages;
            const uint32_t ph = (it / kTqStages) & 1;
            const int64_t r0 = (t % nRT) * 128, c0 = (t / nRT) * 128;
            mbar_wait_role(&empty[s], ph ^ 1);
            if (lane == 0) {
                mbar_arrive_expect_tx(&full[s], kTqA);
                uint8_t* As = smem + s * kTqStage;
                tma_load_2d(As, &tmX, &full[s], (int)c0, (int)r0);
                tma_load_2d(As + 16384, &tmX, &full[s], (int)c0 + 64, (int)r0);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t id_row = idesc_bf16(128, 32, 0), id_col = idesc_bf16(128, 32, 1);
            int it = 0;
            for (int64_t t = blockIdx.x; t < NT; t += gridDim.x, ++it) {
                const int s = it % kTqStages, b = it & 1;
                mbar_wait_role(&tmem_empty[b], ((it >> 1) & 1) ^ 1);
                mbar_wait_role(&full[s], (it / kTqStages) & 1);
                tc_fence_after();
                const uint32_t As = smem_u32(smem + s * kTqStage), Bs = As + kTqA;
                const uint32_t d0 = tmem + b * 256;
#pragma unroll
                for (int g = 0; g < 4; ++g) {
#pragma unroll
                    for (int ks = 0; ks < 2; ++ks) {
                        const uint64_t bd = make_sdesc(Bs + g * 2048 + ks * 256, 128, 512, kLayoutNone);
                        // row pass: A = tile rows, K = columns 32g + 16ks .. (K-major, 128B swizzle)
                        const uint64_t ad = make_sdesc(As + (g >> 1) * 16384 + (g & 1) * 64 + ks * 32, 16, 1024,
                                                       kLayoutSW128);
                        mma_bf16(d0 + 32 * g, ad, bd, id_row, ks);
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
#pragma unroll
                    for (int ks = 0; ks < 2; ++ks) {
                        const uint64_t bd = make_sdesc(Bs + (4 + q) * 2048 + ks * 256, 128, 512, kLayoutNone);
                        // col pass: A = tile^T, M = columns (MN-major: two 64-column boxes 16 KB apart),
                        // K = rows 32q + 16ks .. (8-row groups 1 KB apart)
                        const uint64_t ad = make_sdesc(As + (q * 32 + ks * 16) * 128, 16384, 1024, kLayoutSW128);
                        mma_bf16(d0 + 128 + 32 * q, ad, bd, id_col, ks);
                    }
                }
                tc_commit(&tmem_full[b]);
            }
        }
    } else {
        // ------------------------------------------------------------------ epilogue
        // team (warp - 2) / 8 takes the tiles with it % 2 == team (TMEM buffer b == team), so one team's
        // latency (TMEM loads, stores, barrier hand-offs) hides behind the other's arithmetic
        const int ew = warp - 2, team = ew >> 3, quad = warp & 3, half = (ew >> 2) & 1;
        const int et = ew * 32 + lane - team * 256;   // 0..255 within the team
        const int li = quad * 32 + lane;              // tile row (row pass) / column (col pass)
        int it = team;
        for (int64_t t = blockIdx.x + (int64_t)team * gridDim.x; t < NT; t += 2 * (int64_t)gridDim.x, it += 2) {
            const int s = it % kTqStages, b = team;
            const int64_t r0 = (t % nRT) * 128, c0 = (t / nRT) * 128;
            const int64_t tn = t + (int64_t)kTqStages * gridDim.x;   // next tile of this stage
            uint32_t sw[4];
            if (tn < NT) tq_sign_words(a, tn, nRT, et, sw);        // prefetch: used at the end of the tile
            mbar_wait_hint<1000>(&tmem_full[b], (it >> 1) & 1);
            tc_fence_after();
            const uint8_t* tile = smem + s * kTqStage;
            const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + b * 256;
#pragma unroll 1
            for (int pass = 0; pass < 2; ++pass) {   // 0: row groups of G, 1: column groups of G_t
                uint32_t r0w[32], r1w[32];
                const int g0 = 2 * half;
                tmem_ld32(tbase + pass * 128 + 32 * g0, r0w);
                tmem_ld32(tbase + pass * 128 + 32 * g0 + 32, r1w);
                tmem_ld_wait();
                if (pass == 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tmem_empty[b]);
                }
                if (a.dbg & 1) continue;
                float v0[32], v1[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    v0[j] = __uint_as_float(r0w[j]);
                    v1[j] = __uint_as_float(r1w[j]);
                }
                uint4 c0d, c1d;
                int e0, e1;
                const QuantOut& out = pass ? a.col_out : a.row_out;
                const int64_t orow = pass ? c0 + li : r0 + li;           // output row
                const int64_t kb = pass ? r0 : c0;                      // start of the grouped axis (mult. of 128)
                const uint64_t key = pass ? a.key_c : a.key_r;
                const uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
                // stream position of element 0 of group g0 of this output row
                const uint64_t pos0 = (pass ? a.ctr_c : a.ctr_r) + (uint64_t)(orow * (pass ? a.ld_c : a.ld_r) + kb + 32 * g0);
                bool ok0, ok1;
                if (SRF) {
                    ok0 = srf_checked(v0, a.prescale, k0, k1, pos0, c0d, e0);
                    ok1 = srf_checked(v1, a.prescale, k0, k1, pos0 + 32, c1d, e1);
                } else {
                    ok0 = rtn_checked(v0, a.prescale, c0d, e0);
                    ok1 = rtn_checked(v1, a.prescale, c1d, e1);
                }
                const int64_t lim_k = pass ? a.R : a.C;
                const bool in_row = orow < (pass ? a.C : a.R);
                // undecided groups (~0.1 %): the whole warp recomputes them exactly, one group at a time
                {
                    const uint32_t* sg = pass ? a.sign_r : a.sign_c;
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int64_t gk = kb + 32 * (g0 + u);
                        uint32_t todo = __ballot_sync(0xffffffffu, in_row && !(u ? ok1 : ok0) && gk < lim_k);
                        if (todo && a.fallbacks && lane == 0) atomicAdd(a.fallbacks, __popc(todo));
                        const uint32_t sw = todo && gk < lim_k ? __ldg(sg + (gk >> 5)) : 0u;
                        while (todo) {
                            const int f = __ffs(todo) - 1;
                            todo &= todo - 1;
                            uint4 cx;
                            int ex;
                            const uint64_t pf = SRF ? __shfl_sync(0xffffffffu, pos0, f) + 32 * u : 0;
                            exact_group_warp(tile, pass == 1, quad * 32 + f, g0 + u, sw, a.prescale, out.err, cx, ex,
                                             SRF, k0, k1, pf);
                            if (lane == f) {
                                if (u) {
                                    c1d = cx;
                                    e1 = ex;
                                } else {
                                    c0d = cx;
                                    e0 = ex;
                                }
                            }
                        }
                    }
                }
                if (in_row) {
                    uint8_t* cp = out.codes + orow * out.ldc + (kb >> 5) * 16 + g0 * 16;
                    // scale atom bytes of groups g0, g0 + 1 are adjacent: ((r/128) katoms + k/128) * 512 +
                    // (r % 32) * 16 + ((r / 32) % 4) * 4 + g
                    uint8_t* sp = out.sf + ((orow >> 7) * out.katoms + (kb >> 7)) * 512 + (orow & 31) * 16 +
                                  ((orow >> 5) & 3) * 4 + g0;
                    if ((a.dbg & 8) && orow != -12345) continue;  // timing only: no output stores
                    if (kb + 32 * g0 + 32 < lim_k) {
                        *reinterpret_cast<uint4*>(cp) = c0d;
                        *reinterpret_cast<uint4*>(cp + 16) = c1d;
                        *reinterpret_cast<uint16_t*>(sp) = (uint16_t)(e0 | (e1 << 8));
                    } else if (kb + 32 * g0 < lim_k) {
                        *reinterpret_cast<uint4*>(cp) = c0d;
                        *sp = (uint8_t)e0;
                    }
                }
            }
            // B blocks of the tile that reuses this stage, then release the stage
            if (tn < NT && !(a.dbg & 2)) build_b_chunks(smem_u32(smem + s * kTqStage + kTqA), lut, et, sw);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ---------------------------------------------------------------------------------- host
int g_tcq_dbg = 0;

// row_sign_bits: signs of the row operand (indexed by column), col_sign_bits: of the col operand (by row)
int launch_tcq_dual(const void* x, int64_t ldx, int64_t R, int64_t C, const uint32_t* row_sign_bits,
                    const uint32_t* col_sign_bits, float prescale, const QuantOut& row_out, const QuantOut& col_out,
                    int* fallbacks, cudaStream_t st, const QuantCfg* srf_row, const QuantCfg* srf_col) {
    if (R == 0 || C == 0) return 0;
    CUtensorMap m;
    const int rc = tq_map(&m, x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, R, C, ldx * 2);
    if (rc) return rc;
    static int attr_set[kMaxDevices];
    if (first_use_on_device(attr_set)) {
        cudaFuncSetAttribute(k_tcq_dual<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTqBytes);
        cudaFuncSetAttribute(k_tcq_dual<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTqBytes);
    }
    const int64_t sms = device_sms();
    TqArgs a{R, C, row_sign_bits, col_sign_bits, row_out, col_out, prescale, fallbacks, g_tcq_dbg, 0, 0, 0, 0, 0, C, R};
    if (srf_row && srf_col) {
        a.srf = 1;
        a.key_r = srf_row->sr_base;
        a.key_c = srf_col->sr_base;
        a.ctr_r = srf_row->counter_start;
        a.ctr_c = srf_col->counter_start;
        a.ld_r = srf_row->counter_ld ? srf_row->counter_ld : C;
        a.ld_c = srf_col->counter_ld ? srf_col->counter_ld : R;
    }
    const int64_t tiles = ((R + 127) / 128) * ((C + 127) / 128);
    const unsigned grid = (unsigned)cap_grid(tiles < sms ? tiles : sms);
    if (a.srf)
        k_tcq_dual<true><<<grid, kTqThreads, kTqBytes, st>>>(m, a);
    else
        k_tcq_dual<false><<<grid, kTqThreads, kTqBytes, st>>>(m, a);
    return (int)cudaGetLastError();
}

}  // namespace qt
