// gemm.cu -- MXFP4 block-scaled GEMM on the 5th-gen tensor cores (tcgen05.mma kind::mxf4).
//
//   D[M, N] = deq(A)[M, K] * deq(B)[N, K]^T        (qlinear.gemm_lp, qlinear.py:96-111)
//
// Both operands are K-major MXFP4 operands (see common.cuh): packed E2M1 codes are staged by TMA
// into 128-byte-swizzled shared memory, the E8M0 scale atoms by bulk copies, then tcgen05.cp'd to
// TMEM next to the fp32 accumulator.  Persistent, one CTA per SM; warp roles:
//   warp 0     TMA producer (one elected lane), runs ahead across tiles
//   warp 1     TMEM allocator + MMA issuer (one elected lane)
//   warps 2-9  epilogue: tcgen05.ld of the whole accumulator into registers (freeing TMEM for the
//              next tile at once), then per 64-column pair of chunks (packed f32x2):
//                EPI_STORE      plain fp32 / bf16 store
//                EPI_MASK_H     trust-mask multiply, in-register FWHT-32 along N, x scale
//                EPI_MASK       trust-mask multiply, x scale (hadamard=False layers)
//                               (qlinear.py:229-230 / 249-250: dx = H(dx_q * m_x) * 16/9)
#include "common.cuh"
#include "launch.h"
#include "quant.cuh"  // Pair / fwht_pair / scale_pair (bit-exact packed FWHT-32)

namespace qt {

constexpr int kStages = 4;
constexpr int kBM = 128;
constexpr int kBKBytes = 128;     // 256 E2M1 values per K tile
constexpr int kEpiWarps = 8;      // 2 warps per TMEM lane quadrant, each owning half the columns
constexpr int kThreads = 64 + 32 * kEpiWarps;

template <int BN>
struct GemmSmem {
    static constexpr int A = kBM * kBKBytes;
    static constexpr int B = BN * kBKBytes;
    static constexpr int SFA = 1024;
    static constexpr int SFB = (BN / 128) * 1024;
    static constexpr int STAGE = A + B + SFA + SFB;
    static constexpr int BYTES = kStages * STAGE + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int TMEM_COLS = BN == 256 ? 512 : 256;
};

// Persistent tcgen05 GEMM: one CTA per SM walks tiles blockIdx.x, blockIdx.x + gridDim.x, ...
// The TMA producer runs ahead across tile boundaries (its ring never drains), the MMA warp starts
// tile i+1 as soon as the epilogue warps have copied tile i's accumulator out of TMEM into
// registers, and the epilogue math + stores of tile i overlap the mainloop of tile i+1.
template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_mxf4(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const uint8_t* __restrict__ sfa, int64_t a_katoms, const uint8_t* __restrict__ sfb, int64_t b_katoms,
                int M, int N, int K, EpiParams ep) {
    using L = GemmSmem<BN>;
    constexpr int CW = BN / 2;            // columns per epilogue thread
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = sA + kStages * L::A;
    uint8_t* sSFA = sB + kStages * L::B;
    uint8_t* sSFB = sSFA + kStages * L::SFA;
    uint64_t* full = reinterpret_cast<uint64_t*>(sSFB + kStages * L::SFB);
    uint64_t* empty = full + kStages;
    uint64_t* tmem_full = empty + kStages;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_base_holder = reinterpret_cast<uint32_t*>(tmem_empty + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nk = (K + 255) / 256;
    const int tiles_n = (N + BN - 1) / BN, tiles = ((M + kBM - 1) / kBM) * tiles_n;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, kEpiWarps);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_base_holder, L::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_base_holder;
    const uint32_t t_acc = tmem, t_sfa = tmem + BN, t_sfb = tmem + BN + 8;

    if (warp == 0) {
        if (lane == 0) {
            int it = 0;
            for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
                const int m0 = (tile / tiles_n) * kBM, n0 = (tile % tiles_n) * BN;
                for (int kt = 0; kt < nk; ++kt, ++it) {
                    const int s = it % kStages;
                    const uint32_t ph = (it / kStages) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    const bool skip_sf = (ep.dbg & 2) && kt > 0;
                    const bool skip_b = (ep.dbg & 8) && kt > 0;
                    mbar_arrive_expect_tx(&full[s], L::STAGE - (skip_sf ? L::SFA + L::SFB : 0) - (skip_b ? L::B : 0));
                    tma_load_2d(sA + s * L::A, &tmA, &full[s], kt * kBKBytes, m0);
                    if (!skip_b) tma_load_2d(sB + s * L::B, &tmB, &full[s], kt * kBKBytes, n0);
                    if (!skip_sf) {
                        bulk_load(sSFA + s * L::SFA, sfa + ((int64_t)(m0 / 128) * a_katoms + 2 * kt) * 512, 1024,
                                  &full[s]);
#pragma unroll
                        for (int rb = 0; rb < BN / 128; ++rb)
                            bulk_load(sSFB + s * L::SFB + rb * 1024,
                                      sfb + ((int64_t)(n0 / 128 + rb) * b_katoms + 2 * kt) * 512, 1024, &full[s]);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int it = 0, tcount = 0;
            for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tcount) {
                mbar_wait(tmem_empty, (tcount & 1) ^ 1);  // epilogue has drained the accumulator
                tc_fence_after();
                for (int kt = 0; kt < nk; ++kt, ++it) {
                    const int s = it % kStages;
                    const uint32_t ph = (it / kStages) & 1;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    // scale factors -> TMEM (executes in order with the MMAs below)
                    const uint32_t a_sf = smem_u32(sSFA + s * L::SFA), b_sf = smem_u32(sSFB + s * L::SFB);
                    if (!((ep.dbg & 1) && kt > 0)) {
                    tmem_cp_sf(t_sfa + 0, make_sdesc(a_sf, 0, 128, kLayoutNone));
                    tmem_cp_sf(t_sfa + 4, make_sdesc(a_sf + 512, 0, 128, kLayoutNone));
#pragma unroll
                    for (int rb = 0; rb < BN / 128; ++rb) {
                        tmem_cp_sf(t_sfb + rb * 4, make_sdesc(b_sf + rb * 1024, 0, 128, kLayoutNone));
                        tmem_cp_sf(t_sfb + (BN / 128) * 4 + rb * 4,
                                   make_sdesc(b_sf + rb * 1024 + 512, 0, 128, kLayoutNone));
                    }
                    }
                    const uint32_t a_base = smem_u32(sA + s * L::A), b_base = smem_u32(sB + s * L::B);
                    const int nmma = (ep.dbg & 4) ? 1 : 4;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (j >= nmma) break;
                        const uint64_t ad = make_sdesc(a_base + j * 32, 0, 1024, kLayoutSW128);
                        const uint64_t bd = make_sdesc(b_base + j * 32, 0, 1024, kLayoutSW128);
                        const uint32_t id = idesc_mxf4(kBM, BN, (j & 1) * 2, (j & 1) * 2);
                        mma_mxf4(t_acc, ad, bd, id, t_sfa + (j >> 1) * 4, t_sfb + (j >> 1) * (BN / 128) * 4,
                                 (kt | j) != 0 ? 1u : 0u);
                    }
                    tc_commit(&empty[s]);
                }
                tc_commit(tmem_full);
            }
        }
    } else {
        // epilogue warps 2..9: TMEM lane quadrant warp % 4, column half (warp - 2) / 4
        const int quad = warp % 4, half = (warp - 2) / 4;
        const float2 nz = opaque_nz2();
        int tcount = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tcount) {
            const int m0 = (tile / tiles_n) * kBM, n0 = (tile % tiles_n) * BN;
            const int row = m0 + quad * 32 + lane, cbase = n0 + half * CW;
            mbar_wait(tmem_full, tcount & 1);
            tc_fence_after();
            uint32_t acc[CW / 32][32];
#pragma unroll
            for (int c = 0; c < CW / 32; ++c)
                tmem_ld32(t_acc + ((uint32_t)(quad * 32) << 16) + half * CW + c * 32, acc[c]);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tmem_empty);  // the MMA warp may start the next tile now
            if (row >= M) continue;
#pragma unroll
            for (int pj = 0; pj < CW / 64; ++pj) {
                const int col0 = cbase + pj * 64;  // columns col0 .. col0+63: chunk A, chunk B
                if (col0 >= N) break;
                const bool okB = col0 + 32 < N;
                Pair g;
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    g.p[i] = make_float2(__uint_as_float(acc[2 * pj][i]), __uint_as_float(acc[2 * pj + 1][i]));
                if (ep.mode != kEpiStore) {
                    const uint32_t mA = __ldg(ep.mask + (int64_t)row * ep.ldm + col0 / 32);
                    const uint32_t mB = okB ? __ldg(ep.mask + (int64_t)row * ep.ldm + col0 / 32 + 1) : 0u;
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        g.p[i].x = ((mA >> i) & 1u) ? g.p[i].x : 0.0f;
                        g.p[i].y = ((mB >> i) & 1u) ? g.p[i].y : 0.0f;
                    }
                    if (ep.mode == kEpiMaskH) fwht_pair(g, nz);
                    scale_pair(g, ep.scale);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (h == 1 && !okB) break;
                    const int col = col0 + 32 * h;
                    if (ep.out_bf16) {
                        uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) +
                                                            (int64_t)row * ep.ldo + col);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            uint32_t w[4];
#pragma unroll
                            for (int t = 0; t < 4; ++t) {
                                const int i = q * 8 + 2 * t;
                                __nv_bfloat162 b2 = h ? __floats2bfloat162_rn(g.p[i].y, g.p[i + 1].y)
                                                      : __floats2bfloat162_rn(g.p[i].x, g.p[i + 1].x);
                                w[t] = *reinterpret_cast<uint32_t*>(&b2);
                            }
                            o[q] = make_uint4(w[0], w[1], w[2], w[3]);
                        }
                    } else {
                        float4* o = reinterpret_cast<float4*>(static_cast<float*>(ep.out) + (int64_t)row * ep.ldo + col);
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const int i = 4 * q;
                            o[q] = h ? make_float4(g.p[i].y, g.p[i + 1].y, g.p[i + 2].y, g.p[i + 3].y)
                                     : make_float4(g.p[i].x, g.p[i + 1].x, g.p[i + 2].x, g.p[i + 3].x);
                        }
                    }
                }
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, L::TMEM_COLS);
    }
}

// ---------------------------------------------------------------------------- host side

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    return fn;
}

// 2-D byte tensor [rows, cols_bytes] with row stride ld_bytes; box = 128 bytes x box_rows, 128B swizzle.
static int make_codes_map(CUtensorMap* m, const uint8_t* base, int64_t rows, int64_t cols_bytes, int64_t ld_bytes,
                          int box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return 1001;
    cuuint64_t dims[2] = {(cuuint64_t)cols_bytes, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld_bytes};
    cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : 1002;
}

template <int BN>
static int launch_gemm_bn(const uint8_t* a, int64_t lda, const uint8_t* a_sf, int64_t a_katoms, const uint8_t* b,
                          int64_t ldb, const uint8_t* b_sf, int64_t b_katoms, int64_t M, int64_t N, int64_t K,
                          const EpiParams& ep, cudaStream_t st) {
    using L = GemmSmem<BN>;
    CUtensorMap ta, tb;
    int rc = make_codes_map(&ta, a, M, K / 2, lda, kBM);
    if (rc) return rc;
    rc = make_codes_map(&tb, b, N, K / 2, ldb, BN);
    if (rc) return rc;
    static int sms = 0;
    if (!sms) {
        cudaFuncSetAttribute(k_gemm_mxf4<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t tiles = ((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
    const unsigned grid = (unsigned)(tiles < sms ? tiles : sms);
    k_gemm_mxf4<BN><<<grid, kThreads, L::BYTES, st>>>(ta, tb, a_sf, a_katoms, b_sf, b_katoms, (int)M, (int)N, (int)K,
                                                      ep);
    return (int)cudaGetLastError();
}

int launch_gemm(const uint8_t* a, int64_t lda, const uint8_t* a_sf, int64_t a_katoms, const uint8_t* b, int64_t ldb,
                const uint8_t* b_sf, int64_t b_katoms, int64_t M, int64_t N, int64_t K, const EpiParams& ep,
                cudaStream_t st) {
    if (M == 0 || N == 0) return 0;
    if (N >= 256 && N % 256 == 0)
        return launch_gemm_bn<256>(a, lda, a_sf, a_katoms, b, ldb, b_sf, b_katoms, M, N, K, ep, st);
    return launch_gemm_bn<128>(a, lda, a_sf, a_katoms, b, ldb, b_sf, b_katoms, M, N, K, ep, st);
}

}  // namespace qt
