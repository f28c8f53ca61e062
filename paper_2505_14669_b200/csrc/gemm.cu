// gemm.cu -- MXFP4 block-scaled GEMM on the 5th-gen tensor cores (tcgen05.mma kind::mxf4).
//
//   D[M, N] = deq(A)[M, K] * deq(B)[N, K]^T        (qlinear.gemm_lp, qlinear.py:96-111)
//
// Both operands are K-major MXFP4 operands (see common.cuh): packed E2M1 codes are staged by TMA
// into 128-byte-swizzled shared memory, the E8M0 scale atoms by bulk copies, then tcgen05.cp'd to
// TMEM next to the fp32 accumulator.  Warp roles (one CTA per SM):
//   warp 0     TMA producer (one elected lane)
//   warp 1     TMEM allocator + MMA issuer (one elected lane)
//   warps 2-5  epilogue: tcgen05.ld 32 lanes x 32 columns per thread-row, then
//                EPI_STORE      plain fp32 / bf16 store
//                EPI_MASK_H     trust-mask multiply, in-register FWHT-32 along N, x scale
//                EPI_MASK       trust-mask multiply, x scale (hadamard=False layers)
//                               (qlinear.py:229-230 / 249-250: dx = H(dx_q * m_x) * 16/9)
#include "common.cuh"
#include "launch.h"

namespace qt {

constexpr int kStages = 4;
constexpr int kBM = 128;
constexpr int kBKBytes = 128;  // 256 E2M1 values per K tile

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

template <int BN>
__global__ void __launch_bounds__(192, 1)
    k_gemm_mxf4(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const uint8_t* __restrict__ sfa, int64_t a_katoms, const uint8_t* __restrict__ sfb, int64_t b_katoms,
                int M, int N, int K, EpiParams ep) {
    using L = GemmSmem<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = sA + kStages * L::A;
    uint8_t* sSFA = sB + kStages * L::B;
    uint8_t* sSFB = sSFA + kStages * L::SFA;
    uint64_t* full = reinterpret_cast<uint64_t*>(sSFB + kStages * L::SFB);
    uint64_t* empty = full + kStages;
    uint64_t* tmem_full = empty + kStages;
    uint32_t* tmem_base_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * BN;
    const int nk = (K + 255) / 256;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
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
            for (int kt = 0; kt < nk; ++kt) {
                const int s = kt % kStages;
                const uint32_t ph = (kt / kStages) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], L::STAGE);
                tma_load_2d(sA + s * L::A, &tmA, &full[s], kt * kBKBytes, m0);
                tma_load_2d(sB + s * L::B, &tmB, &full[s], kt * kBKBytes, n0);
                bulk_load(sSFA + s * L::SFA, sfa + ((int64_t)(m0 / 128) * a_katoms + 2 * kt) * 512, 1024, &full[s]);
#pragma unroll
                for (int rb = 0; rb < BN / 128; ++rb)
                    bulk_load(sSFB + s * L::SFB + rb * 1024,
                              sfb + ((int64_t)(n0 / 128 + rb) * b_katoms + 2 * kt) * 512, 1024, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            for (int kt = 0; kt < nk; ++kt) {
                const int s = kt % kStages;
                const uint32_t ph = (kt / kStages) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                // scale factors -> TMEM (executes in order with the MMAs below)
                const uint32_t a_sf = smem_u32(sSFA + s * L::SFA), b_sf = smem_u32(sSFB + s * L::SFB);
                tmem_cp_sf(t_sfa + 0, make_sdesc(a_sf, 0, 128, kLayoutNone));
                tmem_cp_sf(t_sfa + 4, make_sdesc(a_sf + 512, 0, 128, kLayoutNone));
#pragma unroll
                for (int rb = 0; rb < BN / 128; ++rb) {
                    tmem_cp_sf(t_sfb + rb * 4, make_sdesc(b_sf + rb * 1024, 0, 128, kLayoutNone));
                    tmem_cp_sf(t_sfb + (BN / 128) * 4 + rb * 4, make_sdesc(b_sf + rb * 1024 + 512, 0, 128, kLayoutNone));
                }
                const uint32_t a_base = smem_u32(sA + s * L::A), b_base = smem_u32(sB + s * L::B);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
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
    } else {
        // epilogue warps 2..5 -> TMEM lane quadrant warp % 4
        const int quad = warp % 4;
        const int row = m0 + quad * 32 + lane;
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        for (int ch = 0; ch < BN / 32; ++ch) {
            const int col0 = n0 + ch * 32;
            if (col0 >= N) break;
            uint32_t r[32];
            tmem_ld32(t_acc + ((uint32_t)(quad * 32) << 16) + ch * 32, r);
            tmem_ld_wait();
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            if (row < M) {
                if (ep.mode != kEpiStore) {
                    uint32_t mw = __ldg(ep.mask + (int64_t)row * ep.ldm + col0 / 32);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = ((mw >> j) & 1u) ? v[j] : 0.0f;
                    if (ep.mode == kEpiMaskH) fwht32(v);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __fmul_rn(v[j], ep.scale);
                }
                if (ep.out_bf16) {
                    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(ep.out) + (int64_t)row * ep.ldo + col0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t w[4];
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            __nv_bfloat162 b2 = __floats2bfloat162_rn(v[q * 8 + 2 * t], v[q * 8 + 2 * t + 1]);
                            w[t] = *reinterpret_cast<uint32_t*>(&b2);
                        }
                        reinterpret_cast<uint4*>(o)[q] = make_uint4(w[0], w[1], w[2], w[3]);
                    }
                } else {
                    float* o = static_cast<float*>(ep.out) + (int64_t)row * ep.ldo + col0;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        reinterpret_cast<float4*>(o)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                }
            }
        }
        tc_fence_before();
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
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_gemm_mxf4<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES);
        attr_set = true;
    }
    dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + kBM - 1) / kBM));
    k_gemm_mxf4<BN><<<grid, 192, L::BYTES, st>>>(ta, tb, a_sf, a_katoms, b_sf, b_katoms, (int)M, (int)N, (int)K, ep);
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
