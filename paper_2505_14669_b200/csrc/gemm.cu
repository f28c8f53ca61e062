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
#include <algorithm>

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

// Grouped tile rasterization: consecutive tile indices walk GROUP_M row blocks before moving to the next
// column block, so the ~148 tiles in flight share a few A slabs and a few dozen B slabs (L2 reuse instead of
// re-streaming B from HBM for every row block; e.g. the 4096 x 11008 x 16384 dW GEMM read 1 GB of DRAM
// with the plain row-major walk).
// Used for long-K GEMMs (the dW products, K = tokens) where the slabs are large; short-K GEMMs keep the
// row-major walk (group_m = 0), which measured faster there.
__device__ __forceinline__ void tile_mn(int tile, int tiles_m, int tiles_n, int& mb, int& nb, int kGroupM = 8) {
    if (kGroupM == 0) {
        mb = tile / tiles_n;
        nb = tile % tiles_n;
        return;
    }
    const int per_group = kGroupM * tiles_n;
    const int g = tile / per_group, first = g * kGroupM;
    const int gsize = tiles_m - first < kGroupM ? tiles_m - first : kGroupM;
    const int r = tile - g * per_group;
    mb = first + r % gsize;
    nb = r / gsize;
}

// Epilogue of one accumulator row slice: columns cbase .. cbase + CW - 1 of output row `row`, held as
// CW/32 chunks of 32 fp32 values (tcgen05.ld 32x32b); per 64-column pair of chunks (packed f32x2):
// mask multiply, bit-exact FWHT-32 along N, scale, bf16 / fp32 store.
template <int CW>
__device__ __forceinline__ void epi_store(const uint32_t (&acc)[CW / 32][32], int row, int cbase, int N,
                                          const EpiParams& ep, float2 nz) {
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
                uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) + (int64_t)row * ep.ldo + col);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint32_t w[4];
                    uint4 old = ep.accumulate ? o[q] : make_uint4(0, 0, 0, 0);
                    const uint32_t* ow = reinterpret_cast<const uint32_t*>(&old);
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int i = q * 8 + 2 * t;
                        __nv_bfloat162 b2 = h ? __floats2bfloat162_rn(g.p[i].y, g.p[i + 1].y)
                                              : __floats2bfloat162_rn(g.p[i].x, g.p[i + 1].x);
                        if (ep.accumulate) {  // bf16(old + bf16(new)), as out.add_(tmp) in bf16
                            const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ow[t]));
                            const float2 b = __bfloat1622float2(b2);
                            b2 = __floats2bfloat162_rn(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
                        }
                        w[t] = *reinterpret_cast<uint32_t*>(&b2);
                    }
                    o[q] = make_uint4(w[0], w[1], w[2], w[3]);
                }
            } else {
                float4* o = reinterpret_cast<float4*>(static_cast<float*>(ep.out) + (int64_t)row * ep.ldo + col);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int i = 4 * q;
                    float4 v = h ? make_float4(g.p[i].y, g.p[i + 1].y, g.p[i + 2].y, g.p[i + 3].y)
                                 : make_float4(g.p[i].x, g.p[i + 1].x, g.p[i + 2].x, g.p[i + 3].x);
                    if (ep.accumulate) {
                        const float4 a = o[q];
                        v = make_float4(__fadd_rn(a.x, v.x), __fadd_rn(a.y, v.y), __fadd_rn(a.z, v.z),
                                        __fadd_rn(a.w, v.w));
                    }
                    o[q] = v;
                }
            }
        }
    }
}

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
    const int tiles_n = (N + BN - 1) / BN, tiles_m = (M + kBM - 1) / kBM, tiles = tiles_m * tiles_n;

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
        // TMA producer: like the MMA issuer, the whole warp walks the loop (uniform operands) and one elected
        // lane issues the copies
        uint32_t s = 0, ph = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            int mb, nb;
            tile_mn(tile, tiles_m, tiles_n, mb, nb, K >= 8192 ? 8 : 0);
            const int m0 = mb * kBM, n0 = nb * BN;
            const uint8_t* sfa_t = sfa + (int64_t)(m0 / 128) * a_katoms * 512;
            const uint8_t* sfb_t = sfb + (int64_t)(n0 / 128) * b_katoms * 512;
            for (int kt = 0; kt < nk; ++kt) {
                mbar_wait(&empty[s], ph ^ 1);
                const bool skip_sf = (ep.dbg & 2) && kt > 0;
                const bool skip_b = (ep.dbg & 8) && kt > 0;
                if (elect_one()) {
                    mbar_arrive_expect_tx(&full[s], L::STAGE - (skip_sf ? L::SFA + L::SFB : 0) - (skip_b ? L::B : 0));
                    tma_load_2d(sA + s * L::A, &tmA, &full[s], kt * kBKBytes, m0);
                    if (!skip_b) tma_load_2d(sB + s * L::B, &tmB, &full[s], kt * kBKBytes, n0);
                    if (!skip_sf) {
                        bulk_load(sSFA + s * L::SFA, sfa_t + kt * 1024, 1024, &full[s]);
#pragma unroll
                        for (int rb = 0; rb < BN / 128; ++rb)
                            bulk_load(sSFB + s * L::SFB + rb * 1024, sfb_t + (int64_t)rb * b_katoms * 512 + kt * 1024,
                                      1024, &full[s]);
                    }
                }
                __syncwarp();
                s = s + 1 == kStages ? 0u : s + 1;
                ph ^= s == 0 ? 1u : 0u;
            }
        }
    } else if (warp == 1) {
        // The whole warp walks the issue loop (warp-uniform control flow keeps every operand in uniform
        // registers) and one elected lane issues each tcgen05 op.  The single issuing thread was the
        // mainloop's limiter (~200 instructions per K tile, waterfall loops around every tcgen05 op), so
        // descriptors are precomputed once and advanced by adds.
        //
        // Scale factors: the tcgen05.cp of k-tile it + 1 is issued right AFTER the MMAs of k-tile it, into
        // TMEM set (it + 1) % 4, so a copy's latency overlaps a k-tile of MMAs instead of sitting between the
        // copy and its dependent MMAs (measured 14-18 % faster than copy-then-MMA on the same k-tile).  The
        // commit of k-tile it covers the copy of k-tile it (issued one k-tile earlier), so no stage is
        // released before its scale bytes are in TMEM; reusing a set four k-tiles later is ordered behind the
        // MMAs that read it (tcgen05 ops issue in order).  dbg bit 0 (timing only): no copies after the first
        // k-tile of each tile.
        const uint64_t da0 = make_sdesc(smem_u32(sA), 0, 1024, kLayoutSW128);
        const uint64_t db0 = make_sdesc(smem_u32(sB), 0, 1024, kLayoutSW128);
        const uint64_t dsa0 = make_sdesc(smem_u32(sSFA), 0, 128, kLayoutNone);
        const uint64_t dsb0 = make_sdesc(smem_u32(sSFB), 0, 128, kLayoutNone);
        constexpr uint32_t kStA = L::A >> 4, kStB = L::B >> 4, kStSA = L::SFA >> 4, kStSB = L::SFB >> 4;
        const uint32_t id0 = idesc_mxf4(kBM, BN, 0, 0), id2 = idesc_mxf4(kBM, BN, 2, 2);
        const bool no_sf = (ep.dbg & 1) != 0;
        const int nmma = (ep.dbg & 4) ? 1 : 4;
        auto sf_copy = [&](uint32_t sx, uint32_t set) {
            const uint64_t a_sf = dsa0 + sx * kStSA, b_sf = dsb0 + sx * kStSB;
            const uint32_t ta = t_sfa + set * 32, tb = t_sfb + set * 32;
            if (elect_one()) {
                tmem_cp_sf(ta + 0, a_sf);
                tmem_cp_sf(ta + 4, a_sf + (512 >> 4));
#pragma unroll
                for (int rb = 0; rb < BN / 128; ++rb) {
                    tmem_cp_sf(tb + rb * 4, b_sf + rb * (1024 >> 4));
                    tmem_cp_sf(tb + (BN / 128) * 4 + rb * 4, b_sf + (rb * 1024 + 512 >> 4));
                }
            }
            __syncwarp();
        };
        const int my_tiles = tiles > (int)blockIdx.x ? (tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
        const int total = my_tiles * nk;
        // stage / phase of k-tile `it`, advanced incrementally; full[s] of k-tile it is waited for (and its
        // scale factors copied) at the end of iteration it - 1
        uint32_t s = 0, ph = 0;
        int it = 0;
        if (total > 0) {
            mbar_wait(&full[0], 0);
            tc_fence_after();
            sf_copy(0, 0);
        }
        for (int tcount = 0; tcount < my_tiles; ++tcount) {
            mbar_wait(tmem_empty, (tcount & 1) ^ 1);  // epilogue has drained the accumulator
            tc_fence_after();
            for (int kt = 0; kt < nk; ++kt, ++it) {
                const uint64_t ad = da0 + s * kStA, bd = db0 + s * kStB;
                const uint32_t so = (no_sf ? 0u : (uint32_t)(it & 3)) * 32;
                const uint32_t ta = t_sfa + so, tb = t_sfb + so;
                if (elect_one()) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (j >= nmma) break;
                        // K step j: 64 E2M1 = 32 bytes into the 128-byte swizzled rows (+2 in the address field)
                        mma_mxf4(t_acc, ad + 2 * j, bd + 2 * j, (j & 1) ? id2 : id0, ta + (j >> 1) * 4,
                                 tb + (j >> 1) * (BN / 128) * 4, (kt | j) != 0 ? 1u : 0u);
                    }
                    tc_commit(&empty[s]);
                }
                __syncwarp();
                s = s + 1 == kStages ? 0u : s + 1;
                ph ^= s == 0 ? 1u : 0u;
                if (it + 1 < total) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    if (!no_sf || kt + 1 == nk) sf_copy(s, no_sf ? 0u : (uint32_t)((it + 1) & 3));
                }
            }
            if (elect_one()) tc_commit(tmem_full);
            __syncwarp();
        }
    } else {
        // epilogue warps 2..9: TMEM lane quadrant warp % 4, column half (warp - 2) / 4
        const int quad = warp % 4, half = (warp - 2) / 4;
        const float2 nz = opaque_nz2();
        int tcount = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tcount) {
            int mb, nb;
            tile_mn(tile, tiles_m, tiles_n, mb, nb, K >= 8192 ? 8 : 0);
            const int m0 = mb * kBM, n0 = nb * BN;
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
            epi_store<CW>(acc, row, cbase, N, ep, nz);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, L::TMEM_COLS);
    }
}


// ------------------------------------------------------------------ 2-CTA (cta_group::2) GEMM
// A CTA pair (cluster of 2 on one TPC) computes a 256 x 256 tile with tcgen05.mma.cta_group::2
// (M = 256, N = 256, K = 64): CTA r holds A rows m0 + 128 r and B rows n0 + 128 r of each K tile (so
// every SM stages half the B bytes of the 1-CTA kernel per FLOP) plus the scale factors of its A rows
// and of all 256 B rows (the scale-factor TMEM layout is the 1-SM one, duplicated per CTA).  Only the
// leader (rank 0) issues MMAs and scale-factor copies (cta_group::2 acts on both CTAs); both CTAs'
// TMA loads complete on the leader's full barrier, MMA commits multicast to both CTAs' barriers.
namespace sm2 {
constexpr int kStages = 5;
constexpr int kA = 128 * kBKBytes;     // own 128 A rows
constexpr int kB = 128 * kBKBytes;     // own 128 of the 256 B rows
constexpr int kSFA = 1024;             // own 128 rows x 8 groups
constexpr int kSFB = 2048;             // all 256 B rows x 8 groups
constexpr int kStage = kA + kB + kSFA + kSFB;
constexpr int kBox = 128 * 128;        // output staging box: 128 rows x 128 bytes (64 bf16 / 32 fp32 columns)
constexpr int kBytes = kStages * kStage + 2 * kBox + 1024 + 256;
}  // namespace sm2

// Staged epilogue of one accumulator row slice for the 2-CTA kernel: per 64-column pair the values are
// computed as in epi_store, written to a 128-row x 128-byte shared-memory box (SWIZZLE_128B layout, the
// 16-byte chunk k of row r at (k ^ r % 8)) and stored by TMA (full lines, asynchronous, rows/columns past
// M/N clipped by the tensor map).  The 4 warps of a column half share a box: named barrier 1 + half.
__device__ __forceinline__ void fence_proxy_async_cta() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
                 "r"(smem_u32(src)), "r"(x), "r"(y)
                 : "memory");
}
// element-wise out += box through the TMA unit (reduction in L2, one rounding to the map's dtype)
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* src, int x, int y) {
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
                 "r"(smem_u32(src)), "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int CW>
__device__ __forceinline__ void epi_stage(const uint32_t (&acc)[CW / 32][32], int row, int r_box, int cbase, int M,
                                          int N, const EpiParams& ep, float2 nz, const CUtensorMap* tmO, uint8_t* box,
                                          int half, bool issuer, int y0, bool accum) {
#pragma unroll
    for (int pj = 0; pj < CW / 64; ++pj) {
        const int col0 = cbase + pj * 64;
        const bool live = row < M && col0 < N;  // tiles past M / N (cluster padding) compute garbage, stores clip
        Pair g;
#pragma unroll
        for (int i = 0; i < 32; ++i)
            g.p[i] = make_float2(__uint_as_float(acc[2 * pj][i]), __uint_as_float(acc[2 * pj + 1][i]));
        if (ep.mode != kEpiStore && !(ep.dbg & 0x400)) {   // dbg 0x400 (timing only): no mask / FWHT / scale
            const uint32_t mA = live ? __ldg(ep.mask + (int64_t)row * ep.ldm + col0 / 32) : 0u;
            const uint32_t mB = live ? __ldg(ep.mask + (int64_t)row * ep.ldm + col0 / 32 + 1) : 0u;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                g.p[i].x = ((mA >> i) & 1u) ? g.p[i].x : 0.0f;
                g.p[i].y = ((mB >> i) & 1u) ? g.p[i].y : 0.0f;
            }
            if (ep.mode == kEpiMaskH) fwht_pair(g, nz);
            scale_pair(g, ep.scale);
        }
        uint8_t* rowp = box + r_box * 128;
        const int sw = r_box & 7;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            // bf16: one box holds both 32-column chunks; fp32: one box per chunk
            if (ep.out_bf16 ? (h == 0) : true) {
                if (issuer) bulk_wait_read0();  // the previous store out of this box has read it
                named_bar(1 + half, 128);
            }
            if (ep.out_bf16) {
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
                    *reinterpret_cast<uint4*>(rowp + (((h * 4 + q) ^ sw) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
                }
            } else {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int i = 4 * q;
                    *reinterpret_cast<float4*>(rowp + ((q ^ sw) << 4)) =
                        h ? make_float4(g.p[i].y, g.p[i + 1].y, g.p[i + 2].y, g.p[i + 3].y)
                          : make_float4(g.p[i].x, g.p[i + 1].x, g.p[i + 2].x, g.p[i + 3].x);
                }
            }
            if (ep.out_bf16 ? (h == 1) : true) {
                fence_proxy_async_cta();
                named_bar(1 + half, 128);
                if (issuer && !(ep.dbg & 0x200)) {   // dbg 0x200 (timing only): no TMA stores
                    if (accum)
                        tma_reduce_add_2d(tmO, box, ep.out_bf16 ? col0 : col0 + 32 * h, y0);
                    else
                        tma_store_2d(tmO, box, ep.out_bf16 ? col0 : col0 + 32 * h, y0);
                    bulk_commit();
                }
            }
        }
    }
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-SM TMA: data lands in this CTA's smem, completion bytes on the (leader's) barrier `mbar_cluster`
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint32_t mbar_cluster, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(mbar_cluster), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void mma_mxf4_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t sfa_tmem, uint32_t sfb_tmem, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sfa_tmem), "r"(sfb_tmem));
}
__device__ __forceinline__ void tmem_cp_sf_2sm(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc));
}
__device__ __forceinline__ void tc_commit_2sm(uint64_t* bar, uint16_t cta_mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(cta_mask)
        : "memory");
}
// 2-SM TMA multicast: the box lands at the same offset in every CTA of cta_mask, each destination's bytes
// completing on its own pair leader's barrier (mbar_cluster: this pair's leader barrier)
__device__ __forceinline__ void tma_load_2d_2sm_mc(void* dst, const CUtensorMap* map, uint32_t mbar_cluster, int x, int y,
                                                   uint16_t cta_mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
        "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(mbar_cluster), "r"(x), "r"(y), "h"(cta_mask)
        : "memory");
}

// Work unit u of the 2-CTA walk: units below `full` (nfull) are whole tiles; each later tile is two units, its lower
// and upper K half.
__device__ __forceinline__ void gemm_unit(int u, int full, int nk, int& tile, int& kb0, int& kb1) {
    if (u < full) {
        tile = u;
        kb0 = 0;
        kb1 = nk;
    } else {
        const int v = u - full;
        tile = full + (v >> 1);
        kb0 = (v & 1) ? nk / 2 : 0;
        kb1 = (v & 1) ? nk : nk / 2;
    }
}

// Zero the fp32 output blocks (256 x 256, clipped to M x N) of tiles first .. first + n - 1 of the 2-CTA walk.
__global__ void __launch_bounds__(256) k_zero_tiles(float* out, int64_t ldo, int M, int N, int first, int tiles_m,
                                                    int tiles_n, int gm) {
    int mb, nb;
    tile_mn(first + (int)blockIdx.x, tiles_m, tiles_n, mb, nb, gm);
    const int c = nb * 256 + (threadIdx.x & 63) * 4;
    for (int r = mb * 256 + (threadIdx.x >> 6); r < mb * 256 + 256 && r < M; r += 4)
        if (c < N) *reinterpret_cast<float4*>(out + (int64_t)r * ldo + c) = make_float4(0.f, 0.f, 0.f, 0.f);
}

// NP = CTA pairs per cluster: 1 (cluster of 2) or 4 (cluster of 8: a 2 x 2 block of pair tiles whose A rows
// are shared along N and B rows along M, each CTA loading half of its A and B boxes and multicasting them to
// the CTA of the same role in the neighbouring pair, which halves the L2 -> SMEM bytes per FLOP)
template <int NP>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_mxf4_2sm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmSFA, const __grid_constant__ CUtensorMap tmSFB,
                    const __grid_constant__ CUtensorMap tmO, int M, int N, int K, EpiParams ep) {
    constexpr int BN = 256, CW = BN / 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = sA + sm2::kStages * sm2::kA;
    uint8_t* sSFA = sB + sm2::kStages * sm2::kB;
    uint8_t* sSFB = sSFA + sm2::kStages * sm2::kSFA;
    uint8_t* sBox = sSFB + sm2::kStages * sm2::kSFB;  // 2 output staging boxes (one per column half)
    uint64_t* full = reinterpret_cast<uint64_t*>(sBox + 2 * sm2::kBox);
    uint64_t* empty = full + sm2::kStages;
    uint64_t* tmem_full = empty + sm2::kStages;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_base_holder = reinterpret_cast<uint32_t*>(tmem_empty + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_rank();
    const uint32_t q = rank & 1, lead_rank = rank & ~1u;    // CTA within its pair, the pair leader's rank
    const bool leader = q == 0;
    const int pm = NP == 4 ? (int)((rank >> 1) & 1) : 0, pn = NP == 4 ? (int)(rank >> 2) : 0;
    const uint16_t pair_mask = (uint16_t)(3u << lead_rank), all_mask = (uint16_t)((1u << (2 * NP)) - 1);
    const int nk = (K + 255) / 256;
    const int tiles_m = (M + 255) / 256, tiles_n = (N + BN - 1) / BN;
    const int sup_m = NP == 4 ? (tiles_m + 1) / 2 : tiles_m, sup_n = NP == 4 ? (tiles_n + 1) / 2 : tiles_n;
    // work units: the first `nfull` (super-)tiles whole, then the last `split` tiles as two K-half units each
    // (gemm_unit; the launcher zeroes their output blocks and the epilogue adds by TMA reduce-add)
    const int split = NP == 1 ? ep.split_tiles : 0;
    const int nfull = sup_m * sup_n - split;
    const int tiles = nfull + 2 * split;
    const int cid = blockIdx.x / (2 * NP), ncl = gridDim.x / (2 * NP);
    // tile walk: grouped (gm row blocks per column sweep) for long K, row-major otherwise; dbg 0x1000 / 0x2000
    // force grouped-4 / grouped-16 (timing experiments)
    const int gm = (ep.dbg & 0x1000) ? 4 : (ep.dbg & 0x2000) ? 16 : (ep.dbg & 0x4000) ? 2 : (K >= 8192 ? 8 : 0);

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        tma_prefetch(&tmSFA);
        tma_prefetch(&tmSFB);
        for (int s = 0; s < sm2::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NP);  // one commit per pair whose smem this CTA's loads fill
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, 2 * kEpiWarps);
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_holder)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_base_holder;
    const uint32_t t_acc = tmem, t_sfa = tmem + BN, t_sfb = tmem + BN + 8;

    if (warp == 0) {
        // producer (warp-uniform loop, elected issue): this CTA's A half and B half, its A scale atoms and all
        // 256 B rows' atoms, completing on the leader's full barrier
        uint32_t s = 0, ph = 0;
        const uint16_t mask_a = NP == 4 ? (uint16_t)((1u << ((pm << 1) | q)) | (1u << (4 | (pm << 1) | q))) : 0;
        const uint16_t mask_b = NP == 4 ? (uint16_t)((1u << ((pn << 2) | q)) | (1u << ((pn << 2) | 2 | q))) : 0;
        for (int tile = cid; tile < tiles; tile += ncl) {
            int mb, nb;
            int tl, kb0, kb1;
            gemm_unit(tile, nfull, nk, tl, kb0, kb1);
            tile_mn(tl, sup_m, sup_n, mb, nb, gm);
            if (NP == 4) {
                mb = 2 * mb + pm;
                nb = 2 * nb + pn;
            }
            const int m0 = mb * 256 + 128 * (int)q, n0 = nb * BN;
            for (int kt = kb0; kt < kb1; ++kt) {
                mbar_wait(&empty[s], ph ^ 1);
                if (elect_one()) {
                    const uint32_t fb = mapa_shared(smem_u32(&full[s]), lead_rank);
                    if (leader) mbar_arrive_expect_tx(&full[s], 2 * sm2::kStage);
                    if (NP == 4) {
                        // my half of the A box (rows + 64 pn) to both pairs on this M block, my half of the B box
                        // (rows + 64 pm) to both pairs on this N block
                        tma_load_2d_2sm_mc(sA + s * sm2::kA + pn * 8192, &tmA, fb, kt * kBKBytes, m0 + 64 * pn, mask_a);
                        tma_load_2d_2sm_mc(sB + s * sm2::kB + pm * 8192, &tmB, fb, kt * kBKBytes,
                                           n0 + 128 * (int)q + 64 * pm, mask_b);
                    } else {
                        tma_load_2d_2sm(sA + s * sm2::kA, &tmA, fb, kt * kBKBytes, m0);
                        tma_load_2d_2sm(sB + s * sm2::kB, &tmB, fb, kt * kBKBytes, n0 + 128 * (int)q);
                    }
                    // scale atoms (u32 view, 1 KB = 256 words per K tile): A rows of this CTA, all 256 B rows
                    tma_load_2d_2sm(sSFA + s * sm2::kSFA, &tmSFA, fb, kt * 256, m0 / 128);
                    tma_load_2d_2sm(sSFB + s * sm2::kSFB, &tmSFB, fb, kt * 256, n0 / 128);
                }
                __syncwarp();
                s = s + 1 == sm2::kStages ? 0u : s + 1;
                ph ^= s == 0 ? 1u : 0u;
            }
        }
    } else if (warp == 1) {
        if (leader) {
            // issue loop as in k_gemm_mxf4 (warp-uniform, elected issue, scale copies one k-tile ahead into
            // rotating TMEM sets); cta_group::2 MMAs and copies act on both CTAs of the pair
            const uint64_t da0 = make_sdesc(smem_u32(sA), 0, 1024, kLayoutSW128);
            const uint64_t db0 = make_sdesc(smem_u32(sB), 0, 1024, kLayoutSW128);
            const uint64_t dsa0 = make_sdesc(smem_u32(sSFA), 0, 128, kLayoutNone);
            const uint64_t dsb0 = make_sdesc(smem_u32(sSFB), 0, 128, kLayoutNone);
            const uint32_t id0 = idesc_mxf4(256, BN, 0, 0), id2 = idesc_mxf4(256, BN, 2, 2);
            const int my_tiles = tiles > cid ? (tiles - 1 - cid) / ncl + 1 : 0;
            int total = 0;   // k-iterations of this cluster's units
            for (int u = cid; u < tiles; u += ncl) {
                int tl, kb0, kb1;
                gemm_unit(u, nfull, nk, tl, kb0, kb1);
                total += kb1 - kb0;
            }
            // one elected lane walks the whole issue loop: a single divergence region, every loop value uniform
            if (elect_one()) {
                auto sf_copy = [&](uint32_t sx, uint32_t set) {
                    const uint64_t a_sf = dsa0 + sx * (sm2::kSFA >> 4), b_sf = dsb0 + sx * (sm2::kSFB >> 4);
                    const uint32_t ta = t_sfa + set * 32, tb = t_sfb + set * 32;
                    tmem_cp_sf_2sm(ta + 0, a_sf);
                    tmem_cp_sf_2sm(ta + 4, a_sf + (512 >> 4));
#pragma unroll
                    for (int rb = 0; rb < 2; ++rb) {
                        tmem_cp_sf_2sm(tb + rb * 4, b_sf + rb * (1024 >> 4));
                        tmem_cp_sf_2sm(tb + 8 + rb * 4, b_sf + (rb * 1024 + 512 >> 4));
                    }
                };
                uint32_t s = 0, ph = 0;
                int it = 0;
                if (total > 0) {
                    mbar_wait(&full[0], 0);
                    tc_fence_after();
                    sf_copy(0, 0);
                }
                for (int tcount = 0; tcount < my_tiles; ++tcount) {
                    mbar_wait(tmem_empty, (tcount & 1) ^ 1);  // both CTAs' epilogues drained the accumulator
                    tc_fence_after();
                    int tl, kb0, kb1;
                    gemm_unit(cid + tcount * ncl, nfull, nk, tl, kb0, kb1);
                    for (int kt = kb0; kt < kb1; ++kt, ++it) {
                        const uint64_t ad = da0 + s * (sm2::kA >> 4), bd = db0 + s * (sm2::kB >> 4);
                        const uint32_t so = (uint32_t)(it & 3) * 32;
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            mma_mxf4_2sm(t_acc, ad + 2 * j, bd + 2 * j, (j & 1) ? id2 : id0, t_sfa + so + (j >> 1) * 4,
                                         t_sfb + so + (j >> 1) * 8, (kt != kb0 || j != 0) ? 1u : 0u);
                        tc_commit_2sm(&empty[s], all_mask);
                        s = s + 1 == sm2::kStages ? 0u : s + 1;
                        ph ^= s == 0 ? 1u : 0u;
                        if (it + 1 < total) {
                            mbar_wait(&full[s], ph);
                            tc_fence_after();
                            sf_copy(s, (uint32_t)((it + 1) & 3));
                        }
                    }
                    tc_commit_2sm(tmem_full, pair_mask);
                }
            }
            __syncwarp();
        }
    } else {
        const int quad = warp % 4, half = (warp - 2) / 4;
        const bool issuer = ((warp - 2) & 3) == 0 && lane == 0;  // one thread per column half issues the stores
        const float2 nz = opaque_nz2();
        const uint32_t te_leader = mapa_shared(smem_u32(tmem_empty), lead_rank);
        uint8_t* box = sBox + half * sm2::kBox;
        int tcount = 0;
        for (int tile = cid; tile < tiles; tile += ncl, ++tcount) {
            int mb, nb;
            int tl, kb0, kb1;
            gemm_unit(tile, nfull, nk, tl, kb0, kb1);
            tile_mn(tl, sup_m, sup_n, mb, nb, gm);
            if (NP == 4) {
                mb = 2 * mb + pm;
                nb = 2 * nb + pn;
            }
            const int m0 = mb * 256 + 128 * (int)q, n0 = nb * BN;
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
            if (lane == 0) mbar_arrive_remote(te_leader);  // the leader may start the next tile
            if (ep.dbg & 0x100) continue;                   // timing only: no epilogue math/stores
            epi_stage<CW>(acc, row, quad * 32 + lane, cbase, M, N, ep, nz, &tmO, box, half, issuer, m0,
                          ep.accumulate || tile >= nfull);
        }
        if (issuer) bulk_wait0();
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ---------------------------------------------------------------------------- host side
int g_gemm_2sm = 1;  // use the 2-CTA kernel where eligible (launch_gemm); 0: 1-CTA kernel only

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
    static int attr_set[kMaxDevices];
    if (first_use_on_device(attr_set))
        cudaFuncSetAttribute(k_gemm_mxf4<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES);
    const int64_t sms = device_sms();
    const int64_t tiles = ((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
    const unsigned grid = (unsigned)cap_grid(tiles < sms ? tiles : sms);
    k_gemm_mxf4<BN><<<grid, kThreads, L::BYTES, st>>>(ta, tb, a_sf, a_katoms, b_sf, b_katoms, (int)M, (int)N, (int)K,
                                                      ep);
    return (int)cudaGetLastError();
}

// scale atoms viewed as u32 [row blocks][katoms * 128]; box 256 words (one K tile) x box_rows blocks
static int make_sf_map(CUtensorMap* m, const uint8_t* sf, int64_t rows, int64_t katoms, int box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return 1001;
    const int64_t rb = ((rows + 255) / 256) * 2;
    cuuint64_t dims[2] = {(cuuint64_t)(katoms * 128), (cuuint64_t)rb};
    cuuint64_t strides[1] = {(cuuint64_t)(katoms * 512)};
    cuuint32_t box[2] = {256, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, (void*)sf, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : 1002;
}

int g_gemm_cluster8 = 0;  // 1: clusters of 4 pairs with TMA multicast (measured slower: fewer co-resident SMs)
int g_gemm_splitk = 1;    // split-K for under-filled fp32 GEMMs (qt_debug_set_gemm bit 20 disables it)

template <int NP>
static int launch_2sm_np(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tsa, const CUtensorMap& tsb,
                         const CUtensorMap& to, int64_t M, int64_t N, int64_t K, const EpiParams& ep, cudaStream_t st) {
    static int max_clusters_dev[kMaxDevices];
    int& max_clusters = max_clusters_dev[current_device()];
    if (!max_clusters) {
        cudaFuncSetAttribute(k_gemm_mxf4_2sm<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2::kBytes);
        if (NP == 4) cudaFuncSetAttribute(k_gemm_mxf4_2sm<NP>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2 * NP;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(2 * NP * 64, 1, 1);
        cfg.blockDim = dim3(kThreads, 1, 1);
        cfg.dynamicSmemBytes = sm2::kBytes;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_gemm_mxf4_2sm<NP>, &cfg) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = device_sms() / (2 * NP);
        }
        max_clusters = n;
    }
    const int64_t tm = (M + 255) / 256, tn = (N + 255) / 256;
    int64_t tiles = NP == 4 ? ((tm + 1) / 2) * ((tn + 1) / 2) : tm * tn;
    int64_t cl_max = max_clusters;
    if (g_grid_cap > 0) cl_max = std::max<int64_t>(1, std::min<int64_t>(cl_max, g_grid_cap / (2 * NP)));
    // Split-K of the last, partial wave of fp32 GEMMs: its `tail` tiles (tiles mod clusters; all tiles of an
    // under-filled GEMM, e.g. the 25-tile 1280 x 1280 dW of the Llama-200M attention projections) run as two
    // K-half units each, so the wave has twice the units and half the length; their output blocks are zeroed
    // first and the epilogue adds both halves by TMA reduce-add.  Exactly two addends per element
    // (0 + a + b = b + a): deterministic.
    EpiParams epx = ep;
    const int64_t tail = tiles % cl_max;
    if (NP == 1 && g_gemm_splitk && !ep.out_bf16 && !ep.accumulate && tail > 0 && 2 * tail <= cl_max &&
        K >= 8 * 256) {
        const int gm = (ep.dbg & 0x1000) ? 4 : (ep.dbg & 0x2000) ? 16 : (ep.dbg & 0x4000) ? 2 : (K >= 8192 ? 8 : 0);
        k_zero_tiles<<<(unsigned)tail, 256, 0, st>>>(static_cast<float*>(ep.out), ep.ldo, (int)M, (int)N,
                                                     (int)(tiles - tail), (int)tm, (int)tn, gm);
        epx.split_tiles = (int)tail;
        tiles += tail;
    }
    const int64_t clusters = tiles < cl_max ? tiles : cl_max;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2 * NP;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(2 * NP * clusters), 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = sm2::kBytes;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_gemm_mxf4_2sm<NP>, ta, tb, tsa, tsb, to, (int)M, (int)N, (int)K, epx);
    return (int)e;
}

static int launch_gemm_2sm(const uint8_t* a, int64_t lda, const uint8_t* a_sf, int64_t a_katoms, const uint8_t* b,
                           int64_t ldb, const uint8_t* b_sf, int64_t b_katoms, int64_t M, int64_t N, int64_t K,
                           const EpiParams& ep, cudaStream_t st) {
    // cluster of 4 pairs (multicast) when there is at least a 2 x 2 block of pair tiles
    const bool c8 = g_gemm_cluster8 && M >= 512 && N >= 512;
    const int box_rows = c8 ? 64 : 128;
    CUtensorMap ta, tb, tsa, tsb;
    int rc = make_codes_map(&ta, a, M, K / 2, lda, box_rows);
    if (!rc) rc = make_codes_map(&tb, b, N, K / 2, ldb, box_rows);
    if (!rc) rc = make_sf_map(&tsa, a_sf, M, a_katoms, 1);
    if (!rc) rc = make_sf_map(&tsb, b_sf, N, b_katoms, 2);
    if (rc) return rc;
    // output boxes of 128 rows x 128 bytes, 128-byte swizzle (the staging layout of epi_stage)
    CUtensorMap to;
    {
        PFN_encodeTiled enc = get_encode();
        const int esz = ep.out_bf16 ? 2 : 4;
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
        cuuint64_t strides[1] = {(cuuint64_t)(ep.ldo * esz)};
        cuuint32_t box[2] = {(cuuint32_t)(128 / esz), 128};
        cuuint32_t es[2] = {1, 1};
        if (!enc || enc(&to, ep.out_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                        ep.out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return 1002;
    }
    return c8 ? launch_2sm_np<4>(ta, tb, tsa, tsb, to, M, N, K, ep, st)
              : launch_2sm_np<1>(ta, tb, tsa, tsb, to, M, N, K, ep, st);
}

int launch_gemm(const uint8_t* a, int64_t lda, const uint8_t* a_sf, int64_t a_katoms, const uint8_t* b, int64_t ldb,
                const uint8_t* b_sf, int64_t b_katoms, int64_t M, int64_t N, int64_t K, const EpiParams& ep,
                cudaStream_t st) {
    if (M == 0 || N == 0) return 0;
    const int esz = ep.out_bf16 ? 2 : 4;
    // N % 256 == 128 also runs on the pair kernel when K >= 4096: a half-filled last column tile leaves the
    // second CTA's B box entirely past N (TMA zero fill, complete_tx still counts the full box), its B scale
    // atoms in the zeroed 256-row padding of the scale buffer (qt_sf_bytes), and its output columns clipped by
    // the store map -- the same situation as the half-filled last row tile of M % 256 == 128.  Measured at the
    // Llama-30M shapes (d = 640, tools/gemm_30m_probe.py): long-K GEMMs gain (LM-head dx / dW 384 / 408 ->
    // 286 / 287 us, ffn dW 57 -> 48 us), short-K ones (K = 640 / 1792) lose 7-20 % to the wasted half tile.
    const bool pair_n = N % 256 == 0 || (N % 128 == 0 && K >= 4096);
    if (g_gemm_2sm && pair_n && M >= 256 && (reinterpret_cast<uintptr_t>(ep.out) & 15) == 0 &&
        (ep.ldo * esz) % 16 == 0)
        return launch_gemm_2sm(a, lda, a_sf, a_katoms, b, ldb, b_sf, b_katoms, M, N, K, ep, st);
    if (N >= 256 && N % 256 == 0)
        return launch_gemm_bn<256>(a, lda, a_sf, a_katoms, b, ldb, b_sf, b_katoms, M, N, K, ep, st);
    return launch_gemm_bn<128>(a, lda, a_sf, a_katoms, b, ldb, b_sf, b_katoms, M, N, K, ep, st);
}

}  // namespace qt
