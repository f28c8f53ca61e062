// common.cuh -- sm_100a building blocks shared by the Quartet kernels.
//
//   * MXFP4 operand layout (codes, E8M0 scale-factor atoms, QuEST trust masks)
//   * bit-exact fp32 FWHT-32 butterfly (reference: mx4train/_backend/_native.pyx:353-379)
//   * splitmix64 counter RNG (reference: mx4train/rng.py:27-50)
//   * PTX wrappers: mbarrier, TMA (cp.async.bulk[.tensor]), tcgen05 (alloc/mma/cp/ld/commit)
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace qt {

// ------------------------------------------------------------------ MXFP4 operand layout
//
// A quantized operand is a logical [R, K] matrix whose 32-element groups run along K (the
// contraction axis of the GEMM that consumes it):
//   codes : uint8 [R, ldc]   two E2M1 nibbles per byte, element 2k in the LOW nibble
//                            (identical bytes to the reference's pack_nibbles, codec.py:146-153)
//   sf    : uint8 E8M0 scale per group, stored in 512-byte atoms that tcgen05.cp copies to TMEM
//           verbatim.  Atom (rb, ka) covers rows 128*rb..+127 and groups 4*ka..+3; atoms are laid
//           out ka-fastest: ((rb * katoms + ka) * 512).  Inside an atom:
//             (r % 32) * 16 + ((r % 128) / 32) * 4 + (group % 4)
//           Rows are padded to a multiple of 256 and K to a multiple of 256 (katoms even), the
//           padding holds exponent 0 (any finite value: the matching codes are zero).
//   mask  : uint32 [R, K/32]  bit j of word (r, g) = element 32g+j was not clipped (QuEST).
__host__ __device__ __forceinline__ int64_t sf_offset(int64_t r, int64_t grp, int64_t katoms) {
    return ((r >> 7) * katoms + (grp >> 2)) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (grp & 3);
}

// ------------------------------------------------------------------------- rng (rng.py)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kDomainSR = 0x5352ULL;
constexpr uint64_t kDomainSigns = 0x5347ULL;

// ------------------------------------------------------------------------ fp32 helpers
__device__ __forceinline__ float exp2i(int e) {  // 2^e as fp32, e in [-149, 127]
    if (e >= -126) return __uint_as_float((uint32_t)(e + 127) << 23);
    return __uint_as_float(1u << (e + 149));
}

// E2M1 encode of two fp32 values with RNE + satfinite (ties-to-even-mantissa, clamp at 6):
// identical to the reference's midpoint ladder (_numpy.py:26-40).  Returns the byte with `lo`
// in the low nibble.  Negative zero is NOT canonicalised here (see canon8 in qgroup.cuh).
__device__ __forceinline__ uint32_t e2m1x2(float lo, float hi) {
    uint16_t r;
    asm("{\n .reg .b8 t;\n cvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n cvt.u16.u8 %0, t;\n}"
        : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}
// Decode an E2M1 byte pair to fp32 (exact).
__device__ __forceinline__ float2 e2m1x2_to_f32(uint32_t byte) {
    uint32_t h2;
    asm("{\n .reg .b8 t;\n cvt.u8.u32 t, %1;\n cvt.rn.f16x2.e2m1x2 %0, t;\n}" : "=r"(h2) : "r"(byte));
    __half2 h = *reinterpret_cast<__half2*>(&h2);
    return __half22float2(h);  // .x = low nibble
}

// E8M0 exponent of the smallest power of two s with amax / s <= 6 (codec.py:132-143,
// _native.pyx:66-78), from the fp32 bits of amax (exact: see DESIGN.md).
__device__ __forceinline__ int ceil_scale_exp(float amax) {
    uint32_t b = __float_as_uint(amax);
    int E = (int)(b >> 23);
    if (amax <= 0.0f) return 0;
    int e = E - 2 + ((b & 0x7FFFFF) > 0x400000u ? 1 : 0);
    return e < 0 ? 0 : (e > 254 ? 254 : e);
}
// floor(log2(amax / 96)) + 127, clamped (_native.pyx:81-89 applied to amax * 1/16 / 6).
__device__ __forceinline__ int quest_low_exp(float amax) {
    uint32_t b = __float_as_uint(amax);
    int E = (int)(b >> 23);
    int e = E - 7 + ((b & 0x7FFFFF) >= 0x400000u ? 1 : 0);
    return e < 0 ? 0 : (e > 254 ? 254 : e);
}

// ----------------------------------------------------------------------------- mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Wait for the phase with the given parity.  QT_WAIT_HINT (build flag, default 0): 0 = plain try_wait
// loop (the hardware parks the warp inside SYNCS.TRYWAIT until the phase completes or a short timeout),
// 1 = try_wait with a suspend-time hint, which ptxas turns into a NANOSLEEP.SYNCS retry loop.
#ifndef QT_WAIT_HINT
#define QT_WAIT_HINT 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
#if QT_WAIT_HINT
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 10000000;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
#else
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
#endif
}

// Single-thread producer / MMA roles: poll with a fixed sleep between tries (QT_ROLE_SLEEP_NS, build flag), so
// a role that waits a whole tile phase does not take issue slots from the epilogue warps of its scheduler.
#ifndef QT_ROLE_SLEEP_NS
#define QT_ROLE_SLEEP_NS 128
#endif
__device__ __forceinline__ void mbar_wait_role(uint64_t* bar, uint32_t parity) {
#if QT_ROLE_SLEEP_NS > 0
    const uint32_t addr = smem_u32(bar);
    for (;;) {
        uint32_t done;
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(addr), "r"(parity)
                     : "memory");
        if (done) break;
        __nanosleep(QT_ROLE_SLEEP_NS);
    }
#else
    mbar_wait(bar, parity);
#endif
}

template <int HINT_NS>
__device__ __forceinline__ void mbar_wait_hint(uint64_t* bar, uint32_t parity) {
#if QT_WAIT_HINT
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(addr),
        "r"(parity), "n"(HINT_NS)
        : "memory");
#else
    mbar_wait(bar, parity);
#endif
}

// one lane of the (fully active) warp: for issuing single-thread async ops from warp-uniform code
__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n selp.u32 %0, 1, 0, e;\n}" : "=r"(p));
    return p != 0;
}

// ----------------------------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// -------------------------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T with E8M0 block-32 scales from TMEM (MXFP4, K = 64).
__device__ __forceinline__ void mma_mxf4(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t sfa_tmem, uint32_t sfb_tmem, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sfa_tmem), "r"(sfb_tmem));
}
// 32 lanes x 128 bits from smem, broadcast to the 4 lane quadrants (scale-factor staging).
__device__ __forceinline__ void tmem_cp_sf(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc));
}
// Each thread of the warp reads its TMEM lane, 32 consecutive 32-bit columns.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory matrix descriptor (sm100 "version 1").
//   K-major SWIZZLE_128B operand tiles: rows of 128 bytes, 8-row groups 1024 B apart (SBO).
//   Scale-factor staging (SWIZZLE_NONE): 8 x 16-byte core matrices, 128 B apart (SBO).
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version for sm100
    d |= (uint64_t)(layout & 7) << 61;
    return d;
}
constexpr uint32_t kLayoutSW128 = 2;
constexpr uint32_t kLayoutNone = 0;

// Instruction descriptor for kind::mxf4 (E2M1 x E2M1, E8M0 scales, fp32 accumulate, K-major).
__host__ __device__ __forceinline__ uint32_t idesc_mxf4(int M, int N, int a_sf_id, int b_sf_id) {
    uint32_t d = 0;
    d |= (uint32_t)(b_sf_id & 3) << 4;
    d |= 1u << 7;                     // A format: E2M1
    d |= 1u << 10;                    // B format: E2M1
    d |= (uint32_t)(N >> 3) << 17;    // N / 8
    d |= 1u << 23;                    // scale format: UE8M0
    d |= (uint32_t)(M >> 4) << 24;    // M / 16
    d |= (uint32_t)(a_sf_id & 3) << 29;
    return d;
}

}  // namespace qt
