// quant.cu -- fused Hadamard + MXFP4 quantizer kernels (one HBM pass over the input).
//
//   k_signs       sign bitmap of the randomized Hadamard (rng.py:57-62, hadamard.py:77-85)
//   k_quant_tile  128 x 128 smem tile, up to two passes over the same data:
//                   row pass  groups along the contiguous axis: forward X / W (H32 + QuEST,
//                             qlinear.py:139-157) and the backward dy operand G (RHT32 + x0.75 +
//                             RTN/SR, qlinear.py:214-225)
//                   col pass  groups along the strided axis = the transposed operand
//                             (dy^T -> G_t, deq(X_q)^T -> X_t, deq(W_q)^T -> W_t,
//                              qlinear.py:215, 234-246)
//                 so the backward's two dy operands come from ONE read of dy.  Every thread
//                 quantizes two groups in lockstep (packed f32x2, see quant.cuh).
//   k_transform_rows  transform only (the kernels.fwht seam)
#include "launch.h"
#include "quant.cuh"

namespace qt {

__global__ void k_signs(uint32_t* bits, int64_t start, int64_t n, uint64_t base) {
    int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t nw = (n + 31) / 32;
    if (w >= nw) return;
    uint32_t m = 0;
    for (int j = 0; j < 32; ++j) {
        int64_t p = w * 32 + j;
        if (p < n) {
            uint64_t h = mix64(base + ((uint64_t)(start + p) + 1) * kGolden);
            m |= (uint32_t)(h >> 63) << j;
        }
    }
    bits[w] = m;
}

__device__ __forceinline__ void transform_pair(Pair& g, int transform, uint32_t sA, uint32_t sB, float prescale) {
    if (transform == kRandomized) flip_pair(g, sA, sB);
    if (transform != kNone) fwht_pair(g, opaque_nz2());
    if (prescale != 1.0f) scale_pair(g, prescale);
}

// ------------------------------------------------------------------------ transform only
__global__ void __launch_bounds__(256) k_transform_rows(const float* __restrict__ x, float* __restrict__ out,
                                                       int64_t rows, int64_t cols, int transform,
                                                       const uint32_t* sign_bits, float prescale) {
    const int64_t gpr = cols / 32, ppr = (gpr + 1) / 2;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (tid >= rows * ppr) return;
    const int64_t r = tid / ppr, gA = (tid - r * ppr) * 2, gB = gA + 1;
    const bool okB = gB < gpr;
    Pair g;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        g.p[j].x = x[r * cols + gA * 32 + j];
        g.p[j].y = okB ? x[r * cols + gB * 32 + j] : 0.0f;
    }
    transform_pair(g, transform, transform == kRandomized ? sign_bits[gA] : 0u,
                   transform == kRandomized && okB ? sign_bits[gB] : 0u, prescale);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        out[r * cols + gA * 32 + j] = g.p[j].x;
        if (okB) out[r * cols + gB * 32 + j] = g.p[j].y;
    }
}

int launch_transform_rows(const float* x, float* out, int64_t rows, int64_t cols, int transform,
                          const uint32_t* sign_bits, float prescale, cudaStream_t st) {
    if (rows == 0 || cols == 0) return 0;
    const int64_t n = rows * ((cols / 32 + 1) / 2);
    k_transform_rows<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, out, rows, cols, transform, sign_bits,
                                                                   prescale);
    return (int)cudaGetLastError();
}

// ------------------------------------------------------------------------ k_quant_tile
// Persistent kernel over 128 x 128 tiles.  Each CTA double-buffers tiles in dynamic smem with
// cp.async (tile i+1 streams in while tile i is quantized), so HBM latency hides behind compute.
// Dense tiles live in smem as bf16 (ESZ 2, 32 KB) or fp32 (ESZ 4, 64 KB) in 16-byte chunks; chunk
// k of row r sits at k ^ sw(r, k), sw = 2 * ((r + r/32) & 3) ^ ((k / 8) & 1), which keeps (bf16) the
// fill, the row pass (4 rows x 2 group pairs per phase) and the col pass (4 rows 32 apart x 2 chunks
// per 32-lane load) bank-conflict free.  MXFP4 input is staged raw (codes + one 512-B scale atom)
// and decoded exactly into a bf16 tile before the col pass.
constexpr int kTR = 128, kTC = 128;

struct TileArgs {
    const void* x;      // dense input (bf16 / fp32), row stride ldx elements
    int64_t ldx;
    MxIn mx;            // MXFP4 input (in_type kInMXFP4), groups along C
    int64_t R, C;
    QuantCfg row_cfg, col_cfg;
    QuantOut row_out, col_out;
};

__device__ __forceinline__ int tile_chunk(int r, int k) { return k ^ ((((r + (r >> 5)) & 3) << 1) ^ ((k >> 3) & 1)); }

// bf16x2 -> 2 x fp32 on the ALU pipe (PRMT + LOP3), keeping the FMA pipe free for the butterfly.
__device__ __forceinline__ void bf16x2_to_f32(uint32_t w, float& lo, float& hi) {
    lo = __uint_as_float(__byte_perm(w, 0u, 0x1044));
    hi = __uint_as_float(w & 0xFFFF0000u);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <int IN>
struct TileGeom {
    static constexpr int ESZ = IN == kInF32 ? 4 : 2;
    static constexpr int CPR = kTC * ESZ / 16;            // chunks per dense tile row
    static constexpr int DENSE = kTR * CPR;               // chunks per dense tile
    static constexpr int RAW_ROW = kTC / 2 / 16;          // MXFP4: code chunks per row (4)
    static constexpr int RAW = kTR * RAW_ROW + 512 / 16;  // MXFP4: codes + one scale atom
    // buffers: dense -> 2 x DENSE; MXFP4 -> 2 x RAW staging + 1 x DENSE decoded tile
    static constexpr int CHUNKS = IN == kInMXFP4 ? 2 * RAW + DENSE : 2 * DENSE;
    static constexpr int BYTES = CHUNKS * 16;
};

// Issue the cp.async copies of tile (r0, c0) into buffer `buf`.
template <int IN>
__device__ __forceinline__ void tile_fill_async(const TileArgs& a, uint4* buf, int64_t r0, int64_t c0, int tid) {
    using G = TileGeom<IN>;
    const int nr = (int)(a.R - r0 < kTR ? a.R - r0 : kTR), nc = (int)(a.C - c0 < kTC ? a.C - c0 : kTC);
    if (IN == kInMXFP4) {
#pragma unroll
        for (int it = 0; it < kTR * G::RAW_ROW / 256; ++it) {
            const int id = it * 256 + tid, rr = id / G::RAW_ROW, part = id % G::RAW_ROW;
            const bool ok = rr < nr && part * 32 < nc;
            const uint8_t* src = a.mx.codes + (ok ? (r0 + rr) * a.mx.ldc + c0 / 2 + part * 16 : 0);
            cp_async16(buf + id, src, ok);
        }
        if (tid < 32) {
            const uint8_t* src = a.mx.sf + ((r0 / 128) * a.mx.katoms + c0 / 128) * 512 + tid * 16;
            cp_async16(buf + kTR * G::RAW_ROW + tid, src, true);
        }
    } else {
        const uint8_t* xb = static_cast<const uint8_t*>(a.x);
#pragma unroll
        for (int it = 0; it < G::DENSE / 256; ++it) {
            const int id = it * 256 + tid, rr = id / G::CPR, k = id % G::CPR;
            const bool ok = rr < nr && k * (16 / G::ESZ) < nc;
            const uint8_t* src = xb + (ok ? ((r0 + rr) * a.ldx + c0) * G::ESZ + k * 16 : 0);
            cp_async16(buf + rr * G::CPR + tile_chunk(rr, k), src, ok);
        }
    }
}

// MXFP4 staging -> decoded bf16 tile: thread (row t/2, groups 2h, 2h+1), exact code * 2^(e-127).
__device__ __forceinline__ void tile_decode_mxfp4(const uint4* raw, uint4* tile, int tid) {
    constexpr int CPR = kTC * 2 / 16;
    const int rr = tid >> 1, h = tid & 1;
    const uint8_t* sfa = reinterpret_cast<const uint8_t*>(raw + kTR * 4);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int gl = 2 * h + u;
        const uint4 cw = raw[rr * 4 + gl];
        const float s = exp2i((int)sfa[(rr & 31) * 16 + ((rr >> 5) & 3) * 4 + gl] - 127);
        const uint32_t w[4] = {cw.x, cw.y, cw.z, cw.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t bw[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                float2 f = e2m1x2_to_f32((w[q] >> (8 * b)) & 0xFFu);
                bw[b] = (__float_as_uint(f.x * s) >> 16) | (__float_as_uint(f.y * s) & 0xFFFF0000u);
            }
            tile[rr * CPR + tile_chunk(rr, gl * 4 + q)] = make_uint4(bw[0], bw[1], bw[2], bw[3]);
        }
    }
}

// Row pass on one tile: thread -> (row t/2, group pair t%2) = groups A = 2pp, B = 2pp + 1.
template <int ESZ, int ROUND>
__device__ __forceinline__ void tile_row_pass(const TileArgs& a, const uint4* tile, int64_t r0, int64_t c0, int nr,
                                              int nc, int tid) {
    constexpr int CPR = kTC * ESZ / 16;
    const int rr = tid >> 1, pp = tid & 1;
    const bool okA = rr < nr && 64 * pp < nc, okB = rr < nr && 64 * pp + 32 < nc;
    Pair g;
#pragma unroll
    for (int hB = 0; hB < 2; ++hB) {
        const int gl = 2 * pp + hB;
        if (ESZ == 2) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 c = tile[rr * CPR + tile_chunk(rr, gl * 4 + q)];
                const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    float lo, hi;
                    bf16x2_to_f32(w[t], lo, hi);
                    if (hB) {
                        g.p[q * 8 + 2 * t].y = lo;
                        g.p[q * 8 + 2 * t + 1].y = hi;
                    } else {
                        g.p[q * 8 + 2 * t].x = lo;
                        g.p[q * 8 + 2 * t + 1].x = hi;
                    }
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint4 c = tile[rr * CPR + tile_chunk(rr, gl * 8 + q)];
                const float v[4] = {__uint_as_float(c.x), __uint_as_float(c.y), __uint_as_float(c.z),
                                    __uint_as_float(c.w)};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    if (hB)
                        g.p[q * 4 + t].y = v[t];
                    else
                        g.p[q * 4 + t].x = v[t];
                }
            }
        }
    }
    const int64_t row = r0 + rr, gA = c0 / 32 + 2 * pp;
    PairOut o;
    o.sf[0] = o.sf[1] = 0;
    if (okA) {
        const QuantCfg& cf = a.row_cfg;
        transform_pair(g, cf.transform, cf.transform == kRandomized ? __ldg(cf.sign_bits + gA) : 0u,
                       cf.transform == kRandomized && okB ? __ldg(cf.sign_bits + gA + 1) : 0u, cf.prescale);
        const int64_t cld = cf.counter_ld ? cf.counter_ld : a.C;
        const uint64_t idx = cf.counter_start + (uint64_t)(row * cld + gA * 32);
        o = quantize_pair<ROUND>(g, cf.sr_base, idx, idx + 32, a.row_out.err, a.row_out.fallbacks);
        if (!okB) o.sf[1] = 0;
        uint8_t* cp = a.row_out.codes + row * a.row_out.ldc + gA * 16;
        *reinterpret_cast<uint4*>(cp) = o.codes[0];
        if (okB) *reinterpret_cast<uint4*>(cp + 16) = o.codes[1];
        if (a.row_out.mask) {
            a.row_out.mask[row * (a.C / 32) + gA] = o.mask[0];
            if (okB) a.row_out.mask[row * (a.C / 32) + gA + 1] = o.mask[1];
        }
    }
    // the 4 scale bytes of this tile row live in one atom word: combine the two lanes
    const uint32_t mine = o.sf[0] | (o.sf[1] << 8);
    const uint32_t other = __shfl_xor_sync(0xffffffffu, mine, 1);
    if (pp == 0 && okA) {
        uint8_t* sp = a.row_out.sf + sf_offset(row, c0 / 32, a.row_out.katoms);
        const uint32_t w = mine | (other << 16);
        if (nc == kTC)
            *reinterpret_cast<uint32_t*>(sp) = w;
        else
            for (int j = 0; j * 32 < nc; ++j) sp[j] = (uint8_t)(w >> (8 * j));
    }
}

// Col pass on one tile: thread -> (column pair t/4, row group t%4): A = column 2cp, B = 2cp + 1.
template <int ESZ, int ROUND>
__device__ __forceinline__ void tile_col_pass(const TileArgs& a, const uint4* tile, int64_t r0, int64_t c0, int nr,
                                              int nc, int tid) {
    constexpr int CPR = kTC * ESZ / 16;
    const int cp = tid >> 2, q = tid & 3;
    const bool ok = 2 * cp < nc && q * 32 < nr;
    Pair g;
    // the swizzle of row q*32 + i depends on (i + q) & 3 only: 4 precomputed chunk offsets
    const int kc = ESZ == 2 ? (cp >> 2) : (cp >> 1);
    int off[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) off[m] = tile_chunk(q * 32 + m, kc);
    const uint4* base = tile + q * 32 * CPR;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const uint4* chunk = base + i * CPR + off[i & 3];
        if (ESZ == 2) {
            bf16x2_to_f32(reinterpret_cast<const uint32_t*>(chunk)[cp & 3], g.p[i].x, g.p[i].y);
        } else {
            g.p[i] = reinterpret_cast<const float2*>(chunk)[cp & 1];
        }
    }
    const int64_t orow = c0 + 2 * cp, ogrp = r0 / 32 + q;
    PairOut o;
    o.sf[0] = o.sf[1] = 0;
    if (ok) {
        const QuantCfg& cf = a.col_cfg;
        const uint32_t s = cf.transform == kRandomized ? __ldg(cf.sign_bits + ogrp) : 0u;
        transform_pair(g, cf.transform, s, s, cf.prescale);
        const int64_t cld = cf.counter_ld ? cf.counter_ld : a.R;
        const uint64_t idx = cf.counter_start + (uint64_t)(orow * cld + ogrp * 32);
        o = quantize_pair<ROUND>(g, cf.sr_base, idx, idx + (uint64_t)cld, a.col_out.err, a.col_out.fallbacks);
        *reinterpret_cast<uint4*>(a.col_out.codes + orow * a.col_out.ldc + ogrp * 16) = o.codes[0];
        *reinterpret_cast<uint4*>(a.col_out.codes + (orow + 1) * a.col_out.ldc + ogrp * 16) = o.codes[1];
    }
    // gather the 4 scale bytes of each output row (lanes q = 0..3) into one atom word
    uint32_t wA = o.sf[0] << (8 * q), wB = o.sf[1] << (8 * q);
    wA |= __shfl_xor_sync(0xffffffffu, wA, 1);
    wA |= __shfl_xor_sync(0xffffffffu, wA, 2);
    wB |= __shfl_xor_sync(0xffffffffu, wB, 1);
    wB |= __shfl_xor_sync(0xffffffffu, wB, 2);
    if (2 * cp < nc && q < 2) {
        const uint32_t w = q == 0 ? wA : wB;
        uint8_t* sp = a.col_out.sf + sf_offset(orow + q, r0 / 32, a.col_out.katoms);
        if (nr == kTR)
            *reinterpret_cast<uint32_t*>(sp) = w;
        else
            for (int j = 0; j * 32 < nr; ++j) sp[j] = (uint8_t)(w >> (8 * j));
    }
}

template <int IN, bool ROWS, bool COLS, int ROUND>
__global__ void __launch_bounds__(256, IN == kInF32 ? 1 : 2) k_quant_tile(TileArgs a) {
    using G = TileGeom<IN>;
    extern __shared__ __align__(16) uint4 smem[];
    const int tid = threadIdx.x;
    const int64_t nRT = (a.R + kTR - 1) / kTR, nCT = (a.C + kTC - 1) / kTC, T = nRT * nCT;
    constexpr int STAGE = IN == kInMXFP4 ? G::RAW : G::DENSE;
    uint4* dec = smem + 2 * G::RAW;  // MXFP4 decoded tile

    int64_t t = blockIdx.x;
    if (t < T) tile_fill_async<IN>(a, smem, (t % nRT) * kTR, (t / nRT) * kTC, tid);
    cp_async_commit();
    for (int i = 0; t < T; ++i, t += gridDim.x) {
        const int64_t tn = t + gridDim.x;
        if (tn < T) tile_fill_async<IN>(a, smem + ((i + 1) & 1) * STAGE, (tn % nRT) * kTR, (tn / nRT) * kTC, tid);
        cp_async_commit();
        cp_async_wait1();
        __syncthreads();
        const int64_t r0 = (t % nRT) * kTR, c0 = (t / nRT) * kTC;
        const int nr = (int)(a.R - r0 < kTR ? a.R - r0 : kTR), nc = (int)(a.C - c0 < kTC ? a.C - c0 : kTC);
        const uint4* tile = smem + (i & 1) * STAGE;
        if (IN == kInMXFP4) {
            tile_decode_mxfp4(tile, dec, tid);
            __syncthreads();
            tile = dec;
        }
        if (ROWS) tile_row_pass<G::ESZ, ROUND>(a, tile, r0, c0, nr, nc, tid);
        if (COLS) tile_col_pass<G::ESZ, ROUND>(a, tile, r0, c0, nr, nc, tid);
        __syncthreads();
    }
}

}  // namespace qt

// ------------------------------------------------------------------------------- launchers
namespace qt {

int launch_signs(uint32_t* bits, int64_t start, int64_t n, uint64_t xi, cudaStream_t st) {
    if (n <= 0) return 0;
    uint64_t base = mix64(xi ^ mix64(kDomainSigns));
    int64_t nw = (n + 31) / 32;
    k_signs<<<(unsigned)((nw + 255) / 256), 256, 0, st>>>(bits, start, n, base);
    return (int)cudaGetLastError();
}

template <int IN, bool ROWS, bool COLS, int ROUND>
static void tile_launch(const TileArgs& a, dim3 grid, cudaStream_t st) {
    constexpr int smem = TileGeom<IN>::BYTES;
    static int ctas = 0;
    if (!ctas) {
        auto fn = k_quant_tile<IN, ROWS, COLS, ROUND>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int dev = 0, sms = 148, per_sm = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem);
        ctas = sms * (per_sm > 0 ? per_sm : 1);
    }
    const int64_t tiles = (int64_t)grid.x * grid.y;
    const unsigned n = (unsigned)(tiles < ctas ? tiles : ctas);
    k_quant_tile<IN, ROWS, COLS, ROUND><<<n, 256, smem, st>>>(a);
}

template <int IN, bool ROWS, bool COLS>
static void tile_round_dispatch(const TileArgs& a, int round, dim3 grid, cudaStream_t st) {
    if (round == kRtn)
        tile_launch<IN, ROWS, COLS, kRtn>(a, grid, st);
    else if (round == kSr)
        tile_launch<IN, ROWS, COLS, kSr>(a, grid, st);
    else
        tile_launch<IN, ROWS, COLS, kQuest>(a, grid, st);
}

// Row and/or column passes over one read of x[R, C] (both passes share the rounding mode).
int launch_quant_tile(const void* x, int in_type, int64_t ldx, const MxIn& mx, int64_t R, int64_t C,
                      const QuantCfg* row_cfg, const QuantOut* row_out, const QuantCfg* col_cfg,
                      const QuantOut* col_out, cudaStream_t st) {
    if (R == 0 || C == 0) return 0;
    const bool rows = row_cfg != nullptr, cols = col_cfg != nullptr;
    if (!rows && !cols) return 0;
    if (rows && cols && row_cfg->rounding != col_cfg->rounding) return 2003;
    if (in_type == kInMXFP4 && rows) return 2003;  // MXFP4 input is only re-quantized transposed
    TileArgs a{};
    a.x = x;
    a.ldx = ldx;
    a.mx = mx;
    a.R = R;
    a.C = C;
    if (rows) {
        a.row_cfg = *row_cfg;
        a.row_out = *row_out;
    }
    if (cols) {
        a.col_cfg = *col_cfg;
        a.col_out = *col_out;
    }
    const int round = rows ? row_cfg->rounding : col_cfg->rounding;
    dim3 grid((unsigned)((R + kTR - 1) / kTR), (unsigned)((C + kTC - 1) / kTC));
    if (in_type == kInMXFP4) {
        tile_round_dispatch<kInMXFP4, false, true>(a, round, grid, st);
    } else if (in_type == kInBF16) {
        if (rows && cols)
            tile_round_dispatch<kInBF16, true, true>(a, round, grid, st);
        else if (rows)
            tile_round_dispatch<kInBF16, true, false>(a, round, grid, st);
        else
            tile_round_dispatch<kInBF16, false, true>(a, round, grid, st);
    } else {
        if (rows && cols)
            tile_round_dispatch<kInF32, true, true>(a, round, grid, st);
        else if (rows)
            tile_round_dispatch<kInF32, true, false>(a, round, grid, st);
        else
            tile_round_dispatch<kInF32, false, true>(a, round, grid, st);
    }
    return (int)cudaGetLastError();
}

int launch_quant_rows(const void* x, int in_type, int64_t ldx, int64_t rows, int64_t cols, const QuantCfg& cfg,
                      const QuantOut& out, cudaStream_t st) {
    MxIn mx{nullptr, 0, nullptr, 0};
    return launch_quant_tile(x, in_type, ldx, mx, rows, cols, &cfg, &out, nullptr, nullptr, st);
}

}  // namespace qt
