// quant.cu -- fused Hadamard + MXFP4 quantizer kernels (HBM-bound, one pass over the input).
//
//   k_signs        sign bitmap of the randomized Hadamard (rng.py:57-62, hadamard.py:77-85)
//   k_quant_rows   thread-per-group quantizer along the contiguous axis (forward X / W:
//                  H32 + QuEST, qlinear.py:139-157)
//   k_quant_tile   128 x 64 smem tile, up to two passes over the same data:
//                    row pass  groups along the contiguous axis (dy -> G, qlinear.py:214-225)
//                    col pass  groups along the strided axis = the transposed operand
//                              (dy^T -> G_t, deq(X_q)^T -> X_t, deq(W_q)^T -> W_t,
//                               qlinear.py:215, 234-246)
//                  so the backward's two dy operands come from ONE read of dy.
#include "launch.h"
#include "quant.cuh"

namespace qt {

__global__ void k_signs(uint32_t* bits, int64_t n, uint64_t base) {
    int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t nw = (n + 31) / 32;
    if (w >= nw) return;
    uint32_t m = 0;
    for (int j = 0; j < 32; ++j) {
        int64_t p = w * 32 + j;
        if (p < n) {
            uint64_t h = mix64(base + ((uint64_t)p + 1) * kGolden);
            m |= (uint32_t)(h >> 63) << j;
        }
    }
    bits[w] = m;
}

__device__ __forceinline__ void apply_transform(Grp& g, int transform, const uint32_t* sign_bits, int64_t grp,
                                                float prescale) {
    if (transform == kRandomized) flip_signs(g, __ldg(sign_bits + grp));
    if (transform != kNone) fwht32(g);
    if (prescale != 1.0f) scale_grp(g, prescale);
}

__device__ __forceinline__ void unpack_bf16x8(uint4 u, float* dst) {
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        dst[2 * t] = __uint_as_float(w[t] << 16);
        dst[2 * t + 1] = __uint_as_float(w[t] & 0xFFFF0000u);
    }
}

// ------------------------------------------------------------------------ k_quant_rows
template <int IN, int ROUND>
__global__ void __launch_bounds__(256, 3) k_quant_rows(const void* __restrict__ x, int64_t ldx, int64_t rows,
                                                       int64_t cols, QuantCfg cfg, QuantOut out) {
    const int64_t gpr = cols / 32;
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (gid >= rows * gpr) return;
    const int64_t r = gid / gpr, grp = gid - r * gpr;
    Grp g;
    float tmp[8];
    if (IN == kInBF16) {
        const uint4* p = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(x) + r * ldx + grp * 32);
        uint4 u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = __ldg(p + q);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            unpack_bf16x8(u[q], tmp);
#pragma unroll
            for (int t = 0; t < 8; ++t) g.v(q * 8 + t) = tmp[t];
        }
    } else {
        const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(x) + r * ldx + grp * 32);
        float4 f[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) f[q] = __ldg(p + q);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            g.v(4 * q) = f[q].x;
            g.v(4 * q + 1) = f[q].y;
            g.v(4 * q + 2) = f[q].z;
            g.v(4 * q + 3) = f[q].w;
        }
    }
    apply_transform(g, cfg.transform, cfg.sign_bits, grp, cfg.prescale);
    GroupOut o = quantize_grp<ROUND>(g, cfg.sr_base, cfg.counter_start + (uint64_t)(r * cols + grp * 32), out.err,
                                     out.fallbacks);
    *reinterpret_cast<uint4*>(out.codes + r * out.ldc + grp * 16) = o.codes;
    out.sf[sf_offset(r, grp, out.katoms)] = (uint8_t)o.sf;
    if (out.mask) out.mask[r * gpr + grp] = o.mask;
}

// Transform only (kernels.fwht seam, hadamard.py:72-91): out = prescale * H32(x (.) s), fp32 out.
__global__ void __launch_bounds__(256) k_transform_rows(const float* __restrict__ x, float* __restrict__ out,
                                                       int64_t rows, int64_t cols, int transform,
                                                       const uint32_t* sign_bits, float prescale) {
    const int64_t gpr = cols / 32;
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (gid >= rows * gpr) return;
    const int64_t r = gid / gpr, grp = gid - r * gpr;
    Grp g;
#pragma unroll
    for (int j = 0; j < 32; ++j) g.v(j) = x[r * cols + grp * 32 + j];
    apply_transform(g, transform, sign_bits, grp, prescale);
#pragma unroll
    for (int j = 0; j < 32; ++j) out[r * cols + grp * 32 + j] = g.v(j);
}

int launch_transform_rows(const float* x, float* out, int64_t rows, int64_t cols, int transform,
                          const uint32_t* sign_bits, float prescale, cudaStream_t st) {
    if (rows == 0 || cols == 0) return 0;
    int64_t groups = rows * (cols / 32);
    k_transform_rows<<<(unsigned)((groups + 255) / 256), 256, 0, st>>>(x, out, rows, cols, transform, sign_bits,
                                                                        prescale);
    return (int)cudaGetLastError();
}

// ------------------------------------------------------------------------ k_quant_tile
// Tile: 128 rows x 64 columns, held in smem as bf16 (ESZ = 2) or fp32 (ESZ = 4) in 16-byte chunks.
// Chunk k of row r lives at physical chunk k ^ sw(r), sw(r) = ((r & 3) + (r >> 5)) & 3, which makes
// the fill (consecutive chunks of a row), the row pass (4 rows x 2 groups per 8-lane phase) and the
// col pass (one chunk of 4 rows 32 apart per load) bank-conflict free for bf16 tiles.
constexpr int kTR = 128, kTC = 64;

struct TileArgs {
    const void* x;      // dense input (bf16 / fp32), row stride ldx
    int64_t ldx;
    MxIn mx;            // MXFP4 input (in_type kInMXFP4)
    int64_t R, C;
    QuantCfg row_cfg, col_cfg;
    QuantOut row_out, col_out;
};

__device__ __forceinline__ int tile_sw(int r) { return ((r & 3) + (r >> 5)) & 3; }

template <int IN, bool ROWS, bool COLS, int ROUND>
__global__ void __launch_bounds__(256, 3) k_quant_tile(TileArgs a) {
    constexpr int ESZ = IN == kInF32 ? 4 : 2;          // smem element bytes
    constexpr int CPR = kTC * ESZ / 16;                  // 16-byte chunks per row: 8 or 16
    __shared__ __align__(16) uint4 tile[kTR * CPR];
    const int tid = threadIdx.x;
    const int64_t r0 = blockIdx.x * (int64_t)kTR, c0 = blockIdx.y * (int64_t)kTC;
    const int nr = (int)(a.R - r0 < kTR ? a.R - r0 : kTR), nc = (int)(a.C - c0 < kTC ? a.C - c0 : kTC);

    // ---- fill
    if (IN == kInMXFP4) {
        // thread -> (row t/2, group t%2): 16 code bytes + 1 scale, decoded exactly to bf16
        const int rr = tid >> 1, gg = tid & 1;
        uint4 outc[4] = {};
        if (rr < nr && gg * 32 < nc) {
            const int64_t grow = r0 + rr, ggrp = c0 / 32 + gg;
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(a.mx.codes + grow * a.mx.ldc + ggrp * 16));
            const uint32_t e = a.mx.sf[sf_offset(grow, ggrp, a.mx.katoms)];
            const float s = exp2i((int)e - 127);
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t bw[4];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    float2 f = e2m1x2_to_f32((w[q] >> (8 * b)) & 0xFFu);
                    // code * 2^(e-127) is exact in fp32 and in bf16 (<= 3 significant bits)
                    uint32_t lo = __float_as_uint(f.x * s) >> 16, hi = __float_as_uint(f.y * s) >> 16;
                    bw[b] = lo | (hi << 16);
                }
                outc[q] = make_uint4(bw[0], bw[1], bw[2], bw[3]);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) tile[rr * CPR + ((gg * 4 + q) ^ tile_sw(rr))] = outc[q];
    } else {
        const uint8_t* xb = static_cast<const uint8_t*>(a.x);
        uint4 u[kTR * CPR / 256];
#pragma unroll
        for (int it = 0; it < kTR * CPR / 256; ++it) {
            const int id = it * 256 + tid, rr = id / CPR, k = id % CPR;
            u[it] = make_uint4(0, 0, 0, 0);
            if (rr < nr && k * (16 / ESZ) < nc)
                u[it] = __ldg(reinterpret_cast<const uint4*>(xb + ((r0 + rr) * a.ldx + c0) * ESZ + k * 16));
        }
#pragma unroll
        for (int it = 0; it < kTR * CPR / 256; ++it) {
            const int id = it * 256 + tid, rr = id / CPR, k = id % CPR;
            tile[rr * CPR + (k ^ tile_sw(rr))] = u[it];
        }
    }
    __syncthreads();

    // ---- row pass: thread -> (row t/2, group t%2)
    if (ROWS) {
        const int rr = tid >> 1, gg = tid & 1;
        const bool ok = rr < nr && gg * 32 < nc;
        Grp g;
        if (ESZ == 2) {
            float tmp[8];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                unpack_bf16x8(tile[rr * CPR + ((gg * 4 + q) ^ tile_sw(rr))], tmp);
#pragma unroll
                for (int t = 0; t < 8; ++t) g.v(q * 8 + t) = tmp[t];
            }
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                uint4 u = tile[rr * CPR + ((gg * 8 + q) ^ tile_sw(rr))];
                g.v(q * 4) = __uint_as_float(u.x);
                g.v(q * 4 + 1) = __uint_as_float(u.y);
                g.v(q * 4 + 2) = __uint_as_float(u.z);
                g.v(q * 4 + 3) = __uint_as_float(u.w);
            }
        }
        const int64_t row = r0 + rr, grp = c0 / 32 + gg;
        GroupOut o;
        o.sf = 0;
        if (ok) {
            apply_transform(g, a.row_cfg.transform, a.row_cfg.sign_bits, grp, a.row_cfg.prescale);
            o = quantize_grp<ROUND>(g, a.row_cfg.sr_base, a.row_cfg.counter_start + (uint64_t)(row * a.C + grp * 32),
                                    a.row_out.err, a.row_out.fallbacks);
            *reinterpret_cast<uint4*>(a.row_out.codes + row * a.row_out.ldc + grp * 16) = o.codes;
            if (a.row_out.mask) a.row_out.mask[row * (a.C / 32) + grp] = o.mask;
        }
        const uint32_t other = __shfl_xor_sync(0xffffffffu, o.sf, 1);
        if (ok && gg == 0) {
            if (nc > 32)  // groups grp, grp+1 are adjacent bytes of one atom word (grp even)
                *reinterpret_cast<uint16_t*>(a.row_out.sf + sf_offset(row, grp, a.row_out.katoms)) =
                    (uint16_t)(o.sf | (other << 8));
            else
                a.row_out.sf[sf_offset(row, grp, a.row_out.katoms)] = (uint8_t)o.sf;
        }
    }

    // ---- col pass: thread -> (column t/4, row group t%4)
    if (COLS) {
        const int cc = tid >> 2, q = tid & 3;
        const bool ok = cc < nc && q * 32 < nr;
        Grp g;
        const int k = cc / (16 / ESZ), off = cc % (16 / ESZ);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const int rr = q * 32 + i;
            const uint8_t* base = reinterpret_cast<const uint8_t*>(&tile[rr * CPR + (k ^ tile_sw(rr))]);
            if (ESZ == 2)
                g.v(i) = __uint_as_float((uint32_t)(*reinterpret_cast<const uint16_t*>(base + off * 2)) << 16);
            else
                g.v(i) = *reinterpret_cast<const float*>(base + off * 4);
        }
        const int64_t orow = c0 + cc, ogrp = r0 / 32 + q;
        GroupOut o;
        o.sf = 0;
        if (ok) {
            apply_transform(g, a.col_cfg.transform, a.col_cfg.sign_bits, ogrp, a.col_cfg.prescale);
            o = quantize_grp<ROUND>(g, a.col_cfg.sr_base, a.col_cfg.counter_start + (uint64_t)(orow * a.R + ogrp * 32),
                                    a.col_out.err, a.col_out.fallbacks);
            *reinterpret_cast<uint4*>(a.col_out.codes + orow * a.col_out.ldc + ogrp * 16) = o.codes;
        }
        // gather the 4 scale bytes of this column into lane q == 0 (one 32-bit atom word)
        uint32_t sfw = o.sf << (8 * q);
        sfw |= __shfl_xor_sync(0xffffffffu, sfw, 1);
        sfw |= __shfl_xor_sync(0xffffffffu, sfw, 2);
        if (ok && q == 0) {
            if (nr == kTR) {
                *reinterpret_cast<uint32_t*>(a.col_out.sf + sf_offset(orow, ogrp, a.col_out.katoms)) = sfw;
            } else {
                for (int j = 0; j * 32 < nr; ++j)
                    a.col_out.sf[sf_offset(orow, ogrp + j, a.col_out.katoms)] = (uint8_t)(sfw >> (8 * j));
            }
        }
    }
}

}  // namespace qt

// ------------------------------------------------------------------------------- launchers
namespace qt {

int launch_signs(uint32_t* bits, int64_t n, uint64_t xi, cudaStream_t st) {
    if (n <= 0) return 0;
    uint64_t base = mix64(xi ^ mix64(kDomainSigns));
    int64_t nw = (n + 31) / 32;
    k_signs<<<(unsigned)((nw + 255) / 256), 256, 0, st>>>(bits, n, base);
    return (int)cudaGetLastError();
}

template <int IN>
static void rows_dispatch(const void* x, int64_t ldx, int64_t rows, int64_t cols, const QuantCfg& cfg,
                          const QuantOut& out, unsigned grid, cudaStream_t st) {
    if (cfg.rounding == kQuest)
        k_quant_rows<IN, kQuest><<<grid, 256, 0, st>>>(x, ldx, rows, cols, cfg, out);
    else if (cfg.rounding == kRtn)
        k_quant_rows<IN, kRtn><<<grid, 256, 0, st>>>(x, ldx, rows, cols, cfg, out);
    else
        k_quant_rows<IN, kSr><<<grid, 256, 0, st>>>(x, ldx, rows, cols, cfg, out);
}

int launch_quant_rows(const void* x, int in_type, int64_t ldx, int64_t rows, int64_t cols, const QuantCfg& cfg,
                      const QuantOut& out, cudaStream_t st) {
    if (rows == 0 || cols == 0) return 0;
    int64_t groups = rows * (cols / 32);
    unsigned grid = (unsigned)((groups + 255) / 256);
    if (in_type == kInBF16)
        rows_dispatch<kInBF16>(x, ldx, rows, cols, cfg, out, grid, st);
    else
        rows_dispatch<kInF32>(x, ldx, rows, cols, cfg, out, grid, st);
    return (int)cudaGetLastError();
}

template <int IN, bool ROWS, bool COLS>
static void tile_round_dispatch(const TileArgs& a, int round, dim3 grid, cudaStream_t st) {
    if (round == kRtn)
        k_quant_tile<IN, ROWS, COLS, kRtn><<<grid, 256, 0, st>>>(a);
    else if (round == kSr)
        k_quant_tile<IN, ROWS, COLS, kSr><<<grid, 256, 0, st>>>(a);
    else
        k_quant_tile<IN, ROWS, COLS, kQuest><<<grid, 256, 0, st>>>(a);
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

}  // namespace qt
