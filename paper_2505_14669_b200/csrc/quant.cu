// quant.cu -- fused Hadamard + MXFP4 quantizer kernels (HBM-bound, one pass over the input).
//
//   k_signs        sign bitmap of the randomized Hadamard (rng.py:57-62, hadamard.py:77-85)
//   k_quant_rows   groups along the contiguous axis: forward X / W (H32 + QuEST) and the
//                  backward dy row operand (RHT32 + x0.75 + RTN/SR), qlinear.py:139-157, 213-228
//   k_quant_cols   transposing quantizer: groups along the strided axis, input bf16/f32 or an
//                  MXFP4 operand that is dequantized first (dy^T, deq(X_q)^T, deq(W_q)^T),
//                  qlinear.py:213-248
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

__device__ __forceinline__ void apply_transform(float (&v)[32], const QuantCfg& cfg, int64_t grp) {
    if (cfg.transform == kRandomized) {
        uint32_t s = __ldg(cfg.sign_bits + grp);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(__float_as_uint(v[j]) ^ (((s >> j) & 1u) << 31));
    }
    if (cfg.transform != kNone) fwht32(v);
    if (cfg.prescale != 1.0f) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __fmul_rn(v[j], cfg.prescale);
    }
}

// One thread per 32-element group of a row-major [rows, cols] input (cols % 32 == 0).
template <int IN>
__global__ void __launch_bounds__(256) k_quant_rows(const void* __restrict__ x, int64_t ldx, int64_t rows,
                                                    int64_t cols, QuantCfg cfg, QuantOut out) {
    const int64_t gpr = cols / 32;
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (gid >= rows * gpr) return;
    const int64_t r = gid / gpr, grp = gid - r * gpr;
    float v[32];
    if (IN == kInBF16) {
        const uint4* p = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(x) + r * ldx + grp * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint4 u = __ldg(p + q);
            uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                v[q * 8 + 2 * t] = __uint_as_float(w[t] << 16);
                v[q * 8 + 2 * t + 1] = __uint_as_float(w[t] & 0xFFFF0000u);
            }
        }
    } else {
        const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(x) + r * ldx + grp * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            float4 f = __ldg(p + q);
            v[4 * q] = f.x;
            v[4 * q + 1] = f.y;
            v[4 * q + 2] = f.z;
            v[4 * q + 3] = f.w;
        }
    }
    apply_transform(v, cfg, grp);
    GroupOut o = quantize_group(v, cfg.rounding, cfg.sr_base, cfg.counter_start + (uint64_t)(r * cols + grp * 32),
                                out.err, out.fallbacks);
    *reinterpret_cast<uint4*>(out.codes + r * out.ldc + grp * 16) = o.codes;
    out.sf[sf_offset(r, grp, out.katoms)] = (uint8_t)o.sf;
    if (out.mask) out.mask[r * gpr + grp] = o.mask;
}

// Transposing quantizer.  Input M[R, C] (row-major), output Q(T(M^T)) as an MXFP4 operand of
// shape [C, R] with groups along R.  CTA tile: 128 input rows x 64 input columns.
//   warp w: columns (w % 2) * 32 + lane, input rows (w / 2) * 32 .. +31 (one output group)
constexpr int kColTileR = 128, kColTileC = 64;

__device__ __forceinline__ float e2m1_decode(uint32_t nib) {
    uint32_t m = nib & 7u, e = m >> 1, mb = m & 1u;
    uint32_t bits = e == 0 ? (mb ? 0x3F000000u : 0u) : (((e + 126u) << 23) | (mb << 22));
    return __uint_as_float(bits | ((nib & 8u) << 28));
}

template <int IN>
__global__ void __launch_bounds__(256) k_quant_cols(const void* __restrict__ x, int64_t ldx, MxIn mx, int64_t R,
                                                    int64_t C, QuantCfg cfg, QuantOut out) {
    __shared__ float tile[kColTileR][kColTileC + 1];
    __shared__ __align__(16) uint8_t ocodes[kColTileC][80];
    __shared__ uint8_t osf[kColTileC][4];
    const int tid = threadIdx.x;
    const int64_t r0 = blockIdx.y * (int64_t)kColTileR, c0 = blockIdx.x * (int64_t)kColTileC;
    const int nr = (int)(R - r0 < kColTileR ? R - r0 : kColTileR), nc = (int)(C - c0 < kColTileC ? C - c0 : kColTileC);

    // ---- load (coalesced along C) into fp32 smem
    if (IN == kInBF16) {
        const __nv_bfloat16* xb = static_cast<const __nv_bfloat16*>(x);
        for (int i = tid; i < kColTileR * (kColTileC / 8); i += 256) {
            int rr = i / (kColTileC / 8), cc = (i % (kColTileC / 8)) * 8;
            if (rr < nr && cc < nc) {
                uint4 u = __ldg(reinterpret_cast<const uint4*>(xb + (r0 + rr) * ldx + c0 + cc));
                uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    tile[rr][cc + 2 * t] = __uint_as_float(w[t] << 16);
                    tile[rr][cc + 2 * t + 1] = __uint_as_float(w[t] & 0xFFFF0000u);
                }
            }
        }
    } else if (IN == kInF32) {
        const float* xf = static_cast<const float*>(x);
        for (int i = tid; i < kColTileR * (kColTileC / 4); i += 256) {
            int rr = i / (kColTileC / 4), cc = (i % (kColTileC / 4)) * 4;
            if (rr < nr && cc < nc) {
                float4 f = __ldg(reinterpret_cast<const float4*>(xf + (r0 + rr) * ldx + c0 + cc));
                tile[rr][cc] = f.x;
                tile[rr][cc + 1] = f.y;
                tile[rr][cc + 2] = f.z;
                tile[rr][cc + 3] = f.w;
            }
        }
    } else {
        // MXFP4 operand [R, C] (groups along C): dequantize exactly, code * 2^(e-127) in fp32
        // (codec.py:204-211 followed by the f32 cast of qlinear._values).
        int rr = tid / 2, g = tid % 2;
        if (rr < nr && g * 32 < nc) {
            int64_t grow = r0 + rr, ggrp = c0 / 32 + g;
            uint4 u = __ldg(reinterpret_cast<const uint4*>(mx.codes + grow * mx.ldc + ggrp * 16));
            float s = exp2i((int)mx.sf[sf_offset(grow, ggrp, mx.katoms)] - 127);
            uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int n = 0; n < 8; ++n) tile[rr][g * 32 + q * 8 + n] = e2m1_decode(w[q] >> (4 * n)) * s;
        }
    }
    __syncthreads();

    // ---- one output group per thread
    const int warp = tid / 32, lane = tid % 32;
    const int cc = (warp % 2) * 32 + lane, q = warp / 2;
    if (cc < nc && q * 32 < nr) {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = tile[q * 32 + i][cc];
        const int64_t ogrp = r0 / 32 + q;  // group index along R
        apply_transform(v, cfg, ogrp);
        const int64_t orow = c0 + cc;
        GroupOut o = quantize_group(v, cfg.rounding, cfg.sr_base, cfg.counter_start + (uint64_t)(orow * R + ogrp * 32),
                                    out.err, out.fallbacks);
        *reinterpret_cast<uint4*>(&ocodes[cc][q * 16]) = o.codes;
        osf[cc][q] = (uint8_t)o.sf;
        if (out.mask) out.mask[orow * (R / 32) + ogrp] = o.mask;
    }
    __syncthreads();

    // ---- coalesced stores: each output row gets up to 64 contiguous code bytes + 4 SF bytes
    {
        int row = tid / 4, chunk = tid % 4;
        if (row < nc && chunk * 32 < nr) {
            int64_t orow = c0 + row;
            *reinterpret_cast<uint4*>(out.codes + orow * out.ldc + (r0 / 32 + chunk) * 16) =
                *reinterpret_cast<const uint4*>(&ocodes[row][chunk * 16]);
        }
        if (tid < nc) {
            int64_t orow = c0 + tid, g0 = r0 / 32;
            int ng = (nr + 31) / 32;
            if (ng == 4) {
                uint32_t w = osf[tid][0] | (osf[tid][1] << 8) | (osf[tid][2] << 16) | ((uint32_t)osf[tid][3] << 24);
                *reinterpret_cast<uint32_t*>(out.sf + sf_offset(orow, g0, out.katoms)) = w;
            } else {
                for (int g = 0; g < ng; ++g) out.sf[sf_offset(orow, g0 + g, out.katoms)] = osf[tid][g];
            }
        }
    }
}

}  // namespace qt

// ------------------------------------------------------------------------------- launchers
using namespace qt;

namespace qt {
int launch_signs(uint32_t* bits, int64_t n, uint64_t xi, cudaStream_t st) {
    if (n <= 0) return 0;
    uint64_t base = mix64(xi ^ mix64(kDomainSigns));
    int64_t nw = (n + 31) / 32;
    k_signs<<<(unsigned)((nw + 255) / 256), 256, 0, st>>>(bits, n, base);
    return (int)cudaGetLastError();
}

int launch_quant_rows(const void* x, int in_type, int64_t ldx, int64_t rows, int64_t cols, const QuantCfg& cfg,
                      const QuantOut& out, cudaStream_t st) {
    if (rows == 0 || cols == 0) return 0;
    int64_t groups = rows * (cols / 32);
    unsigned grid = (unsigned)((groups + 255) / 256);
    if (in_type == kInBF16)
        k_quant_rows<kInBF16><<<grid, 256, 0, st>>>(x, ldx, rows, cols, cfg, out);
    else
        k_quant_rows<kInF32><<<grid, 256, 0, st>>>(x, ldx, rows, cols, cfg, out);
    return (int)cudaGetLastError();
}

int launch_quant_cols(const void* x, int in_type, int64_t ldx, const MxIn& mx, int64_t R, int64_t C,
                      const QuantCfg& cfg, const QuantOut& out, cudaStream_t st) {
    if (R == 0 || C == 0) return 0;
    dim3 grid((unsigned)((C + kColTileC - 1) / kColTileC), (unsigned)((R + kColTileR - 1) / kColTileR));
    if (in_type == kInBF16)
        k_quant_cols<kInBF16><<<grid, 256, 0, st>>>(x, ldx, mx, R, C, cfg, out);
    else if (in_type == kInF32)
        k_quant_cols<kInF32><<<grid, 256, 0, st>>>(x, ldx, mx, R, C, cfg, out);
    else
        k_quant_cols<kInMXFP4><<<grid, 256, 0, st>>>(x, ldx, mx, R, C, cfg, out);
    return (int)cudaGetLastError();
}
}  // namespace qt
