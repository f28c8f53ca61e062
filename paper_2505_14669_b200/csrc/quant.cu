// quant.cu -- fused Hadamard + MXFP4 quantizer kernels (v3: scalar one-group pipeline, qgroup.cuh).
//
//   k_signs       sign bitmap of the randomized Hadamard (rng.py:57-62, hadamard.py:77-85)
//   k_quant       persistent tile kernel; per 128 x 128 tile (64 x 128 for fp32 input) up to two passes:
//                   row pass  groups along the contiguous axis: forward X / W (H32 + QuEST,
//                             qlinear.py:139-157), the backward dy operand G (RHT32 + x0.75 + RTN/SR,
//                             qlinear.py:214-225), or any quantize_{rtn,sr,quest} of the plugin seam
//                   col pass  groups along the strided axis = the transposed operand, fed by
//                             * the dense tile  (dy^T -> G_t, qlinear.py:234-245: one read of dy
//                               gives both dy operands), or
//                             * MXFP4 codes     deq(X_q)^T -> X_t and deq(W_q)^T -> W_t
//                               (qlinear.py:206-207, 215, 235), either straight from the row pass of
//                               the same tile (fused forward: X is read once for X_q AND X_t) or
//                               from a saved operand in HBM (lazy requantization)
//   k_transform_rows  transform only (the kernels.fwht seam)
//
// Thread mapping (256 threads):
//   row pass  thread -> one tile row, 2 groups (processed one after the other; fp32 tiles: 1 group)
//   col pass  thread -> column pair cp = t % 64 (groups A = column 2cp, B = 2cp+1), row group t / 64
// Shared-memory layouts are XOR-swizzled so that the fill, both passes and the code exchange between
// them are bank-conflict free (see tile_chunk / codes_chunk).
#include "launch.h"
#include "qgroup.cuh"

namespace qt {

__device__ __forceinline__ void signs_word(uint32_t* bits, int64_t start, int64_t n, uint64_t base, int64_t w) {
    uint32_t m = 0;
    for (int j = 0; j < 32; ++j) {
        const int64_t p = w * 32 + j;
        if (p < n) {
            const uint64_t h = mix64(base + ((uint64_t)(start + p) + 1) * kGolden);
            m |= (uint32_t)(h >> 63) << j;
        }
    }
    bits[w] = m;
}
// two sign vectors of one seed in one launch (a layer's d_out and token signs): blocks [0, nba) -> a
__global__ void k_signs2(uint32_t* a, int64_t sa, int64_t na, int64_t nba, uint32_t* b, int64_t sb, int64_t nb,
                         uint64_t base) {
    const bool first = blockIdx.x < nba;
    const int64_t w = (first ? blockIdx.x : blockIdx.x - nba) * (int64_t)blockDim.x + threadIdx.x;
    if (first) {
        if (w < (na + 31) / 32) signs_word(a, sa, na, base, w);
    } else if (w < (nb + 31) / 32) {
        signs_word(b, sb, nb, base, w);
    }
}
// k_signs2 with the seed read from device memory: the per-step layer seeds of a captured training step
__global__ void k_signs2_dev(uint32_t* a, int64_t sa, int64_t na, int64_t nba, uint32_t* b, int64_t sb, int64_t nb,
                             const uint64_t* xi) {
    const uint64_t base = mix64(*xi ^ mix64(kDomainSigns));
    const bool first = blockIdx.x < nba;
    const int64_t w = (first ? blockIdx.x : blockIdx.x - nba) * (int64_t)blockDim.x + threadIdx.x;
    if (first) {
        if (w < (na + 31) / 32) signs_word(a, sa, na, base, w);
    } else if (w < (nb + 31) / 32) {
        signs_word(b, sb, nb, base, w);
    }
}

__device__ __forceinline__ uint64_t derive2(uint64_t acc, uint64_t p) {  // one fold of rng.derive_seed
    return mix64(acc ^ p) + kGolden;
}
// xi[l] = derive_seed(derive_seed(seed, 4, *step), ids[l]) (train.py:346-348), then ++*step: one block
__global__ void k_layer_seeds(uint64_t* xi, const uint64_t* ids, int n, uint64_t seed, int64_t* step, int inc) {
    const uint64_t s = (uint64_t)*step;
    const uint64_t d = mix64(derive2(derive2(derive2(0x243F6A8885A308D3ULL, seed), 4), s));
    for (int l = threadIdx.x; l < n; l += blockDim.x) xi[l] = mix64(derive2(derive2(0x243F6A8885A308D3ULL, d), ids[l]));
    __syncthreads();
    if (threadIdx.x == 0 && inc) *step = (int64_t)(s + 1);
}

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

// --------------------------------------------------------------------------------- k_quant
enum RowMode : int { kRowOff = -1 };           // otherwise the rounding (kQuest / kRtn / kSr)
enum ColSrc : int { kColOff = 0, kColDense = 1, kColCodes = 2 };

constexpr int kTC = 128;  // tile columns (4 groups)

struct TileArgs {
    const void* x;      // dense input (bf16 / fp32), row stride ldx elements
    int64_t ldx;
    MxIn mx;            // MXFP4 input (in_type kInMXFP4), groups along C
    int64_t R, C;
    QuantCfg row_cfg, col_cfg;
    QuantOut row_out, col_out;
};

// dense tile: 16-byte chunk k of row r lives at chunk tile_chunk(r, k) of that row
template <int ESZ>
__device__ __forceinline__ int tile_chunk(int r, int k) {
    if (ESZ == 2) return k ^ ((((r + (r >> 5)) & 3) << 1) ^ ((k >> 3) & 1));
    return k ^ ((k >> 3) & 3) ^ ((r & 1) << 2);
}
// codes tile ([rows][64 B]): 16-byte chunk g (= group g of the row) at chunk g ^ ((r >> 1) & 1)
__device__ __forceinline__ int codes_byte(int r, int b) { return r * 64 + (b ^ (((r >> 1) & 1) << 4)); }

template <int IN>
struct Geom {
    static constexpr int ESZ = IN == kInF32 ? 4 : 2;
    static constexpr int TR = IN == kInF32 ? 64 : 128;     // tile rows
    static constexpr int CPR = kTC * ESZ / 16;              // dense chunks per row
    static constexpr int DENSE = TR * CPR;                  // dense chunks per tile
    static constexpr int RAW = TR * 4 + 512 / 16;           // MXFP4: code chunks + one scale atom
    static constexpr int STAGE = IN == kInMXFP4 ? RAW : DENSE;
    static constexpr int TSTRIDE = TR + 4;                  // floats per scale-table row (4 groups)
    // smem: 2 input stages | codes tile (TR x 64 B) | scale table [4][TSTRIDE] f32 | row LUT [64] | col LUT [TR]
    static constexpr int OFF_CODES = 2 * STAGE * 16;
    static constexpr int OFF_T = OFF_CODES + TR * 64;
    static constexpr int OFF_RLUT = OFF_T + 4 * TSTRIDE * 4;
    static constexpr int OFF_CLUT = OFF_RLUT + 64 * 4;
    static constexpr int BYTES = OFF_CLUT + TR * 4;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <int IN>
__device__ __forceinline__ void tile_fill_async(const TileArgs& a, uint8_t* buf, int64_t r0, int64_t c0, int tid) {
    using G = Geom<IN>;
    const int nr = (int)(a.R - r0 < G::TR ? a.R - r0 : G::TR), nc = (int)(a.C - c0 < kTC ? a.C - c0 : kTC);
    uint4* b16 = reinterpret_cast<uint4*>(buf);
    if (IN == kInMXFP4) {
#pragma unroll
        for (int it = 0; it < G::TR * 4 / 256; ++it) {
            const int id = it * 256 + tid, rr = id >> 2, part = id & 3;
            const bool ok = rr < nr && part * 32 < nc;
            const uint8_t* src = a.mx.codes + (ok ? (r0 + rr) * a.mx.ldc + c0 / 2 + part * 16 : 0);
            cp_async16(buf + codes_byte(rr, part * 16), src, ok);
        }
        if (tid < 32) {
            const uint8_t* src = a.mx.sf + ((r0 / 128) * a.mx.katoms + c0 / 128) * 512 + tid * 16;
            cp_async16(b16 + G::TR * 4 + tid, src, true);
        }
    } else {
        const uint8_t* xb = static_cast<const uint8_t*>(a.x);
#pragma unroll
        for (int it = 0; it < G::DENSE / 256; ++it) {
            const int id = it * 256 + tid, rr = id / G::CPR, k = id % G::CPR;
            const bool ok = rr < nr && k * (16 / G::ESZ) < nc;
            const uint8_t* src = xb + (ok ? ((r0 + rr) * a.ldx + c0) * G::ESZ + k * 16 : 0);
            cp_async16(b16 + rr * G::CPR + tile_chunk<G::ESZ>(rr, k), src, ok);
        }
    }
}

// ---------------------------------------------------------------------- group loaders
// Row group g of tile row rr into v, with the transform's first butterfly stage fused into the load.
template <int IN>
__device__ __forceinline__ void load_row_group(const uint4* tile, int rr, int g, int transform, const uint32_t* rlut,
                                               const uint32_t* sign_bits, int64_t gglob, float (&v)[32]) {
    using G = Geom<IN>;
    if (IN == kInBF16) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 c = tile[rr * G::CPR + tile_chunk<2>(rr, g * 4 + q)];
            uint4 m = make_uint4(0, 0, 0, 0);
            if (transform == kRandomized) m = reinterpret_cast<const uint4*>(rlut)[g * 4 + q];
            const uint32_t w[4] = {c.x ^ m.x, c.y ^ m.y, c.z ^ m.z, c.w ^ m.w};
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
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint4 c = tile[rr * G::CPR + tile_chunk<4>(rr, g * 8 + q)];
            v[4 * q] = __uint_as_float(c.x);
            v[4 * q + 1] = __uint_as_float(c.y);
            v[4 * q + 2] = __uint_as_float(c.z);
            v[4 * q + 3] = __uint_as_float(c.w);
        }
        if (transform == kRandomized) {
            const uint32_t s = __ldg(sign_bits + gglob);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(__float_as_uint(v[j]) ^ ((s >> j) << 31));
        }
        if (transform != kNone) fwht_full(v);
    }
}

// Column pair (columns 2cp, 2cp+1; tile rows q*32 .. q*32+31) of a dense tile into a / b.
template <int IN>
__device__ __forceinline__ void load_col_pair(const uint4* tile, int cp, int q, int transform, const uint32_t* clut,
                                              float (&a)[32], float (&b)[32]) {
    using G = Geom<IN>;
    const int r0 = q * 32;
    if (IN == kInBF16) {
        const uint32_t* t32 = reinterpret_cast<const uint32_t*>(tile) + r0 * G::CPR * 4 + (cp & 3);
        const int kc = cp >> 2;
        // the swizzle of row q*32 + i depends on (i + q) & 3 only: 4 word offsets, hoisted
        int off[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) off[m] = tile_chunk<2>(r0 + m, kc) * 4;
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            const int r = r0 + i;
            uint32_t w0 = t32[i * G::CPR * 4 + off[i & 3]];
            uint32_t w1 = t32[(i + 1) * G::CPR * 4 + off[(i + 1) & 3]];
            if (transform == kRandomized) {
                const uint2 m = *reinterpret_cast<const uint2*>(clut + r);
                w0 ^= m.x;
                w1 ^= m.y;
            }
            if (transform != kNone) {
                const float nA = bf_lo(w1), nB = bf_hi(w1);
                a[i] = __fmul_rn(fh_add_lo(w0, nA), kHc);
                a[i + 1] = __fmul_rn(fh_sub_lo(w0, nA), kHc);
                b[i] = __fmul_rn(fh_add_hi(w0, nB), kHc);
                b[i + 1] = __fmul_rn(fh_sub_hi(w0, nB), kHc);
            } else {
                a[i] = bf_lo(w0);
                b[i] = bf_hi(w0);
                a[i + 1] = bf_lo(w1);
                b[i + 1] = bf_hi(w1);
            }
        }
        if (transform != kNone) {
            fwht_tail(a);
            fwht_tail(b);
        }
    } else {
        const float2* t64 = reinterpret_cast<const float2*>(tile);
        const int kc = cp >> 1, hf = cp & 1;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const int r = r0 + i;
            float2 f = t64[(r * G::CPR + tile_chunk<4>(r, kc)) * 2 + hf];
            if (transform == kRandomized) {
                const uint32_t m = clut[r] & 0x80000000u;
                f.x = __uint_as_float(__float_as_uint(f.x) ^ m);
                f.y = __uint_as_float(__float_as_uint(f.y) ^ m);
            }
            a[i] = f.x;
            b[i] = f.y;
        }
        if (transform != kNone) {
            fwht_full(a);
            fwht_full(b);
        }
    }
}

// Column pair from an MXFP4 codes tile: value = code * T[g][r] (T = +-2^(e-127), sign = RHT flip).
__device__ __forceinline__ void load_col_codes(const uint8_t* codes, const float* T, int tstride, int cp, int q,
                                               int transform, float (&a)[32], float (&b)[32]) {
    const int g = cp >> 4;
    const float4* trow = reinterpret_cast<const float4*>(T + g * tstride + q * 32);
#pragma unroll
    for (int i4 = 0; i4 < 8; ++i4) {
        const float4 s = trow[i4];
        const float sv[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i4 * 4 + u, r = q * 32 + i;
            const float2 f = e2m1x2_to_f32(codes[codes_byte(r, cp)]);
            a[i] = __fmul_rn(f.x, sv[u]);
            b[i] = __fmul_rn(f.y, sv[u]);
        }
    }
    if (transform != kNone) {
        fwht_full(a);
        fwht_full(b);
    }
}

// One column c (rows 32q .. 32q+31) of the staged codes tile: the nibble c % 2 of byte pair c / 2.
__device__ __forceinline__ void load_col_code1(const uint8_t* codes, const float* T, int tstride, int c, int q,
                                               int transform, float (&v)[32]) {
    const int cp = c >> 1, hi = c & 1;
    const float4* trow = reinterpret_cast<const float4*>(T + (c >> 5) * tstride + q * 32);
#pragma unroll
    for (int i4 = 0; i4 < 8; ++i4) {
        const float4 s = trow[i4];
        const float sv[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i4 * 4 + u, r = q * 32 + i;
            const float2 f = e2m1x2_to_f32(codes[codes_byte(r, cp)]);
            v[i] = __fmul_rn(hi ? f.y : f.x, sv[u]);
        }
    }
    if (transform != kNone) fwht_full(v);
}

// ------------------------------------------------------------------------------- kernel
template <int IN, int ROW, int COL, int CROUND>
__global__ void __launch_bounds__(256, 2) k_quant(TileArgs a) {
    using G = Geom<IN>;
    constexpr int TR = G::TR;
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t* codes_s = smem + G::OFF_CODES;
    float* T = reinterpret_cast<float*>(smem + G::OFF_T);
    uint32_t* rlut = reinterpret_cast<uint32_t*>(smem + G::OFF_RLUT);
    uint32_t* clut = reinterpret_cast<uint32_t*>(smem + G::OFF_CLUT);
    const int tid = threadIdx.x;
    const int64_t nRT = (a.R + TR - 1) / TR, nCT = (a.C + kTC - 1) / kTC, NT = nRT * nCT;
    const QuantCfg& rc = a.row_cfg;
    const QuantCfg& cc = a.col_cfg;

    int64_t t = blockIdx.x;
    if (t < NT) tile_fill_async<IN>(a, smem, (t % nRT) * TR, (t / nRT) * kTC, tid);
    cp_async_commit();
    for (int it = 0; t < NT; ++it, t += gridDim.x) {
        const int64_t tn = t + gridDim.x;
        if (tn < NT) tile_fill_async<IN>(a, smem + ((it + 1) & 1) * G::STAGE * 16, (tn % nRT) * TR, (tn / nRT) * kTC, tid);
        cp_async_commit();
        const int64_t r0 = (t % nRT) * TR, c0 = (t / nRT) * kTC;
        const int nr = (int)(a.R - r0 < TR ? a.R - r0 : TR), nc = (int)(a.C - c0 < kTC ? a.C - c0 : kTC);
        // per-tile sign LUTs: row pass (bf16 words along C), col pass (rows)
        if (ROW != kRowOff && IN == kInBF16 && rc.transform == kRandomized && tid < 64) {
            const int64_t col = c0 + 2 * tid;
            uint32_t m = 0;
            if (col < a.C) {
                const uint32_t s = __ldg(rc.sign_bits + (col >> 5));
                const int b = (int)(col & 31);
                m = (((s >> b) & 1u) << 15) | (((s >> (b + 1)) & 1u) << 31);
            }
            rlut[tid] = m;
        }
        if (COL != kColOff && cc.transform == kRandomized && tid < TR) {
            const int64_t row = r0 + tid;
            uint32_t m = 0;
            if (row < a.R) m = ((__ldg(cc.sign_bits + (row >> 5)) >> (row & 31)) & 1u) ? 0x80008000u : 0u;
            clut[tid] = m;
        }
        cp_async_wait1();
        __syncthreads();
        const uint8_t* stage = smem + (it & 1) * G::STAGE * 16;
        const uint4* tile = reinterpret_cast<const uint4*>(stage);

        if (IN == kInMXFP4) {
            // scale table of the staged operand: T[g][r] = (+-) 2^(e - 127)
            const uint8_t* atom = stage + TR * 64;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int id = tid + 256 * u, r = id & 127, g = id >> 7;
                const int e = atom[(r & 31) * 16 + ((r >> 5) & 3) * 4 + g];
                float s = exp2i(e - 127);
                if (cc.transform == kRandomized && (clut[r] & 1u << 31)) s = -s;
                T[g * G::TSTRIDE + r] = s;
            }
            __syncthreads();
        }

        // ---------------------------------------------------------------- row pass
        if (ROW != kRowOff) {
            constexpr int GPT = TR == 128 ? 2 : 1;  // groups per thread
            const int rr = TR == 128 ? tid >> 1 : tid >> 2;
            const int64_t row = r0 + rr;
            uint32_t sfw = 0;
#pragma unroll
            for (int h = 0; h < GPT; ++h) {
                const int g = TR == 128 ? 2 * (tid & 1) + h : (tid & 3);
                const bool ok = rr < nr && g * 32 < nc;
                const int64_t gg = c0 / 32 + g;
                int e = 0;
                if (ok) {
                    float v[32];
                    load_row_group<IN>(tile, rr, g, rc.transform, rlut, rc.sign_bits, gg, v);
                    const int64_t cld = rc.counter_ld ? rc.counter_ld : a.C;
                    uint4 codes;
                    uint32_t mask;
                    e = quant_group<ROW>(v, rc, rc.counter_start + (uint64_t)(row * cld + gg * 32), a.row_out.err,
                                         a.row_out.fallbacks, codes, mask);
                    *reinterpret_cast<uint4*>(a.row_out.codes + row * a.row_out.ldc + gg * 16) = codes;
                    if (a.row_out.mask) a.row_out.mask[row * (a.C / 32) + gg] = mask;
                    if (COL == kColCodes) {
                        *reinterpret_cast<uint4*>(codes_s + codes_byte(rr, g * 16)) = codes;
                        float s = exp2i(e - 127);
                        if (cc.transform == kRandomized && (clut[rr] & 1u << 31)) s = -s;
                        T[g * G::TSTRIDE + rr] = s;
                    }
                }
                sfw |= (uint32_t)e << (8 * g);
            }
            // the 4 scale bytes of this tile row form one atom word
            if (TR == 128) {
                sfw |= __shfl_xor_sync(0xffffffffu, sfw, 1);
            } else {
                sfw |= __shfl_xor_sync(0xffffffffu, sfw, 1);
                sfw |= __shfl_xor_sync(0xffffffffu, sfw, 2);
            }
            if ((tid & (TR == 128 ? 1 : 3)) == 0 && rr < nr) {
                uint8_t* sp = a.row_out.sf + sf_offset(row, c0 / 32, a.row_out.katoms);
                if (nc == kTC)
                    *reinterpret_cast<uint32_t*>(sp) = sfw;
                else
                    for (int j = 0; j * 32 < nc; ++j) sp[j] = (uint8_t)(sfw >> (8 * j));
            }
            if (COL == kColCodes) __syncthreads();
        }

        // ---------------------------------------------------------------- col pass
        if (COL == kColCodes && TR == 64) {
            // 64-row (fp32) tiles hold 2 column groups per column: one column per thread keeps all 256 threads
            // busy (the pair layout below would leave half of them idle)
            const int c = tid & 127, q = tid >> 7;
            if (c < nc && q * 32 < nr) {
                float v[32];
                load_col_code1(codes_s, T, G::TSTRIDE, c, q, cc.transform, v);
                const int64_t orow = c0 + c, ogrp = r0 / 32 + q;
                const int64_t cld = cc.counter_ld ? cc.counter_ld : a.R;
                uint4 codes;
                uint32_t mask;
                const int e = quant_group<CROUND, ROW == kQuest>(v, cc, cc.counter_start + (uint64_t)(orow * cld + ogrp * 32),
                                                  a.col_out.err, nullptr, codes, mask);
                *reinterpret_cast<uint4*>(a.col_out.codes + orow * a.col_out.ldc + ogrp * 16) = codes;
                a.col_out.sf[sf_offset(orow, ogrp, a.col_out.katoms)] = (uint8_t)e;
            }
        } else if (COL != kColOff) {
            const int cp = tid & 63, q = tid >> 6;
            if (q < TR / 32 && 2 * cp < nc && q * 32 < nr) {
                float va[32], vb[32];
                if (COL == kColDense)
                    load_col_pair<IN>(tile, cp, q, cc.transform, clut, va, vb);
                else
                    load_col_codes(IN == kInMXFP4 ? stage : codes_s, T, G::TSTRIDE, cp, q, cc.transform, va, vb);
                const int64_t orow = c0 + 2 * cp, ogrp = r0 / 32 + q;
                const int64_t cld = cc.counter_ld ? cc.counter_ld : a.R;
                const uint64_t idx = cc.counter_start + (uint64_t)(orow * cld + ogrp * 32);
                uint4 codes;
                uint32_t mask;
                const int eA = quant_group<CROUND, ROW == kQuest>(va, cc, idx, a.col_out.err, nullptr, codes, mask);
                *reinterpret_cast<uint4*>(a.col_out.codes + orow * a.col_out.ldc + ogrp * 16) = codes;
                const int eB = quant_group<CROUND, ROW == kQuest>(vb, cc, idx + (uint64_t)cld, a.col_out.err, nullptr, codes, mask);
                *reinterpret_cast<uint4*>(a.col_out.codes + (orow + 1) * a.col_out.ldc + ogrp * 16) = codes;
                a.col_out.sf[sf_offset(orow, ogrp, a.col_out.katoms)] = (uint8_t)eA;
                a.col_out.sf[sf_offset(orow + 1, ogrp, a.col_out.katoms)] = (uint8_t)eB;
            }
        }
        // Before the next iteration refills this stage buffer (cp.async at its top) and rewrites the LUTs, every
        // thread must be done with this tile.  The fused forward (codes-sourced col pass from a dense tile) needs
        // no barrier here: its col pass reads only codes_s / T, which the next tile rewrites after the barrier
        // that follows cp_async_wait1, and the row pass that read the stage and rlut ended at the mid barrier.
        if (!(COL == kColCodes && IN != kInMXFP4)) __syncthreads();
    }
}

}  // namespace qt

// ------------------------------------------------------------------------------- launchers
namespace qt {

int launch_signs2(uint32_t* a, int64_t sa, int64_t na, uint32_t* b, int64_t sb, int64_t nb, uint64_t xi,
                  cudaStream_t st) {
    const uint64_t base = mix64(xi ^ mix64(kDomainSigns));
    const int64_t nba = ((na + 31) / 32 + 255) / 256, nbb = ((nb + 31) / 32 + 255) / 256;
    if (nba + nbb == 0) return 0;
    k_signs2<<<(unsigned)(nba + nbb), 256, 0, st>>>(a, sa, na, nba, b, sb, nb, base);
    return (int)cudaGetLastError();
}

int launch_signs2_dev(uint32_t* a, int64_t sa, int64_t na, uint32_t* b, int64_t sb, int64_t nb, const uint64_t* xi,
                      cudaStream_t st) {
    const int64_t nba = ((na + 31) / 32 + 255) / 256, nbb = ((nb + 31) / 32 + 255) / 256;
    if (nba + nbb == 0) return 0;
    k_signs2_dev<<<(unsigned)(nba + nbb), 256, 0, st>>>(a, sa, na, nba, b, sb, nb, xi);
    return (int)cudaGetLastError();
}

int launch_layer_seeds(uint64_t* xi, const uint64_t* ids, int n, uint64_t seed, int64_t* step, int inc,
                       cudaStream_t st) {
    k_layer_seeds<<<1, 256, 0, st>>>(xi, ids, n, seed, step, inc);
    return (int)cudaGetLastError();
}

int launch_signs(uint32_t* bits, int64_t start, int64_t n, uint64_t xi, cudaStream_t st) {
    if (n <= 0) return 0;
    uint64_t base = mix64(xi ^ mix64(kDomainSigns));
    int64_t nw = (n + 31) / 32;
    k_signs<<<(unsigned)((nw + 255) / 256), 256, 0, st>>>(bits, start, n, base);
    return (int)cudaGetLastError();
}

template <int IN, int ROW, int COL, int CROUND>
static int quant_launch(const TileArgs& a, cudaStream_t st) {
    using G = Geom<IN>;
    auto fn = k_quant<IN, ROW, COL, CROUND>;
    static int per_sm[kMaxDevices];
    const int dev = current_device();
    if (!per_sm[dev]) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, G::BYTES);
        int n = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, 256, G::BYTES);
        per_sm[dev] = n > 0 ? n : 1;
    }
    const int64_t ctas = (int64_t)device_sms() * per_sm[dev];
    const int64_t tiles = ((a.R + G::TR - 1) / G::TR) * ((a.C + kTC - 1) / kTC);
    const unsigned n = (unsigned)cap_grid(tiles < ctas ? tiles : ctas);
    fn<<<n, 256, G::BYTES, st>>>(a);
    return 0;
}

template <int IN, int ROW, int COL>
static int dispatch_cround(const TileArgs& a, int cround, cudaStream_t st) {
    if (COL == kColOff) return quant_launch<IN, ROW, COL, kRtn>(a, st);
    if (cround == kSr) return quant_launch<IN, ROW, COL, kSr>(a, st);
    if (cround == kRtn) return quant_launch<IN, ROW, COL, kRtn>(a, st);
    return 2003;
}

template <int IN, int ROW>
static int dispatch_col(const TileArgs& a, int col_src, int cround, cudaStream_t st) {
    if (col_src == kColOff) return dispatch_cround<IN, ROW, kColOff>(a, cround, st);
    if (col_src == kColCodes) {
        if (ROW == kRowOff) return 2003;
        return dispatch_cround<IN, ROW, kColCodes>(a, cround, st);
    }
    if (ROW == kQuest) return 2003;  // no dense col pass next to a QuEST row pass
    return dispatch_cround<IN, ROW, kColDense>(a, cround, st);
}

template <int IN>
static int dispatch_row(const TileArgs& a, int row, int col_src, int cround, cudaStream_t st) {
    switch (row) {
        case kRowOff: return dispatch_col<IN, kRowOff>(a, col_src, cround, st);
        case kQuest: return dispatch_col<IN, kQuest>(a, col_src, cround, st);
        case kRtn: return dispatch_col<IN, kRtn>(a, col_src, cround, st);
        case kSr: return dispatch_col<IN, kSr>(a, col_src, cround, st);
    }
    return 2003;
}

// Row and/or column passes over one read of x[R, C].  col_from_codes: the col pass quantizes the
// transpose of the row pass's dequantized result (fused forward) instead of the dense tile.
int launch_quant_tile(const void* x, int in_type, int64_t ldx, const MxIn& mx, int64_t R, int64_t C,
                      const QuantCfg* row_cfg, const QuantOut* row_out, const QuantCfg* col_cfg,
                      const QuantOut* col_out, int col_from_codes, cudaStream_t st) {
    if (R == 0 || C == 0) return 0;
    const bool rows = row_cfg != nullptr, cols = col_cfg != nullptr;
    if (!rows && !cols) return 0;
    if (in_type == kInMXFP4 && rows) return 2003;  // MXFP4 input is only re-quantized transposed
    if (cols && col_cfg->rounding == kQuest) return 2003;
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
    const int row = rows ? row_cfg->rounding : (int)kRowOff;
    const int col_src = !cols ? kColOff : (in_type == kInMXFP4 || col_from_codes) ? kColCodes : kColDense;
    const int cround = cols ? col_cfg->rounding : kRtn;
    int rc;
    if (in_type == kInMXFP4) {
        rc = cround == kSr ? quant_launch<kInMXFP4, kRowOff, kColCodes, kSr>(a, st)
                           : quant_launch<kInMXFP4, kRowOff, kColCodes, kRtn>(a, st);
    } else if (in_type == kInBF16) {
        rc = dispatch_row<kInBF16>(a, row, col_src, cround, st);
    } else {
        rc = dispatch_row<kInF32>(a, row, col_src, cround, st);
    }
    if (rc) return rc;
    return (int)cudaGetLastError();
}

int launch_quant_rows(const void* x, int in_type, int64_t ldx, int64_t rows, int64_t cols, const QuantCfg& cfg,
                      const QuantOut& out, cudaStream_t st) {
    MxIn mx{nullptr, 0, nullptr, 0};
    return launch_quant_tile(x, in_type, ldx, mx, rows, cols, &cfg, &out, nullptr, nullptr, 0, st);
}

}  // namespace qt
