// glue.cu -- fused elementwise kernels of the Llama training loop around the Quartet linears (llama.py):
// rotary embedding (forward / backward) and SwiGLU (forward / backward), bf16 in / out, fp32 math, one HBM
// pass each.  Not part of the Quartet hot path; they replace 4-6 torch elementwise passes per op.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <algorithm>

#include "../../include/quartet_b200.h"
#include "launch.h"

namespace {

__device__ __forceinline__ float bf(uint32_t w, int hi) {
    return __uint_as_float(hi ? (w & 0xFFFF0000u) : (w << 16));
}
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
    __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&b);
}
// 8 bf16 + 8 bf16, each sum in fp32 rounded once to bf16 (what torch's bf16 add computes)
__device__ __forceinline__ uint4 add_bf8(uint4 a, uint4 b) {
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
    uint32_t o[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) o[t] = pack_bf2(bf(aw[t], 0) + bf(bw[t], 0), bf(aw[t], 1) + bf(bw[t], 1));
    return make_uint4(o[0], o[1], o[2], o[3]);
}

// Half-split (GPT-NeoX) rotary embedding on x [rows = B*S, H, dh] (row r at sequence position r % S),
// tables cos/sin [S, dh].  Each thread rotates 8 (j, j + dh/2) pairs.  Backward applies the transposed
// rotation to dy.
__global__ void k_rope(const uint4* __restrict__ x, uint4* __restrict__ out, const uint4* __restrict__ cs,
                       const uint4* __restrict__ sn, int64_t rows, int H, int dh, int S, int backward, int64_t sb,
                       int64_t ss, int64_t sh) {
    const int half8 = dh / 16;                          // uint4 chunks per half row
    const int64_t total = rows * H * half8;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % half8);
        const int64_t rh = i / half8;                   // (row, head)
        const int64_t row = rh / H;
        const int pos = (int)(row % S);
        const int64_t base = rh * (dh / 8);             // uint4 index of this (row, head) in the output
        // input element (b, s, h, :) at b sb + s ss + h sh (uint4 units; dh contiguous)
        const int64_t ib = (row / S) * sb + (int64_t)pos * ss + (rh % H) * sh;
        const uint4 a = x[ib + c], b = x[ib + half8 + c];
        const uint4 ca = cs[(int64_t)pos * (dh / 8) + c], cb = cs[(int64_t)pos * (dh / 8) + half8 + c];
        const uint4 sa = sn[(int64_t)pos * (dh / 8) + c], sb = sn[(int64_t)pos * (dh / 8) + half8 + c];
        const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
        const uint32_t caw[4] = {ca.x, ca.y, ca.z, ca.w}, cbw[4] = {cb.x, cb.y, cb.z, cb.w};
        const uint32_t saw[4] = {sa.x, sa.y, sa.z, sa.w}, sbw[4] = {sb.x, sb.y, sb.z, sb.w};
        uint32_t lo[4], hi[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float o_lo[2], o_hi[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const float xl = bf(aw[k], t), xh = bf(bw[k], t);
                const float cl = bf(caw[k], t), ch = bf(cbw[k], t), sl = bf(saw[k], t), sh = bf(sbw[k], t);
                if (!backward) {
                    o_lo[t] = xl * cl - xh * sl;
                    o_hi[t] = xh * ch + xl * sh;
                } else {
                    o_lo[t] = xl * cl + xh * sh;
                    o_hi[t] = xh * ch - xl * sl;
                }
            }
            lo[k] = pack_bf2(o_lo[0], o_lo[1]);
            hi[k] = pack_bf2(o_hi[0], o_hi[1]);
        }
        out[base + c] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        out[base + half8 + c] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    }
}

// SwiGLU: y = silu(g) * u; backward dg = dy * u * silu'(g), du = dy * silu(g).  8 elements per thread.
__global__ void k_swiglu(const uint4* __restrict__ g, const uint4* __restrict__ u, const uint4* __restrict__ dy,
                         uint4* __restrict__ o0, uint4* __restrict__ o1, int64_t n8, int backward) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 gv = g[i], uv = u[i];
        const uint32_t gw[4] = {gv.x, gv.y, gv.z, gv.w}, uw[4] = {uv.x, uv.y, uv.z, uv.w};
        uint32_t dw[4] = {0, 0, 0, 0};
        if (backward) {
            const uint4 dv = dy[i];
            dw[0] = dv.x;
            dw[1] = dv.y;
            dw[2] = dv.z;
            dw[3] = dv.w;
        }
        uint32_t r0[4], r1[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float a[2], b[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const float x = bf(gw[k], t), up = bf(uw[k], t);
                const float sg = 1.0f / (1.0f + __expf(-x));
                const float silu = x * sg;
                if (!backward) {
                    a[t] = silu * up;
                    b[t] = 0.0f;
                } else {
                    const float d = bf(dw[k], t);
                    a[t] = d * up * sg * (1.0f + x * (1.0f - sg));  // dg
                    b[t] = d * silu;                                // du
                }
            }
            r0[k] = pack_bf2(a[0], a[1]);
            r1[k] = pack_bf2(b[0], b[1]);
        }
        o0[i] = make_uint4(r0[0], r0[1], r0[2], r0[3]);
        if (backward) o1[i] = make_uint4(r1[0], r1[1], r1[2], r1[3]);
    }
}

// RMSNorm over rows of x [rows, d] bf16 with an fp32 weight, one warp per row (d % 8 == 0, d <= 2048):
// forward y = x * rstd * w (rstd = 1/sqrt(mean(x^2) + eps) in fp32, saved); backward dx = rstd (g - xh mean(g xh))
// with g = dy * w, xh = x * rstd, and dw += sum_rows dy * xh (per-warp partials in shared memory -> one atomic per
// column per block).  Lane `lane` owns the 16-byte chunks v * 32 + lane (v < NV) that lie inside the row.
// Optional residual stream (qt_rmsnorm_res): forward normalises h = x + res and writes h; backward adds res to dx.
// Kept lean in registers (rows held as packed bf16, w re-read through L1, dw partials in shared memory) so that
// 2-4 blocks of 8 warps fit per SM (no spills): one row per warp is a full memory round trip, and with 16-32 warps the
// loads of many rows overlap (at 8 resident warps the kernel was latency-bound at 2-3 TB/s).
__device__ __forceinline__ void w8(const float* __restrict__ w, int chunk, float (&o)[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(w) + 2 * chunk);
    const float4 b = __ldg(reinterpret_cast<const float4*>(w) + 2 * chunk + 1);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
template <int NV>  // uint4 chunks of 8 bf16 per lane: d <= 256 * NV
__global__ void __launch_bounds__(256, NV <= 2 ? 4 : 2) k_rmsnorm(const uint4* __restrict__ x, const float* __restrict__ w,
                                                    const uint4* __restrict__ dy, uint4* __restrict__ out,
                                                    float* __restrict__ rstd_io, float* __restrict__ dw, int64_t rows,
                                                    int d, float eps, int backward, const uint4* __restrict__ res,
                                                    uint4* __restrict__ h_out) {
    extern __shared__ float red[];  // [warps][d] partial dw (backward)
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nch = d / 8;          // chunks per row
    float* my = red + wib * d;
    if (backward) {
#pragma unroll
        for (int v = 0; v < NV; ++v)
            if (v * 32 + lane < nch)
#pragma unroll
                for (int t = 0; t < 8; ++t) my[(v * 32 + lane) * 8 + t] = 0.f;
    }
    for (int64_t r = (int64_t)blockIdx.x * nw + wib; r < rows; r += (int64_t)gridDim.x * nw) {
        uint4 cx[NV], cd[NV], cr[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const bool ok = v * 32 + lane < nch;
            cx[v] = ok ? x[r * nch + v * 32 + lane] : make_uint4(0, 0, 0, 0);
            if (res) cr[v] = ok ? res[r * nch + v * 32 + lane] : make_uint4(0, 0, 0, 0);
            if (backward) cd[v] = ok ? dy[r * nch + v * 32 + lane] : make_uint4(0, 0, 0, 0);
        }
        if (!backward) {
            if (res) {   // fused residual add: h = bf16(x + y), normalised and written
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    cx[v] = add_bf8(cx[v], cr[v]);
                    if (v * 32 + lane < nch) h_out[r * nch + v * 32 + lane] = cx[v];
                }
            }
            float ss = 0.f;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const uint32_t cw[4] = {cx[v].x, cx[v].y, cx[v].z, cx[v].w};
#pragma unroll
                for (int t = 0; t < 8; ++t) ss = fmaf(bf(cw[t >> 1], t & 1), bf(cw[t >> 1], t & 1), ss);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            const float rs = rsqrtf(ss / (float)d + eps);
            if (lane == 0) rstd_io[r] = rs;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if (v * 32 + lane >= nch) continue;
                float wv[8];
                w8(w, v * 32 + lane, wv);
                const uint32_t cw[4] = {cx[v].x, cx[v].y, cx[v].z, cx[v].w};
                uint32_t o4[4];
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    o4[t] = pack_bf2(bf(cw[t], 0) * rs * wv[2 * t], bf(cw[t], 1) * rs * wv[2 * t + 1]);
                out[r * nch + v * 32 + lane] = make_uint4(o4[0], o4[1], o4[2], o4[3]);
            }
        } else {
            const float rs = rstd_io[r];
            float dot = 0.f;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if (v * 32 + lane >= nch) continue;
                float wv[8];
                w8(w, v * 32 + lane, wv);
                const uint32_t xw[4] = {cx[v].x, cx[v].y, cx[v].z, cx[v].w};
                const uint32_t dw4[4] = {cd[v].x, cd[v].y, cd[v].z, cd[v].w};
                float* pp = my + (v * 32 + lane) * 8;
                float4 p0 = *reinterpret_cast<float4*>(pp), p1 = *reinterpret_cast<float4*>(pp + 4);
                float pv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const float dd = bf(dw4[t >> 1], t & 1), xh = bf(xw[t >> 1], t & 1) * rs;
                    dot = fmaf(dd * wv[t], xh, dot);
                    pv[t] = fmaf(dd, xh, pv[t]);
                }
                *reinterpret_cast<float4*>(pp) = make_float4(pv[0], pv[1], pv[2], pv[3]);
                *reinterpret_cast<float4*>(pp + 4) = make_float4(pv[4], pv[5], pv[6], pv[7]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            const float mdot = dot / (float)d;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if (v * 32 + lane >= nch) continue;
                float wv[8];
                w8(w, v * 32 + lane, wv);
                const uint32_t xw[4] = {cx[v].x, cx[v].y, cx[v].z, cx[v].w};
                const uint32_t dw4[4] = {cd[v].x, cd[v].y, cd[v].z, cd[v].w};
                uint32_t o4[4];
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    o4[t] = pack_bf2(rs * (bf(dw4[t], 0) * wv[2 * t] - bf(xw[t], 0) * rs * mdot),
                                     rs * (bf(dw4[t], 1) * wv[2 * t + 1] - bf(xw[t], 1) * rs * mdot));
                uint4 o = make_uint4(o4[0], o4[1], o4[2], o4[3]);
                if (res) o = add_bf8(o, cr[v]);   // + the residual stream's gradient
                out[r * nch + v * 32 + lane] = o;
            }
        }
    }
    if (backward) {
        __syncthreads();
        for (int c = threadIdx.x; c < d; c += blockDim.x) {
            float sum = 0.f;
            for (int k = 0; k < nw; ++k) sum += red[k * d + c];
            atomicAdd(dw + c, sum);
        }
    }
}

// Cross-entropy over rows of logits [rows, V] bf16 (V % 8 == 0), one 256-thread block per row.
// forward: online max / sum-exp in one pass -> lse[r] and loss[r] = lse - logit[target] (fp32);
// backward: dlogits = (exp(x - lse) - [j == target]) * (*dloss) * scale, one read + one write.
__device__ __forceinline__ void ce_merge(float& m, float& s, float m2, float s2) {
    const float mn = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mn));
    m = mn;
}
// Forward: one warp per row, online log-sum-exp; four independent 16-byte loads per lane and iteration
// (memory-level parallelism) and one merge per 32 values (out-of-range chunks read as -inf, adding nothing);
// shuffle-only reduction (no block barrier per row).
__global__ void __launch_bounds__(256) k_xent_fwd(const uint4* __restrict__ logits, const int64_t* __restrict__ tgt,
                                                  float* __restrict__ lse, float* __restrict__ loss, int64_t rows,
                                                  int V) {
    const int V8 = V / 8, lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nw) {
        const uint4* row = logits + r * V8;
        float m = -INFINITY, sum = 0.f;
        for (int i0 = lane; i0 < V8; i0 += 4 * 32) {
            uint4 c[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + 32 * u;
                c[u] = i < V8 ? row[i] : make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
            }
            float v[32], cm = -INFINITY;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t w[4] = {c[u].x, c[u].y, c[u].z, c[u].w};
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    v[8 * u + k] = bf(w[k >> 1], k & 1);
                    cm = fmaxf(cm, v[8 * u + k]);
                }
            }
            float cs = 0.f;
            if (cm != -INFINITY) {
#pragma unroll
                for (int k = 0; k < 32; ++k) cs += __expf(v[k] - cm);
            }
            ce_merge(m, sum, cm, cs);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
            ce_merge(m, sum, m2, s2);
        }
        if (lane == 0) {
            const float l = m + __logf(sum);
            lse[r] = l;
            const int64_t t = tgt[r];
            if (t >= 0 && t < V) {   // otherwise ignored (loss 0, gradient 0), like ignore_index
                const uint32_t tw = reinterpret_cast<const uint32_t*>(row)[t >> 1];
                loss[r] = l - bf(tw, (int)(t & 1));
            } else {
                loss[r] = 0.f;
            }
        }
    }
}

// Backward: dlogits = (softmax - onehot) * dloss * scale, one block per row (streaming).
__global__ void k_xent_bwd(const uint4* __restrict__ logits, const int64_t* __restrict__ tgt,
                           const float* __restrict__ lse, uint4* __restrict__ dlogits, const float* __restrict__ dloss,
                           float scale, int64_t rows, int V) {
    const int V8 = V / 8;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const uint4* row = logits + r * V8;
        const int64_t t = tgt[r];
        const bool valid = t >= 0 && t < V;   // otherwise ignored (loss 0, gradient 0), like ignore_index
        const float l = lse[r], g = valid ? *dloss * scale : 0.f;
        uint4* drow = dlogits + r * V8;
        for (int i = threadIdx.x; i < V8; i += blockDim.x) {
            const uint4 c = row[i];
            const uint32_t w[4] = {c.x, c.y, c.z, c.w};
            uint32_t o[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t j0 = (int64_t)i * 8 + 2 * k;
                const float p0 = __expf(bf(w[k], 0) - l) - (j0 == t ? 1.f : 0.f);
                const float p1 = __expf(bf(w[k], 1) - l) - (j0 + 1 == t ? 1.f : 0.f);
                o[k] = pack_bf2(p0 * g, p1 * g);
            }
            drow[i] = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
}

// Wide rows (d = 2048 * NV, one 256-thread block per row, 8 * NV elements per thread): same math as
// k_rmsnorm; dw partials stay in registers across the block's rows, one atomic per column per block.
template <int NV>
__global__ void __launch_bounds__(256) k_rmsnorm_wide(const uint4* __restrict__ x, const float* __restrict__ w,
                                                      const uint4* __restrict__ dy, uint4* __restrict__ out,
                                                      float* __restrict__ rstd_io, float* __restrict__ dw,
                                                      int64_t rows, float eps, int backward,
                                                      const uint4* __restrict__ res, uint4* __restrict__ h_out) {
    constexpr int D = 2048 * NV;
    __shared__ float red[8];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    float wv[NV][8], dwp[NV][8];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            wv[v][t] = w[(v * 256 + tid) * 8 + t];
            dwp[v][t] = 0.f;
        }
    auto block_sum = [&](float val) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        __syncthreads();
        if (lane == 0) red[wid] = val;
        __syncthreads();
        float tot = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) tot += red[k];
        return tot;
    };
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        float xv[NV][8], ss = 0.f;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            uint4 c = x[r * (D / 8) + v * 256 + tid];
            if (!backward && res) {
                c = add_bf8(c, res[r * (D / 8) + v * 256 + tid]);
                h_out[r * (D / 8) + v * 256 + tid] = c;
            }
            const uint32_t cw[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                xv[v][t] = bf(cw[t >> 1], t & 1);
                ss = fmaf(xv[v][t], xv[v][t], ss);
            }
        }
        if (!backward) {
            const float rs = rsqrtf(block_sum(ss) / (float)D + eps);
            if (tid == 0) rstd_io[r] = rs;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                uint32_t o4[4];
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    o4[t] = pack_bf2(xv[v][2 * t] * rs * wv[v][2 * t], xv[v][2 * t + 1] * rs * wv[v][2 * t + 1]);
                out[r * (D / 8) + v * 256 + tid] = make_uint4(o4[0], o4[1], o4[2], o4[3]);
            }
        } else {
            const float rs = rstd_io[r];
            float gv[NV][8], dot = 0.f;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const uint4 c = dy[r * (D / 8) + v * 256 + tid];
                const uint32_t cw[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const float dd = bf(cw[t >> 1], t & 1), xh = xv[v][t] * rs;
                    gv[v][t] = dd * wv[v][t];
                    dot = fmaf(gv[v][t], xh, dot);
                    dwp[v][t] = fmaf(dd, xh, dwp[v][t]);
                }
            }
            const float mdot = block_sum(dot) / (float)D;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                uint32_t o4[4];
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    o4[t] = pack_bf2(rs * (gv[v][2 * t] - xv[v][2 * t] * rs * mdot),
                                     rs * (gv[v][2 * t + 1] - xv[v][2 * t + 1] * rs * mdot));
                uint4 o = make_uint4(o4[0], o4[1], o4[2], o4[3]);
                if (res) o = add_bf8(o, res[r * (D / 8) + v * 256 + tid]);
                out[r * (D / 8) + v * 256 + tid] = o;
            }
        }
    }
    if (backward)
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int t = 0; t < 8; ++t) atomicAdd(dw + (v * 256 + tid) * 8 + t, dwp[v][t]);
}

int grid_for(int64_t work) {
    const int64_t sms = qt::device_sms();
    const int64_t blocks = (work + 255) / 256;
    return (int)(blocks < (int64_t)sms * 8 ? blocks : (int64_t)sms * 8);
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" {

QT_API int qt_rope(const void* x, void* out, int64_t rows, int heads, int head_dim, int seq, const void* cos,
                   const void* sin, int backward, int64_t stride_b, int64_t stride_s, int64_t stride_h, void* stream) {
    if (rows < 0 || heads <= 0 || head_dim % 16 != 0 || seq <= 0 || rows % seq != 0) return QT_ERR_SHAPE;
    if (!al16(x) || !al16(out) || !al16(cos) || !al16(sin) || stride_b % 8 || stride_s % 8 || stride_h % 8)
        return QT_ERR_ALIGN;
    const int64_t work = rows * heads * (head_dim / 16);
    if (work == 0) return 0;
    k_rope<<<grid_for(work), 256, 0, (cudaStream_t)stream>>>(
        static_cast<const uint4*>(x), static_cast<uint4*>(out), static_cast<const uint4*>(cos),
        static_cast<const uint4*>(sin), rows, heads, head_dim, seq, backward, stride_b / 8, stride_s / 8,
        stride_h / 8);
    return (int)cudaGetLastError();
}

QT_API int qt_rmsnorm(const void* x, const float* w, const void* dy, void* out, float* rstd, float* dw, int64_t rows,
                      int d, float eps, int backward, void* stream) {
    return qt_rmsnorm_res(x, nullptr, w, dy, out, nullptr, rstd, dw, rows, d, eps, backward, stream);
}

QT_API int qt_rmsnorm_res(const void* x, const void* res, const float* w, const void* dy, void* out, void* h_out,
                          float* rstd, float* dw, int64_t rows, int d, float eps, int backward, void* stream) {
    if (rows < 0 || d % 8 != 0 || d < 8 || (d > 2048 && (d % 2048 != 0 || d > 8192))) return QT_ERR_SHAPE;
    if (!al16(x) || !al16(out) || (backward && (!al16(dy) || !dw))) return QT_ERR_ALIGN;
    if (res && (!al16(res) || (!backward && (!h_out || !al16(h_out))))) return QT_ERR_ALIGN;
    if (rows == 0) return 0;
    if (d > 2048) {
        int blocks = grid_for(rows * 256);
        if (blocks > 1184) blocks = 1184;
        auto wide = [&](auto kern) {
            int per_sm = 0;   // backward: one wave of resident blocks (one dw atomic per column per block)
            if (backward && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0) == cudaSuccess &&
                per_sm > 0)
                blocks = std::min<int>(blocks, per_sm * (int)qt::device_sms());
            kern<<<blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<const uint4*>(x), w, static_cast<const uint4*>(dy),
                                                           static_cast<uint4*>(out), rstd, dw, rows, eps, backward,
                                                           static_cast<const uint4*>(res), static_cast<uint4*>(h_out));
        };
        switch (d / 2048) {
            case 2: wide(k_rmsnorm_wide<2>); break;
            case 3: wide(k_rmsnorm_wide<3>); break;
            default: wide(k_rmsnorm_wide<4>); break;
        }
        return (int)cudaGetLastError();
    }
    const int warps = 8;
    int blocks = grid_for(rows * 32);
    if (blocks > 1184) blocks = 1184;
    const size_t smem = backward ? (size_t)warps * d * sizeof(float) : 0;
    auto go = [&](auto kern) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        // backward: one wave of resident blocks, so one dw atomic per column per resident block (1184 blocks
        // issued 4x the atomics: d = 1280 backward 72 -> 63 us); the forward keeps the wider grid (measured faster)
        int per_sm = 0;
        if (backward && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem) == cudaSuccess &&
            per_sm > 0)
            blocks = std::min<int>(blocks, per_sm * (int)qt::device_sms());
        kern<<<blocks, warps * 32, smem, (cudaStream_t)stream>>>(static_cast<const uint4*>(x), w,
                                                               static_cast<const uint4*>(dy), static_cast<uint4*>(out),
                                                               rstd, dw, rows, d, eps, backward,
                                                               static_cast<const uint4*>(res), static_cast<uint4*>(h_out));
    };
    switch ((d + 255) / 256) {
        case 1: go(k_rmsnorm<1>); break;
        case 2: go(k_rmsnorm<2>); break;
        case 3: go(k_rmsnorm<3>); break;
        case 4: go(k_rmsnorm<4>); break;
        case 5: go(k_rmsnorm<5>); break;
        case 6: go(k_rmsnorm<6>); break;
        case 7: go(k_rmsnorm<7>); break;
        default: go(k_rmsnorm<8>); break;
    }
    return (int)cudaGetLastError();
}

QT_API int qt_cross_entropy(const void* logits, const int64_t* targets, int64_t rows, int vocab, float* lse,
                            float* loss, void* dlogits, const float* dloss, float scale, int backward, void* stream) {
    if (rows < 0 || vocab <= 0 || vocab % 8 != 0) return QT_ERR_SHAPE;
    if (!al16(logits) || (backward && !al16(dlogits))) return QT_ERR_ALIGN;
    if (rows == 0) return 0;
    const int64_t sms = qt::device_sms();
    if (!backward) {
        const int64_t wb = (rows + 7) / 8;   // 8 rows (warps) per block
        const int64_t blocks = wb < (int64_t)sms * 8 ? wb : (int64_t)sms * 8;
        k_xent_fwd<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<const uint4*>(logits), targets,
                                                                        lse, loss, rows, vocab);
    } else {
        const int64_t blocks = rows < (int64_t)sms * 8 ? rows : (int64_t)sms * 8;
        k_xent_bwd<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<const uint4*>(logits), targets,
                                                                        lse, static_cast<uint4*>(dlogits), dloss,
                                                                        scale, rows, vocab);
    }
    return (int)cudaGetLastError();
}

QT_API int qt_swiglu(const void* gate, const void* up, const void* dy, void* out0, void* out1, int64_t n,
                     int backward, void* stream) {
    if (n < 0 || n % 8 != 0) return QT_ERR_SHAPE;
    if (!al16(gate) || !al16(up) || !al16(out0) || (backward && (!al16(dy) || !al16(out1)))) return QT_ERR_ALIGN;
    if (n == 0) return 0;
    k_swiglu<<<grid_for(n / 8), 256, 0, (cudaStream_t)stream>>>(
        static_cast<const uint4*>(gate), static_cast<const uint4*>(up), static_cast<const uint4*>(dy),
        static_cast<uint4*>(out0), static_cast<uint4*>(out1), n / 8, backward);
    return (int)cudaGetLastError();
}

}  // extern "C"
