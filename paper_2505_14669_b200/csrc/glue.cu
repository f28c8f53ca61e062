// glue.cu -- fused elementwise kernels of the Llama training loop around the Quartet linears (llama.py):
// rotary embedding (forward / backward) and SwiGLU (forward / backward), bf16 in / out, fp32 math, one HBM
// pass each.  Not part of the Quartet hot path; they replace 4-6 torch elementwise passes per op.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/quartet_b200.h"

namespace {

__device__ __forceinline__ float bf(uint32_t w, int hi) {
    return __uint_as_float(hi ? (w & 0xFFFF0000u) : (w << 16));
}
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
    __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&b);
}

// Half-split (GPT-NeoX) rotary embedding on x [rows = B*S, H, dh] (row r at sequence position r % S),
// tables cos/sin [S, dh].  Each thread rotates 8 (j, j + dh/2) pairs.  Backward applies the transposed
// rotation to dy.
__global__ void k_rope(const uint4* __restrict__ x, uint4* __restrict__ out, const uint4* __restrict__ cs,
                       const uint4* __restrict__ sn, int64_t rows, int H, int dh, int S, int backward) {
    const int half8 = dh / 16;                          // uint4 chunks per half row
    const int64_t total = rows * H * half8;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % half8);
        const int64_t rh = i / half8;                   // (row, head)
        const int64_t row = rh / H;
        const int pos = (int)(row % S);
        const int64_t base = rh * (dh / 8);             // uint4 index of this (row, head)
        const uint4 a = x[base + c], b = x[base + half8 + c];
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

int grid_for(int64_t work) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t blocks = (work + 255) / 256;
    return (int)(blocks < (int64_t)sms * 8 ? blocks : (int64_t)sms * 8);
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" {

QT_API int qt_rope(const void* x, void* out, int64_t rows, int heads, int head_dim, int seq, const void* cos,
                   const void* sin, int backward, void* stream) {
    if (rows < 0 || heads <= 0 || head_dim % 16 != 0 || seq <= 0) return QT_ERR_SHAPE;
    if (!al16(x) || !al16(out) || !al16(cos) || !al16(sin)) return QT_ERR_ALIGN;
    const int64_t work = rows * heads * (head_dim / 16);
    if (work == 0) return 0;
    k_rope<<<grid_for(work), 256, 0, (cudaStream_t)stream>>>(
        static_cast<const uint4*>(x), static_cast<uint4*>(out), static_cast<const uint4*>(cos),
        static_cast<const uint4*>(sin), rows, heads, head_dim, seq, backward);
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
