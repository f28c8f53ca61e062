// sfb_layout.cu -- which TMEM (lane, column) does tcgen05.mma kind::mxf4.block32 read as the B scale of
// output column n when N = 256, and does the lane field of the SFB address move it?  (not product code)
//
// A, B codes all 1.0, every A scale 2^0: D[0][n] = 32 (2^(s1-127) + 2^(s2-127)), s1/s2 the two B scale
// bytes of column n.  Both bytes of a TMEM word carry the same value, planted with one 128x256b copy
// (lane L <- 32 source bytes = 8 columns): pattern 0 -> 60 + L % 32, pattern 1 -> 60 + 8 (L / 32) + column.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2505_14669_b200/csrc/common.cuh"
using namespace qt;

__global__ void k(float* out, int pattern, int lane_off) {
    __shared__ __align__(1024) uint8_t codes[16384];
    __shared__ __align__(128) uint8_t sfa[2048];
    __shared__ __align__(128) uint8_t sfb[4096];
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    const int t = threadIdx.x, warp = t / 32;
    for (int i = t; i < 16384; i += blockDim.x) codes[i] = 0x22;
    for (int i = t; i < 2048; i += blockDim.x) sfa[i] = 127;
    for (int i = t; i < 4096; i += blockDim.x) {
        const int h = i / 2048, L = (i / 16) % 128, c = 4 * h + (i % 16) / 4;
        sfb[i] = (uint8_t)(pattern == 0 ? 60 + L % 32 : 60 + 8 * (L / 32) + c);
    }
    if (t == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&holder, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = holder;
    if (t == 0) {
        const uint32_t t_sfa = tmem + 256, t_sfb = tmem + 384;
        asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(t_sfa),
                     "l"(make_sdesc(smem_u32(sfa), 0, 128, kLayoutNone)));
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(t_sfb),
                     "l"(make_sdesc(smem_u32(sfb), 2048, 128, kLayoutNone)));
        const uint64_t ad = make_sdesc(smem_u32(codes), 128, 256, kLayoutNone);
        const uint64_t bd = make_sdesc(smem_u32(codes + 4096), 128, 256, kLayoutNone);
        mma_mxf4(tmem, ad, bd, idesc_mxf4(128, 256, 0, 0), t_sfa, t_sfb + ((uint32_t)lane_off << 16), 0u);
        tc_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    tc_fence_after();
    if (warp == 0) {
        uint32_t r[32];
        for (int c = 0; c < 8; ++c) {
            tmem_ld32(tmem + c * 32, r);
            tmem_ld_wait();
            if (t == 0)
                for (int j = 0; j < 32; ++j) out[c * 32 + j] = __uint_as_float(r[j]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int main(int argc, char** argv) {
    const int lane_off = argc > 1 ? atoi(argv[1]) : 0;
    float* out;
    cudaMalloc(&out, 256 * 4);
    float h[2][256];
    for (int p = 0; p < 2; ++p) {
        k<<<1, 128>>>(out, p, lane_off);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h[p], out, 1024, cudaMemcpyDeviceToHost);
    }
    printf("SFB address lane offset %d\n", lane_off);
    for (int n = 0; n < 256; n += (n % 32 == 0 ? 1 : 15)) {
        // both bytes equal: D = 64 * 2^(v - 127)
        int v[2];
        for (int p = 0; p < 2; ++p) v[p] = h[p][n] > 0 ? (int)std::lround(std::log2(h[p][n] / 64.0)) + 127 : -1;
        printf("  n %3d: lane %%32 = %2d, lane/32 = %d, column %d   (D %g %g)\n", n, v[0] - 60, (v[1] - 60) / 8,
               (v[1] - 60) % 8, h[0][n], h[1][n]);
    }
    return 0;
}
