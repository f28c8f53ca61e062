// sf_layout.cu -- which TMEM bytes does tcgen05.mma kind::mxf4 block32 read as the A scale factors?
// (not product code; answers whether the scale staging can use fewer / larger tcgen05.cp copies)
//
// A and B codes are all 1.0 and every B scale is 2^0, so D[m][n] = 32 (2^(s1-127) + 2^(s2-127)) where
// s1, s2 are the two A scale bytes the MMA used for row m (K = 64 = 2 groups).  The A scale bytes are
// planted in TMEM with one tcgen05.cp 128x128b (lane L <- 16 source bytes, no broadcast) or
// 32x128b.warpx4 (lanes q*32+i <- source row i), each byte encoding where it sits.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2505_14669_b200/csrc/common.cuh"
using namespace qt;

__device__ __forceinline__ void cp_128x128b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc));
}

// pattern 0: byte j of lane L = 60 + 16 (L / 32) + j;  pattern 1: = 60 + (L % 32)
__global__ void k(float* out, int pattern, int use_warpx4, int sf_id, int col_off) {
    __shared__ __align__(1024) uint8_t codes[8192];
    __shared__ __align__(128) uint8_t sfa[4096];
    __shared__ __align__(128) uint8_t sfb[2048];
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    const int t = threadIdx.x, warp = t / 32;
    for (int i = t; i < 8192; i += blockDim.x) codes[i] = 0x22;  // E2M1 1.0, 1.0
    for (int i = t; i < 2048; i += blockDim.x) {
        const int L = i / 16, j = i % 16;
        sfa[i] = (uint8_t)(pattern == 0 ? 60 + 16 * (L / 32) + j : 60 + (L % 32));
        sfb[i] = 127;
    }
    if (use_warpx4 == 2)  // 128x256b source: half h (2 KB) x lane L x 4 columns x 4 bytes; byte = 60 + 4 c + b
        for (int i = t; i < 4096; i += blockDim.x) {
            const int h = i / 2048, L = (i / 16) % 128, c = 4 * h + (i % 16) / 4, b = i % 4;
            sfa[i] = (uint8_t)(pattern == 0 ? 60 + 4 * c + b : 60 + (L % 32));
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
        if (use_warpx4 == 2)
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(t_sfa),
                         "l"(make_sdesc(smem_u32(sfa), 2048, 128, kLayoutNone)));
        else if (use_warpx4)
            tmem_cp_sf(t_sfa, make_sdesc(smem_u32(sfa), 0, 128, kLayoutNone));
        else
            cp_128x128b(t_sfa, make_sdesc(smem_u32(sfa), 0, 128, kLayoutNone));
        cp_128x128b(t_sfb, make_sdesc(smem_u32(sfb), 0, 128, kLayoutNone));
        cp_128x128b(t_sfb + 4, make_sdesc(smem_u32(sfb), 0, 128, kLayoutNone));
        const uint64_t ad = make_sdesc(smem_u32(codes), 128, 256, kLayoutNone);
        const uint64_t bd = make_sdesc(smem_u32(codes + 4096), 128, 256, kLayoutNone);
        mma_mxf4(tmem, ad, bd, idesc_mxf4(128, 128, sf_id, 0), t_sfa + col_off, t_sfb, 0u);
        tc_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    tc_fence_after();
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), r);
    tmem_ld_wait();
    out[warp * 32 + (t % 32)] = __uint_as_float(r[0]);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

static void decode(float d, int& v1, int& v2) {
    const double x = d / 32.0;
    if (!(x > 0)) { v1 = v2 = -1; return; }
    int e = (int)std::floor(std::log2(x));
    double r = x - std::ldexp(1.0, e);
    if (r == 0) { v1 = v2 = e + 127 - 1; return; }
    v1 = e + 127;
    v2 = (int)std::lround(std::log2(r)) + 127;
}

int main(int argc, char** argv) {
    const int only_co = argc > 1 ? atoi(argv[1]) : -1;
    float* out;
    cudaMalloc(&out, 128 * 4);
    float h[128];
    const char* names[] = {"128x128b", "32x128b.warpx4", "128x256b"};
    if (argc > 2) {  // 128x256b: row m with base offset co reads column (c) bytes (b)
        for (int co = 0; co <= 6; co += 2) {
            k<<<1, 128>>>(out, 0, 2, 0, co);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(h, out, 512, cudaMemcpyDeviceToHost);
            printf("== 128x256b base +%d\n", co);
            for (int m = 0; m < 128; m += 32) {
                int v1, v2;
                decode(h[m], v1, v2);
                printf("  row %3d: col %d bytes %d,%d\n", m, (v1 - 60) / 4, (v1 - 60) % 4, (v2 - 60) % 4);
            }
        }
        return 0;
    }
    for (int wx = 0; wx < 2; ++wx)
        for (int sf_id = 0; sf_id <= 2; sf_id += 2)
            for (int co = 0; co <= 4; ++co) {
                if (only_co >= 0 && co != only_co) continue;
                if (only_co < 0 && co != 0) continue;
                int res[2][128][2];
                for (int p = 0; p < 2; ++p) {
                    k<<<1, 128>>>(out, p, wx, sf_id, co);
                    cudaError_t e = cudaDeviceSynchronize();
                    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                    cudaMemcpy(h, out, 512, cudaMemcpyDeviceToHost);
                    for (int m = 0; m < 128; ++m) decode(h[m], res[p][m][0], res[p][m][1]);
                }
                printf("== %s sf_id %d col+%d\n", names[wx], sf_id, co);
                for (int m = 0; m < 128; m += (m % 32 == 0 ? 1 : 31)) {
                    // pattern 0 -> (quadrant, byte j), pattern 1 -> lane % 32
                    printf("  row %3d: reads (q%d j%2d | l%2d) and (q%d j%2d | l%2d)\n", m, (res[0][m][0] - 60) / 16,
                           (res[0][m][0] - 60) % 16, res[1][m][0] - 60, (res[0][m][1] - 60) / 16,
                           (res[0][m][1] - 60) % 16, res[1][m][1] - 60);
                }
            }
    return 0;
}
