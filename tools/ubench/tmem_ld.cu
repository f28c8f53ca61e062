// tmem_ld.cu -- tcgen05.ld throughput per SM on B200 (not product code).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2505_14669_b200/csrc/common.cuh"
using namespace qt;
template <int WARPS, int X>
__global__ void __launch_bounds__(WARPS * 32, 1) k(uint32_t* out, int iters) {
    __shared__ uint32_t holder;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc(&holder, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = holder;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint32_t r[32];
#pragma unroll
        for (int c = 0; c < X; ++c) {
            tmem_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + ((warp >> 2) * 32 * X + c * 32) % 512, r);
            tmem_ld_wait();
            acc += r[0] ^ r[31];
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}
template <int W, int X>
void run() {
    uint32_t* out;
    cudaMalloc(&out, 148 * 1024 * 4);
    int iters = 2000;
    k<W, X><<<148, W * 32>>>(out, 10);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<W, X><<<148, W * 32>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double bytes_per_sm = (double)W * 32 * 32 * 4 * X * iters;
    printf("warps %2d x%d: %.3f ms  %.1f B/clk/SM (1.965 GHz)  err=%s\n", W, X, ms, bytes_per_sm / (ms * 1e-3 * 1.965e9),
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}
int main() {
    run<4, 1>(); run<4, 4>(); run<8, 2>(); run<16, 1>(); run<16, 2>();
}
