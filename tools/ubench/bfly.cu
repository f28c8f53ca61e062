// bfly.cu -- scalar vs packed f32x2 FWHT butterfly throughput on B200 (not product code).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int ITERS = 1024;
__device__ float g_nz = -0.0f;

// scalar: v[t] = (a+b)*c, v[t+1] = (a-b)*c  over 16 values, 4 instr per butterfly (8 butterflies)
template <int LOPS>
__global__ void k_scalar(float* out, float seed) {
    float v[16];
    uint32_t m = __float_as_uint(seed);
    for (int i = 0; i < 16; ++i) v[i] = seed + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int t = 0; t < 16; t += 2) {
            float a = v[t], b = v[t + 1];
            v[t] = __fmul_rn(__fadd_rn(a, b), 0.70710677f);
            v[t + 1] = __fmul_rn(__fsub_rn(a, b), 0.70710677f);
            if (LOPS) { m = (m ^ __float_as_uint(v[t])) & 0x7fffffffu; }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) { float x = v[t]; v[t] = v[t + 8]; v[t + 8] = x; }
    }
    float s = 0;
    for (int i = 0; i < 16; ++i) s += v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + __uint_as_float(m);
}
// packed: 16 float2, 8 butterflies of float2 -> 4 packed instr per butterfly (processes 4 values)
template <int LOPS>
__global__ void k_packed(float* out, float seed) {
    uint64_t v[16];
    const float z = *const_cast<volatile float*>(&g_nz);
    uint64_t nz = ((uint64_t)__float_as_uint(z) << 32) | __float_as_uint(z);
    uint64_t c2 = ((uint64_t)0x3F3504F3u << 32) | 0x3F3504F3u;
    uint32_t m = __float_as_uint(seed);
    for (int i = 0; i < 16; ++i) v[i] = ((uint64_t)__float_as_uint(seed + i) << 32) | __float_as_uint(seed - i);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int t = 0; t < 16; t += 2) {
            uint64_t s, d;
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s) : "l"(v[t]), "l"(v[t + 1]));
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(v[t]), "l"(v[t + 1]));
            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(v[t]) : "l"(s), "l"(c2), "l"(nz));
            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(v[t + 1]) : "l"(d), "l"(c2), "l"(nz));
            if (LOPS) { m = (m ^ (uint32_t)v[t]) & 0x7fffffffu; m = (m ^ (uint32_t)(v[t] >> 32)) | 1u; }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) { uint64_t x = v[t]; v[t] = v[t + 8]; v[t + 8] = x; }
    }
    uint64_t s = 0;
    for (int i = 0; i < 16; ++i) s ^= v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float((uint32_t)s ^ m);
}

template <typename K>
void run(const char* name, K k, double values_per_thread_iter, int block) {
    float* out;
    cudaMalloc(&out, 148 * 8 * 1024 * 4);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int blocks = sms * (2048 / block);
    k<<<blocks, block>>>(out, 1.0f);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<<<blocks, block>>>(out, 1.0f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double elem_stages = (double)blocks * block * ITERS * values_per_thread_iter * 5;
    printf("%-16s block %4d: %7.3f ms  %6.2f value-stages/clk/SM (at 1.965 GHz)\n", name, block, ms,
           elem_stages / sms / (ms * 1e-3 * 1.965e9));
    cudaFree(out);
}
int main() {
    for (int blk : {256, 512, 1024}) {
        run("scalar", k_scalar<0>, 16, blk);
        run("scalar+lop", k_scalar<1>, 16, blk);
        run("packed", k_packed<0>, 32, blk);
        run("packed+lop", k_packed<1>, 32, blk);
    }
}
