// Which bits of rbits drive each element of cvt.rs.satfinite.e2m1x4.f32, and the exact up-probability it
// realises for a value between two grid points (hardware stochastic rounding, sm_100a).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t cvt_rs(float a, float b, float c, float d, uint32_t rb) {
    uint16_t o;
    asm("cvt.rs.satfinite.e2m1x4.f32 %0, {%1, %2, %3, %4}, %5;" : "=h"(o) : "f"(a), "f"(b), "f"(c), "f"(d), "r"(rb));
    return o;
}
__device__ uint32_t lowbias(uint32_t h) {
    h ^= h >> 16; h *= 0x7FEB352Du; h ^= h >> 15; h *= 0x846CA68Bu; h ^= h >> 16; return h;
}
// influence[p][b]: how many of 4096 random rbits flip element p's code when bit b flips
__global__ void k_infl(const float* v, unsigned* infl) {
    const int b = threadIdx.x;  // 32 threads = bits
    for (int s = 0; s < 4096; ++s) {
        const uint32_t r = lowbias(s * 7919u + 17u);
        const uint32_t o0 = cvt_rs(v[0], v[1], v[2], v[3], r), o1 = cvt_rs(v[0], v[1], v[2], v[3], r ^ (1u << b));
        for (int p = 0; p < 4; ++p)
            if (((o0 >> (4 * p)) ^ (o1 >> (4 * p))) & 0xF) atomicAdd(&infl[p * 32 + b], 1u);
    }
}
// count of "upper neighbour" outcomes per element over n rbits values r = lowbias(i)
__global__ void k_prob(const float* v, unsigned long long* hist, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t o = cvt_rs(v[0], v[1], v[2], v[3], lowbias((uint32_t)i));
        for (int p = 0; p < 4; ++p) atomicAdd(&hist[p * 16 + ((o >> (4 * p)) & 0xF)], 1ull);
    }
}
// exhaustive over all 2^32 rbits is too long; over the 2^24 values (i << 8) | 0x5A and (i) for low-bit checks
__global__ void k_exh(const float* v, const unsigned* upcode, unsigned long long* cnt, uint32_t shift, uint32_t fill) {
    unsigned long long c[4] = {0, 0, 0, 0};
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (1u << 24); i += gridDim.x * blockDim.x) {
        const uint32_t o = cvt_rs(v[0], v[1], v[2], v[3], (i << shift) | fill);
        for (int p = 0; p < 4; ++p) c[p] += (((o >> (4 * p)) & 0xF) == upcode[p]);
    }
    for (int p = 0; p < 4; ++p) atomicAdd(&cnt[p], c[p]);
}

int main() {
    // element values: 1.25 (1 | 1.5, p = .5), 0.3 (0 | 0.5, p = .6), 4.4 (4 | 6, p = .2), 2.0000002 (2 | 3)
    float hv[4] = {1.25f, 0.3f, 4.4f, 2.75f};
    unsigned hup[4] = {3u, 1u, 7u, 5u};   // codes of 1.5, 0.5, 6, 3
    double exact[4] = {0.5, 0.6, 0.2, (2.0000002 - 2.0) / 1.0};
    float* v; unsigned* infl; unsigned* up; unsigned long long* cnt;
    cudaMalloc(&v, 16); cudaMalloc(&infl, 4 * 32 * 4); cudaMalloc(&up, 16); cudaMalloc(&cnt, 32);
    cudaMemcpy(v, hv, 16, cudaMemcpyHostToDevice); cudaMemcpy(up, hup, 16, cudaMemcpyHostToDevice);
    cudaMemset(infl, 0, 512);
    k_infl<<<1, 32>>>(v, infl);
    unsigned hi[128];
    cudaMemcpy(hi, infl, 512, cudaMemcpyDeviceToHost);
    for (int p = 0; p < 4; ++p) {
        printf("element %d (v=%g) influenced by bits:", p, hv[p]);
        for (int b = 0; b < 32; ++b) if (hi[p * 32 + b]) printf(" %d(%u)", b, hi[p * 32 + b]);
        printf("\n");
    }
    const int n = 1 << 26;
    unsigned long long* hist;
    cudaMalloc(&hist, 64 * 8);
    cudaMemset(hist, 0, 64 * 8);
    k_prob<<<148 * 8, 256>>>(v, hist, n);
    unsigned long long hh[64];
    cudaMemcpy(hh, hist, 64 * 8, cudaMemcpyDeviceToHost);
    for (int p = 0; p < 4; ++p) {
        printf("nibble %d:", p);
        for (int c = 0; c < 16; ++c) if (hh[p * 16 + c]) printf("  code %d: %.8f", c, (double)hh[p * 16 + c] / n);
        printf("\n");
    }
    return 0;
}
