// Exact up-probabilities of the hardware stochastic rounding cvt.rs.satfinite.e2m1x4.f32 (sm_100a): every one of
// the 2^32 rbits values, for values v with long binary expansions of p = (v - lo) / (hi - lo); prints P_hw - p.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t cvt_rs(float a, float b, float c, float d, uint32_t rb) {
    uint16_t o;
    asm("cvt.rs.satfinite.e2m1x4.f32 %0, {%1, %2, %3, %4}, %5;" : "=h"(o) : "f"(a), "f"(b), "f"(c), "f"(d), "r"(rb));
    return o;
}
// nibble 3 <- a, 2 <- b, 1 <- c, 0 <- d; count outcomes equal to the upper neighbour's code
__global__ void k(const float* v, const unsigned* up, unsigned long long* cnt) {
    unsigned long long c[4] = {0, 0, 0, 0};
    const uint64_t n = 1ull << 32;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t o = cvt_rs(v[0], v[1], v[2], v[3], (uint32_t)i);
        c[0] += ((o >> 12) & 0xF) == up[0];
        c[1] += ((o >> 8) & 0xF) == up[1];
        c[2] += ((o >> 4) & 0xF) == up[2];
        c[3] += (o & 0xF) == up[3];
    }
    for (int p = 0; p < 4; ++p) atomicAdd(&cnt[p], c[p]);
}

static const float grid[8] = {0.f, 0.5f, 1.f, 1.5f, 2.f, 3.f, 4.f, 6.f};

int main() {
    float *v; unsigned* up; unsigned long long* cnt;
    cudaMalloc(&v, 16); cudaMalloc(&up, 16); cudaMalloc(&cnt, 32);
    double worst = 0;
    // 3 tuples x 4 slots: v = lo + frac * span with irrational-ish fractions, in every grid interval
    const double fr[12] = {1 / 3.0, 0.1, 0.7071067811865476, 0.9999, 1e-4, 0.31830988618379, 0.5772156649,
                           0.0078125 + 1e-6, 0.99609375 + 1e-6, 0.6180339887, 0.2718281828, 0.1414213562};
    for (int t = 0; t < 7; ++t) {   // grid intervals 0..6
        for (int q = 0; q < 3; ++q) {
            float hv[4]; unsigned hu[4]; double p[4];
            for (int s = 0; s < 4; ++s) {
                const double f = fr[(q * 4 + s) % 12];
                const double lo = grid[t], hi = grid[t + 1];
                hv[s] = (float)(lo + f * (hi - lo));
                p[s] = ((double)hv[s] - lo) / (hi - lo);
                hu[s] = t + 1;
                if (s & 1) { hv[s] = -hv[s]; hu[s] |= 8; }   // negative values: sign-symmetric SR
            }
            cudaMemcpy(v, hv, 16, cudaMemcpyHostToDevice);
            cudaMemcpy(up, hu, 16, cudaMemcpyHostToDevice);
            cudaMemset(cnt, 0, 32);
            k<<<148 * 16, 256>>>(v, up, cnt);
            unsigned long long hc[4];
            cudaMemcpy(hc, cnt, 32, cudaMemcpyDeviceToHost);
            for (int s = 0; s < 4; ++s) {
                const double ph = (double)hc[s] / 4294967296.0, d = ph - p[s];
                if (fabs(d) > worst) worst = fabs(d);
                printf("[%g,%g] v=%+.9g p=%.10f P_hw=%.10f diff=%+.3e (x2^14 = %+.3f)\n", grid[t], grid[t + 1], hv[s],
                       p[s], ph, d, d * 16384.0);
            }
        }
    }
    printf("max |P_hw - p| = %.3e = 2^%.2f\n", worst, log2(worst));
    return 0;
}
