// Pairwise correlation of the four up/down decisions of one cvt.rs.satfinite.e2m1x4.f32 (shared 32 rbits),
// over 2^28 random rbits, for several probabilities p (hardware stochastic rounding, sm_100a).
#include <cmath>
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
// s[i] = #up of slot i, s[4 + 4i + j] = #(up_i and up_j)
__global__ void k(float va, float vb, float vc, float vd, unsigned long long* s, int n) {
    unsigned long long c[20] = {};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t o = cvt_rs(va, vb, vc, vd, lowbias((uint32_t)i * 2654435761u + 12345u));
        int up[4];
        up[0] = ((o >> 12) & 7) == 3;   // a, b, c, d in (1, 1.5): up = code 3
        up[1] = ((o >> 8) & 7) == 3;
        up[2] = ((o >> 4) & 7) == 3;
        up[3] = (o & 7) == 3;
        for (int a = 0; a < 4; ++a) {
            c[a] += up[a];
            for (int b = 0; b < 4; ++b) c[4 + 4 * a + b] += up[a] & up[b];
        }
    }
    for (int a = 0; a < 20; ++a) atomicAdd(&s[a], c[a]);
}
int main() {
    unsigned long long* s;
    cudaMalloc(&s, 20 * 8);
    const int n = 1 << 28;
    const float ps[5][4] = {{.5f, .5f, .5f, .5f}, {.3f, .3f, .3f, .3f}, {.7f, .2f, .55f, .9f}, {.01f, .5f, .99f, .25f},
                            {.123f, .456f, .789f, .321f}};
    double worst = 0;
    for (int t = 0; t < 5; ++t) {
        cudaMemset(s, 0, 160);
        k<<<148 * 8, 256>>>(1 + .5f * ps[t][0], 1 + .5f * ps[t][1], 1 + .5f * ps[t][2], 1 + .5f * ps[t][3], s, n);
        unsigned long long h[20];
        cudaMemcpy(h, s, 160, cudaMemcpyDeviceToHost);
        printf("p = %.3f %.3f %.3f %.3f  P_hw = %.5f %.5f %.5f %.5f\n  corr:", ps[t][0], ps[t][1], ps[t][2], ps[t][3],
               (double)h[0] / n, (double)h[1] / n, (double)h[2] / n, (double)h[3] / n);
        for (int a = 0; a < 4; ++a)
            for (int b = a + 1; b < 4; ++b) {
                const double pa = (double)h[a] / n, pb = (double)h[b] / n, pab = (double)h[4 + 4 * a + b] / n;
                const double r = (pab - pa * pb) / sqrt(pa * (1 - pa) * pb * (1 - pb));
                if (fabs(r) > worst) worst = fabs(r);
                printf(" (%d,%d) %+.4f", a, b, r);
            }
        printf("\n");
    }
    printf("max |corr| = %.4f (sampling sd ~ %.1e)\n", worst, 1 / sqrt((double)n));
    return 0;
}
