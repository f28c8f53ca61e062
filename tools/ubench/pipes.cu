// pipes.cu -- issue/throughput microbenchmark of the instructions the quantizers lean on (B200).
// Not product code.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;
constexpr int CH = 8;  // independent chains per thread

#define KERNEL(NAME, DECL, BODY, OUT)                                                  \
    __global__ void NAME(uint32_t* out, uint32_t seed) {                                 \
        DECL;                                                                           \
        for (int it = 0; it < ITERS; ++it) {                                            \
            _Pragma("unroll") for (int c = 0; c < CH; ++c) { BODY; }                    \
        }                                                                               \
        OUT;                                                                            \
    }

// FFMA2 (3 x 64-bit regs)
KERNEL(k_ffma2, uint64_t v[CH]; uint64_t m = seed * 0x100000001ull; for (int c = 0; c < CH; ++c) v[c] = m + c,
       asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(v[c]) : "l"(m)),
       uint64_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c]; out[threadIdx.x] = (uint32_t)s)
KERNEL(k_fadd2, uint64_t v[CH]; uint64_t m = seed * 0x100000001ull; for (int c = 0; c < CH; ++c) v[c] = m + c,
       asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(v[c]) : "l"(m)),
       uint64_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c]; out[threadIdx.x] = (uint32_t)s)
KERNEL(k_fmul2, uint64_t v[CH]; uint64_t m = seed * 0x100000001ull; for (int c = 0; c < CH; ++c) v[c] = m + c,
       asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(v[c]) : "l"(m)),
       uint64_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c]; out[threadIdx.x] = (uint32_t)s)
KERNEL(k_ffma, float v[CH]; float m = __uint_as_float(seed); for (int c = 0; c < CH; ++c) v[c] = m + c,
       asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[c]) : "f"(m), "f"(v[(c + 1) % CH])),
       uint32_t s = 0; for (int c = 0; c < CH; ++c) s ^= __float_as_uint(v[c]); out[threadIdx.x] = s)
KERNEL(k_fadd, float v[CH]; float m = __uint_as_float(seed); for (int c = 0; c < CH; ++c) v[c] = m + c,
       asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(v[c]) : "f"(m)),
       uint32_t s = 0; for (int c = 0; c < CH; ++c) s ^= __float_as_uint(v[c]); out[threadIdx.x] = s)
KERNEL(k_lop3, uint32_t v[CH]; for (int c = 0; c < CH; ++c) v[c] = seed + c,
       asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(seed), "r"(v[(c + 3) % CH])),
       uint32_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c]; out[threadIdx.x] = s)
KERNEL(k_prmt, uint32_t v[CH]; for (int c = 0; c < CH; ++c) v[c] = seed + c,
       asm volatile("prmt.b32 %0, %0, %1, 0x1044;" : "+r"(v[c]) : "r"(seed)),
       uint32_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c]; out[threadIdx.x] = s)
KERNEL(k_shf, uint32_t v[CH]; for (int c = 0; c < CH; ++c) v[c] = seed + c,
       asm volatile("shf.l.wrap.b32 %0, %0, %1, 1;" : "+r"(v[c]) : "r"(seed)),
       uint32_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c]; out[threadIdx.x] = s)
KERNEL(k_fmnmx, float v[CH]; float m = __uint_as_float(seed); for (int c = 0; c < CH; ++c) v[c] = m + c,
       asm volatile("max.f32 %0, %0, %1;" : "+f"(v[c]) : "f"(v[(c + 1) % CH])),
       uint32_t s = 0; for (int c = 0; c < CH; ++c) s ^= __float_as_uint(v[c]); out[threadIdx.x] = s)
// e2m1x2 pack: 2 f32 -> 1 byte
KERNEL(k_cvt_e2m1, float v[CH]; uint32_t acc = 0; float m = __uint_as_float(seed); for (int c = 0; c < CH; ++c) v[c] = m + c,
       { uint16_t r; asm volatile("{\n .reg .b8 t;\n cvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n cvt.u16.u8 %0, t;\n}" : "=h"(r) : "f"(v[c]), "f"(v[(c+1)%CH])); acc += r; v[c] = __uint_as_float(__float_as_uint(v[c]) ^ r); },
       out[threadIdx.x] = acc)
// e2m1x2 -> f16x2
KERNEL(k_cvt_f16, uint32_t v[CH]; for (int c = 0; c < CH; ++c) v[c] = seed + c,
       asm volatile("{\n .reg .b8 t;\n cvt.u8.u32 t, %0;\n cvt.rn.f16x2.e2m1x2 %0, t;\n}" : "+r"(v[c])),
       uint32_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c]; out[threadIdx.x] = s)
// f16 -> f32
KERNEL(k_h2f, uint32_t v[CH]; for (int c = 0; c < CH; ++c) v[c] = seed + c,
       { float f; asm volatile("{\n .reg .b16 lo, hi;\n mov.b32 {lo, hi}, %1;\n cvt.f32.f16 %0, lo;\n}" : "=f"(f) : "r"(v[c])); v[c] = __float_as_uint(f); },
       uint32_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c]; out[threadIdx.x] = s)
// mixed: 1 FFMA2 + 1 LOP3 per step (dual pipe)
KERNEL(k_mix, uint64_t v[CH]; uint32_t w[CH]; uint64_t m = seed * 0x100000001ull; for (int c = 0; c < CH; ++c) { v[c] = m + c; w[c] = seed + c; },
       asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(v[c]) : "l"(m)); asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(w[c]) : "r"(seed), "r"(w[(c + 3) % CH])),
       uint64_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c] ^ w[c]; out[threadIdx.x] = (uint32_t)s)
// mixed: FADD2 + FFMA2 alternating (butterfly pattern)
KERNEL(k_bfly, uint64_t v[CH]; uint64_t m = seed * 0x100000001ull; for (int c = 0; c < CH; ++c) v[c] = m + c,
       asm volatile("add.rn.f32x2 %0, %0, %1;\n fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[c]) : "l"(m), "l"(v[(c+1)%CH])),
       uint64_t s = 0; for (int c = 0; c < CH; ++c) s ^= v[c]; out[threadIdx.x] = (uint32_t)s)

template <typename K>
void run(const char* name, K k, double ops_per_body) {
    uint32_t* out;
    cudaMalloc(&out, 1024 * 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    dim3 grid(sms * 4), block(512);  // 64 warps / SM
    k<<<grid, block>>>(out, 0x3f800001u);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k<<<grid, block>>>(out, 0x3f800001u);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    double warp_instr = (double)grid.x * block.x / 32 * ITERS * CH * ops_per_body * reps;
    double per_sm_per_ns = warp_instr / sms / (ms * 1e6);
    printf("%-10s %8.3f ms  %6.3f warp-instr/ns/SM  (= %5.2f /clk/SM at %d MHz max)\n", name, ms, per_sm_per_ns,
           per_sm_per_ns / (clk_khz / 1e6), clk_khz / 1000);
    cudaFree(out);
}

int main() {
    run("ffma2", k_ffma2, 1);
    run("fadd2", k_fadd2, 1);
    run("fmul2", k_fmul2, 1);
    run("ffma", k_ffma, 1);
    run("fadd", k_fadd, 1);
    run("lop3", k_lop3, 1);
    run("prmt", k_prmt, 1);
    run("shf", k_shf, 1);
    run("fmnmx", k_fmnmx, 1);
    run("cvt_e2m1", k_cvt_e2m1, 1);
    run("cvt_f16", k_cvt_f16, 1);
    run("h2f", k_h2f, 1);
    run("mix", k_mix, 2);
    run("bfly", k_bfly, 2);
    return 0;
}
