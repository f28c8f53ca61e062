/*
 * quartet_oracle.c -- CPU restatement of the reference's Quartet linear-layer kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200 path: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load it.
 * The product path (paper_2505_14669_b200) never calls it.
 *
 * Every function restates, operation for operation, the reference implementation in
 * /root/reference/pkg/src/mx4train/_backend/_native.pyx (abbreviated `_native.pyx`) and
 * rng.py, so results are bit-identical: same f64/f32 op order, no FMA contraction
 * (compile with -ffp-contract=off, as the reference's setup.py:5-12 does).
 *
 * The only deviation is an optional OpenMP loop over independent rows (nthreads > 1),
 * which does not change any per-element operation order.
 *
 * Parity pins: tests/test_oracle_golden.py checks every entry point against golden vectors
 * produced by the reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_API __attribute__((visibility("default")))

static const double GRID_C[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};       /* _native.pyx:24-25 */
static const double SGRID_C[15] = {-6.0, -4.0, -3.0, -2.0, -1.5, -1.0, -0.5, 0.0,
                                   0.5,  1.0,  1.5,  2.0,  3.0,  4.0,  6.0};      /* _native.pyx:26-27 */
static const uint8_t SGRID_CODE_C[15] = {15, 14, 13, 12, 11, 10, 9, 0, 1, 2, 3, 4, 5, 6, 7}; /* :28-29 */

#define DOMAIN_SR 0x5352ULL      /* rng.py:21 */
#define DOMAIN_SIGNS 0x5347ULL   /* rng.py:22 */
#define GOLDEN 0x9E3779B97F4A7C15ULL
static const double U53 = 1.0 / 9007199254740992.0;

static void set_threads(int nthreads) {
#ifdef _OPENMP
    omp_set_num_threads(nthreads > 0 ? nthreads : 1);
#else
    (void)nthreads;
#endif
}

/* ---------------------------------------------------------------- rng.py */

/* rng.py:27-31 / _native.pyx:35-38 */
ORC_API uint64_t orc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* rng.py:34-37 */
ORC_API uint64_t orc_stream_base(uint64_t seed, uint64_t domain) {
    return orc_mix64(seed ^ orc_mix64(domain));
}

/* rng.py:40-44 */
ORC_API uint64_t orc_raw_at(uint64_t seed, uint64_t domain, uint64_t index) {
    return orc_mix64(orc_stream_base(seed, domain) + (index + 1) * GOLDEN);
}

/* rng.py:47-50 (vectorised over a contiguous index range) */
ORC_API void orc_uniform(uint64_t seed, uint64_t domain, uint64_t start, int64_t count, double* out) {
    uint64_t base = orc_stream_base(seed, domain);
    for (int64_t i = 0; i < count; ++i) {
        uint64_t h = orc_mix64(base + ((start + (uint64_t)i) + 1) * GOLDEN);
        out[i] = (double)(h >> 11) * U53;
    }
}

/* rng.py:57-62: +1 / -1 from the top bit of raw_at(seed, DOMAIN_SIGNS, i) */
ORC_API void orc_signs_f32(uint64_t seed, uint64_t start, int64_t count, float* out) {
    uint64_t base = orc_stream_base(seed, DOMAIN_SIGNS);
    for (int64_t i = 0; i < count; ++i) {
        uint64_t h = orc_mix64(base + ((start + (uint64_t)i) + 1) * GOLDEN);
        out[i] = (h >> 63) ? -1.0f : 1.0f;
    }
}

/* rng.py:72-78 */
ORC_API uint64_t orc_derive_seed(const uint64_t* parts, int nparts) {
    uint64_t acc = 0x243F6A8885A308D3ULL;
    for (int i = 0; i < nparts; ++i) {
        acc = orc_mix64(acc ^ parts[i]);
        acc = acc + GOLDEN;
    }
    return orc_mix64(acc);
}

/* ------------------------------------------------------- _native.pyx helpers */

/* _native.pyx:46-63 */
static inline int grid_index(double a) {
    int idx = 0;
    if (a > 0.25) idx += 1;
    if (a >= 0.75) idx += 1;
    if (a > 1.25) idx += 1;
    if (a >= 1.75) idx += 1;
    if (a > 2.5) idx += 1;
    if (a >= 3.5) idx += 1;
    if (a > 5.0) idx += 1;
    return idx;
}

/* _native.pyx:66-78 */
static inline int ceil_scale_exponent(double amax) {
    int e2, e;
    double m;
    if (amax <= 0.0) return 0;
    m = frexp(amax / 6.0, &e2);
    e = 127 + e2 - (m == 0.5 ? 1 : 0);
    if (e < 0) e = 0;
    if (e > 254) e = 254;
    return e;
}

/* _native.pyx:81-89 */
static inline int floor_exponent_clamped(double t) {
    int e2;
    frexp(t, &e2);
    int e = 127 + e2 - 1;
    if (e < 0) e = 0;
    if (e > 254) e = 254;
    return e;
}

/* _native.pyx:92-101 */
static inline double group_absmax(const double* row, int64_t lo, int64_t hi) {
    double amax = 0.0, a;
    for (int64_t j = lo; j < hi; ++j) {
        a = row[j] >= 0.0 ? row[j] : -row[j];
        if (a > amax) amax = a;
    }
    return amax;
}

/* --------------------------------------------------------------- quantizers */

/* _native.pyx:104-131.  codes: unpacked nibbles [rows, cols]; scales [rows, ceil(cols/g)] */
ORC_API void orc_quantize_rtn(const double* x, int64_t rows, int64_t cols, int g, uint8_t* codes,
                              uint8_t* scales, int nthreads) {
    int64_t ngroups = (cols + g - 1) / g;
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
        const double* xr = x + i * cols;
        for (int64_t gi = 0; gi < ngroups; ++gi) {
            int64_t lo = gi * g, hi = lo + g;
            if (hi > cols) hi = cols;
            int e = ceil_scale_exponent(group_absmax(xr, lo, hi));
            scales[i * ngroups + gi] = (uint8_t)e;
            double s = ldexp(1.0, e - 127);
            for (int64_t j = lo; j < hi; ++j) {
                double v = xr[j] / s;
                int idx = grid_index(v >= 0.0 ? v : -v);
                codes[i * cols + j] = idx == 0 ? 0 : (uint8_t)(idx | (v < 0.0 ? 8 : 0));
            }
        }
    }
}

/* _native.pyx:134-168.  Element (i, j) draws stream position counter_start + i*cols + j. */
ORC_API void orc_quantize_sr(const double* x, int64_t rows, int64_t cols, int g, uint64_t seed,
                             uint64_t counter_start, uint8_t* codes, uint8_t* scales, int nthreads) {
    int64_t ngroups = (cols + g - 1) / g;
    uint64_t base = orc_mix64(seed ^ orc_mix64(DOMAIN_SR));
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
        const double* xr = x + i * cols;
        for (int64_t gi = 0; gi < ngroups; ++gi) {
            int64_t lo = gi * g, hi = lo + g;
            if (hi > cols) hi = cols;
            int e = ceil_scale_exponent(group_absmax(xr, lo, hi));
            scales[i * ngroups + gi] = (uint8_t)e;
            double s = ldexp(1.0, e - 127);
            for (int64_t j = lo; j < hi; ++j) {
                double v = xr[j] / s;
                int k = 1;
                while (k < 14 && SGRID_C[k] < v) k += 1;
                double p = (v - SGRID_C[k - 1]) / (SGRID_C[k] - SGRID_C[k - 1]);
                uint64_t h = orc_mix64(base + ((counter_start + (uint64_t)(i * cols + j)) + 1) * GOLDEN);
                double u = (double)(h >> 11) * U53;
                codes[i * cols + j] = u < p ? SGRID_CODE_C[k] : SGRID_CODE_C[k - 1];
            }
        }
    }
}

/* _native.pyx:171-203 */
static int quest_best_exponent(const double* xr, int64_t lo, int64_t hi, double amax,
                               double ratio_lo, double* vbuf) {
    int e_hi = ceil_scale_exponent(amax);
    int e_lo = floor_exponent_clamped((amax * ratio_lo) / 6.0);
    double s_hi = ldexp(1.0, e_hi - 127);
    int64_t n = hi - lo;
    for (int64_t j = 0; j < n; ++j) vbuf[j] = xr[lo + j] / s_hi;
    int best_e = e_hi;
    double best_err = -1.0;
    for (int e = e_hi; e >= e_lo; --e) {
        double s2 = ldexp(1.0, 2 * (e - 127));
        double acc = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            double v = vbuf[j];
            double a = v >= 0.0 ? v : -v;
            int idx = grid_index(a);
            double t = a - GRID_C[idx];
            acc += t * t;
        }
        double err = s2 * acc;
        if (best_err < 0.0 || err < best_err) {
            best_err = err;
            best_e = e;
        }
        for (int64_t j = 0; j < n; ++j) vbuf[j] = vbuf[j] * 2.0;
    }
    return best_e;
}

/* _native.pyx:206-245.  mask[i, j] = 1 where |x/s| <= 6 at the chosen scale. */
ORC_API void orc_quantize_quest(const double* x, int64_t rows, int64_t cols, int g, double ratio_lo,
                                uint8_t* codes, uint8_t* scales, uint8_t* mask, int nthreads) {
    int64_t ngroups = (cols + g - 1) / g;
    set_threads(nthreads);
#pragma omp parallel
    {
        double* vbuf = (double*)malloc(sizeof(double) * (size_t)g);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < rows; ++i) {
            const double* xr = x + i * cols;
            for (int64_t gi = 0; gi < ngroups; ++gi) {
                int64_t lo = gi * g, hi = lo + g;
                if (hi > cols) hi = cols;
                double amax = group_absmax(xr, lo, hi);
                if (amax <= 0.0) {
                    scales[i * ngroups + gi] = 0;
                    for (int64_t j = lo; j < hi; ++j) {
                        codes[i * cols + j] = 0;
                        mask[i * cols + j] = 1;
                    }
                    continue;
                }
                int best_e = quest_best_exponent(xr, lo, hi, amax, ratio_lo, vbuf);
                scales[i * ngroups + gi] = (uint8_t)best_e;
                double s = ldexp(1.0, best_e - 127);
                for (int64_t j = lo; j < hi; ++j) {
                    double v = xr[j] / s;
                    double a = v >= 0.0 ? v : -v;
                    mask[i * cols + j] = a <= 6.0 ? 1 : 0;
                    int idx = grid_index(a);
                    codes[i * cols + j] = idx == 0 ? 0 : (uint8_t)(idx | (v < 0.0 ? 8 : 0));
                }
            }
        }
        free(vbuf);
    }
}

/* -------------------------------------------------------------------- fwht */

/* _native.pyx:353-379: in-place blockwise orthonormal FWHT, ascending stride, (a+b)*c, (a-b)*c */
ORC_API void orc_fwht_f32(float* x, int64_t rows, int64_t n, int g, int nthreads) {
    const float c = (float)(1.0 / sqrt(2.0));
    int64_t nblk_row = n / g;
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
        for (int64_t b = 0; b < nblk_row; ++b) {
            float* flat = x + r * n + b * g;
            for (int h = 1; h < g; h *= 2) {
                for (int start = 0; start < g; start += 2 * h) {
                    for (int t = start; t < start + h; ++t) {
                        float a = flat[t], bb = flat[t + h];
                        flat[t] = (a + bb) * c;
                        flat[t + h] = (a - bb) * c;
                    }
                }
            }
        }
    }
}

ORC_API void orc_fwht_f64(double* x, int64_t rows, int64_t n, int g, int nthreads) {
    const double c = 1.0 / sqrt(2.0);
    int64_t nblk_row = n / g;
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
        for (int64_t b = 0; b < nblk_row; ++b) {
            double* flat = x + r * n + b * g;
            for (int h = 1; h < g; h *= 2) {
                for (int start = 0; start < g; start += 2 * h) {
                    for (int t = start; t < start + h; ++t) {
                        double a = flat[t], bb = flat[t + h];
                        flat[t] = (a + bb) * c;
                        flat[t + h] = (a - bb) * c;
                    }
                }
            }
        }
    }
}

/* -------------------------------------------------------------------- gemm */

/* _native.pyx:382-396: C = A B^T, i-k-j loops, sequential += per output, no FMA.
 * The j loop auto-vectorises; each c[i,j] still sees its k terms in ascending order. */
ORC_API void orc_gemm_nt_f32(const float* a, const float* b, int64_t m, int64_t n, int64_t k,
                             float* c, int nthreads) {
    float* bt = (float*)malloc(sizeof(float) * (size_t)(n * k > 0 ? n * k : 1));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t kk = 0; kk < k; ++kk) bt[kk * n + j] = b[j * k + kk];
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        float* ci = c + i * n;
        for (int64_t j = 0; j < n; ++j) ci[j] = 0.0f;
        for (int64_t kk = 0; kk < k; ++kk) {
            float av = a[i * k + kk];
            const float* br = bt + kk * n;
            for (int64_t j = 0; j < n; ++j) ci[j] = ci[j] + av * br[j];
        }
    }
    free(bt);
}

ORC_API void orc_gemm_nt_f64(const double* a, const double* b, int64_t m, int64_t n, int64_t k,
                             double* c, int nthreads) {
    double* bt = (double*)malloc(sizeof(double) * (size_t)(n * k > 0 ? n * k : 1));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t kk = 0; kk < k; ++kk) bt[kk * n + j] = b[j * k + kk];
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        double* ci = c + i * n;
        for (int64_t j = 0; j < n; ++j) ci[j] = 0.0;
        for (int64_t kk = 0; kk < k; ++kk) {
            double av = a[i * k + kk];
            const double* br = bt + kk * n;
            for (int64_t j = 0; j < n; ++j) ci[j] = ci[j] + av * br[j];
        }
    }
    free(bt);
}
