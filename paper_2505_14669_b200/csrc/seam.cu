// seam.cu -- the reference's kernel-plugin seam for EVERY input its kernels accept.
//
// The layer path runs on the tiled kernels (quant.cu, tcq.cu, gemm.cu), which take bf16 / fp32 matrices,
// group 32 and FWHT-32.  The reference's `kernels` module (mx4train/_backend/_native.pyx) is more general:
// f64 matrices, any group size, any power-of-two FWHT block in f32 or f64, and a GEMM with a fixed
// ascending-k order.  These kernels replay _native.pyx operation for operation in scalar f64 / f32 code
// (the library is built with --fmad=false, so no multiply-add is contracted, like setup.py:5-12), one
// thread per group, transform block or output element -- bit-identical for every input, including
// ragged trailing groups, subnormal and huge values:
//
//   k_seam_quant<ROUND, VALUES>  quantize_rtn / quantize_sr / quantize_quest   _native.pyx:104-245
//                                rtn_values / sr_values / quest_values         _native.pyx:248-350
//   k_seam_fwht<T>               fwht (in place, ascending stride h)           _native.pyx:353-379
//   k_seam_gemm_nt<T>            gemm_nt (c = c + a*b, ascending k)            _native.pyx:382-396
//   k_seam_row_sums              numpy's pairwise add.reduce along rows of (a-b)^2 or a*b, the reductions
//                                of diagnostics.gaussian_mse / misalignment_suite (diagnostics.py:84, 161-165)
//
// They are not on the layer's hot path (the B200 layer never sees f64), so they favour exactness over
// speed: the per-thread loops read global memory through L1.
#include "launch.h"
#include "quant.cuh"  // Rounding

namespace qt {

__constant__ double kGridC[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};                        // _native.pyx:24
__constant__ double kSGridC[15] = {-6.0, -4.0, -3.0, -2.0, -1.5, -1.0, -0.5, 0.0,
                                   0.5,  1.0,  1.5,  2.0,  3.0,  4.0,  6.0};                     // _native.pyx:26
__constant__ uint8_t kSGridCode[15] = {15, 14, 13, 12, 11, 10, 9, 0, 1, 2, 3, 4, 5, 6, 7};      // _native.pyx:28

// _native.pyx:46-63
__device__ __forceinline__ int seam_grid_index(double a) {
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

// C frexp (glibc semantics: zero / inf / nan -> exponent 0, value returned unchanged)
__device__ __forceinline__ double seam_frexp(double t, int* e2) {
    if (t == 0.0 || !isfinite(t)) {
        *e2 = 0;
        return t;
    }
    return frexp(t, e2);
}

// _native.pyx:66-78
__device__ __forceinline__ int seam_ceil_scale_exponent(double amax) {
    if (amax <= 0.0) return 0;
    int e2;
    const double m = seam_frexp(amax / 6.0, &e2);
    int e = 127 + e2 - (m == 0.5 ? 1 : 0);
    return e < 0 ? 0 : (e > 254 ? 254 : e);
}

// _native.pyx:81-89
__device__ __forceinline__ int seam_floor_exponent_clamped(double t) {
    int e2;
    seam_frexp(t, &e2);
    const int e = 127 + e2 - 1;
    return e < 0 ? 0 : (e > 254 ? 254 : e);
}

__device__ __forceinline__ double seam_pow2(int k) { return ldexp(1.0, k); }

// _native.pyx:171-203: the candidate error accumulated in the divided domain (vbuf doubled per candidate;
// v_j * 2^k is exact for any value, normal or subnormal, so it is recomputed instead of stored).
__device__ int seam_quest_best_exponent(const double* xr, int64_t lo, int64_t hi, double amax, double ratio_lo) {
    const int e_hi = seam_ceil_scale_exponent(amax);
    const int e_lo = seam_floor_exponent_clamped((amax * ratio_lo) / 6.0);
    const double s_hi = seam_pow2(e_hi - 127);
    int best_e = e_hi;
    double best_err = -1.0, mult = 1.0;
    for (int e = e_hi; e >= e_lo; --e) {
        const double s2 = seam_pow2(2 * (e - 127));
        double acc = 0.0;
        for (int64_t j = lo; j < hi; ++j) {
            const double v = __dmul_rn(__ddiv_rn(xr[j], s_hi), mult);
            const double a = v >= 0.0 ? v : -v;
            const double t = __dsub_rn(a, kGridC[seam_grid_index(a)]);
            acc = __dadd_rn(acc, __dmul_rn(t, t));
        }
        const double err = __dmul_rn(s2, acc);
        if (best_err < 0.0 || err < best_err) {
            best_err = err;
            best_e = e;
        }
        mult = __dmul_rn(mult, 2.0);
    }
    return best_e;
}

__device__ __forceinline__ double seam_absmax(const double* xr, int64_t lo, int64_t hi) {  // _native.pyx:92-101
    double amax = 0.0;
    for (int64_t j = lo; j < hi; ++j) {
        const double a = xr[j] >= 0.0 ? xr[j] : -xr[j];
        if (a > amax) amax = a;
    }
    return amax;
}

__device__ __forceinline__ double seam_uniform(uint64_t base, uint64_t idx) {  // rng.py:47-50, _native.pyx:41-43
    const uint64_t h = mix64(base + (idx + 1) * kGolden);
    return __dmul_rn((double)(h >> 11), 1.0 / 9007199254740992.0);
}

struct SeamQuantArgs {
    const double* x;
    int64_t rows, cols, group;
    uint64_t sr_base, counter_start;
    double ratio_lo;
    uint8_t* codes;   // [rows, cols] (codes mode)
    uint8_t* scales;  // [rows, ngroups] (codes mode)
    uint8_t* mask;    // [rows, cols] (QuEST)
    double* values;   // [rows, cols] (values mode)
};

// One thread per (row, group).  ROUND: kQuest / kRtn / kSr; VALUES: the *_values variant.
template <int ROUND, bool VALUES>
__global__ void __launch_bounds__(128) k_seam_quant(SeamQuantArgs a) {
    const int64_t ng = (a.cols + a.group - 1) / a.group;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= a.rows * ng) return;
    const int64_t i = t / ng, gi = t - i * ng;
    const int64_t lo = gi * a.group, hi = lo + a.group < a.cols ? lo + a.group : a.cols;
    const double* xr = a.x + i * a.cols;
    const int64_t o = i * a.cols;
    if (ROUND == kQuest) {
        const double amax = seam_absmax(xr, lo, hi);
        if (amax <= 0.0) {  // _native.pyx:228-233 / 321-325
            if (!VALUES) a.scales[i * ng + gi] = 0;
            for (int64_t j = lo; j < hi; ++j) {
                if (VALUES)
                    a.values[o + j] = 0.0;
                else
                    a.codes[o + j] = 0;
                a.mask[o + j] = 1;
            }
            return;
        }
        int best_e;
        if (!VALUES) {
            best_e = seam_quest_best_exponent(xr, lo, hi, amax, a.ratio_lo);
            a.scales[i * ng + gi] = (uint8_t)best_e;
        } else {  // quest_values: error in the value domain (_native.pyx:326-339)
            const int e_hi = seam_ceil_scale_exponent(amax);
            const int e_lo = seam_floor_exponent_clamped((amax * a.ratio_lo) / 6.0);
            best_e = e_hi;
            double best_err = -1.0;
            for (int e = e_hi; e >= e_lo; --e) {
                const double s = seam_pow2(e - 127);
                double err = 0.0;
                for (int64_t j = lo; j < hi; ++j) {
                    const double v = __ddiv_rn(xr[j], s);
                    const double mag = __dmul_rn(kGridC[seam_grid_index(v >= 0.0 ? v : -v)], s);
                    const double d = __dsub_rn(xr[j], xr[j] < 0.0 ? -mag : mag);
                    err = __dadd_rn(err, __dmul_rn(d, d));
                }
                if (best_err < 0.0 || err < best_err) {
                    best_err = err;
                    best_e = e;
                }
            }
        }
        const double s = seam_pow2(best_e - 127);
        for (int64_t j = lo; j < hi; ++j) {
            const double v = __ddiv_rn(xr[j], s);
            const double av = v >= 0.0 ? v : -v;
            a.mask[o + j] = av <= 6.0 ? 1 : 0;
            const int idx = seam_grid_index(av);
            if (VALUES) {
                const double mag = __dmul_rn(kGridC[idx], s);
                a.values[o + j] = v < 0.0 ? -mag : mag;
            } else {
                a.codes[o + j] = idx == 0 ? 0 : (uint8_t)(idx | (v < 0.0 ? 8 : 0));
            }
        }
    } else {
        const int e = seam_ceil_scale_exponent(seam_absmax(xr, lo, hi));
        if (!VALUES) a.scales[i * ng + gi] = (uint8_t)e;
        const double s = seam_pow2(e - 127);
        for (int64_t j = lo; j < hi; ++j) {
            const double v = __ddiv_rn(xr[j], s);
            if (ROUND == kRtn) {  // _native.pyx:124-131 / 262-271
                const int idx = seam_grid_index(v >= 0.0 ? v : -v);
                if (VALUES) {
                    const double mag = __dmul_rn(kGridC[idx], s);
                    a.values[o + j] = v < 0.0 ? -mag : mag;
                } else {
                    a.codes[o + j] = idx == 0 ? 0 : (uint8_t)(idx | (v < 0.0 ? 8 : 0));
                }
            } else {  // _native.pyx:155-168 / 293-301
                int k = 1;
                while (k < 14 && kSGridC[k] < v) k += 1;
                const double p = __ddiv_rn(__dsub_rn(v, kSGridC[k - 1]), __dsub_rn(kSGridC[k], kSGridC[k - 1]));
                const double u = seam_uniform(a.sr_base, a.counter_start + (uint64_t)(i * a.cols + j));
                if (VALUES)
                    a.values[o + j] = u < p ? __dmul_rn(kSGridC[k], s) : __dmul_rn(kSGridC[k - 1], s);
                else
                    a.codes[o + j] = u < p ? kSGridCode[k] : kSGridCode[k - 1];
            }
        }
    }
}

// _native.pyx:353-379: one thread per block of g, in place, stages h = 1, 2, .. g/2, (a+b)*c and (a-b)*c.
template <typename T>
__device__ __forceinline__ T seam_add(T a, T b);
template <>
__device__ __forceinline__ float seam_add(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double seam_add(double a, double b) { return __dadd_rn(a, b); }
template <typename T>
__device__ __forceinline__ T seam_sub(T a, T b);
template <>
__device__ __forceinline__ float seam_sub(float a, float b) { return __fsub_rn(a, b); }
template <>
__device__ __forceinline__ double seam_sub(double a, double b) { return __dsub_rn(a, b); }
template <typename T>
__device__ __forceinline__ T seam_mul(T a, T b);
template <>
__device__ __forceinline__ float seam_mul(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double seam_mul(double a, double b) { return __dmul_rn(a, b); }

template <typename T>
__global__ void __launch_bounds__(128) k_seam_fwht(T* x, int64_t nblk, int64_t g, T c) {
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nblk) return;
    T* flat = x + b * g;
    for (int64_t h = 1; h < g; h *= 2)
        for (int64_t start = 0; start < g; start += 2 * h)
            for (int64_t t = start; t < start + h; ++t) {
                const T u = flat[t], v = flat[t + h];
                flat[t] = seam_mul(seam_add(u, v), c);
                flat[t + h] = seam_mul(seam_sub(u, v), c);
            }
}

// _native.pyx:382-396: c[i, j] = c[i, j] + a[i, k] * b[j, k] for k ascending, starting from zero.
template <typename T>
__global__ void __launch_bounds__(256) k_seam_gemm_nt(const T* a, const T* b, T* c, int64_t m, int64_t n, int64_t k) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= m * n) return;
    const int64_t i = t / n, j = t - i * n;
    const T* ar = a + i * k;
    const T* br = b + j * k;
    T acc = T(0);
    for (int64_t kk = 0; kk < k; ++kk) acc = seam_add(acc, seam_mul(ar[kk], br[kk]));
    c[t] = acc;
}

// numpy's pairwise summation (umath loops_utils.h: blocks of <= 128 summed with 8 interleaved partial
// sums, longer runs split at n/2 rounded down to a multiple of 8), which is what add.reduce does along a
// contiguous row; verified against numpy's row sums in tests/test_seam.py.  Element e_i = (a-b)^2 or a*b,
// each rounded once like numpy's materialised temporary.
__device__ __forceinline__ double seam_elem(const double* a, const double* b, int op, int64_t i) {
    if (op == 0) {
        const double d = __dsub_rn(a[i], b[i]);
        return __dmul_rn(d, d);
    }
    return __dmul_rn(a[i], b[i]);
}
__device__ double seam_pairwise(const double* a, const double* b, int op, int64_t n) {
    // iterative form of the recursion: the split points only depend on n, so walk the leaves left to
    // right with an explicit stack of (start, length, partial) frames
    struct Frame {
        int64_t lo, n;
        int state;     // 0: fresh, 1: left done
        double left;
    } st[40];
    int sp = 0;
    st[0] = {0, n, 0, 0.0};
    double ret = 0.0;
    while (sp >= 0) {
        Frame& f = st[sp];
        if (f.n <= 128) {
            double res;
            if (f.n < 8) {
                res = 0.0;
                for (int64_t i = 0; i < f.n; ++i) res = __dadd_rn(res, seam_elem(a, b, op, f.lo + i));
            } else {
                double r[8];
                for (int j = 0; j < 8; ++j) r[j] = seam_elem(a, b, op, f.lo + j);
                int64_t i = 8;
                for (; i < f.n - (f.n % 8); i += 8)
                    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], seam_elem(a, b, op, f.lo + i + j));
                res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
                for (; i < f.n; ++i) res = __dadd_rn(res, seam_elem(a, b, op, f.lo + i));
            }
            ret = res;
            --sp;
        } else if (f.state == 0) {
            int64_t n2 = f.n / 2;
            n2 -= n2 % 8;
            f.state = 1;
            st[sp + 1] = {f.lo, n2, 0, 0.0};
            ++sp;
            continue;
        } else if (f.state == 1) {
            int64_t n2 = f.n / 2;
            n2 -= n2 % 8;
            f.left = ret;
            f.state = 2;
            st[sp + 1] = {f.lo + n2, f.n - n2, 0, 0.0};
            ++sp;
            continue;
        } else {
            ret = __dadd_rn(f.left, ret);
            --sp;
        }
        // a finished child hands `ret` to its parent (state 1 or 2 above)
    }
    return ret;
}

__global__ void __launch_bounds__(128) k_seam_row_sums(const double* a, const double* b, int op, int64_t rows,
                                                       int64_t n, double* out) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= rows) return;
    out[r] = seam_pairwise(a + r * n, b ? b + r * n : nullptr, op, n);
}

// ----------------------------------------------------------------------------------- launchers
static unsigned seam_blocks(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

int launch_seam_quant(const double* x, int64_t rows, int64_t cols, int64_t group, int rounding, bool values,
                      uint64_t seed, uint64_t counter_start, double ratio_lo, uint8_t* codes, uint8_t* scales,
                      uint8_t* mask, double* out, cudaStream_t st) {
    if (rows == 0 || cols == 0) return 0;
    SeamQuantArgs a{x, rows, cols, group, mix64(seed ^ mix64(kDomainSR)), counter_start, ratio_lo,
                    codes, scales, mask, out};
    const int64_t n = rows * ((cols + group - 1) / group);
    const unsigned nb = seam_blocks(n, 128);
#define QT_SEAM_LAUNCH(R, V) k_seam_quant<R, V><<<nb, 128, 0, st>>>(a)
    switch (rounding) {
        case kQuest: values ? QT_SEAM_LAUNCH(kQuest, true) : QT_SEAM_LAUNCH(kQuest, false); break;
        case kRtn: values ? QT_SEAM_LAUNCH(kRtn, true) : QT_SEAM_LAUNCH(kRtn, false); break;
        case kSr: values ? QT_SEAM_LAUNCH(kSr, true) : QT_SEAM_LAUNCH(kSr, false); break;
        default: return 2003;
    }
#undef QT_SEAM_LAUNCH
    return (int)cudaGetLastError();
}

int launch_seam_fwht(void* x, bool f64, int64_t rows, int64_t n, int64_t g, cudaStream_t st) {
    if (rows == 0 || n == 0) return 0;
    const int64_t nblk = rows * (n / g);
    if (f64)
        k_seam_fwht<double><<<seam_blocks(nblk, 128), 128, 0, st>>>(static_cast<double*>(x), nblk, g,
                                                                     1.0 / sqrt(2.0));
    else
        k_seam_fwht<float><<<seam_blocks(nblk, 128), 128, 0, st>>>(static_cast<float*>(x), nblk, g,
                                                                    (float)(1.0 / sqrt(2.0)));
    return (int)cudaGetLastError();
}

int launch_seam_gemm_nt(const void* a, const void* b, void* c, bool f64, int64_t m, int64_t n, int64_t k,
                        cudaStream_t st) {
    if (m == 0 || n == 0) return 0;
    const unsigned nb = seam_blocks(m * n, 256);
    if (f64)
        k_seam_gemm_nt<double><<<nb, 256, 0, st>>>(static_cast<const double*>(a), static_cast<const double*>(b),
                                                   static_cast<double*>(c), m, n, k);
    else
        k_seam_gemm_nt<float><<<nb, 256, 0, st>>>(static_cast<const float*>(a), static_cast<const float*>(b),
                                                  static_cast<float*>(c), m, n, k);
    return (int)cudaGetLastError();
}

int launch_seam_row_sums(const double* a, const double* b, int op, int64_t rows, int64_t n, double* out,
                         cudaStream_t st) {
    if (rows == 0) return 0;
    k_seam_row_sums<<<seam_blocks(rows, 128), 128, 0, st>>>(a, b, op, rows, n, out);
    return (int)cudaGetLastError();
}

}  // namespace qt
