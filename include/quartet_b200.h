/*
 * quartet_b200.h -- C ABI of the B200-native Quartet linear-layer hot path (libquartet_b200.so).
 *
 * Drop-in boundary for the reference's operator-plugin seam: the duck-typed `kernels` backend
 * module of mx4train (/root/reference/pkg/src/mx4train/_backend/__init__.py:13-35) whose entry
 * points are quantize_rtn / quantize_sr / quantize_quest / fwht / gemm_nt
 * (_backend/_native.pyx:104-396), composed by qlinear.forward / qlinear.backward
 * (qlinear.py:114-252).  Each entry point below cites the reference interface it replaces.
 *
 * Conventions (all functions):
 *   - plain device pointers, sizes in elements unless a name says bytes; no allocation, no throw;
 *   - stream-ordered on the caller's `stream` (a cudaStream_t passed as void*); reentrant.  Process
 *     state: a lazily resolved driver entry point, per-device caches of launch facts (SM count,
 *     occupancy, one-time kernel attributes; any device of the process may be current), and the
 *     qt_debug_set_* test knobs (production value 0, never set by the product path);
 *   - return 0 on success, a cudaError_t value (1..999) on a CUDA error, or a QT_ERR_* code;
 *   - `err` (nullable, device int) gets bit 0 set when a quantizer sees a non-finite input: the
 *     analogue of the reference's ValueError("non-finite input") (codec.py:164-170), checked by
 *     the host wrapper after the call;
 *   - every quantized axis length must be a multiple of 32 (the reference requires the same on the
 *     layer path: qlinear.py:136-137, 200-204).
 *
 * MXFP4 operand layout (one [R, K] matrix quantized in groups of 32 along K):
 *   codes  uint8 [R, K/2], element 2k in the low nibble of byte k (== reference pack_nibbles,
 *          codec.py:146-153, so `codes` bytes equal QuantizedTensor.codes bytes)
 *   sf     uint8 E8M0 scale bytes (== QuantizedTensor.scales values) in tcgen05 scale atoms:
 *          byte offset of (row r, group g) = ((r/128)*katoms + g/4)*512 + (r%32)*16
 *                                            + ((r%128)/32)*4 + g%4
 *          with katoms = qt_sf_katoms(K); buffer size qt_sf_bytes(R, K), zero-initialised by the
 *          caller (padding must hold a finite exponent).
 *   mask   uint32 [R, K/32], bit j of word (r, g): |x/s| <= 6 at the chosen scale (LayerContext
 *          m_x / m_w, qlinear.py:74-87, as a bitmap instead of a bool matrix).
 */
#ifndef QUARTET_B200_H
#define QUARTET_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define QT_API __attribute__((visibility("default")))
#else
#define QT_API
#endif

#define QT_ABI_VERSION 1

/* Empty dimensions (rows, cols or a GEMM's M / N = 0; the reference accepts batch = 0) are valid: after the
 * shape and enum checks the call returns 0 without reading any pointer.  A GEMM with K = 0 writes zeros
 * (every epilogue of a zero product is zero) or, with QT_EPI_ACCUMULATE, leaves D unchanged. */

/* error codes beyond cudaError_t */
#define QT_ERR_SHAPE 2001  /* axis not a multiple of 32 / mismatched operands (ValueError upstream) */
#define QT_ERR_ALIGN 2002  /* pointer or leading dimension not 16-byte aligned */
#define QT_ERR_ARG 2003    /* unknown enum value */
#define QT_ERR_TMA 2004    /* tensor-map creation failed */

/* dtype / mode enums */
#define QT_IN_BF16 0
#define QT_IN_F32 1
#define QT_IN_MXFP4 2
#define QT_TRANSFORM_NONE 0        /* no rotation */
#define QT_TRANSFORM_HADAMARD 1    /* hadamard.transform_last_axis, g = 32 (hadamard.py:72-74) */
#define QT_TRANSFORM_RANDOMIZED 2  /* randomized_transform_last_axis (hadamard.py:82-85) */
#define QT_ROUND_QUEST 0           /* quantize_quest, ratio_lo = 1/16 (_native.pyx:206-245) */
#define QT_ROUND_RTN 1             /* quantize_rtn (_native.pyx:104-131) */
#define QT_ROUND_SR 2              /* quantize_sr (_native.pyx:134-168) */
#define QT_ROUND_SR_FAST 3         /* B200 extension: stochastic rounding to the same two neighbours as QT_ROUND_SR by
                                      the hardware conversion cvt.rs.satfinite.e2m1x4.f32 (32 hashed random bits of
                                      (seed, stream position) per 4 elements): P(upper) = floor(p * 2^16) / 2^16,
                                      unbiased up to 2^-16 of a grid step, not the reference's splitmix64 draws
                                      (quantizer entry points only; the seam and the diagnostics keep the
                                      reference's streams) */
#define QT_EPI_STORE 0             /* D = A B^T */
#define QT_EPI_MASK_H 1            /* D = H32(A B^T (.) mask) * scale (qlinear.py:229-230, 249-250) */
#define QT_EPI_MASK 2              /* D = (A B^T (.) mask) * scale (hadamard=False layers) */
#define QT_EPI_ACCUMULATE 0x10     /* flag OR'ed into any epilogue: D += E, E first rounded to D's dtype (the sum
                                      of several layers' dx in one buffer, as out.add_(tmp); 2-CTA kernel: TMA
                                      reduce-add into L2) */
#define QT_OUT_F32 0
#define QT_OUT_BF16 1

QT_API int qt_abi_version(void);
QT_API const char* qt_error_string(int code);

/* ---- geometry helpers (host) */
QT_API int64_t qt_codes_ld(int64_t k);            /* bytes per codes row: k/2 */
QT_API int64_t qt_sf_katoms(int64_t k);           /* scale atoms per 128-row block: 2*ceil(k/256) */
QT_API int64_t qt_sf_bytes(int64_t rows, int64_t k);

/* ---- counter RNG (host), rng.py:27-78 */
QT_API uint64_t qt_mix64(uint64_t z);                                   /* rng.mix64 */
QT_API uint64_t qt_derive_seed(const uint64_t* parts, int nparts);      /* rng.derive_seed */

/* Sign bitmap of rng.signs(xi, 0, n) (rng.py:57-62): bit p%32 of word p/32 is 1 where the
 * randomized Hadamard flips position p.  d_bits holds ceil(n/32) words. */
QT_API int qt_sign_bits(uint32_t* d_bits, int64_t n, uint64_t xi, void* stream);
/* Same for rng.signs(xi, start, n): positions start .. start+n-1 (data-parallel token shards). */
QT_API int qt_sign_bits_at(uint32_t* d_bits, int64_t start, int64_t n, uint64_t xi, void* stream);
/* Both sign vectors of one seed in one launch: rng.signs(xi, start_a, n_a) into a, rng.signs(xi, start_b, n_b)
 * into b (a layer's d_out and token signs; same bitmaps as two qt_sign_bits_at calls). */
QT_API int qt_sign_bits_pair(uint32_t* a, int64_t start_a, int64_t n_a, uint32_t* b, int64_t start_b, int64_t n_b,
                             uint64_t xi, void* stream);

/* Device-resident seeds, for a training step captured as one CUDA graph (the seed changes every step):
 * qt_layer_seeds writes d_xi[l] = derive_seed(derive_seed(seed, 4, *d_step), d_layer_ids[l]) for l < n -- the
 * per-step, per-layer backward seed of the reference's training loop (train.py:346-348) -- and then increments
 * *d_step if `increment`; qt_sign_bits_pair_dev is qt_sign_bits_pair with xi = *d_xi read on the device. */
QT_API int qt_layer_seeds(uint64_t* d_xi, const uint64_t* d_layer_ids, int n, uint64_t seed, int64_t* d_step,
                          int increment, void* stream);
QT_API int qt_sign_bits_pair_dev(uint32_t* a, int64_t start_a, int64_t n_a, uint32_t* b, int64_t start_b, int64_t n_b,
                                 const uint64_t* d_xi, void* stream);

/* Blockwise transform only (the kernels.fwht plugin entry, _native.pyx:353-379, with the
 * randomized variant of hadamard.py:82-85): out[r, :] = prescale * FWHT32(x[r, :] (.) s), fp32,
 * bit-identical to the reference's fp32 butterfly.  x and out are dense [rows, cols]. */
QT_API int qt_fwht32(const float* x, float* out, int64_t rows, int64_t cols, int transform,
                     const uint32_t* sign_bits, float prescale, void* stream);

/* ---- general quantizers ---------------------------------------------------------------
 * qt_quant_rows: groups along the contiguous axis of x[rows, cols] (row stride ldx elements).
 *   transform (+ sign_bits for RANDOMIZED, indexed by column), then * prescale (1.0 or 0.75,
 *   qlinear.py:219-220), then quantize with `rounding` (SR: seed = per-tensor seed, stream
 *   position counter_start + r*ld + c with ld = counter_ld or cols, quantizers.py:79-84).
 *   Replaces: kernels.fwht + kernels.quantize_{quest,rtn,sr} on a row-major matrix. */
QT_API int qt_quant_rows(const void* x, int in_dtype, int64_t ldx, int64_t rows, int64_t cols, int transform,
                  const uint32_t* sign_bits, float prescale, int rounding, uint64_t sr_seed, uint64_t counter_start,
                  int64_t counter_ld, uint8_t* codes, int64_t ldc, uint8_t* sf, int64_t katoms, uint32_t* mask, int* err,
                  int* fallbacks, void* stream);

/* qt_quant_cols: quantize the TRANSPOSE of x[rows, cols]: output operand [cols, rows] with groups
 *   along `rows`; sign_bits indexed by row; SR stream position counter_start + c*ld + r with
 *   ld = counter_ld (0 -> rows; a token shard of a larger matrix passes the full length).
 *   in_dtype QT_IN_MXFP4 reads x as an MXFP4 operand (mx_codes/mx_ldc/mx_sf/mx_katoms; x unused)
 *   and dequantizes it exactly first (qlinear._values, qlinear.py:90-93). */
QT_API int qt_quant_cols(const void* x, int in_dtype, int64_t ldx, const uint8_t* mx_codes, int64_t mx_ldc,
                  const uint8_t* mx_sf, int64_t mx_katoms, int64_t rows, int64_t cols, int transform,
                  const uint32_t* sign_bits, float prescale, int rounding, uint64_t sr_seed, uint64_t counter_start,
                  int64_t counter_ld, uint8_t* codes, int64_t ldc, uint8_t* sf, int64_t katoms, int* err,
                  void* stream);

/* qt_quant_dual: both backward dy operands from ONE read of x[rows, cols]:
 *   row operand  [rows, cols] groups along cols (row_sign_bits by column, SR seed seed_rows,
 *                stream position row_counter_start + r*cols + c)          -- qlinear.py:214, 219, 225
 *   col operand  [cols, rows] groups along rows (col_sign_bits by row, SR seed seed_cols,
 *                stream position col_counter_start + c*ld + r, ld = col_counter_ld or rows)
 *                                                                        -- qlinear.py:234, 239, 245
 * A data-parallel token shard passes global sign offsets / counters so that its operands equal the
 * corresponding slices of the single-GPU operands. */
QT_API int qt_quant_dual(const void* x, int in_dtype, int64_t ldx, int64_t rows, int64_t cols, int transform,
                         const uint32_t* row_sign_bits, const uint32_t* col_sign_bits, float prescale, int rounding,
                         uint64_t seed_rows, uint64_t row_counter_start, uint64_t seed_cols,
                         uint64_t col_counter_start, int64_t col_counter_ld, uint8_t* row_codes, int64_t row_ldc,
                         uint8_t* row_sf, int64_t row_katoms, uint32_t* row_mask, uint8_t* col_codes,
                         int64_t col_ldc, uint8_t* col_sf, int64_t col_katoms, int* err, void* stream);

/* qt_quant_fused: a forward operand AND its transposed backward requantization from ONE read of x:
 *   row operand [rows, cols] = Q_row(T_row(x) * row_prescale)        e.g. QuEST(H32(x)), qlinear.py:139-157
 *   col operand [cols, rows] = Q_col(T_col(deq(row operand)^T) * col_prescale)
 *                              == qt_requant_t of the row operand: X_t / W_t (qlinear.py:206-207, 215, 235)
 * so the layer can produce X_t and W_t at forward time, when the backward seed xi is known (the training
 * loop derives it per step and layer, train.py:346-348), instead of re-reading the saved operands.
 * col_sign_bits are indexed by row (the contraction axis of the backward GEMM); col_rounding is RTN or SR
 * (SR stream position col_counter_start + c*ld + r, ld = col_counter_ld or rows). */
QT_API int qt_quant_fused(const void* x, int in_dtype, int64_t ldx, int64_t rows, int64_t cols, int row_transform,
                          const uint32_t* row_sign_bits, float row_prescale, int row_rounding, uint64_t row_seed,
                          uint64_t row_counter_start, int64_t row_counter_ld, uint8_t* row_codes, int64_t row_ldc,
                          uint8_t* row_sf, int64_t row_katoms, uint32_t* row_mask, int col_transform,
                          const uint32_t* col_sign_bits, float col_prescale, int col_rounding, uint64_t col_seed,
                          uint64_t col_counter_start, int64_t col_counter_ld, uint8_t* col_codes, int64_t col_ldc,
                          uint8_t* col_sf, int64_t col_katoms, int* err, int* fallbacks, void* stream);

/* ---- named hot-path entry points (dense row-major inputs, ld == cols) ------------------- */

/* Forward operand quantizer: x_h = H32(x) (if hadamard), QuEST -> codes/sf/mask.
 * Replaces qlinear.py:139-141 + apply_scheme(x_h, QUEST) (quantizers.py:87-92). */
QT_API int qt_quant_fwd_quest(const void* x, int in_dtype, int64_t rows, int64_t cols, int hadamard, uint8_t* codes,
                       uint8_t* sf, uint32_t* mask, int* err, void* stream);

/* Backward row operand: Q(H32(dy (.) s_xi) * 0.75) along d_out (qlinear.py:214, 219, 225). */
QT_API int qt_quant_bwd_rows(const void* dy, int in_dtype, int64_t rows, int64_t cols, const uint32_t* sign_bits,
                      int rounding, uint64_t sr_seed, uint8_t* codes, uint8_t* sf, int* err, void* stream);

/* Backward transposed operand: Q(H32(dy^T (.) s_xi) * 0.75) along tokens (qlinear.py:234, 239, 245). */
QT_API int qt_quant_bwd_cols(const void* dy, int in_dtype, int64_t rows, int64_t cols, const uint32_t* sign_bits,
                      int rounding, uint64_t sr_seed, uint8_t* codes, uint8_t* sf, int* err, void* stream);

/* Requant-transpose of a saved MXFP4 operand [rows, cols]:
 * Q(H32(deq(q)^T (.) s_xi) * 0.75) -> operand [cols, rows] (qlinear.py:206-207, 215, 235). */
QT_API int qt_requant_t(const uint8_t* codes, const uint8_t* sf, int64_t rows, int64_t cols, const uint32_t* sign_bits,
                 int rounding, uint64_t sr_seed, uint8_t* out_codes, uint8_t* out_sf, int* err, void* stream);

/* MXFP4 GEMM D[M,N] = deq(A)[M,K] deq(B)[N,K]^T on tcgen05 (gemm_lp, qlinear.py:96-111), with an
 * optional fused epilogue (QT_EPI_MASK_H: mask[M, N/32], FWHT-32 along N, * scale). */
QT_API int qt_gemm_mxf4(const uint8_t* a_codes, const uint8_t* a_sf, const uint8_t* b_codes, const uint8_t* b_sf,
                 int64_t M, int64_t N, int64_t K, void* out, int out_dtype, int64_t ldo, int epilogue,
                 const uint32_t* mask, float scale, void* stream);

/* Experiment hook for the GEMM mainloop studies in tools/gemm_probe.py (0 = production; bit 18 forces the
 * 1-CTA kernel where the 2-CTA pair kernel is the default, bit 19 runs the pairs in clusters of 8 with TMA
 * multicast of A and B, bit 20 turns off the split-K of the last wave of fp32 GEMMs -- all for A/B parity tests).
 * qt_gemm_mxf4 with an fp32 output, no QT_EPI_ACCUMULATE and K >= 2048 may launch a second kernel (zero-fill of
 * the split tiles' output blocks) on the same stream. */
QT_API void qt_debug_set_gemm(int dbg);
/* Quantizer path selection for A/B parity tests: mode 0 (production; 3 is an alias) runs the tensor-core
 * Hadamard quantizers where they apply -- the backward dual operands (bf16, RTN, randomized) and the bf16 QuEST
 * forward of qt_quant_fused with an RTN randomized transposed requantization (checked QuEST + checked RTN);
 * mode 1 forces the CUDA-core kernels everywhere.  `fallbacks` (nullable device ints, 3 of them) counts the
 * groups a tensor-core path re-decided exactly: [0] dual groups / forward QuEST searches, [1] forward X_t
 * groups, [2] forward codes-only re-encodes.  Not thread-safe; tests only. */
QT_API void qt_debug_set_quant(int mode, int* fallbacks);
/* Parity-test hook: cap every persistent grid (quantizer and GEMM kernels) at max_ctas CTAs (the 2-CTA GEMM
 * at max_ctas/2 pairs, at least one), so that each CTA walks many tiles; 0 restores the production grid.
 * Not thread-safe; tests only. */
QT_API void qt_debug_set_grid(int max_ctas);

/* ---- exact plugin seam: every input the reference's kernels accept ---------------------------
 * The reference's `kernels` module takes f64 matrices, any group size, any power-of-two FWHT block in f32
 * or f64, and a fixed-order GEMM (_native.pyx:104-396).  These entry points replay it operation for
 * operation in scalar f64 / f32 device code (one thread per group / block / output element), bit-identical
 * for every input; the layer path uses the tiled kernels above.  Codes, masks and scales are UNPACKED,
 * the reference's own layout: codes / mask uint8 [rows, cols], scales uint8 [rows, ceil(cols / group)].
 *
 * qt_seam_quantize: rounding QT_ROUND_RTN  -> quantize_rtn   (_native.pyx:104-131), codes + scales
 *                            QT_ROUND_SR   -> quantize_sr    (_native.pyx:134-168), stream position
 *                                             counter_start + i*cols + j of seed `seed`
 *                            QT_ROUND_QUEST-> quantize_quest (_native.pyx:171-245, clip ratio ratio_lo), + mask
 *   values != 0: the *_values variants instead (_native.pyx:248-350): `out` f64 [rows, cols] gets the
 *   dequantized values (codes / scales unused; QuEST still writes mask).
 * qt_seam_fwht: in-place blockwise FWHT of x [rows, n] (f64 != 0: double, else float), block g a power of
 *   two dividing n (_native.pyx:353-379).
 * qt_seam_gemm_nt: c [m, n] = a [m, k] b [n, k]^T, each output summed c = c + a*b over ascending k from zero
 *   (_native.pyx:382-396), f32 or f64.
 * qt_seam_row_sums: out[r] = numpy add.reduce of row r of e = (a - b)^2 (op 0) or a * b (op 1) -- numpy's
 *   pairwise order, so the results equal the reference's ((x - d) ** 2).mean(axis=1) * n and
 *   (y * qy).sum(axis=1) bit for bit (diagnostics.py:84, 161-165). */
QT_API int qt_seam_quantize(const double* x, int64_t rows, int64_t cols, int64_t group, int rounding, int values,
                            uint64_t seed, uint64_t counter_start, double ratio_lo, uint8_t* codes, uint8_t* scales,
                            uint8_t* mask, double* out, void* stream);
QT_API int qt_seam_fwht(void* x, int f64, int64_t rows, int64_t n, int64_t g, void* stream);
QT_API int qt_seam_gemm_nt(const void* a, const void* b, void* c, int f64, int64_t m, int64_t n, int64_t k,
                           void* stream);
QT_API int qt_seam_row_sums(const double* a, const double* b, int op, int64_t rows, int64_t n, double* out,
                            void* stream);

/* ---- Llama-loop glue (not on the Quartet path; llama.py): fused bf16 elementwise kernels, fp32 math.
 * qt_rope: half-split rotary embedding of x [batch, seq, heads, head_dim] (rows = batch * seq; element
 *   strides stride_b / stride_s / stride_h, head_dim contiguous) with cos/sin tables [seq, head_dim], into a
 *   contiguous out; backward != 0 applies the transposed rotation (dx from dy).
 * qt_swiglu: forward out0 = silu(gate) * up; backward (dy given) out0 = d gate, out1 = d up.  n % 8 == 0.
 * qt_rmsnorm: rows of x [rows, d] bf16 (d % 8 == 0 up to 2048, or d in {4096, 6144, 8192}), fp32 weight w: forward out = x rstd w and
 *   rstd[rows] saved; backward (dy, rstd given) out = dx, dw[d] += sum over rows (caller zeroes dw).
 * qt_rmsnorm_res: qt_rmsnorm fused with the residual stream around it (bf16 sums rounded once, as torch's add):
 *   forward h_out = x + res and out = rmsnorm(h_out); backward out = dx + res (res = the gradient that reaches
 *   the residual stream past the norm, so autograd needs no separate accumulation).  res == NULL: qt_rmsnorm.
 * qt_cross_entropy: rows of logits [rows, vocab] bf16 (vocab % 8 == 0), int64 targets: forward writes lse and
 *   the per-row loss (fp32); backward writes dlogits = (softmax - onehot) * (*dloss) * scale (bf16). */
QT_API int qt_rope(const void* x, void* out, int64_t rows, int heads, int head_dim, int seq, const void* cos,
                   const void* sin, int backward, int64_t stride_b, int64_t stride_s, int64_t stride_h, void* stream);
QT_API int qt_rmsnorm(const void* x, const float* w, const void* dy, void* out, float* rstd, float* dw, int64_t rows,
                      int d, float eps, int backward, void* stream);
QT_API int qt_rmsnorm_res(const void* x, const void* res, const float* w, const void* dy, void* out, void* h_out,
                          float* rstd, float* dw, int64_t rows, int d, float eps, int backward, void* stream);
QT_API int qt_cross_entropy(const void* logits, const int64_t* targets, int64_t rows, int vocab, float* lse,
                            float* loss, void* dlogits, const float* dloss, float scale, int backward, void* stream);
QT_API int qt_swiglu(const void* gate, const void* up, const void* dy, void* out0, void* out1, int64_t n,
                     int backward, void* stream);

#ifdef __cplusplus
}
#endif
#endif
