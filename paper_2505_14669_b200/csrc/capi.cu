// capi.cu -- extern "C" boundary of libquartet_b200.so (declared in include/quartet_b200.h).
#include "../../include/quartet_b200.h"
#include "common.cuh"

#include "launch.h"

using namespace qt;

static inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static inline uint64_t sr_base_of(uint64_t seed) { return mix64(seed ^ mix64(kDomainSR)); }
// QT_ROUND_SR_FAST runs the SR kernels with the hash uniforms (QuantCfg::sr_fast)
static inline int round_kind(int r) { return r == QT_ROUND_SR_FAST ? QT_ROUND_SR : r; }

static int g_gemm_dbg = 0;  // experiment knobs for qt_debug_set_gemm (never set in production)
static int g_quant_mode = 0;  // qt_debug_set_quant: 0 production (tensor-core quantizers where they apply), 1 CUDA cores only
static int* g_quant_fallbacks = nullptr;

namespace qt {
int g_grid_cap = 0;

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev < 0 || dev >= kMaxDevices ? 0 : dev;
}
int device_sms() {
    static int sms[kMaxDevices];  // 0 = not yet queried (a benign race: every writer stores the same value)
    const int dev = current_device();
    if (!sms[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        sms[dev] = n > 0 ? n : 148;
    }
    return sms[dev];
}
bool first_use_on_device(int (&flags)[kMaxDevices]) {
    const int dev = current_device();
    if (flags[dev]) return false;
    flags[dev] = 1;
    return true;
}
}  // namespace qt

extern "C" {

void qt_debug_set_grid(int max_ctas) { qt::g_grid_cap = max_ctas > 0 ? max_ctas : 0; }

void qt_debug_set_gemm(int dbg) {
    g_gemm_dbg = dbg & 0xFFFF;
    qt::g_gemm_2sm = (dbg & 0x40000) ? 0 : 1;       // bit 18: force the 1-CTA kernel (A/B tests)
    qt::g_gemm_cluster8 = (dbg & 0x80000) ? 1 : 0;  // bit 19: clusters of 4 pairs with TMA multicast
    qt::g_gemm_splitk = (dbg & 0x100000) ? 0 : 1;   // bit 20: no split-K for under-filled fp32 GEMMs
}

void qt_debug_set_quant(int mode, int* fallbacks) {
    qt::g_tcq_dbg = mode >> 4;
    g_quant_mode = mode & 15;
    g_quant_fallbacks = fallbacks;
}

int qt_abi_version(void) { return QT_ABI_VERSION; }

const char* qt_error_string(int code) {
    switch (code) {
        case 0: return "ok";
        case QT_ERR_SHAPE: return "shape: quantized axis not a multiple of 32 or operand mismatch";
        case QT_ERR_ALIGN: return "alignment: pointer or leading dimension not 16-byte aligned";
        case QT_ERR_ARG: return "bad enum argument";
        case QT_ERR_TMA: return "tensor map creation failed";
        default: return cudaGetErrorString((cudaError_t)code);
    }
}

int64_t qt_codes_ld(int64_t k) { return k / 2; }
int64_t qt_sf_katoms(int64_t k) { return 2 * ((k + 255) / 256); }
int64_t qt_sf_bytes(int64_t rows, int64_t k) { return ((rows + 255) / 256) * 2 * qt_sf_katoms(k) * 512; }

uint64_t qt_mix64(uint64_t z) { return mix64(z); }

uint64_t qt_derive_seed(const uint64_t* parts, int nparts) {
    uint64_t acc = 0x243F6A8885A308D3ULL;
    for (int i = 0; i < nparts; ++i) {
        acc = mix64(acc ^ parts[i]);
        acc = acc + kGolden;
    }
    return mix64(acc);
}

int qt_sign_bits(uint32_t* d_bits, int64_t n, uint64_t xi, void* stream) {
    return launch_signs(d_bits, 0, n, xi, (cudaStream_t)stream);
}

int qt_sign_bits_at(uint32_t* d_bits, int64_t start, int64_t n, uint64_t xi, void* stream) {
    if (start < 0) return QT_ERR_ARG;
    return launch_signs(d_bits, start, n, xi, (cudaStream_t)stream);
}

int qt_sign_bits_pair(uint32_t* a, int64_t start_a, int64_t n_a, uint32_t* b, int64_t start_b, int64_t n_b,
                      uint64_t xi, void* stream) {
    if (start_a < 0 || start_b < 0 || n_a < 0 || n_b < 0) return QT_ERR_ARG;
    return launch_signs2(a, start_a, n_a, b, start_b, n_b, xi, (cudaStream_t)stream);
}

int qt_sign_bits_pair_dev(uint32_t* a, int64_t start_a, int64_t n_a, uint32_t* b, int64_t start_b, int64_t n_b,
                          const uint64_t* d_xi, void* stream) {
    if (start_a < 0 || start_b < 0 || n_a < 0 || n_b < 0 || !d_xi) return QT_ERR_ARG;
    return launch_signs2_dev(a, start_a, n_a, b, start_b, n_b, d_xi, (cudaStream_t)stream);
}

int qt_layer_seeds(uint64_t* d_xi, const uint64_t* d_layer_ids, int n, uint64_t seed, int64_t* d_step, int increment,
                   void* stream) {
    if (n < 0 || (n > 0 && (!d_xi || !d_layer_ids)) || !d_step) return QT_ERR_ARG;
    return launch_layer_seeds(d_xi, d_layer_ids, n, seed, d_step, increment, (cudaStream_t)stream);
}

// ---- exact plugin seam (seam.cu): f64 / any-group replays of _native.pyx:104-396
int qt_seam_quantize(const double* x, int64_t rows, int64_t cols, int64_t group, int rounding, int values,
                     uint64_t seed, uint64_t counter_start, double ratio_lo, uint8_t* codes, uint8_t* scales,
                     uint8_t* mask, double* out, void* stream) {
    if (rows < 0 || cols < 0 || group < 1) return QT_ERR_SHAPE;
    if (rounding < 0 || rounding > 2) return QT_ERR_ARG;
    if (rows == 0 || cols == 0) return 0;
    if (!x || (values ? !out : (!codes || !scales)) || (rounding == QT_ROUND_QUEST && !mask)) return QT_ERR_ARG;
    return launch_seam_quant(x, rows, cols, group, rounding, values != 0, seed, counter_start, ratio_lo, codes,
                             scales, mask, out, (cudaStream_t)stream);
}

int qt_seam_fwht(void* x, int f64, int64_t rows, int64_t n, int64_t g, void* stream) {
    if (rows < 0 || n < 0 || g < 1 || (g & (g - 1)) != 0 || n % g != 0) return QT_ERR_SHAPE;
    if (rows == 0 || n == 0) return 0;
    return launch_seam_fwht(x, f64 != 0, rows, n, g, (cudaStream_t)stream);
}

int qt_seam_gemm_nt(const void* a, const void* b, void* c, int f64, int64_t m, int64_t n, int64_t k, void* stream) {
    if (m < 0 || n < 0 || k < 0) return QT_ERR_SHAPE;
    return launch_seam_gemm_nt(a, b, c, f64 != 0, m, n, k, (cudaStream_t)stream);
}

int qt_seam_row_sums(const double* a, const double* b, int op, int64_t rows, int64_t n, double* out, void* stream) {
    if (rows < 0 || n < 0) return QT_ERR_SHAPE;
    if (op != 0 && op != 1) return QT_ERR_ARG;
    if (op == 0 && !b && rows > 0 && n > 0) return QT_ERR_ARG;
    return launch_seam_row_sums(a, op == 1 && !b ? a : b, op, rows, n, out, (cudaStream_t)stream);
}

int qt_fwht32(const float* x, float* out, int64_t rows, int64_t cols, int transform, const uint32_t* sign_bits,
             float prescale, void* stream) {
    if (cols % 32 != 0 || rows < 0) return QT_ERR_SHAPE;
    if (transform < 0 || transform > 2) return QT_ERR_ARG;
    if (rows == 0 || cols == 0) return 0;  // nothing to quantize: no pointer is read (empty sign vectors are null)
    if (transform == QT_TRANSFORM_RANDOMIZED && !sign_bits) return QT_ERR_ARG;
    return launch_transform_rows(x, out, rows, cols, transform, sign_bits, prescale, (cudaStream_t)stream);
}

int qt_quant_rows(const void* x, int in_dtype, int64_t ldx, int64_t rows, int64_t cols, int transform,
                  const uint32_t* sign_bits, float prescale, int rounding, uint64_t sr_seed, uint64_t counter_start,
                  int64_t counter_ld, uint8_t* codes, int64_t ldc, uint8_t* sf, int64_t katoms, uint32_t* mask, int* err, int* fallbacks,
                  void* stream) {
    if (cols % 32 != 0 || rows < 0) return QT_ERR_SHAPE;
    if (in_dtype != QT_IN_BF16 && in_dtype != QT_IN_F32) return QT_ERR_ARG;
    if (rounding < 0 || rounding > 3 || transform < 0 || transform > 2) return QT_ERR_ARG;
    if (rows == 0 || cols == 0) return 0;  // nothing to quantize: no pointer is read (empty sign vectors are null)
    if (transform == QT_TRANSFORM_RANDOMIZED && !sign_bits) return QT_ERR_ARG;
    int esz = in_dtype == QT_IN_BF16 ? 2 : 4;
    if (!al16(x) || (ldx * esz) % 16 || !al16(codes) || ldc % 16) return QT_ERR_ALIGN;
    QuantCfg cfg{transform, sign_bits, prescale, round_kind(rounding), sr_base_of(sr_seed), counter_start, counter_ld,
                 rounding == QT_ROUND_SR_FAST};
    QuantOut out{codes, ldc, sf, katoms, mask, err, fallbacks};
    return launch_quant_rows(x, in_dtype, ldx, rows, cols, cfg, out, (cudaStream_t)stream);
}

int qt_quant_cols(const void* x, int in_dtype, int64_t ldx, const uint8_t* mx_codes, int64_t mx_ldc,
                  const uint8_t* mx_sf, int64_t mx_katoms, int64_t rows, int64_t cols, int transform,
                  const uint32_t* sign_bits, float prescale, int rounding, uint64_t sr_seed, uint64_t counter_start,
                  int64_t counter_ld, uint8_t* codes, int64_t ldc, uint8_t* sf, int64_t katoms, int* err,
                  void* stream) {
    if (rows % 32 != 0 || cols % 32 != 0 || rows < 0 || cols < 0) return QT_ERR_SHAPE;
    if (in_dtype < 0 || in_dtype > 2 || rounding < 0 || rounding > 3 || transform < 0 || transform > 2)
        return QT_ERR_ARG;
    if (rows == 0 || cols == 0) return 0;  // nothing to quantize: no pointer is read (empty sign vectors are null)
    if (transform == QT_TRANSFORM_RANDOMIZED && !sign_bits) return QT_ERR_ARG;
    if (in_dtype == QT_IN_MXFP4) {
        if (!al16(mx_codes) || mx_ldc % 16) return QT_ERR_ALIGN;
    } else {
        int esz = in_dtype == QT_IN_BF16 ? 2 : 4;
        if (!al16(x) || (ldx * esz) % 16) return QT_ERR_ALIGN;
    }
    if (!al16(codes) || ldc % 16) return QT_ERR_ALIGN;
    QuantCfg cfg{transform, sign_bits, prescale, round_kind(rounding), sr_base_of(sr_seed), counter_start, counter_ld,
                 rounding == QT_ROUND_SR_FAST};
    QuantOut out{codes, ldc, sf, katoms, nullptr, err, nullptr};
    MxIn mx{mx_codes, mx_ldc, mx_sf, mx_katoms};
    return launch_quant_tile(x, in_dtype, ldx, mx, rows, cols, nullptr, nullptr, &cfg, &out, 0, (cudaStream_t)stream);
}

int qt_quant_dual(const void* x, int in_dtype, int64_t ldx, int64_t rows, int64_t cols, int transform,
                  const uint32_t* row_sign_bits, const uint32_t* col_sign_bits, float prescale, int rounding,
                  uint64_t seed_rows, uint64_t row_counter_start, uint64_t seed_cols, uint64_t col_counter_start,
                  int64_t col_counter_ld, uint8_t* row_codes, int64_t row_ldc, uint8_t* row_sf, int64_t row_katoms,
                  uint32_t* row_mask, uint8_t* col_codes, int64_t col_ldc, uint8_t* col_sf, int64_t col_katoms,
                  int* err, void* stream) {
    if (rows % 32 != 0 || cols % 32 != 0 || rows < 0 || cols < 0) return QT_ERR_SHAPE;
    if ((in_dtype != QT_IN_BF16 && in_dtype != QT_IN_F32) || rounding < 0 || rounding > 3 || transform < 0 ||
        transform > 2)
        return QT_ERR_ARG;
    if (rows == 0 || cols == 0) return 0;  // nothing to quantize: no pointer is read (empty sign vectors are null)
    if (transform == QT_TRANSFORM_RANDOMIZED && (!row_sign_bits || !col_sign_bits)) return QT_ERR_ARG;
    int esz = in_dtype == QT_IN_BF16 ? 2 : 4;
    if (!al16(x) || (ldx * esz) % 16 || !al16(row_codes) || row_ldc % 16 || !al16(col_codes) || col_ldc % 16)
        return QT_ERR_ALIGN;
    QuantCfg rc{transform, row_sign_bits, prescale, round_kind(rounding), sr_base_of(seed_rows), row_counter_start, 0,
                rounding == QT_ROUND_SR_FAST};
    QuantCfg cc{transform, col_sign_bits, prescale, round_kind(rounding), sr_base_of(seed_cols), col_counter_start,
                col_counter_ld, rounding == QT_ROUND_SR_FAST};
    QuantOut ro{row_codes, row_ldc, row_sf, row_katoms, row_mask, err, nullptr};
    QuantOut co{col_codes, col_ldc, col_sf, col_katoms, nullptr, err, nullptr};
    if (g_quant_mode != 1 && in_dtype == QT_IN_BF16 && (rounding == QT_ROUND_RTN || rounding == QT_ROUND_SR_FAST) &&
        transform == QT_TRANSFORM_RANDOMIZED && !row_mask) {
        // tensor-core Hadamard + checked RTN (bit-identical; exact fallback per group) or fast SR
        const bool srf = rounding == QT_ROUND_SR_FAST;
        int rc2 = launch_tcq_dual(x, ldx, rows, cols, row_sign_bits, col_sign_bits, prescale, ro, co,
                                  g_quant_fallbacks, (cudaStream_t)stream, srf ? &rc : nullptr, srf ? &cc : nullptr);
        return rc2 == 1001 || rc2 == 1002 ? QT_ERR_TMA : rc2;
    }
    MxIn mx{nullptr, 0, nullptr, 0};
    return launch_quant_tile(x, in_dtype, ldx, mx, rows, cols, &rc, &ro, &cc, &co, 0, (cudaStream_t)stream);
}

int qt_quant_fused(const void* x, int in_dtype, int64_t ldx, int64_t rows, int64_t cols, int row_transform,
                   const uint32_t* row_sign_bits, float row_prescale, int row_rounding, uint64_t row_seed,
                   uint64_t row_counter_start, int64_t row_counter_ld, uint8_t* row_codes, int64_t row_ldc,
                   uint8_t* row_sf, int64_t row_katoms, uint32_t* row_mask, int col_transform,
                   const uint32_t* col_sign_bits, float col_prescale, int col_rounding, uint64_t col_seed,
                   uint64_t col_counter_start, int64_t col_counter_ld, uint8_t* col_codes, int64_t col_ldc,
                   uint8_t* col_sf, int64_t col_katoms, int* err, int* fallbacks, void* stream) {
    if (rows % 32 != 0 || cols % 32 != 0 || rows < 0 || cols < 0) return QT_ERR_SHAPE;
    if (in_dtype != QT_IN_BF16 && in_dtype != QT_IN_F32) return QT_ERR_ARG;
    if (row_rounding < 0 || row_rounding > 3 || col_rounding < 1 || col_rounding > 3) return QT_ERR_ARG;
    if (row_transform < 0 || row_transform > 2 || col_transform < 0 || col_transform > 2) return QT_ERR_ARG;
    if (rows == 0 || cols == 0) return 0;  // nothing to quantize: no pointer is read (empty sign vectors are null)
    if ((row_transform == QT_TRANSFORM_RANDOMIZED && !row_sign_bits) ||
        (col_transform == QT_TRANSFORM_RANDOMIZED && !col_sign_bits))
        return QT_ERR_ARG;
    int esz = in_dtype == QT_IN_BF16 ? 2 : 4;
    if (!al16(x) || (ldx * esz) % 16 || !al16(row_codes) || row_ldc % 16 || !al16(col_codes) || col_ldc % 16)
        return QT_ERR_ALIGN;
    QuantCfg rc{row_transform, row_sign_bits, row_prescale, round_kind(row_rounding), sr_base_of(row_seed),
                row_counter_start, row_counter_ld, row_rounding == QT_ROUND_SR_FAST};
    QuantCfg cc{col_transform, col_sign_bits, col_prescale, round_kind(col_rounding), sr_base_of(col_seed),
                col_counter_start, col_counter_ld, col_rounding == QT_ROUND_SR_FAST};
    QuantOut ro{row_codes, row_ldc, row_sf, row_katoms, row_mask, err, fallbacks};
    QuantOut co{col_codes, col_ldc, col_sf, col_katoms, nullptr, err, nullptr};
    if (g_quant_mode != 1 && in_dtype == QT_IN_BF16 && row_rounding == QT_ROUND_QUEST &&
        row_transform == QT_TRANSFORM_HADAMARD && row_prescale == 1.0f &&
        (col_rounding == QT_ROUND_RTN || col_rounding == QT_ROUND_SR_FAST) && col_transform == QT_TRANSFORM_RANDOMIZED) {
        // X_q and X_t both on the tensor cores (checked QuEST / RTN, exact per-group fallback; or fast-SR X_t)
        int rc3 = launch_tcq_xq(x, ldx, rows, cols, ro, col_sign_bits, col_prescale, co, g_quant_fallbacks,
                                (cudaStream_t)stream, col_rounding == QT_ROUND_SR_FAST ? &cc : nullptr);
        return rc3 == 1001 || rc3 == 1002 ? QT_ERR_TMA : rc3;
    }
    MxIn mx{nullptr, 0, nullptr, 0};
    return launch_quant_tile(x, in_dtype, ldx, mx, rows, cols, &rc, &ro, &cc, &co, 1, (cudaStream_t)stream);
}

int qt_quant_fwd_quest(const void* x, int in_dtype, int64_t rows, int64_t cols, int hadamard, uint8_t* codes,
                       uint8_t* sf, uint32_t* mask, int* err, void* stream) {
    return qt_quant_rows(x, in_dtype, cols, rows, cols, hadamard ? QT_TRANSFORM_HADAMARD : QT_TRANSFORM_NONE, nullptr,
                         1.0f, QT_ROUND_QUEST, 0, 0, 0, codes, qt_codes_ld(cols), sf, qt_sf_katoms(cols), mask, err,
                         nullptr, stream);
}

int qt_quant_bwd_rows(const void* dy, int in_dtype, int64_t rows, int64_t cols, const uint32_t* sign_bits,
                      int rounding, uint64_t sr_seed, uint8_t* codes, uint8_t* sf, int* err, void* stream) {
    if (rounding == QT_ROUND_QUEST) return QT_ERR_ARG;
    return qt_quant_rows(dy, in_dtype, cols, rows, cols, sign_bits ? QT_TRANSFORM_RANDOMIZED : QT_TRANSFORM_NONE,
                         sign_bits, 0.75f, rounding, sr_seed, 0, 0, codes, qt_codes_ld(cols), sf, qt_sf_katoms(cols),
                         nullptr, err, nullptr, stream);
}

int qt_quant_bwd_cols(const void* dy, int in_dtype, int64_t rows, int64_t cols, const uint32_t* sign_bits,
                      int rounding, uint64_t sr_seed, uint8_t* codes, uint8_t* sf, int* err, void* stream) {
    if (rounding == QT_ROUND_QUEST) return QT_ERR_ARG;
    return qt_quant_cols(dy, in_dtype, cols, nullptr, 0, nullptr, 0, rows, cols,
                         sign_bits ? QT_TRANSFORM_RANDOMIZED : QT_TRANSFORM_NONE, sign_bits, 0.75f, rounding, sr_seed,
                         0, 0, codes, qt_codes_ld(rows), sf, qt_sf_katoms(rows), err, stream);
}

int qt_requant_t(const uint8_t* codes, const uint8_t* sf, int64_t rows, int64_t cols, const uint32_t* sign_bits,
                 int rounding, uint64_t sr_seed, uint8_t* out_codes, uint8_t* out_sf, int* err, void* stream) {
    if (rounding == QT_ROUND_QUEST) return QT_ERR_ARG;
    return qt_quant_cols(nullptr, QT_IN_MXFP4, 0, codes, qt_codes_ld(cols), sf, qt_sf_katoms(cols), rows, cols,
                         sign_bits ? QT_TRANSFORM_RANDOMIZED : QT_TRANSFORM_NONE, sign_bits, 0.75f, rounding, sr_seed,
                         0, 0, out_codes, qt_codes_ld(rows), out_sf, qt_sf_katoms(rows), err, stream);
}

int qt_gemm_mxf4(const uint8_t* a_codes, const uint8_t* a_sf, const uint8_t* b_codes, const uint8_t* b_sf, int64_t M,
                 int64_t N, int64_t K, void* out, int out_dtype, int64_t ldo, int epilogue, const uint32_t* mask,
                 float scale, void* stream) {
    if (K % 32 != 0 || K < 0 || N % 32 != 0 || N < 0 || M < 0) return QT_ERR_SHAPE;
    const int accumulate = (epilogue & QT_EPI_ACCUMULATE) ? 1 : 0;
    epilogue &= ~QT_EPI_ACCUMULATE;
    if (epilogue < QT_EPI_STORE || epilogue > QT_EPI_MASK) return QT_ERR_ARG;
    if (out_dtype != QT_OUT_F32 && out_dtype != QT_OUT_BF16) return QT_ERR_ARG;
    if (M == 0 || N == 0) return 0;
    int esz = out_dtype == QT_OUT_BF16 ? 2 : 4;
    if (K == 0) {  // empty contraction: every epilogue of a zero product is zero (D += 0 leaves D as it is)
        if (accumulate) return 0;
        if ((ldo < N) || !out) return QT_ERR_ARG;
        return (int)cudaMemset2DAsync(out, (size_t)(ldo * esz), 0, (size_t)(N * esz), (size_t)M, (cudaStream_t)stream);
    }
    if (epilogue != QT_EPI_STORE && !mask) return QT_ERR_ARG;
    if (!al16(a_codes) || !al16(b_codes) || !al16(out) || (ldo * esz) % 16) return QT_ERR_ALIGN;
    EpiParams ep{out, ldo, out_dtype == QT_OUT_BF16, epilogue, mask, N / 32, scale, g_gemm_dbg, accumulate};
    int rc = launch_gemm(a_codes, qt_codes_ld(K), a_sf, qt_sf_katoms(K), b_codes, qt_codes_ld(K), b_sf,
                         qt_sf_katoms(K), M, N, K, ep, (cudaStream_t)stream);
    return rc == 1001 || rc == 1002 ? QT_ERR_TMA : rc;
}

}  // extern "C"
