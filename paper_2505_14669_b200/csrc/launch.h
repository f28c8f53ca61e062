// launch.h -- host-side launcher interface shared by the kernel TUs and the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qt {

enum InType : int { kInBF16 = 0, kInF32 = 1, kInMXFP4 = 2 };
enum Transform : int { kNone = 0, kHadamard = 1, kRandomized = 2 };
enum EpiMode : int { kEpiStore = 0, kEpiMaskH = 1, kEpiMask = 2 };

struct QuantOut {
    uint8_t* codes;
    int64_t ldc;      // bytes per output row
    uint8_t* sf;
    int64_t katoms;   // scale-factor atoms per 128-row block
    uint32_t* mask;   // nullable; [rows, K/32]
    int* err;         // nullable; bit 0 = non-finite input seen
    int* fallbacks;   // nullable; QuEST exact-search count
};

struct QuantCfg {
    int transform;
    const uint32_t* sign_bits;  // bit p%32 of word p/32 = 1 -> flip sign at axis position p
    float prescale;             // 1.0 or 0.75
    int rounding;
    uint64_t sr_base;           // mix64(seed ^ mix64(DOMAIN_SR))
    uint64_t counter_start;
    int64_t counter_ld;         // SR stream row stride (0 = the quantized matrix's own row length)
    int sr_fast;                // rounding kSr only: 1 = QT_ROUND_SR_FAST (hash uniforms, not the reference stream)
};

struct MxIn {
    const uint8_t* codes;
    int64_t ldc;
    const uint8_t* sf;
    int64_t katoms;
};

struct EpiParams {
    void* out;
    int64_t ldo;             // elements
    int out_bf16;
    int mode;
    const uint32_t* mask;    // [M, N/32] words (kEpiMaskH)
    int64_t ldm;             // words per mask row
    float scale;
    int dbg;                 // experiment knobs (0 in production)
    int accumulate;          // D += epilogue result (rounded to D's dtype first), QT_EPI_ACCUMULATE
    int split_tiles = 0;     // 2-CTA kernel: the last split_tiles tiles of the walk run as two K-half work units each,
                             // added into their zeroed fp32 D blocks by TMA reduce-add
};

// ---- per-device launch facts (the library serves any device of the process; no single-device caches)
constexpr int kMaxDevices = 64;
int current_device();
int device_sms();                       // SM count of the current device (cached per device)
// true exactly once per device for the given flag array (one-time cudaFuncSetAttribute per device)
bool first_use_on_device(int (&flags)[kMaxDevices]);
// qt_debug_set_grid: cap on the persistent grid of every tile kernel (0 = no cap, production).  Tests set a
// small cap so that each CTA walks many tiles (multi-tile pipelines, stage reuse, TMEM phases).
extern int g_grid_cap;
inline int64_t cap_grid(int64_t want) { return g_grid_cap > 0 && want > g_grid_cap ? g_grid_cap : want; }

int launch_transform_rows(const float* x, float* out, int64_t rows, int64_t cols, int transform,
                          const uint32_t* sign_bits, float prescale, cudaStream_t st);
int launch_signs(uint32_t* bits, int64_t start, int64_t n, uint64_t xi, cudaStream_t st);
int launch_signs2(uint32_t* a, int64_t sa, int64_t na, uint32_t* b, int64_t sb, int64_t nb, uint64_t xi,
                  cudaStream_t st);
int launch_signs2_dev(uint32_t* a, int64_t sa, int64_t na, uint32_t* b, int64_t sb, int64_t nb, const uint64_t* xi,
                      cudaStream_t st);
int launch_layer_seeds(uint64_t* xi, const uint64_t* ids, int n, uint64_t seed, int64_t* step, int inc,
                       cudaStream_t st);
int launch_quant_rows(const void* x, int in_type, int64_t ldx, int64_t rows, int64_t cols, const QuantCfg& cfg,
                      const QuantOut& out, cudaStream_t st);
int launch_quant_tile(const void* x, int in_type, int64_t ldx, const MxIn& mx, int64_t R, int64_t C,
                      const QuantCfg* row_cfg, const QuantOut* row_out, const QuantCfg* col_cfg,
                      const QuantOut* col_out, int col_from_codes, cudaStream_t st);
int launch_tcq_xq(const void* x, int64_t ldx, int64_t R, int64_t C, const QuantOut& row_out,
                  const uint32_t* col_sign_bits, float col_prescale, const QuantOut& col_out, int* fallbacks,
                  cudaStream_t st, const QuantCfg* srf_col = nullptr);   // srf_col: X_t by QT_ROUND_SR_FAST
extern int g_tcq_dbg;  // experiment knobs of the tensor-core quantizer (0 in production)
// srf_row / srf_col (both or neither): QT_ROUND_SR_FAST with these keys / stream layouts instead of RTN
int launch_tcq_dual(const void* x, int64_t ldx, int64_t R, int64_t C, const uint32_t* row_sign_bits,
                    const uint32_t* col_sign_bits, float prescale, const QuantOut& row_out, const QuantOut& col_out,
                    int* fallbacks, cudaStream_t st, const QuantCfg* srf_row = nullptr,
                    const QuantCfg* srf_col = nullptr);
extern int g_gemm_2sm;
extern int g_gemm_cluster8;
extern int g_gemm_splitk;
int launch_gemm(const uint8_t* a, int64_t lda, const uint8_t* a_sf, int64_t a_katoms, const uint8_t* b, int64_t ldb,
                const uint8_t* b_sf, int64_t b_katoms, int64_t M, int64_t N, int64_t K, const EpiParams& ep,
                cudaStream_t st);

// seam.cu: exact scalar replays of the reference's kernels for f64 / any-group inputs
int launch_seam_quant(const double* x, int64_t rows, int64_t cols, int64_t group, int rounding, bool values,
                      uint64_t seed, uint64_t counter_start, double ratio_lo, uint8_t* codes, uint8_t* scales,
                      uint8_t* mask, double* out, cudaStream_t st);
int launch_seam_fwht(void* x, bool f64, int64_t rows, int64_t n, int64_t g, cudaStream_t st);
int launch_seam_gemm_nt(const void* a, const void* b, void* c, bool f64, int64_t m, int64_t n, int64_t k,
                        cudaStream_t st);
int launch_seam_row_sums(const double* a, const double* b, int op, int64_t rows, int64_t n, double* out,
                         cudaStream_t st);

}  // namespace qt
