/* turbofno.h — C ABI of the B200-native TurboFNO Fourier layer (libturbofno.so).
 *
 * Drop-in boundary for the reference package's hot path (arxiv 2504.11681,
 * reference package `fnofuse`, paths relative to /root/reference/pkg/src/fnofuse):
 *
 *   tfno_layer_forward   replaces pipeline.run_layer / run_fused / run_staged
 *                        (pipeline.py:129-131, 297-306): same layer, same
 *                        five modes, same [B,H,dx,dy] -> [B,N,dx,dy] c64
 *                        shapes, first-keep truncation, shared W[H,N],
 *                        unnormalised forward, 1/n inverse.
 *   tfno_config_violations  mirrors core.config_violations (core.py:192-222)
 *                        and build_schedule's k_tb == bs check
 *                        (pipeline.py:106-116) as a bitmask of codes.
 *   tfno_plan_counts     mirrors fft.plan's prune masks and op/twiddle
 *                        budgets (fft.py:97-182, 194-209).
 *   tfno_fft_execute     replaces fft.execute / batched_execute
 *                        (fft.py:258-315) on device pencils with arbitrary
 *                        strides.
 *   tfno_cgemm           replaces cgemm.gemm_tiled / gemm_kloop
 *                        (cgemm.py:83-114) on device matrices with strides.
 *
 * All pointers passed to compute entry points are DEVICE pointers to
 * interleaved complex64 (float re, float im) data.  Calls are asynchronous
 * on `stream` (a cudaStream_t, NULL = legacy default stream), never allocate
 * on the hot call (workspace is caller-provided), take no ownership and are
 * reentrant per stream.  Return 0 on success, else a TFNO_E* code
 * (tfno_strerror).  There is no CPU fallback: without a CUDA device every
 * compute entry point returns TFNO_ECUDA.
 */
#ifndef TURBOFNO_H
#define TURBOFNO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* FnoLayerConfig (core.py:101-124), field order preserved. rank 1 => dim_x = keep_x = 1. */
typedef struct {
  int32_t batch, hidden_dim, output_dim, dim_x, dim_y, keep_x, keep_y, rank;
} tfno_cfg;

/* TileConfig (core.py:127-145). Validated for parity; GPU kernels pick their own tiles. */
typedef struct {
  int32_t m_tb, n_tb, k_tb, m_w, n_w, m_t, n_t;
} tfno_tiles;

/* pipeline.MODES (pipeline.py:41-42), same order. */
enum {
  TFNO_STAGED = 0,          /* cuFFT + truncate + cuBLAS + pad + cuFFT^-1 (unfused baseline) */
  TFNO_FFT_OPTIMIZED = 1,   /* truncating FFT, CGEMM, padded iFFT as separate kernels */
  TFNO_FUSED_FFT_GEMM = 2,  /* FFT inside the GEMM k-loop, C to HBM, padded iFFT */
  TFNO_FUSED_GEMM_IFFT = 3, /* truncating FFT to HBM, GEMM with iFFT epilogue */
  TFNO_FULLY_FUSED = 4      /* FFT -> CGEMM -> iFFT, only input and output touch HBM (rank 1) */
};

/* arithmetic of the channel contraction (FFTs are always FP32):
 *   FP32   FP32 SIMT CGEMM (the exact path; default)
 *   TF32   tcgen05.mma kind::tf32, one pass (stated tolerance 1e-3)
 *   TF32X3 tcgen05 3xTF32 split (hi*hi + hi*lo + lo*hi), fp32-level accuracy (1e-5)
 *   BF16   tcgen05.mma kind::f16 with bf16 operands, fp32 accumulation (stated tolerance 5e-3)
 * Only schedules with a separate contraction kernel use the tensor cores
 * (rank-2 plane path, unfused 1D); the fused row kernels always run FP32. */
enum { TFNO_FP32 = 0, TFNO_TF32 = 1, TFNO_BF16 = 2, TFNO_TF32X3 = 3 };

/* violation bits (core.py ConstraintViolation codes) */
enum {
  TFNO_V_INVALID_RANK_SHAPE = 1u << 0,
  TFNO_V_NON_POWER_OF_TWO = 1u << 1,
  TFNO_V_TRUNCATION_EXCEEDS = 1u << 2,
  TFNO_V_TILE_DIVISIBILITY = 1u << 3,
  TFNO_V_BATCH_SIZE_MISMATCH = 1u << 4
};

/* status codes */
enum {
  TFNO_OK = 0,
  TFNO_EINVAL = 1,      /* config violates constraints / bad argument */
  TFNO_EUNSUPPORTED = 2,/* valid but outside this build's limits (e.g. length > 8192) */
  TFNO_ECUDA = 3,       /* CUDA runtime error (incl. no device) */
  TFNO_EWORKSPACE = 4,  /* workspace too small */
  TFNO_ECUFFT = 5,      /* cuFFT error (staged baseline) */
  TFNO_ECUBLAS = 6      /* cuBLAS error (staged baseline) */
};

const char* tfno_strerror(int code);
const char* tfno_version(void);

/* Bitmask of violated constraints (0 = valid).  tiles may be NULL (skip tile checks). */
uint32_t tfno_config_violations(const tfno_cfg* cfg, const tfno_tiles* tiles, int fft_batch_size);

/* fft.plan(n, direction, keep, src_len): direction -1 forward, +1 inverse.
 * masks (nullable) receives log2(n) * n bytes (stage-major, 1 = executed). */
int tfno_plan_counts(int n, int direction, int keep, int src_len, int64_t* op_budget,
                     int64_t* twiddle_budget, int64_t* full_ops, uint8_t* masks);

/* Device workspace bytes tfno_layer_forward needs for (cfg, mode, prec). */
size_t tfno_workspace_bytes(const tfno_cfg* cfg, int mode, int prec);

/* One Fourier layer: y[B,N,dx,dy] = iFFT_pad( W-mix( FFT_trunc( x[B,H,dx,dy] ))).
 * w is row-major [H][N] (the Python wrapper transposes the reference's
 * column-major ComplexMatrix). */
int tfno_layer_forward(const tfno_cfg* cfg, int mode, int prec, const void* x, const void* w, void* y,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Tensor-core weight packing (SURVEY.md §8b tfno_prepare_weights; no reference
 * equivalent -- the reference's W is a plain ComplexMatrix, cgemm.py:21-58).
 * The real-embedded W' image [[Wr, Wi], [-Wi, Wr]] of W[H][N] in the exact
 * shared-memory layout of the tcgen05 contraction (TF32 / 3xTF32: hi and lo
 * tiles; BF16), built once per weight tensor instead of once per call.
 * tfno_packed_weight_bytes: 0 for TFNO_FP32 (the SIMT path needs no packing).
 * w_packed must be 16-byte aligned device memory. */
size_t tfno_packed_weight_bytes(const tfno_cfg* cfg, int prec);
int tfno_prepare_weights(const tfno_cfg* cfg, int prec, const void* w, void* w_packed, void* stream);
/* tfno_layer_forward with W' from tfno_prepare_weights (same cfg.hidden_dim /
 * output_dim and prec): skips the per-call image build launch. */
int tfno_layer_forward_packed(const tfno_cfg* cfg, int mode, int prec, const void* x, const void* w,
                              const void* w_packed, void* y, void* workspace, size_t workspace_bytes, void* stream);

/* Spectrum-level entry points (building blocks of the hidden-dim split and
 * of layer chains).  modes are natural-order [planes][keep_x][keep_y] c64.
 *   forward: modes[B][H] = first-keep 2D (rank 2) / 1D (rank 1) DFT of x[B][H]
 *   inverse: y[B][N] = scale * zero-padded inverse (1/(dx*dy) normalised) of modes[B][N]
 * Workspace: tfno_spectrum_workspace_bytes(cfg, -1 forward / +1 inverse). */
size_t tfno_spectrum_workspace_bytes(const tfno_cfg* cfg, int direction);
int tfno_spectrum_forward(const tfno_cfg* cfg, const void* x, void* modes, void* workspace, size_t workspace_bytes,
                          void* stream);
int tfno_spectrum_inverse(const tfno_cfg* cfg, const void* modes, void* y, float scale, void* workspace,
                          size_t workspace_bytes, void* stream);

/* Batched pencils FFT: pencil p (p < P) of `in` starts at (p / in_P0) * in_s1 + (p % in_P0) * in_s0
 * and element e is at start + e * in_es (complex elements); same for `out`.
 * Reads src_len elements, writes keep elements; direction -1 forward, +1 inverse (x 1/n). */
int tfno_fft_execute(int n, int direction, int keep, int src_len, int64_t P, const void* in, int64_t in_P0,
                     int64_t in_s1, int64_t in_s0, int64_t in_es, void* out, int64_t out_P0, int64_t out_s1,
                     int64_t out_s0, int64_t out_es, void* stream);

/* C[b] = alpha * A[b] @ W[b], complex64, FP32 accumulation in ascending k.
 * Element (i,j) of X[b] is at X + b*x_bs + i*x_{row} + j*x_{col}. */
int tfno_cgemm(int64_t M, int64_t N, int64_t K, int64_t batch, const void* A, int64_t a_ms, int64_t a_ks,
               int64_t a_bs, const void* W, int64_t w_ks, int64_t w_ns, int64_t w_bs, void* C, int64_t c_ms,
               int64_t c_ns, int64_t c_bs, float alpha, void* stream);

/* tfno_cgemm with a contraction precision (TFNO_FP32 / TFNO_TF32 / TFNO_TF32X3 / TFNO_BF16).
 * The tensor-core path needs the mode layout: a_ms = c_ms = w_ns = 1, w_bs = 0 (N > 128 runs in
 * 128-channel blocks). */
int tfno_cgemm_prec(int64_t M, int64_t N, int64_t K, int64_t batch, const void* A, int64_t a_ms, int64_t a_ks,
                    int64_t a_bs, const void* W, int64_t w_ks, int64_t w_ns, int64_t w_bs, void* C, int64_t c_ms,
                    int64_t c_ns, int64_t c_bs, float alpha, int prec, void* stream);

/* out[i] = sum_{b < batch} in[b*n + i] (complex64, ascending b: deterministic); the batch
 * reduction of the per-element grad_W partials of the backward pass (extension). */
int tfno_batch_sum(const void* in, int64_t batch, int64_t n, void* out, void* stream);

/* Per-mode channel mix (extension: per-mode weights, einsum bhq,hnq->bnq):
 * C[b][n][q] = alpha * sum_h A[b][h][q] * W[h][n][q], complex64, q < modes fastest in all three
 * (A = the truncated spectrum [batch][hidden][kx*ky], W = [hidden][out][kx][ky] weights,
 * C = the modes the padded inverse reads).  FP32 accumulation in ascending h. */
int tfno_permode_mix(int64_t batch, int64_t hidden, int64_t out, int64_t modes, const void* A, const void* W,
                     void* C, float alpha, void* stream);

/* Plane modulation (symmetric +-mode truncation, an extension beyond the reference):
 * out[p][x][y] = scale * in[p][x][y] * exp(sign * 2*pi*i * (sx*x/dx + sy*y/dy)), sign = +1 / -1.
 * Modulating by (+keep_x/2, +keep_y/2) before and (-keep_x/2, -keep_y/2) after the first-keep
 * layer keeps the frequencies [-keep/2, keep/2) on each axis.  in == out is allowed. */
int tfno_modulate(int64_t planes, int dx, int dy, int sx, int sy, int sign, const void* in, void* out,
                  float scale, void* stream);

/* Real-field FNO block (extension beyond the reference, which is complex-to-complex only).
 * The real layer irfft2(rfft2(x)[:kx, :ky] W, s=(dx, dy)), ky <= dy/2 + 1, is composed on the
 * spectrum ABI: tfno_real_to_complex -> tfno_spectrum_forward -> tfno_half_spectrum_weight ->
 * tfno_cgemm -> tfno_spectrum_inverse -> tfno_real_epilogue (see paper_2504_11681_b200/realfield.py).
 *   tfno_real_to_complex:      z[i] = x[i] + 0i, n reals (16-byte aligned pointers)
 *   tfno_half_spectrum_weight: modes[r][k] *= 2 for 0 < k < dy/2 (rows x ky complex, in place)
 *   tfno_real_epilogue:        out[b][n][p] = act(Re z[b][n][p] + bypass[b][n][p] + bias[n]);
 *                              bypass / bias may be NULL; activation TFNO_ACT_*. */
enum { TFNO_ACT_NONE = 0, TFNO_ACT_RELU = 1, TFNO_ACT_GELU = 2 };
int tfno_real_to_complex(const float* x, void* z, int64_t n, void* stream);
int tfno_half_spectrum_weight(void* modes, int64_t rows, int ky, int dy, void* stream);
int tfno_real_epilogue(const void* z, const float* bypass, const float* bias, int64_t batch, int N, int64_t P,
                       int activation, float* out, void* stream);

/* Kernels of this library launched by the calling thread since load (library
 * kernels of the staged baseline, cuFFT/cuBLAS, are not counted). */
long long tfno_launch_count(void);

/* Profiling hook (calling thread): when events != NULL, tfno_layer_forward
 * records events[0] before its first launch and events[i+1] after its i-th
 * stage, on its stream (cudaEvent_t handles; count = capacity). */
void tfno_set_stage_events(void** events, int count);

/* Kernel schedule tfno_layer_forward will use: number of launches and a
 * short description (e.g. "x-fft|fused-rows|x-ifft").  desc may be NULL. */
int tfno_layer_schedule(const tfno_cfg* cfg, int mode, int prec, char* desc, size_t desc_len);

#ifdef __cplusplus
}
#endif
#endif /* TURBOFNO_H */
