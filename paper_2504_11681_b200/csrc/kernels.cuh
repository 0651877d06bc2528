// Kernel argument structs and launch helpers shared by kernels.cu / api.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tfno {

// Pencil p of a batched transform starts at (p / P0) * s1 + (p % P0) * s0 and
// its element e lives at base + e * es (all in complex elements).
struct PencilMap {
  int64_t P0, s1, s0, es;
};

struct FftPencilArgs {
  int n, keep, src_len, PB, pencil_major;
  int64_t P;
  float scale;
  const float2* in;
  PencilMap im;
  float2* out;
  PencilMap om;
  const float2* twg;
};

struct GemmArgs {
  int64_t M, N, K, batch;
  const float2* A;
  int64_t a_ms, a_ks, a_bs;
  const float2* W;
  int64_t w_ks, w_ns, w_bs;
  float2* C;
  int64_t c_ms, c_ns, c_bs;
  float alpha;
  int64_t fold;  // batch elements folded into one M tile (0/1 = none; mode-layout fast path only)
  void* wimg;    // tcgen05 paths: caller scratch for the real-embedded W' image (nullptr: build per CTA)
  int wimg_ready;  // wimg already holds the image of W (tfno_prepare_weights): skip the build launch
};

// Row-fused layer kernel (FFT along contiguous rows -> CGEMM over the
// channel axis -> padded iFFT along rows).  A "row group" g = b*gx + p owns
// H input rows (one per channel h) and N output rows.
struct FusedArgs {
  int n, keep, H, N, gx;
  int64_t G;
  const float2* x;
  int64_t x_sb, x_sp, x_sh;  // input row (g,h): x + b*x_sb + p*x_sp + h*x_sh
  const float2* A;
  int64_t a_sb, a_sp, a_sh;  // A panel row (g,h), contiguous keep
  const float2* W;           // [H][N] row-major
  float2* y;
  int64_t y_sb, y_sp, y_sn;  // output row (g,n), contiguous n
  float2* C;
  int64_t c_sb, c_sp, c_sn;  // C row (g,n), contiguous keep
  int NT, KC, EC;
  int nsplit;  // fused1d: output channels split over nsplit CTAs per row group (forward recomputed)
  int cluster;  // fused1d: hidden channels split over a cluster of CTAs, partial C reduced over DSMEM
  int part;     // fused1d: 0 full layer, 1 FFT + GEMM -> C (K4), 2 A -> GEMM + iFFT (K5)
  const float2* twg;
  float inv_scale;
};

size_t fused_smem_bytes(const FusedArgs& a);
size_t fft_pencils_smem_bytes(int n, int PB, int pencil_major);

cudaError_t launch_fft_pencils(const FftPencilArgs& a, int dir, cudaStream_t s);
cudaError_t launch_cgemm(const GemmArgs& g, cudaStream_t s);
// tcgen05 TF32 contraction (cgemm_tc.cu): passes 1 = TF32, 3 = 3xTF32 (fp32-level accuracy)
bool cgemm_tc_supported(const GemmArgs& g);
cudaError_t launch_cgemm_tc(const GemmArgs& g, int passes, cudaStream_t s);
// bytes of the W' image (TF32 / 3xTF32) for an N x K channel mix; 0 for other precisions
size_t cgemm_tc_wimg_bytes(int64_t N, int64_t K, int prec);
// build the W' image of g.W (precision 1 TF32, 2 BF16, 3 3xTF32) into img
cudaError_t build_cgemm_wimg(const GemmArgs& g, int prec, void* img, cudaStream_t s);
// precision dispatch: 0 FP32 SIMT, 1 TF32 tcgen05, 2 BF16 tcgen05, 3 3xTF32 tcgen05
// (launch_cgemm_tc passes: 1 TF32, 3 3xTF32, 0 BF16)
inline cudaError_t launch_cgemm_prec(const GemmArgs& g, int prec, cudaStream_t s) {
  if (prec == 0) return launch_cgemm(g, s);
  if (prec == 1 || prec == 3) return launch_cgemm_tc(g, prec == 1 ? 1 : 3, s);
  if (prec == 2) return launch_cgemm_tc(g, 0, s);
  return cudaErrorNotSupported;
}
cudaError_t launch_fused(const FusedArgs& a, bool fuse_fft, bool fuse_ifft, cudaStream_t s);
// per-mode channel mix C[b][n][q] = alpha sum_h A[b][h][q] W[h][n][q] (permode.cu)
cudaError_t launch_permode_mix(const float2* A, const float2* W, float2* C, int64_t B, int64_t H, int64_t N,
                               int64_t MQ, float alpha, cudaStream_t s);
cudaError_t launch_batch_sum(const float2* in, int64_t batch, int64_t n, float2* out, cudaStream_t s);
cudaError_t launch_modulate(const float2* in, float2* out, int64_t planes, int dx, int dy, int sx, int sy, int sign,
                            float scale, const float2* tw, cudaStream_t s);
// warp-synchronous register FFT rows (warpfft.cu): n in {256, 1024}, keep / src_len <= n/4
bool warp_fft_supported(int n, int dir, int keep, int src_len);
cudaError_t launch_warp_fft(int n, int dir, const float2* in, int64_t is, float2* out, int64_t os, int64_t P,
                            int keep, int src_len, float scale, const float2* tw, cudaStream_t s);
// fully fused 1D layer on warp FFTs (K6): whole k-loop per CTA, W resident in smem
bool warp_fused_supported(int n, int keep, int H, int NO);
// fully fused 1D layer, k-loop over channel chunks with a TMA producer warp (fused1d.cu)
bool fused1d_supported(int n, int keep, int H, int NO);
// output-channel split for fused1d so that small batches still fill the SMs (0 = unsupported)
int fused1d_split(int n, int keep, int H, int NO, int64_t G);
int fused1d_split_gemm_ifft(int n, int keep, int H, int NO);  // K5: output-channel split, any batch (0: none)
// hidden-channel cluster split for fused1d (0/1 = none); takes precedence over the output split
int fused1d_cluster(int n, int keep, int H, int NO, int64_t G);
cudaError_t launch_fused1d(const FusedArgs& a, cudaStream_t s);
cudaError_t launch_warp_fused(const FusedArgs& a, cudaStream_t s);
cudaError_t launch_pad_truncate(const float2* src, int64_t planes, int sx, int sy, int64_t s_plane,
                                float2* dst, int dx2, int dy2, int64_t d_plane, int cx, int cy,
                                float scale, cudaStream_t s);

extern thread_local long long g_launches;  // our kernels launched by this thread
int device_sms();
// programmatic dependent launch (TFNO_PDL: 0 off, 1 = the fused 1D layer kernel only (default),
// 2 = also the plane / mode-CGEMM kernels).  Measured (profiles/r02/pdl_ab.txt): C1 graph
// replay 13.5-15.3 -> 12.4 us with it; the 2D kernels gain nothing eagerly (C3, C4) and the
// C5 4-layer graph slows 12.9 -> 20.7 ms with PDL edges between the plane kernels.
bool pdl_enabled(int level = 1);
// launch with the programmatic-stream-serialization attribute: ONLY for kernels
// that call pdl_wait() (ptx.cuh) before touching memory an earlier kernel writes
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {  // the level-2 kernels (plane / mode CGEMM)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled(2) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
// the same with PDL at level 1 (on by default): the 1D layer kernels
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl1(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                               Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled(1) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
// small latency-bound 1D layers (N = 128 / 256 / 1024): one kernel, CTA = (batch element, 8 / 32 / 64
// output channels) with the grid within one wave of SMs
bool tiny1d_supported(int n, int keep, int B, int H, int N);
int tiny1d_channels_per_cta(int B, int N);  // 8 / 32 / 64 (0: no one-wave grid)
cudaError_t launch_tiny1d(const float2* x, const float2* W, float2* y, int n, int B, int H, int N, int keep,
                          const float2* tw, cudaStream_t s);  // SM count of the current device (cached per device)

}  // namespace tfno
