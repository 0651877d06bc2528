// C ABI of libturbofno.so: validation, workspace sizing, the per-mode
// kernel schedule of the Fourier layer, the standalone FFT / CGEMM entry
// points and the staged (cuFFT + cuBLAS) unfused baseline.
//
// Layer schedule (all modes compute pipeline.run_layer's values,
// pipeline.py:129-294; which passes cross HBM follows the mode):
//   rank 2 stage 1   x-FFT, truncating to keep_x      (pipeline.py:150-168)
//   stage 2          y-FFT -> CGEMM -> y-iFFT, fused per mode
//                    (pipeline.py:185-275)
//   rank 2 stage 3   x-iFFT, zero-padded from keep_x   (pipeline.py:277-292)
// Rank-2 fully_fused uses the per-plane 2D kernels (plane2d.cu) when the
// shape qualifies: 2D-FFT(plane) -> CGEMM over modes -> 2D-iFFT(plane), so
// only the input, the output and two 1/64-size mode tensors touch HBM.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cufft.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/turbofno.h"
#include "common.cuh"
#include "kernels.cuh"
#include "plane2d.cuh"
#include "rows1d.cuh"

using namespace tfno;

namespace {

std::mutex g_mu;

// optional per-stage profiling events (tfno_set_stage_events)
thread_local cudaEvent_t* t_events = nullptr;
thread_local int t_nevents = 0;
thread_local int t_mark = 0;
inline void stage_begin(cudaStream_t st) {
  t_mark = 0;
  if (t_nevents > 0) cudaEventRecord(t_events[t_mark++], st);
}
inline void stage_mark(cudaStream_t st) {
  if (t_mark < t_nevents) cudaEventRecord(t_events[t_mark++], st);
}
float2* g_tw[64] = {nullptr};  // per-device master twiddle table w_{TW_MAX}^k

const float2* twiddle_table(int& err) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || dev < 0 || dev >= 64) {
    err = TFNO_ECUDA;
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_tw[dev]) {
    std::vector<float2> h(TFNO_TW_MAX);
    for (int k = 0; k < TFNO_TW_MAX; ++k) {
      double ang = -2.0 * M_PI * (double)k / (double)TFNO_TW_MAX;
      h[k] = make_float2((float)cos(ang), (float)sin(ang));
    }
    float2* d = nullptr;
    if (cudaMalloc(&d, sizeof(float2) * TFNO_TW_MAX) != cudaSuccess) {
      err = TFNO_ECUDA;
      return nullptr;
    }
    if (cudaMemcpy(d, h.data(), sizeof(float2) * TFNO_TW_MAX, cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaFree(d);
      err = TFNO_ECUDA;
      return nullptr;
    }
    g_tw[dev] = d;
  }
  err = 0;
  return g_tw[dev];
}

bool pow2(int n) { return n >= 1 && (n & (n - 1)) == 0; }

inline int cuda_status(cudaError_t e) { return e == cudaSuccess ? TFNO_OK : TFNO_ECUDA; }

struct Geo {
  int64_t B, H, N, dx, dy, kx, ky;
  int rank;
};

Geo geo_of(const tfno_cfg* c) {
  return Geo{c->batch, c->hidden_dim, c->output_dim, c->dim_x, c->dim_y, c->keep_x, c->keep_y, c->rank};
}

// ---------------- fused-rows tiling ----------------
bool fused_tiling(int n, int keep, int N, FusedArgs& a) {
  if (n > 4096 || keep > 1024) return false;
  int KC = 4096 / n;
  KC = KC < 1 ? 1 : (KC > 8 ? 8 : KC);
  int EC = 4096 / n;
  EC = EC < 1 ? 1 : (EC > 32 ? 32 : EC);
  int MT = (keep + 3) / 4;
  int ntg_max = 256 / MT;
  if (ntg_max < 1) return false;
  int NT = ((N + 3) / 4) * 4;
  if (NT > 4 * ntg_max) NT = 4 * ntg_max;
  int cap = (8192 / keep) & ~3;
  if (cap < 1) cap = 1;
  if (NT > cap) NT = cap;
  if (NT < 1) NT = 1;
  a.n = n;
  a.keep = keep;
  a.N = N;
  a.KC = KC;
  a.EC = EC;
  a.NT = NT;
  while (fused_smem_bytes(a) > 220 * 1024 && (a.EC > 1 || a.NT > 1)) {
    if (a.EC > 1)
      a.EC /= 2;
    else
      a.NT = a.NT > 4 ? a.NT - 4 : a.NT - 1;
  }
  return fused_smem_bytes(a) <= 220 * 1024;
}

// compile-time row kernels (rows1d.cu): C tile [keep x NT] in registers of 512 threads
bool rows_tiling(int n, int keep, int N, int& NT) {
  if (!rows_supported(n) || keep > 2048) return false;
  const int MT = (keep + 3) / 4;
  const int ntg_max = 512 / MT;
  if (ntg_max < 1) return false;
  NT = ((N + 3) / 4) * 4;
  if (NT > 4 * ntg_max) NT = 4 * ntg_max;
  while (rows_fused_smem_bytes(n, keep, NT) > 220 * 1024 && NT > 4) NT -= 4;
  return rows_fused_smem_bytes(n, keep, NT) <= 220 * 1024;
}

// FFT over pencils: contiguous rows of a specialised length go to the
// compile-time row kernel, everything else to the general pencil kernel
cudaError_t launch_pencils_auto(const FftPencilArgs& a, int dir, cudaStream_t st) {
  const bool rows = a.im.P0 == 1 && a.im.s0 == 0 && a.im.es == 1 && a.om.P0 == 1 && a.om.s0 == 0 && a.om.es == 1;
  const int dir_ = dir < 0 ? -1 : 1;
  if (rows && warp_fft_supported(a.n, dir_, a.keep, a.src_len))
    return launch_warp_fft(a.n, dir_, a.in, a.im.s1, a.out, a.om.s1, a.P, a.keep, a.src_len, a.scale, a.twg, st);
  if (rows && rows_supported(a.n))
    return launch_rows_fft(a.n, dir, a.in, a.im.s1, a.out, a.om.s1, a.P, a.keep, a.src_len, a.scale, a.twg, st);
  return launch_fft_pencils(a, dir, st);
}

// schedule decision shared by workspace sizing and the forward
struct Sched {
  bool staged = false, plane2d = false, rows_fast = false, warp_fused = false, f1 = false;
  bool plane_mix = false;  // rank-2 plane path with the channel mix fused into the inverse
  bool tiny = false;       // small latency-bound 1D layer: tiny1d kernel
  int rows_NT = 0, f1_split = 1, f1_cluster = 1, f1_part = 0;
  bool fg = false, gi = false;  // which row fusions actually run
  bool need_A = false, need_C = false, need_s1 = false, need_mid = false;
  int launches = 0;
  std::string desc;
};

int num_sms_api() { return device_sms(); }  // per device

Sched make_sched(const tfno_cfg* c, int mode, int prec = 0, bool allow_f1 = true) {
  Sched s;
  Geo g = geo_of(c);
  if (mode == TFNO_STAGED) {
    s.staged = true;
    s.launches = 2;
    s.desc = "cufft|truncate|cublas|pad|cufft-inv";
    return s;
  }
  bool want_fg = (mode == TFNO_FUSED_FFT_GEMM || mode == TFNO_FULLY_FUSED);
  bool want_gi = (mode == TFNO_FUSED_GEMM_IFFT || mode == TFNO_FULLY_FUSED);
  // rank 2 on the per-plane kernels: fully_fused, and fused_gemm_ifft as the fused channel mix +
  // inverse kernel (the GEMM-iFFT fusion of the mode, plane_invmix_g)
  if (g.rank == 2 && plane2d_supported(c) &&
      (mode == TFNO_FULLY_FUSED || (mode == TFNO_FUSED_GEMM_IFFT && plane2d_fusedmix(c, prec, mode)))) {
    s.plane2d = true;
    s.need_A = s.need_C = true;
    if (plane2d_fusedmix(c, prec, mode)) {
      s.plane_mix = true;
      s.launches = 2;
      s.desc = "plane-fft2d|plane-mix-ifft2d";
    } else {
      s.launches = 3;
      s.desc = "plane-fft2d|cgemm-modes|plane-ifft2d";
    }
    return s;
  }
  {
    // latency-bound small 1D layers (C1): one independent CTA per (batch element, 8 output
    // channels), forward FFTs recomputed per CTA; only while the CTAs fit one wave
    static int tiny_env = -2;
    if (tiny_env == -2) {
      const char* e = getenv("TFNO_TINY1D");
      tiny_env = e ? atoi(e) : -1;
    }
    // default where measured faster than the persistent fused kernel (profiles/r02/tiny2_ab.txt):
    // N <= 256 rows, H <= 64, at most 32 output channels per CTA (C1 12.7 -> 6.9 us, N256-H64-B64
    // 15.2 -> 13.0 us; N256-H128-B64 and N1024-H64-B64 are slower: 22.7 -> 30.6, 31.8 -> 42.1 us);
    // TFNO_TINY1D=1 wherever the kernel fits, 0 never
    const bool tiny_ok = tiny1d_supported((int)g.dy, (int)g.ky, (int)g.B, (int)g.H, (int)g.N);
    const bool tiny_win = g.dy <= 256 && g.H <= 64 && tiny1d_channels_per_cta((int)g.B, (int)g.N) <= 32;
    if (g.rank == 1 && mode == TFNO_FULLY_FUSED && prec == TFNO_FP32 && tiny_env != 0 && tiny_ok &&
        (tiny_env == 1 || tiny_win)) {
      s.tiny = true;
      s.launches = 1;
      s.desc = "tiny1d-fft-cgemm-ifft";
      return s;
    }
  }
  FusedArgs fa{};
  int NT = 0;
  bool ok;
  static int f1_env = -2;
  if (f1_env == -2) {
    const char* e = getenv("TFNO_FUSED1D");
    f1_env = e ? atoi(e) : -1;
  }
  // tensor-core precisions on contraction-heavy shapes: the fused 1D kernel's
  // contraction is FP32 SIMT, so the unfused schedule with the tcgen05 CGEMM wins
  const bool tc_heavy = prec != TFNO_FP32 && g.H * g.N >= 128 * 128;
  const bool f1_full = fused1d_supported((int)g.dy, (int)g.ky, (int)g.H, (int)g.N);
  const int f1_forced = f1_full ? 0 : fused1d_split((int)g.dy, (int)g.ky, (int)g.H, (int)g.N, g.B * g.kx);
  // the partial fusions (K4 fused_fft_gemm / K5 fused_gemm_ifft) on the same kernel: its FFT + GEMM
  // half writing C, or its GEMM + iFFT half reading the y-FFT's A (even keep: 16-byte bulk rows)
  const bool part_mode = mode == TFNO_FUSED_FFT_GEMM || mode == TFNO_FUSED_GEMM_IFFT;
  const int gi_split = mode == TFNO_FUSED_GEMM_IFFT
                           ? fused1d_split_gemm_ifft((int)g.dy, (int)g.ky, (int)g.H, (int)g.N) : 0;
  if (allow_f1 && part_mode && f1_env != 0 && !tc_heavy && (f1_full || f1_forced > 1 || gi_split > 1) &&
      g.ky % 2 == 0) {
    s.f1 = true;
    s.f1_part = mode == TFNO_FUSED_FFT_GEMM ? 1 : 2;
    s.f1_cluster = 1;
    s.f1_split = f1_full ? 1 : (s.f1_part == 2 ? std::max(gi_split, f1_forced) : f1_forced);
    s.fg = s.f1_part == 1;
    s.gi = s.f1_part == 2;
    s.need_s1 = s.need_mid = (g.rank == 2);
    s.need_A = !s.fg;
    s.need_C = !s.gi;
    const char* mid = s.fg ? "fused1d-fft-cgemm|y-ifft" : "y-fft|fused1d-cgemm-ifft";
    s.desc = g.rank == 2 ? std::string("x-fft|") + mid + "|x-ifft" : std::string(mid);
    s.launches = g.rank == 2 ? 4 : 2;
    return s;
  }
  if (allow_f1 && mode == TFNO_FULLY_FUSED && f1_env != 0 && !tc_heavy && (f1_full || f1_forced > 1)) {
    s.f1 = true;
    s.f1_cluster = f1_full ? fused1d_cluster((int)g.dy, (int)g.ky, (int)g.H, (int)g.N, g.B * g.kx) : 1;
    s.f1_split = s.f1_cluster > 1 ? 1 : fused1d_split((int)g.dy, (int)g.ky, (int)g.H, (int)g.N, g.B * g.kx);
    s.fg = s.gi = true;
    s.need_s1 = s.need_mid = (g.rank == 2);
    s.launches = (g.rank == 2) ? 3 : 1;
    s.desc = g.rank == 2 ? "x-fft|fused1d-fft-cgemm-ifft|x-ifft" : "fused1d-fft-cgemm-ifft";
    return s;
  }
  if (mode == TFNO_FULLY_FUSED && !tc_heavy && warp_fused_supported((int)g.dy, (int)g.ky, (int)g.H, (int)g.N)) {
    s.warp_fused = true;
    s.fg = s.gi = true;
    s.need_s1 = s.need_mid = (g.rank == 2);
    s.launches = (g.rank == 2) ? 3 : 1;
    s.desc = g.rank == 2 ? "x-fft|fused-fft-cgemm-ifft|x-ifft" : "fused-fft-cgemm-ifft";
    return s;
  }
  if (rows_tiling((int)g.dy, (int)g.ky, (int)g.N, NT)) {
    // fused only while the C tile covers all of N (else the FFT would be
    // recomputed per n-tile): otherwise the unfused schedule of fast kernels
    ok = (g.N + NT - 1) / NT <= 1;  // measured: a second n-tile (recomputed FFTs) loses to the unfused schedule
    // ...except when there are too few row groups to fill the SMs (C1: 16):
    // then split N into tiles so G * tiles approaches one wave (FFT recompute
    // is cheap next to the idle SMs)
    const int64_t G = g.B * g.kx;
    const int sms = num_sms_api();
    if (ok && 2 * G <= sms) {
      int tiles = (int)(sms / G);
      int nt = (int)((g.N + tiles - 1) / tiles);
      nt = ((nt + 3) / 4) * 4;
      if (nt < 4) nt = 4;
      if (nt < NT) NT = nt;
    }
    s.rows_fast = ok;
    s.rows_NT = NT;
  } else {
    ok = fused_tiling((int)g.dy, (int)g.ky, (int)g.N, fa);
  }
  if (tc_heavy) ok = false;  // the standalone tcgen05 CGEMM beats the fused SIMT contraction
  s.fg = want_fg && ok;
  s.gi = want_gi && ok;
  s.need_s1 = s.need_mid = (g.rank == 2);
  s.need_A = !s.fg;
  s.need_C = !s.gi;
  std::string d;
  int L = 0;
  if (g.rank == 2) {
    d += "x-fft|";
    ++L;
  }
  if (!s.fg) {
    d += "y-fft|";
    ++L;
  }
  if (s.fg || s.gi) {
    d += s.fg && s.gi ? "fused-fft-cgemm-ifft|" : (s.fg ? "fused-fft-cgemm|" : "fused-cgemm-ifft|");
    ++L;
  } else {
    d += "cgemm|";
    ++L;
  }
  if (!s.gi) {
    d += "y-ifft|";
    ++L;
  }
  if (g.rank == 2) {
    d += "x-ifft|";
    ++L;
  }
  if (!d.empty()) d.pop_back();
  s.desc = d;
  s.launches = L;
  return s;
}

// ---------------- staged baseline: cuFFT + cuBLAS ----------------
// Plans and cuBLAS handles are per (device, stream): a cuFFT plan's work area
// and a cuBLAS handle's workspace are used by the kernels they enqueue, so two
// streams running the staged layer concurrently (HostPipeline) must not share them.
struct BaselineCtx {
  std::map<cudaStream_t, cublasHandle_t> blas;
  std::map<std::tuple<int, int, int, int64_t, cudaStream_t>, cufftHandle> plans;
};
BaselineCtx g_base[64];
std::mutex g_base_mu[64];  // guards the per-device caches (enqueue only)

int staged_chunk(const Geo& g) {
  // batch chunk so that the full forward spectrum of a chunk is <= 8 GiB
  int64_t per = g.H * g.dx * g.dy * 8;
  int64_t cap = (8LL << 30) / (per > 0 ? per : 1);
  if (cap < 1) cap = 1;
  return (int)(cap < g.B ? cap : g.B);
}

size_t staged_ws(const Geo& g) {
  int64_t bc = staged_chunk(g);
  return (size_t)(bc * g.H * g.dx * g.dy + g.B * g.H * g.kx * g.ky + g.B * g.N * g.kx * g.ky) * 8;
}

// cuBLAS handles and cuFFT plans are created on first use per stream; when that
// first use happens while the stream is being captured into a CUDA graph, their
// (uncaptured) setup allocations run in relaxed capture mode for this thread
struct RelaxedCapture {
  cudaStreamCaptureMode m = cudaStreamCaptureModeRelaxed;
  RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&m); }
  ~RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&m); }
};

int get_plan(int dev, int rank, int dx, int dy, int64_t batch, cudaStream_t st, cufftHandle* out) {
  auto key = std::make_tuple(rank, dx, dy, batch, st);
  auto& ctx = g_base[dev];
  auto it = ctx.plans.find(key);
  if (it != ctx.plans.end()) {
    *out = it->second;
    return 0;
  }
  RelaxedCapture relax;
  cufftHandle h;
  if (cufftCreate(&h) != CUFFT_SUCCESS) return TFNO_ECUFFT;
  size_t wsz = 0;
  cufftResult r;
  if (rank == 2) {
    long long dims[2] = {dx, dy};
    r = cufftMakePlanMany64(h, 2, dims, nullptr, 1, (long long)dx * dy, nullptr, 1, (long long)dx * dy, CUFFT_C2C,
                            batch, &wsz);
  } else {
    long long dims[1] = {dy};
    r = cufftMakePlanMany64(h, 1, dims, nullptr, 1, dy, nullptr, 1, dy, CUFFT_C2C, batch, &wsz);
  }
  if (r != CUFFT_SUCCESS) {
    cufftDestroy(h);
    return TFNO_ECUFFT;
  }
  ctx.plans[key] = h;
  *out = h;
  return 0;
}

int staged_forward(const tfno_cfg* c, const float2* x, const float2* w, float2* y, float2* ws, size_t ws_bytes,
                   cudaStream_t st) {
  Geo g = geo_of(c);
  if (ws_bytes < staged_ws(g)) return TFNO_EWORKSPACE;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TFNO_ECUDA;
  if (dev < 0 || dev >= 64) return TFNO_ECUDA;
  std::lock_guard<std::mutex> lk(g_base_mu[dev]);
  auto& ctx = g_base[dev];
  cublasHandle_t& blas = ctx.blas[st];
  if (!blas) {
    RelaxedCapture relax;
    if (cublasCreate(&blas) != CUBLAS_STATUS_SUCCESS) {
      ctx.blas.erase(st);
      return TFNO_ECUBLAS;
    }
    cublasSetMathMode(blas, CUBLAS_DEFAULT_MATH);  // true FP32, no TF32
    // a per-handle workspace allocated here, so no GEMM allocates lazily (inside a capture)
    void* bws = nullptr;
    if (cudaMalloc(&bws, 32u << 20) == cudaSuccess) cublasSetWorkspace(blas, bws, 32u << 20);
  }
  const int64_t bc = staged_chunk(g);
  float2* full = ws;
  float2* A = full + bc * g.H * g.dx * g.dy;
  float2* Cm = A + g.B * g.H * g.kx * g.ky;
  const int64_t plane = g.dx * g.dy, modes = g.kx * g.ky;
  stage_begin(st);
  // forward FFT + truncate, chunked over batch
  for (int64_t b0 = 0; b0 < g.B; b0 += bc) {
    int64_t nb = (g.B - b0 < bc) ? g.B - b0 : bc;
    cufftHandle p;
    int e = get_plan(dev, g.rank, (int)g.dx, (int)g.dy, nb * g.H, st, &p);
    if (e) return e;
    cufftSetStream(p, st);
    if (cufftExecC2C(p, (cufftComplex*)(x + b0 * g.H * plane), (cufftComplex*)full, CUFFT_FORWARD) !=
        CUFFT_SUCCESS)
      return TFNO_ECUFFT;
    cudaError_t ce = launch_pad_truncate(full, nb * g.H, (int)g.dx, (int)g.dy, plane, A + b0 * g.H * modes,
                                         (int)g.kx, (int)g.ky, modes, (int)g.kx, (int)g.ky, 1.0f, st);
    if (ce != cudaSuccess) return TFNO_ECUDA;
  }
  stage_mark(st);
  // CGEMM over the channel axis, 1/(dx*dy) folded into alpha
  cublasSetStream(blas, st);
  cuComplex alpha = make_cuComplex((float)(1.0 / (double)(g.dx * g.dy)), 0.f), beta = make_cuComplex(0.f, 0.f);
  cublasStatus_t bs = cublasCgemmStridedBatched(blas, CUBLAS_OP_N, CUBLAS_OP_T, (int)modes, (int)g.N, (int)g.H,
                                                &alpha, (const cuComplex*)A, (int)modes, g.H * modes,
                                                (const cuComplex*)w, (int)g.N, 0, &beta, (cuComplex*)Cm,
                                                (int)modes, g.N * modes, (int)g.B);
  if (bs != CUBLAS_STATUS_SUCCESS) return TFNO_ECUBLAS;
  stage_mark(st);
  // pad into y, then in-place inverse FFT over the whole output
  cudaError_t ce = launch_pad_truncate(Cm, g.B * g.N, (int)g.kx, (int)g.ky, modes, y, (int)g.dx, (int)g.dy, plane,
                                       (int)g.kx, (int)g.ky, 1.0f, st);
  if (ce != cudaSuccess) return TFNO_ECUDA;
  int64_t obc = bc * g.H / (g.N > 0 ? g.N : 1);
  if (obc < 1) obc = 1;
  for (int64_t b0 = 0; b0 < g.B; b0 += obc) {
    int64_t nb = (g.B - b0 < obc) ? g.B - b0 : obc;
    cufftHandle p;
    int e = get_plan(dev, g.rank, (int)g.dx, (int)g.dy, nb * g.N, st, &p);
    if (e) return e;
    cufftSetStream(p, st);
    cufftComplex* yy = (cufftComplex*)(y + b0 * g.N * plane);
    if (cufftExecC2C(p, yy, yy, CUFFT_INVERSE) != CUFFT_SUCCESS) return TFNO_ECUFFT;
  }
  stage_mark(st);
  return cuda_status(cudaGetLastError());
}

// the channel mix runs as a standalone CGEMM (plane2d path or the unfused row schedule)
bool sched_has_cgemm(const Sched& s) {
  return (s.plane2d && !s.plane_mix) || (!s.plane2d && !s.tiny && !s.staged && !s.fg && !s.gi);
}

size_t wimg_bytes_for(const tfno_cfg* c, int mode, int prec) {
  Sched s = make_sched(c, mode, prec);
  if (!sched_has_cgemm(s)) return 0;
  Geo g = geo_of(c);
  const size_t b = cgemm_tc_wimg_bytes(g.N, g.H, prec);
  return (b + 255) & ~(size_t)255;
}

size_t base_ws_bytes(const tfno_cfg* c, int mode, int prec) {  // intermediates only
  Geo g = geo_of(c);
  Sched s = make_sched(c, mode, prec);
  if (s.staged) return staged_ws(g);
  size_t e = 0;
  if (s.need_s1) e += g.B * g.H * g.kx * g.dy;
  if (s.need_mid) e += g.B * g.N * g.kx * g.dy;
  const int64_t mq = s.plane2d ? plane2d_modes(c) : g.kx * g.ky;  // generic plane kernels: KP^2 padded modes
  if (s.need_A) e += g.B * g.H * mq;
  if (s.need_C) e += s.plane2d ? plane2d_c_elems(c, prec, mode) : g.B * g.N * mq;
  return e * sizeof(float2);
}

size_t ws_bytes_for(const tfno_cfg* c, int mode, int prec = 0) {
  return base_ws_bytes(c, mode, prec) + wimg_bytes_for(c, mode, prec);
}

FftPencilArgs pencil_args(int n, int keep, int src_len, int64_t P, const float2* in, PencilMap im, float2* out,
                          PencilMap om, float scale, const float2* tw) {
  FftPencilArgs a{};
  a.n = n;
  a.keep = keep;
  a.src_len = src_len;
  a.P = P;
  a.in = in;
  a.im = im;
  a.out = out;
  a.om = om;
  a.scale = scale;
  a.twg = tw;
  // coalesce across pencils when elements are strided and pencils adjacent
  a.pencil_major = (im.es != 1 && om.es != 1) ? 1 : 0;
  int PB = 4096 / n;
  if (PB < 1) PB = 1;
  if (a.pencil_major && PB > 64) PB = 64;
  if (PB > P) PB = (int)P;
  if (PB < 1) PB = 1;
  a.PB = PB;
  return a;
}

}  // namespace

extern "C" {

const char* tfno_strerror(int code) {
  switch (code) {
    case TFNO_OK: return "ok";
    case TFNO_EINVAL: return "invalid configuration or argument";
    case TFNO_EUNSUPPORTED: return "unsupported shape for this build";
    case TFNO_ECUDA: return "CUDA error (or no CUDA device)";
    case TFNO_EWORKSPACE: return "workspace too small";
    case TFNO_ECUFFT: return "cuFFT error";
    case TFNO_ECUBLAS: return "cuBLAS error";
    default: return "unknown error";
  }
}

const char* tfno_version(void) { return "turbofno-b200 0.1.0 sm_100a"; }

long long tfno_launch_count(void) { return tfno::g_launches; }

void tfno_set_stage_events(void** events, int count) {
  t_events = (cudaEvent_t*)events;
  t_nevents = events ? count : 0;
}

uint32_t tfno_config_violations(const tfno_cfg* c, const tfno_tiles* t, int fft_batch_size) {
  if (!c) return TFNO_V_INVALID_RANK_SHAPE;
  uint32_t v = 0;
  if (c->rank != 1 && c->rank != 2) v |= TFNO_V_INVALID_RANK_SHAPE;
  if (c->batch < 1 || c->hidden_dim < 1 || c->output_dim < 1) v |= TFNO_V_INVALID_RANK_SHAPE;
  if (!pow2(c->dim_x) || !pow2(c->dim_y)) v |= TFNO_V_NON_POWER_OF_TWO;
  if (c->keep_x < 1 || c->keep_x > c->dim_x || c->keep_y < 1 || c->keep_y > c->dim_y)
    v |= TFNO_V_TRUNCATION_EXCEEDS;
  if (c->rank == 1 && (c->dim_x != 1 || c->keep_x != 1)) v |= TFNO_V_INVALID_RANK_SHAPE;
  if (t) {
    const int32_t* f = &t->m_tb;
    bool pos = true;
    for (int i = 0; i < 7; ++i) pos = pos && f[i] >= 1;
    if (!pos) {
      v |= TFNO_V_TILE_DIVISIBILITY;
    } else {
      bool div = (t->m_tb % t->m_w == 0) && (t->n_tb % t->n_w == 0) && (t->m_w % t->m_t == 0) &&
                 (t->n_w % t->n_t == 0);
      if (!div || (t->m_w / t->m_t) * (t->n_w / t->n_t) != 32) v |= TFNO_V_TILE_DIVISIBILITY;
    }
    if (t->k_tb != fft_batch_size) v |= TFNO_V_BATCH_SIZE_MISMATCH;
  }
  return v;
}

size_t tfno_workspace_bytes(const tfno_cfg* c, int mode, int prec) {
  if (!c || tfno_config_violations(c, nullptr, 8)) return 0;
  return ws_bytes_for(c, mode, prec);
}

int tfno_layer_schedule(const tfno_cfg* c, int mode, int prec, char* desc, size_t len) {
  if (!c || mode < 0 || mode > 4 || tfno_config_violations(c, nullptr, 8)) return -1;
  Sched s = make_sched(c, mode, prec);
  if (desc && len) {
    strncpy(desc, s.desc.c_str(), len - 1);
    desc[len - 1] = 0;
  }
  // the TF32 / 3xTF32 contraction adds one launch building the W' image (same stage)
  return s.launches + (wimg_bytes_for(c, mode, prec) ? 1 : 0);
}

int tfno_fft_execute(int n, int direction, int keep, int src_len, int64_t P, const void* in, int64_t in_P0,
                     int64_t in_s1, int64_t in_s0, int64_t in_es, void* out, int64_t out_P0, int64_t out_s1,
                     int64_t out_s0, int64_t out_es, void* stream) {
  if (!pow2(n) || keep < 1 || keep > n || src_len < 1 || src_len > n || P < 0 || in_P0 < 1 || out_P0 < 1)
    return TFNO_EINVAL;
  if (n > TFNO_TW_MAX) return TFNO_EUNSUPPORTED;
  if (P == 0) return TFNO_OK;
  if (!in || !out) return TFNO_EINVAL;
  int err = 0;
  const float2* tw = twiddle_table(err);
  if (err) return err;
  FftPencilArgs a = pencil_args(n, keep, src_len, P, (const float2*)in, PencilMap{in_P0, in_s1, in_s0, in_es},
                                (float2*)out, PencilMap{out_P0, out_s1, out_s0, out_es},
                                direction < 0 ? 1.0f : (float)(1.0 / n), tw);
  return cuda_status(launch_pencils_auto(a, direction < 0 ? -1 : 1, (cudaStream_t)stream));
}

int tfno_cgemm_prec(int64_t M, int64_t N, int64_t K, int64_t batch, const void* A, int64_t a_ms, int64_t a_ks,
                    int64_t a_bs, const void* W, int64_t w_ks, int64_t w_ns, int64_t w_bs, void* C, int64_t c_ms,
                    int64_t c_ns, int64_t c_bs, float alpha, int prec, void* stream) {
  if (prec == TFNO_FP32)
    return tfno_cgemm(M, N, K, batch, A, a_ms, a_ks, a_bs, W, w_ks, w_ns, w_bs, C, c_ms, c_ns, c_bs, alpha, stream);
  if (prec != TFNO_TF32 && prec != TFNO_TF32X3 && prec != TFNO_BF16) return TFNO_EUNSUPPORTED;
  if (M < 0 || N < 0 || K < 0 || batch < 0) return TFNO_EINVAL;
  if (M == 0 || N == 0 || batch == 0) return TFNO_OK;
  if (!A || !W || !C) return TFNO_EINVAL;
  GemmArgs g{M, N, K, batch, (const float2*)A, a_ms, a_ks, a_bs, (const float2*)W, w_ks, w_ns, w_bs,
             (float2*)C, c_ms, c_ns, c_bs, alpha};
  if (!cgemm_tc_supported(g)) return TFNO_EUNSUPPORTED;
  return cuda_status(launch_cgemm_prec(g, prec, (cudaStream_t)stream));
}

int tfno_cgemm(int64_t M, int64_t N, int64_t K, int64_t batch, const void* A, int64_t a_ms, int64_t a_ks,
               int64_t a_bs, const void* W, int64_t w_ks, int64_t w_ns, int64_t w_bs, void* C, int64_t c_ms,
               int64_t c_ns, int64_t c_bs, float alpha, void* stream) {
  if (M < 0 || N < 0 || K < 0 || batch < 0) return TFNO_EINVAL;
  if (M == 0 || N == 0 || batch == 0) return TFNO_OK;
  if (!A || !W || !C || batch > 65535) return TFNO_EINVAL;
  GemmArgs g{M, N, K, batch, (const float2*)A, a_ms, a_ks, a_bs, (const float2*)W, w_ks, w_ns, w_bs,
             (float2*)C, c_ms, c_ns, c_bs, alpha};
  return cuda_status(launch_cgemm(g, (cudaStream_t)stream));
}

int tfno_batch_sum(const void* in, int64_t batch, int64_t n, void* out, void* stream) {
  if (batch < 0 || n < 0) return TFNO_EINVAL;
  if (n == 0) return TFNO_OK;
  if (!in || !out) return TFNO_EINVAL;
  return cuda_status(launch_batch_sum((const float2*)in, batch, n, (float2*)out, (cudaStream_t)stream));
}

int tfno_permode_mix(int64_t batch, int64_t hidden, int64_t out, int64_t modes, const void* A, const void* W,
                     void* C, float alpha, void* stream) {
  if (batch < 0 || hidden < 0 || out < 0 || modes < 0) return TFNO_EINVAL;
  if (batch == 0 || out == 0 || modes == 0) return TFNO_OK;
  if (!A || !W || !C) return TFNO_EINVAL;
  return cuda_status(launch_permode_mix((const float2*)A, (const float2*)W, (float2*)C, batch, hidden, out, modes,
                                        alpha, (cudaStream_t)stream));
}

int tfno_modulate(int64_t planes, int dx, int dy, int sx, int sy, int sign, const void* in, void* out, float scale,
                  void* stream) {
  if (planes < 0 || !pow2(dx) || !pow2(dy) || dx > TFNO_TW_MAX || dy > TFNO_TW_MAX || (sign != 1 && sign != -1))
    return TFNO_EINVAL;
  if (planes == 0) return TFNO_OK;
  if (!in || !out) return TFNO_EINVAL;
  int err = 0;
  const float2* tw = twiddle_table(err);
  if (err) return err;
  return cuda_status(launch_modulate((const float2*)in, (float2*)out, planes, dx, dy, sx, sy, sign, scale, tw,
                                     (cudaStream_t)stream));
}

size_t tfno_spectrum_workspace_bytes(const tfno_cfg* c, int direction) {
  if (!c || tfno_config_violations(c, nullptr, 8)) return 0;
  if (c->rank != 2 || plane2d_spectrum_ok(c)) return 0;
  Geo g = geo_of(c);
  return (size_t)((direction < 0 ? g.H : g.N) * g.B * g.kx * g.dy) * sizeof(float2);
}

int tfno_spectrum_forward(const tfno_cfg* c, const void* xv, void* modes, void* wsv, size_t ws_bytes, void* stream) {
  if (!c || tfno_config_violations(c, nullptr, 8) || !xv || !modes) return TFNO_EINVAL;
  if (c->dim_x > TFNO_TW_MAX || c->dim_y > TFNO_TW_MAX) return TFNO_EUNSUPPORTED;
  if (ws_bytes < tfno_spectrum_workspace_bytes(c, -1)) return TFNO_EWORKSPACE;
  int err = 0;
  const float2* tw = twiddle_table(err);
  if (err) return err;
  cudaStream_t st = (cudaStream_t)stream;
  Geo g = geo_of(c);
  const float2* x = (const float2*)xv;
  float2* A = (float2*)modes;
  if (plane2d_spectrum_ok(c)) return cuda_status(launch_plane2d_fwd(c, x, A, tw, st));
  const float2* src = x;
  if (g.rank == 2) {
    float2* s1 = (float2*)wsv;
    FftPencilArgs a = pencil_args((int)g.dx, (int)g.kx, (int)g.dx, g.B * g.H * g.dy, x,
                                  PencilMap{g.dy, g.dx * g.dy, 1, g.dy}, s1, PencilMap{g.dy, g.kx * g.dy, 1, g.dy},
                                  1.0f, tw);
    if (launch_pencils_auto(a, -1, st) != cudaSuccess) return TFNO_ECUDA;
    src = s1;
  }
  FftPencilArgs a = pencil_args((int)g.dy, (int)g.ky, (int)g.dy, g.B * g.H * g.kx, src, PencilMap{1, g.dy, 0, 1}, A,
                                PencilMap{1, g.ky, 0, 1}, 1.0f, tw);
  return cuda_status(launch_pencils_auto(a, -1, st));
}

int tfno_spectrum_inverse(const tfno_cfg* c, const void* modes, void* yv, float scale, void* wsv, size_t ws_bytes,
                          void* stream) {
  if (!c || tfno_config_violations(c, nullptr, 8) || !yv || !modes) return TFNO_EINVAL;
  if (c->dim_x > TFNO_TW_MAX || c->dim_y > TFNO_TW_MAX) return TFNO_EUNSUPPORTED;
  if (ws_bytes < tfno_spectrum_workspace_bytes(c, 1)) return TFNO_EWORKSPACE;
  int err = 0;
  const float2* tw = twiddle_table(err);
  if (err) return err;
  cudaStream_t st = (cudaStream_t)stream;
  Geo g = geo_of(c);
  const float2* Cm = (const float2*)modes;
  float2* y = (float2*)yv;
  if (plane2d_spectrum_ok(c))
    return cuda_status(launch_plane2d_inv(c, Cm, y, (float)(scale / ((double)g.dx * g.dy)), tw, st));
  float2* dst = g.rank == 2 ? (float2*)wsv : y;
  float sy = (float)(1.0 / (double)g.dy) * (g.rank == 2 ? 1.0f : scale);
  FftPencilArgs a = pencil_args((int)g.dy, (int)g.dy, (int)g.ky, g.B * g.N * g.kx, Cm, PencilMap{1, g.ky, 0, 1}, dst,
                                PencilMap{1, g.dy, 0, 1}, sy, tw);
  if (launch_pencils_auto(a, 1, st) != cudaSuccess) return TFNO_ECUDA;
  if (g.rank == 2) {
    FftPencilArgs b = pencil_args((int)g.dx, (int)g.dx, (int)g.kx, g.B * g.N * g.dy, dst,
                                  PencilMap{g.dy, g.kx * g.dy, 1, g.dy}, y, PencilMap{g.dy, g.dx * g.dy, 1, g.dy},
                                  (float)(scale / (double)g.dx), tw);
    if (launch_pencils_auto(b, 1, st) != cudaSuccess) return TFNO_ECUDA;
  }
  return TFNO_OK;
}

size_t tfno_packed_weight_bytes(const tfno_cfg* c, int prec) {
  if (!c || tfno_config_violations(c, nullptr, 8)) return 0;
  if (prec != TFNO_TF32 && prec != TFNO_TF32X3 && prec != TFNO_BF16) return 0;
  return cgemm_tc_wimg_bytes(c->output_dim, c->hidden_dim, prec);
}

int tfno_prepare_weights(const tfno_cfg* c, int prec, const void* wv, void* packed, void* stream) {
  if (!c || tfno_config_violations(c, nullptr, 8) || !wv || !packed) return TFNO_EINVAL;
  if (prec != TFNO_TF32 && prec != TFNO_TF32X3 && prec != TFNO_BF16) return TFNO_EINVAL;
  if (((uintptr_t)packed & 15) != 0) return TFNO_EINVAL;
  GemmArgs ga{};
  ga.M = 1;
  ga.N = c->output_dim;
  ga.K = c->hidden_dim;
  ga.batch = 1;
  ga.a_ms = 1;
  ga.W = (const float2*)wv;
  ga.w_ks = c->output_dim;
  ga.w_ns = 1;
  ga.c_ms = 1;
  return cuda_status(build_cgemm_wimg(ga, prec, packed, (cudaStream_t)stream));
}

static int layer_forward_impl(const tfno_cfg* c, int mode, int prec, const void* xv, const void* wv,
                              const void* packed, void* yv, void* wsv, size_t ws_bytes, void* stream);

int tfno_layer_forward(const tfno_cfg* c, int mode, int prec, const void* xv, const void* wv, void* yv,
                       void* wsv, size_t ws_bytes, void* stream) {
  return layer_forward_impl(c, mode, prec, xv, wv, nullptr, yv, wsv, ws_bytes, stream);
}

int tfno_layer_forward_packed(const tfno_cfg* c, int mode, int prec, const void* xv, const void* wv,
                              const void* w_packed, void* yv, void* wsv, size_t ws_bytes, void* stream) {
  if (!w_packed || ((uintptr_t)w_packed & 15) != 0) return TFNO_EINVAL;
  return layer_forward_impl(c, mode, prec, xv, wv, w_packed, yv, wsv, ws_bytes, stream);
}

static int layer_forward_impl(const tfno_cfg* c, int mode, int prec, const void* xv, const void* wv,
                              const void* packed, void* yv, void* wsv, size_t ws_bytes, void* stream) {
  if (!c || mode < TFNO_STAGED || mode > TFNO_FULLY_FUSED) return TFNO_EINVAL;
  if (tfno_config_violations(c, nullptr, 8)) return TFNO_EINVAL;
  if (prec != TFNO_FP32 && prec != TFNO_TF32 && prec != TFNO_TF32X3 && prec != TFNO_BF16) return TFNO_EINVAL;
  if (!xv || !wv || !yv) return TFNO_EINVAL;
  if (c->dim_x > TFNO_TW_MAX || c->dim_y > TFNO_TW_MAX) return TFNO_EUNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  const float2* x = (const float2*)xv;
  const float2* w = (const float2*)wv;
  float2* y = (float2*)yv;
  float2* ws = (float2*)wsv;
  // a workspace sized without the W' image (older callers) still works: the
  // tensor-core contraction then builds W' per CTA
  size_t need = base_ws_bytes(c, mode, prec);
  if (ws_bytes < need || (need && !ws)) return TFNO_EWORKSPACE;
  const size_t wimg_need = wimg_bytes_for(c, mode, prec);
  Geo g = geo_of(c);
  Sched s = make_sched(c, mode, prec);
  if (s.f1 && ((((uintptr_t)x | (uintptr_t)w | (uintptr_t)y) & 15) != 0 || (g.rank == 2 && (g.dy * 8) % 16))) {
    // the fused 1D kernel moves rows with 16-byte TMA bulk copies: a valid but
    // misaligned view (e.g. w_all[i] with odd H*N) takes the next schedule
    Sched s2 = make_sched(c, mode, prec, false);
    size_t need2 = 0;
    {
      if (s2.need_s1) need2 += g.B * g.H * g.kx * g.dy;
      if (s2.need_mid) need2 += g.B * g.N * g.kx * g.dy;
      if (s2.need_A) need2 += g.B * g.H * g.kx * g.ky;
      if (s2.need_C) need2 += g.B * g.N * g.kx * g.ky;
      need2 *= sizeof(float2);
    }
    if (ws_bytes < need2 || (need2 && !ws)) return TFNO_EUNSUPPORTED;
    s = s2;
  }
  if (s.plane2d && ((((uintptr_t)x | (uintptr_t)y) & 15) != 0)) return TFNO_EUNSUPPORTED;  // TMA rows
  if (s.staged) return staged_forward(c, x, w, y, ws, ws_bytes, st);
  int err = 0;
  const float2* tw = twiddle_table(err);
  if (err) return err;

  // workspace carve-up
  float2* p = ws;
  float2* s1 = nullptr;
  float2* mid = nullptr;
  float2* A = nullptr;
  float2* Cm = nullptr;
  if (s.need_s1) { s1 = p; p += g.B * g.H * g.kx * g.dy; }
  if (s.need_mid) { mid = p; p += g.B * g.N * g.kx * g.dy; }
  const int64_t mq = s.plane2d ? plane2d_modes(c) : g.kx * g.ky;
  if (s.need_A) { A = p; p += g.B * g.H * mq; }
  if (s.need_C) { Cm = p; p += s.plane2d ? plane2d_c_elems(c, prec, mode) : g.B * g.N * mq; }
  // W' image: the caller's packed weights (tfno_prepare_weights) or built per call in the workspace tail
  const int wimg_ready = (packed && wimg_need) ? 1 : 0;
  void* wimg = wimg_ready ? const_cast<void*>(packed)
                          : ((wimg_need && ws_bytes >= need + wimg_need) ? (void*)p : nullptr);

  stage_begin(st);
  if (s.plane2d)
    return cuda_status(launch_plane2d_layer(c, x, w, y, A, Cm, tw, prec, wimg, wimg_ready, st, &stage_mark, mode));
  if (s.tiny) {
    const cudaError_t te = launch_tiny1d(x, w, y, (int)g.dy, (int)g.B, (int)g.H, (int)g.N, (int)g.ky, tw, st);
    if (te == cudaSuccess) stage_mark(st);
    return cuda_status(te);
  }

  cudaError_t e;
  const float2* src = x;
  if (g.rank == 2) {
    // stage 1: x-FFT over B*H*dy strided pencils, keep kx -> s1[B,H,kx,dy]
    FftPencilArgs a = pencil_args((int)g.dx, (int)g.kx, (int)g.dx, g.B * g.H * g.dy, x,
                                  PencilMap{g.dy, g.dx * g.dy, 1, g.dy}, s1, PencilMap{g.dy, g.kx * g.dy, 1, g.dy},
                                  1.0f, tw);
    if ((e = launch_pencils_auto(a, -1, st)) != cudaSuccess) return TFNO_ECUDA;
    stage_mark(st);
    src = s1;
  }
  float2* dst_mid = (g.rank == 2) ? mid : y;
  const int64_t rows_in = g.B * g.H * g.kx, rows_out = g.B * g.N * g.kx;
  if (!s.fg) {
    // y-FFT of every source row -> A[B,H,kx,ky]
    FftPencilArgs a = pencil_args((int)g.dy, (int)g.ky, (int)g.dy, rows_in, src, PencilMap{1, g.dy, 0, 1}, A,
                                  PencilMap{1, g.ky, 0, 1}, 1.0f, tw);
    if ((e = launch_pencils_auto(a, -1, st)) != cudaSuccess) return TFNO_ECUDA;
    stage_mark(st);
  }
  if (s.fg || s.gi) {
    FusedArgs fa{};
    if (s.rows_fast || s.warp_fused || s.f1) {
      fa.n = (int)g.dy;
      fa.keep = (int)g.ky;
      fa.N = (int)g.N;
      fa.NT = (s.warp_fused || s.f1) ? (int)g.N : s.rows_NT;
      fa.nsplit = s.f1 ? s.f1_split : 1;
      fa.cluster = s.f1 ? s.f1_cluster : 1;
      fa.part = s.f1 ? s.f1_part : 0;
      fa.KC = rows_chunk((int)g.dy);
      fa.EC = fa.KC;
    } else {
      fused_tiling((int)g.dy, (int)g.ky, (int)g.N, fa);
    }
    fa.H = (int)g.H;
    fa.gx = (int)g.kx;
    fa.G = g.B * g.kx;
    fa.x = src;
    fa.x_sb = g.H * g.kx * g.dy;
    fa.x_sp = g.dy;
    fa.x_sh = g.kx * g.dy;
    fa.A = A;
    fa.a_sb = g.H * g.kx * g.ky;
    fa.a_sp = g.ky;
    fa.a_sh = g.kx * g.ky;
    fa.W = w;
    fa.y = dst_mid;
    fa.y_sb = g.N * g.kx * g.dy;
    fa.y_sp = g.dy;
    fa.y_sn = g.kx * g.dy;
    fa.C = Cm;
    fa.c_sb = g.N * g.kx * g.ky;
    fa.c_sp = g.ky;
    fa.c_sn = g.kx * g.ky;
    fa.twg = tw;
    fa.inv_scale = (float)(1.0 / (double)g.dy);
    if (fa.G > 2147483647LL || (g.N + fa.NT - 1) / fa.NT > 65535) return TFNO_EUNSUPPORTED;
    e = s.f1 ? launch_fused1d(fa, st)
             : s.warp_fused ? launch_warp_fused(fa, st)
                            : (s.rows_fast ? launch_rows_fused(fa, s.fg, s.gi, st) : launch_fused(fa, s.fg, s.gi, st));
    if (e != cudaSuccess) return TFNO_ECUDA;
    stage_mark(st);
  } else {
    // C[b, n, pq] = sum_h A[b, h, pq] W[h, n]
    GemmArgs ga{g.kx * g.ky, g.N, g.H, g.B, A, 1, g.kx * g.ky, g.H * g.kx * g.ky, w, g.N, 1, 0,
                Cm, 1, g.kx * g.ky, g.N * g.kx * g.ky, 1.0f};
    ga.wimg = wimg;
    ga.wimg_ready = wimg_ready;
    if (g.B > 65535) return TFNO_EUNSUPPORTED;
    if ((e = launch_cgemm_prec(ga, prec, st)) != cudaSuccess) return e == cudaErrorNotSupported ? TFNO_EUNSUPPORTED : TFNO_ECUDA;
    stage_mark(st);
  }
  if (!s.gi) {
    FftPencilArgs a = pencil_args((int)g.dy, (int)g.dy, (int)g.ky, rows_out, Cm, PencilMap{1, g.ky, 0, 1}, dst_mid,
                                  PencilMap{1, g.dy, 0, 1}, (float)(1.0 / (double)g.dy), tw);
    if ((e = launch_pencils_auto(a, 1, st)) != cudaSuccess) return TFNO_ECUDA;
    stage_mark(st);
  }
  if (g.rank == 2) {
    FftPencilArgs a = pencil_args((int)g.dx, (int)g.dx, (int)g.kx, g.B * g.N * g.dy, mid,
                                  PencilMap{g.dy, g.kx * g.dy, 1, g.dy}, y, PencilMap{g.dy, g.dx * g.dy, 1, g.dy},
                                  (float)(1.0 / (double)g.dx), tw);
    if ((e = launch_pencils_auto(a, 1, st)) != cudaSuccess) return TFNO_ECUDA;
    stage_mark(st);
  }
  return TFNO_OK;
}

}  // extern "C"
