// Compile-time-specialised row kernels (contiguous pencils of length N):
//
//   rows_fused_kernel<N, FUSE_FFT, FUSE_IFFT>  K6 / K4 / K5 — the paper's fused
//       Fourier layer over rows (pipeline.py:185-206 k-loop, :245-250
//       epilogue): for each k-chunk of KC channel rows the inputs of the NEXT
//       chunk are prefetched into registers while the current chunk's
//       truncated FFT lands in the shared-memory A panel and updates the
//       register C tile; the epilogue runs the zero-padded iFFT of the C tile
//       straight from shared memory and writes output rows.
//   rows_fft_kernel<N, DIR>  K1/K2 for contiguous rows: persistent, next block
//       prefetched into registers, truncating / zero-padded.
//
// Chunk size KC*N = 8*NTH complex, so every thread owns 8 first-pass inputs.
#include <cuda_runtime.h>

#include "fft_ct.cuh"
#include "kernels.cuh"
#include "rows1d.cuh"

namespace tfno {

constexpr int kRowsNTH = 512;

template <int N>
struct RowsGeo {
  using P = ct::Plan<N>;
  static constexpr int NTH = kRowsNTH;
  static constexpr int KC = (8 * NTH / N) < 1 ? 1 : 8 * NTH / N;  // rows per chunk
  static constexpr int NB0 = N / P::R0;
  static constexpr int IT0 = (KC * NB0) / NTH;   // first-pass butterflies per thread
  static constexpr int VPT = IT0 * P::R0;        // prefetched values per thread
  static_assert((KC * NB0) % NTH == 0, "chunk shape");
  static constexpr int BUF = KC * P::PSTRIDE;    // one ping-pong buffer (complex)
};

// first-pass inputs of a KC-row chunk: thread t, iteration it -> butterfly
// idx = t + it*NTH, pencil p = idx / NB0, k = idx % NB0, elements k + m*NB0
template <int N>
__device__ __forceinline__ void prefetch_chunk(float2 (&pre)[RowsGeo<N>::VPT], const float2* __restrict__ base,
                                               int64_t row_stride, int rows, int src_len, int tid) {
  using Gm = RowsGeo<N>;
  constexpr int R0 = ct::Plan<N>::R0, NB0 = Gm::NB0;
#pragma unroll
  for (int it = 0; it < Gm::IT0; ++it) {
    const int idx = tid + it * Gm::NTH;
    const int p = idx / NB0, k = idx % NB0;
#pragma unroll
    for (int m = 0; m < R0; ++m) {
      const int e = k + m * NB0;
      pre[it * R0 + m] = (p < rows && e < src_len) ? __ldg(&base[(int64_t)p * row_stride + e]) : make_float2(0.f, 0.f);
    }
  }
}

// pass 0 from the register prefetch, then the remaining passes through smem
template <int N, int DIR, class Dst>
__device__ __forceinline__ void transform_from_regs(const float2 (&pre)[RowsGeo<N>::VPT], int tid,
                                                    const float2* twp, const Dst& dst, float2* b0, float2* b1,
                                                    int keep, float scale) {
  using Gm = RowsGeo<N>;
  using P = ct::Plan<N>;
  constexpr int R0 = P::R0, NB0 = Gm::NB0;
  static_assert(P::NP > 1, "row kernels are instantiated for N >= 64");
  {
    const ct::PadBuf o{b0, P::PSTRIDE};
#pragma unroll
    for (int it = 0; it < Gm::IT0; ++it) {
      const int idx = tid + it * Gm::NTH;
      const int p = idx / NB0, k = idx % NB0;
      float2 v[R0];
#pragma unroll
      for (int m = 0; m < R0; ++m) v[m] = pre[it * R0 + m];
      ct::dftR<R0, DIR>(v);
#pragma unroll
      for (int m = 0; m < R0; ++m) o.store(p, k * R0 + m, v[m]);
    }
    __syncthreads();
    ct::run_from<N, 1, DIR, Gm::NTH>(Gm::KC, tid, twp, o, dst, b1, b0, keep, N, scale);
  }
}

struct PanelDst1 {
  float2* as;
  int keep;
  __device__ __forceinline__ void store(int p, int o, float2 v) const { as[p * keep + o] = v; }
};
struct ColSrc1 {
  const float2* cs;
  int ldc, c0;
  __device__ __forceinline__ float2 load(int p, int e) const { return cs[(c0 + p) * ldc + e]; }
};
struct RowOut1 {
  float2* __restrict__ base;
  int64_t sn;
  int c0, ncols;
  __device__ __forceinline__ void store(int p, int o, float2 v) const {
    if (c0 + p < ncols) base[(int64_t)(c0 + p) * sn + o] = v;
  }
};

template <int N>
size_t rows_fused_smem(int keep, int NT) {
  using Gm = RowsGeo<N>;
  using P = ct::Plan<N>;
  size_t e = P::TWN + 2 * (size_t)Gm::BUF + (size_t)Gm::KC * keep + (size_t)Gm::KC * NT + (size_t)NT * (keep + 1);
  return e * sizeof(float2);
}

template <int N, bool FUSE_FFT, bool FUSE_IFFT>
__global__ void __launch_bounds__(kRowsNTH, 1) rows_fused_kernel(FusedArgs a) {
  using Gm = RowsGeo<N>;
  using P = ct::Plan<N>;
  constexpr int NTH = Gm::NTH, KC = Gm::KC;
  extern __shared__ __align__(16) float2 sm[];
  float2* twp = sm;
  float2* b0 = twp + P::TWN;
  float2* b1 = b0 + Gm::BUF;
  const int keep = a.keep, NT = a.NT, H = a.H, NO = a.N;
  float2* As = b1 + Gm::BUF;
  float2* Ws = As + KC * keep;
  float2* Cs = Ws + KC * NT;
  const int ldc = keep + 1;
  const int tid = threadIdx.x;
  const int ntiles = (NO + NT - 1) / NT;
  const int64_t items = a.G * ntiles;
  const int MT = (keep + 3) / 4, NTg = (NT + 3) / 4;
  const bool gemm_thread = tid < MT * NTg;
  const int tm = tid % MT, tn = tid / MT;
  if (FUSE_FFT || FUSE_IFFT) ct::build_twiddles<N, NTH>(twp, a.twg, tid);
  __syncthreads();
  const int nchunks = (H + KC - 1) / KC;

  float2 pre[Gm::VPT];
  auto chunk_base = [&](int64_t item, int c) {
    const int64_t g = item / ntiles;
    return a.x + (g / a.gx) * a.x_sb + (g % a.gx) * a.x_sp + (int64_t)c * KC * a.x_sh;
  };
  int64_t item = blockIdx.x;
  if (FUSE_FFT && item < items) prefetch_chunk<N>(pre, chunk_base(item, 0), a.x_sh, min(KC, H), N, tid);

  for (; item < items; item += gridDim.x) {
    const int64_t g = item / ntiles;
    const int64_t bb = g / a.gx, pp = g % a.gx;
    const int n0 = (int)(item % ntiles) * NT;
    const int ntc = min(NT, NO - n0);
    float2 acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);

    for (int c = 0; c < nchunks; ++c) {
      const int kc = c * KC, kcn = min(KC, H - kc);
      for (int i = tid; i < KC * NT; i += NTH) {
        const int k = i / NT, j = i % NT;
        Ws[i] = (k < kcn && j < ntc) ? a.W[(int64_t)(kc + k) * NO + n0 + j] : make_float2(0.f, 0.f);
      }
      if (FUSE_FFT) {
        float2 cur[Gm::VPT];
#pragma unroll
        for (int v = 0; v < Gm::VPT; ++v) cur[v] = pre[v];
        // prefetch the next chunk (or the first chunk of the next work item)
        if (c + 1 < nchunks) {
          prefetch_chunk<N>(pre, chunk_base(item, c + 1), a.x_sh, min(KC, H - kc - KC), N, tid);
        } else if (item + gridDim.x < items) {
          prefetch_chunk<N>(pre, chunk_base(item + gridDim.x, 0), a.x_sh, min(KC, H), N, tid);
        }
        transform_from_regs<N, -1>(cur, tid, twp, PanelDst1{As, keep}, b0, b1, keep, 1.0f);
        // rows kcn..KC were zero-filled by the prefetch -> their panel rows are 0
      } else {
        const float2* Ab = a.A + bb * a.a_sb + pp * a.a_sp + (int64_t)kc * a.a_sh;
        for (int i = tid; i < KC * keep; i += NTH) {
          const int k = i / keep, q = i % keep;
          As[i] = k < kcn ? Ab[(int64_t)k * a.a_sh + q] : make_float2(0.f, 0.f);
        }
        __syncthreads();
      }
      if (gemm_thread) {
#pragma unroll 4
        for (int k = 0; k < KC; ++k) {
          float2 av[4], bv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int q = tm + MT * i;
            av[i] = q < keep ? As[k * keep + q] : make_float2(0.f, 0.f);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int cc = tn + NTg * j;
            bv[j] = cc < NT ? Ws[k * NT + cc] : make_float2(0.f, 0.f);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) cmac(acc[i][j], av[i], bv[j]);
        }
      }
      __syncthreads();
    }

    if (FUSE_IFFT) {
      if (gemm_thread) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int q = tm + MT * i;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int cc = tn + NTg * j;
            if (q < keep && cc < NT) Cs[cc * ldc + q] = acc[i][j];
          }
        }
      }
      __syncthreads();
      float2* ybase = a.y + bb * a.y_sb + pp * a.y_sp + (int64_t)n0 * a.y_sn;
      for (int c0 = 0; c0 < ntc; c0 += KC) {
        const int pb = min(KC, ntc - c0);
        ct::transform<N, 1, NTH>(pb, tid, twp, ColSrc1{Cs, ldc, c0}, RowOut1{ybase, a.y_sn, c0, ntc}, b0, b1, N,
                                 keep, a.inv_scale);
      }
    } else {
      if (gemm_thread) {
        float2* cbase = a.C + bb * a.c_sb + pp * a.c_sp + (int64_t)n0 * a.c_sn;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int q = tm + MT * i;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int cc = tn + NTg * j;
            if (q < keep && cc < ntc) cbase[(int64_t)cc * a.c_sn + q] = acc[i][j];
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- rows FFT
struct RowsOut {
  float2* __restrict__ base;
  int64_t stride;
  int rows;
  __device__ __forceinline__ void store(int p, int o, float2 v) const {
    if (p < rows) base[(int64_t)p * stride + o] = v;
  }
};

template <int N>
size_t rows_fft_smem() {
  using Gm = RowsGeo<N>;
  return sizeof(float2) * ((size_t)ct::Plan<N>::TWN + 2 * (size_t)Gm::BUF);
}

template <int N, int DIR>
__global__ void __launch_bounds__(kRowsNTH, 1) rows_fft_kernel(const float2* __restrict__ in, int64_t in_stride,
                                                               float2* __restrict__ out, int64_t out_stride, int64_t P,
                                                               int keep, int src_len, float scale,
                                                               const float2* __restrict__ twg) {
  using Gm = RowsGeo<N>;
  constexpr int NTH = Gm::NTH, KC = Gm::KC;
  extern __shared__ __align__(16) float2 sm[];
  float2* twp = sm;
  float2* b0 = twp + ct::Plan<N>::TWN;
  float2* b1 = b0 + Gm::BUF;
  const int tid = threadIdx.x;
  ct::build_twiddles<N, NTH>(twp, twg, tid);
  __syncthreads();
  const int64_t nblk = (P + KC - 1) / KC;
  float2 pre[Gm::VPT];
  int64_t blk = blockIdx.x;
  if (blk < nblk) prefetch_chunk<N>(pre, in + blk * KC * in_stride, in_stride, (int)min((int64_t)KC, P - blk * KC), src_len, tid);
  for (; blk < nblk; blk += gridDim.x) {
    float2 cur[Gm::VPT];
#pragma unroll
    for (int v = 0; v < Gm::VPT; ++v) cur[v] = pre[v];
    const int64_t nx = blk + gridDim.x;
    if (nx < nblk)
      prefetch_chunk<N>(pre, in + nx * KC * in_stride, in_stride, (int)min((int64_t)KC, P - nx * KC), src_len, tid);
    const int rows = (int)min((int64_t)KC, P - blk * KC);
    transform_from_regs<N, DIR>(cur, tid, twp, RowsOut{out + blk * KC * out_stride, out_stride, rows}, b0, b1, keep,
                                scale);
  }
}

// ---------------------------------------------------------------- dispatch
static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

bool rows_supported(int n) { return n >= 64 && n <= 4096 && (n & (n - 1)) == 0; }

template <int N, bool F, bool I>
static cudaError_t launch_rf(const FusedArgs& a, cudaStream_t s) {
  size_t smem = rows_fused_smem<N>(a.keep, a.NT);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(rows_fused_kernel<N, F, I>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t items = a.G * ((a.N + a.NT - 1) / a.NT);
  const int grid = (int)(items < sm_count() ? items : sm_count());
  rows_fused_kernel<N, F, I><<<grid, kRowsNTH, smem, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch_rf_n(const FusedArgs& a, bool f, bool i, cudaStream_t s) {
  if (f && i) return launch_rf<N, true, true>(a, s);
  if (f) return launch_rf<N, true, false>(a, s);
  if (i) return launch_rf<N, false, true>(a, s);
  return launch_rf<N, false, false>(a, s);
}

size_t rows_fused_smem_bytes(int n, int keep, int NT) {
  switch (n) {
    case 64: return rows_fused_smem<64>(keep, NT);
    case 128: return rows_fused_smem<128>(keep, NT);
    case 256: return rows_fused_smem<256>(keep, NT);
    case 512: return rows_fused_smem<512>(keep, NT);
    case 1024: return rows_fused_smem<1024>(keep, NT);
    case 2048: return rows_fused_smem<2048>(keep, NT);
    case 4096: return rows_fused_smem<4096>(keep, NT);
  }
  return (size_t)-1;
}

int rows_chunk(int n) {
  int kc = 8 * kRowsNTH / n;
  return kc < 1 ? 1 : kc;
}

cudaError_t launch_rows_fused(const FusedArgs& a, bool fuse_fft, bool fuse_ifft, cudaStream_t s) {
  switch (a.n) {
    case 64: return launch_rf_n<64>(a, fuse_fft, fuse_ifft, s);
    case 128: return launch_rf_n<128>(a, fuse_fft, fuse_ifft, s);
    case 256: return launch_rf_n<256>(a, fuse_fft, fuse_ifft, s);
    case 512: return launch_rf_n<512>(a, fuse_fft, fuse_ifft, s);
    case 1024: return launch_rf_n<1024>(a, fuse_fft, fuse_ifft, s);
    case 2048: return launch_rf_n<2048>(a, fuse_fft, fuse_ifft, s);
    case 4096: return launch_rf_n<4096>(a, fuse_fft, fuse_ifft, s);
  }
  return cudaErrorNotSupported;
}

template <int N, int DIR>
static cudaError_t launch_rows_t(const float2* in, int64_t is, float2* out, int64_t os, int64_t P, int keep,
                                 int src_len, float scale, const float2* tw, cudaStream_t s) {
  size_t smem = rows_fft_smem<N>();
  cudaError_t e = cudaFuncSetAttribute(rows_fft_kernel<N, DIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t nblk = (P + RowsGeo<N>::KC - 1) / RowsGeo<N>::KC;
  const int grid = (int)(nblk < sm_count() ? nblk : sm_count());
  if (grid < 1) return cudaSuccess;
  rows_fft_kernel<N, DIR><<<grid, kRowsNTH, smem, s>>>(in, is, out, os, P, keep, src_len, scale, tw);
  ++g_launches;
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch_rows_n(int dir, const float2* in, int64_t is, float2* out, int64_t os, int64_t P, int keep,
                                 int src_len, float scale, const float2* tw, cudaStream_t s) {
  return dir < 0 ? launch_rows_t<N, -1>(in, is, out, os, P, keep, src_len, scale, tw, s)
                 : launch_rows_t<N, 1>(in, is, out, os, P, keep, src_len, scale, tw, s);
}

cudaError_t launch_rows_fft(int n, int dir, const float2* in, int64_t in_stride, float2* out, int64_t out_stride,
                            int64_t P, int keep, int src_len, float scale, const float2* tw, cudaStream_t s) {
  switch (n) {
    case 64: return launch_rows_n<64>(dir, in, in_stride, out, out_stride, P, keep, src_len, scale, tw, s);
    case 128: return launch_rows_n<128>(dir, in, in_stride, out, out_stride, P, keep, src_len, scale, tw, s);
    case 256: return launch_rows_n<256>(dir, in, in_stride, out, out_stride, P, keep, src_len, scale, tw, s);
    case 512: return launch_rows_n<512>(dir, in, in_stride, out, out_stride, P, keep, src_len, scale, tw, s);
    case 1024: return launch_rows_n<1024>(dir, in, in_stride, out, out_stride, P, keep, src_len, scale, tw, s);
    case 2048: return launch_rows_n<2048>(dir, in, in_stride, out, out_stride, P, keep, src_len, scale, tw, s);
    case 4096: return launch_rows_n<4096>(dir, in, in_stride, out, out_stride, P, keep, src_len, scale, tw, s);
  }
  return cudaErrorNotSupported;
}

}  // namespace tfno
