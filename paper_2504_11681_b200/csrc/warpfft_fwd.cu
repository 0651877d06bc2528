// Unfused truncating forward row FFT for N = 256 / 1024 (warp-register, one row per L lanes:
// DFT_L over j in registers, twiddle w_N^{t k1}, padded smem transpose, first KP outputs of the
// second DFT_L).  This translation unit is compiled with the scalar complex primitives
// (TFNO_SCALAR_COMPLEX): for this kernel they measured faster than the packed f32x2 form
// (N1024 forward 0.422 -> 0.379 ms at H256 B1024, neutral at N = 256), while the other
// warpfft.cu kernels (inverse, team FFTs) are faster packed (profiles/r01/plane_loop_ab.txt).
// -DTFNO_WF_FWD_PACKED restores the packed form for A/B.
#ifndef TFNO_WF_FWD_PACKED
#ifndef TFNO_SCALAR_COMPLEX
#define TFNO_SCALAR_COMPLEX
#endif
#endif

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.cuh"
#include "warpfft.cuh"
#include "wf_dft.cuh"

namespace tfno {

// forward: rows [P][src stride] -> out [P][keep] (out stride), src_len = N
template <int L, int KP>
__global__ void __launch_bounds__(WfGeo<L>::NTH) warp_fft_fwd_kernel(const float2* __restrict__ in,
                                                                   int64_t in_stride, float2* __restrict__ out,
                                                                   int64_t out_stride, int64_t P, int keep,
                                                                   const float2* __restrict__ twg) {
  using G = WfGeo<L>;
  constexpr int N = G::N;
  extern __shared__ __align__(16) float2 sm[];
  float2* twL = sm;                 // w_L^k
  float2* twN = twL + L;            // [k1][t] = w_N^{t k1}
  float2* tr = twN + L * L;         // ROWS x L x TSTR
  const int tid = threadIdx.x, lane = tid % L, rloc = tid / L;
  const unsigned tmask = L == 32 ? 0xffffffffu : (0xffffu << (16 * (rloc & 1)));
  for (int k = tid; k < L; k += G::NTH) twL[k] = __ldg(&twg[(size_t)k * (TFNO_TW_MAX / L)]);
  for (int i = tid; i < L * L; i += G::NTH) {
    const int k1 = i / L, t = i % L;
    twN[i] = __ldg(&twg[(size_t)((t * k1) % N) * (TFNO_TW_MAX / N)]);
  }
  __syncthreads();
  float2* trr = tr + rloc * L * G::TSTR;
  for (int64_t row = (int64_t)blockIdx.x * G::ROWS + rloc; row < P; row += (int64_t)gridDim.x * G::ROWS) {
    const float2* src = in + row * in_stride;
    float2 v[L];
#pragma unroll
    for (int j = 0; j < L; ++j) v[j] = __ldg(&src[lane + L * j]);
    wf::dftL<L, -1>(v, twL);
#pragma unroll
    for (int k1 = 1; k1 < L; ++k1) v[k1] = cmul(v[k1], twN[k1 * L + lane]);  // consecutive lanes
    __syncwarp(tmask);
#pragma unroll
    for (int k1 = 0; k1 < L; ++k1) trr[k1 * G::TSTR + lane] = v[k1];
    __syncwarp(tmask);
    // lane = k1 now: gather Y_t[k1] over t, first KP outputs of DFT_L over t
#pragma unroll
    for (int t = 0; t < L; ++t) v[t] = trr[lane * G::TSTR + t];
    float2 o[KP];
    wf::dftL_first<L, KP>(v, o, twL);
    float2* dst = out + row * out_stride;
#pragma unroll
    for (int k2 = 0; k2 < KP; ++k2) {
      const int k = lane + L * k2;
      if (k < keep) dst[k] = o[k2];
    }
  }
}

template <int L, int KP>
static cudaError_t launch_wf_fwd(const float2* in, int64_t is, float2* out, int64_t os, int64_t P, int keep,
                                 const float2* tw, cudaStream_t s) {
  using G = WfGeo<L>;
  const size_t smem = G::smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(warp_fft_fwd_kernel<L, KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = (P + G::ROWS - 1) / G::ROWS;
  const int grid = (int)(blocks < (int64_t)sms * 8 ? blocks : (int64_t)sms * 8);
  warp_fft_fwd_kernel<L, KP><<<grid, G::NTH, smem, s>>>(in, is, out, os, P, keep, tw);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_warp_fft_fwd_rows(int L, int kp, const float2* in, int64_t is, float2* out, int64_t os,
                                     int64_t P, int keep, const float2* tw, cudaStream_t s) {
#define WF_CASE(LL, KK) \
  if (L == LL && kp == KK) return launch_wf_fwd<LL, KK>(in, is, out, os, P, keep, tw, s);
  WF_CASE(16, 1) WF_CASE(16, 2) WF_CASE(16, 3) WF_CASE(16, 4) WF_CASE(16, 5) WF_CASE(16, 6) WF_CASE(16, 7)
  WF_CASE(16, 8)
  WF_CASE(32, 1) WF_CASE(32, 2) WF_CASE(32, 3) WF_CASE(32, 4) WF_CASE(32, 5) WF_CASE(32, 6) WF_CASE(32, 7)
  WF_CASE(32, 8)
#undef WF_CASE
  return cudaErrorNotSupported;
}

}  // namespace tfno
