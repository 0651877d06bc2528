// Real-field FNO block pieces (extension beyond the reference):
// R2C input expansion, the half-spectrum weights that turn the first-keep complex
// inverse into irfft, and the block epilogue Re(.) + bypass + bias -> activation.
//
// The real layer is composed on the spectrum ABI (paper_2504_11681_b200/realfield.py):
//   X = DFT_trunc(x + 0i)               (first kx rows / ky columns == rfft2(x)[:kx, :ky])
//   C = (c_k X) W,  c_0 = 1, c_k = 2 for 0 < k < dy/2, c_{dy/2} = 1
//   y = Re(iDFT_pad(C))                  (== irfft2(X W, s=(dx, dy)) for ky <= dy/2 + 1)
// because irfft over y of bins 0..ky-1 is Re(sum_k c_k Z_k e^{2 pi i k t / dy}) / dy.
// All three kernels are HBM-bound streams: 16-byte accesses, grid = SMs x 8 CTAs, grid-stride.

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/turbofno.h"
#include "kernels.cuh"

namespace tfno {
namespace {

inline int grid_for(int64_t work) {
  const int sms = tfno::device_sms();
  int64_t g = (work + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// z[i] = (x[i], 0); 4 reals -> 4 complex per thread step
__global__ void real_to_complex_kernel(const float* __restrict__ x, float2* __restrict__ z, int64_t n) {
  const int64_t n4 = n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float4* z4 = reinterpret_cast<float4*>(z);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = __ldcs(&x4[i]);
    __stcs(&z4[2 * i], make_float4(v.x, 0.f, v.y, 0.f));
    __stcs(&z4[2 * i + 1], make_float4(v.z, 0.f, v.w, 0.f));
  }
  for (int64_t i = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    z[i] = make_float2(x[i], 0.f);
}

// modes[r][k] *= c_k (k < ky), c_k = 2 for 0 < k and 2k < dy, else 1
__global__ void half_spectrum_weight_kernel(float2* __restrict__ m, int64_t total, int ky, int dy) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % ky);
    if (k > 0 && 2 * k < dy) {
      const float2 v = m[i];
      m[i] = make_float2(2.f * v.x, 2.f * v.y);
    }
  }
}

__device__ __forceinline__ float activate(float v, int act) {
  if (act == TFNO_ACT_RELU) return fmaxf(v, 0.f);
  if (act == TFNO_ACT_GELU) return 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
  return v;
}

// out[b][n][p] = act(Re z[b][n][p] + bypass[b][n][p] + bias[n]); P % 4 == 0 path (16-byte accesses)
__global__ void real_epilogue4_kernel(const float2* __restrict__ z, const float* __restrict__ bypass,
                                      const float* __restrict__ bias, int64_t total4, int N, int64_t P4, int act,
                                      float* __restrict__ out) {
  const float4* z4 = reinterpret_cast<const float4*>(z);
  const float4* b4 = reinterpret_cast<const float4*>(bypass);
  float4* o4 = reinterpret_cast<float4*>(out);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = __ldcs(&z4[2 * i]), c = __ldcs(&z4[2 * i + 1]);
    float4 v = make_float4(a.x, a.z, c.x, c.z);
    if (bypass) {
      const float4 q = __ldcs(&b4[i]);
      v.x += q.x, v.y += q.y, v.z += q.z, v.w += q.w;
    }
    if (bias) {
      const float s = __ldg(&bias[(i / P4) % N]);
      v.x += s, v.y += s, v.z += s, v.w += s;
    }
    v = make_float4(activate(v.x, act), activate(v.y, act), activate(v.z, act), activate(v.w, act));
    __stcs(&o4[i], v);
  }
}

__global__ void real_epilogue_kernel(const float2* __restrict__ z, const float* __restrict__ bypass,
                                     const float* __restrict__ bias, int64_t total, int N, int64_t P, int act,
                                     float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    float v = z[i].x;
    if (bypass) v += bypass[i];
    if (bias) v += bias[(i / P) % N];
    out[i] = activate(v, act);
  }
}

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }
inline int status(cudaError_t e) { return e == cudaSuccess ? TFNO_OK : TFNO_ECUDA; }

}  // namespace
}  // namespace tfno

using namespace tfno;

extern "C" {

int tfno_real_to_complex(const float* x, void* z, int64_t n, void* stream) {
  if (n < 0 || (n && (!x || !z))) return TFNO_EINVAL;
  if (n == 0) return TFNO_OK;
  if (!aligned16(x) || !aligned16(z)) return TFNO_EINVAL;
  real_to_complex_kernel<<<grid_for((n + 3) / 4), 256, 0, (cudaStream_t)stream>>>(x, (float2*)z, n);
  ++g_launches;
  return status(cudaGetLastError());
}

int tfno_half_spectrum_weight(void* modes, int64_t rows, int ky, int dy, void* stream) {
  if (rows < 0 || ky < 1 || dy < 1 || ky > dy / 2 + 1 || (rows && !modes)) return TFNO_EINVAL;
  if (rows == 0) return TFNO_OK;
  const int64_t total = rows * ky;
  half_spectrum_weight_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>((float2*)modes, total, ky, dy);
  ++g_launches;
  return status(cudaGetLastError());
}

int tfno_real_epilogue(const void* z, const float* bypass, const float* bias, int64_t batch, int N, int64_t P,
                       int activation, float* out, void* stream) {
  if (batch < 0 || N < 0 || P < 0 || activation < TFNO_ACT_NONE || activation > TFNO_ACT_GELU) return TFNO_EINVAL;
  const int64_t total = batch * N * P;
  if (total == 0) return TFNO_OK;
  if (!z || !out) return TFNO_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (P % 4 == 0 && aligned16(z) && aligned16(out) && (!bypass || aligned16(bypass)))
    real_epilogue4_kernel<<<grid_for(total / 4), 256, 0, s>>>((const float2*)z, bypass, bias, total / 4, N, P / 4,
                                                             activation, out);
  else
    real_epilogue_kernel<<<grid_for(total), 256, 0, s>>>((const float2*)z, bypass, bias, total, N, P, activation,
                                                         out);
  ++g_launches;
  return status(cudaGetLastError());
}

}  // extern "C"
