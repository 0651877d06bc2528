// Geometry of the warp-register row FFTs (N = L*L, one row per L lanes) shared by
// warpfft.cu and warpfft_fwd.cu, and the forward launcher the latter exports.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tfno {

template <int L>
struct WfGeo {
  static constexpr int N = L * L;
  static constexpr int NTH = 256;
  static constexpr int ROWS = NTH / L;        // rows in flight per CTA pass
  static constexpr int TSTR = L + 1;          // padded transpose stride (complex)
  static constexpr size_t smem_bytes() {
    return sizeof(float2) * ((size_t)L + (size_t)L * L + (size_t)ROWS * L * TSTR);
  }
};

// unfused truncating forward row FFT, N = L*L (L = 16 / 32), kp = ceil(keep / L) <= 8
cudaError_t launch_warp_fft_fwd_rows(int L, int kp, const float2* in, int64_t is, float2* out, int64_t os,
                                     int64_t P, int keep, const float2* tw, cudaStream_t s);

}  // namespace tfno
