// Compile-time-specialised row kernels (rows1d.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace tfno {
bool rows_supported(int n);                               // 64 <= n <= 4096, power of two
int rows_chunk(int n);                                    // rows per k-chunk (KC)
size_t rows_fused_smem_bytes(int n, int keep, int NT);
cudaError_t launch_rows_fused(const FusedArgs& a, bool fuse_fft, bool fuse_ifft, cudaStream_t s);
cudaError_t launch_rows_fft(int n, int dir, const float2* in, int64_t in_stride, float2* out, int64_t out_stride,
                            int64_t P, int keep, int src_len, float scale, const float2* tw, cudaStream_t s);
}  // namespace tfno
