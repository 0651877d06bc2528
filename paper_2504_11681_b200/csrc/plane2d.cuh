// Per-plane 2D Fourier-layer kernels (rank 2, fully_fused fast path).
#pragma once
#include <cuda_runtime.h>

#include "../../include/turbofno.h"

namespace tfno {
bool plane2d_supported(const tfno_cfg* c);
cudaError_t launch_plane2d_layer(const tfno_cfg* c, const float2* x, const float2* w, float2* y, float2* A,
                                 float2* Cm, const float2* tw, int prec, cudaStream_t s,
                                 void (*mark)(cudaStream_t));
}  // namespace tfno
