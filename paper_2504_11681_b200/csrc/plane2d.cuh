// Per-plane 2D Fourier-layer kernels (rank 2, fully_fused fast path).
#pragma once
#include <cuda_runtime.h>

#include "../../include/turbofno.h"

namespace tfno {
bool plane2d_supported(const tfno_cfg* c);
// mode count per plane of the A / C workspace tensors (kx*ky, or KP^2 on the generic kernels)
int64_t plane2d_modes(const tfno_cfg* c);
// the natural [kx][ky] mode layout of the spectrum API is what the plane kernels produce
bool plane2d_spectrum_ok(const tfno_cfg* c);
int plane_g_kp(const tfno_cfg* c);
// rank-2 FP32 layer as plane-fft2d | plane-mix-ifft2d (channel mix fused into the inverse)
bool plane2d_fusedmix(const tfno_cfg* c, int prec, int mode = TFNO_FULLY_FUSED);
// complex elements of the C workspace region: the full [B][N][modes] tensor, or
// the fused kernel's per-CTA two-task ring
int64_t plane2d_c_elems(const tfno_cfg* c, int prec, int mode = TFNO_FULLY_FUSED);
cudaError_t launch_plane2d_layer(const tfno_cfg* c, const float2* x, const float2* w, float2* y, float2* A,
                                 float2* Cm, const float2* tw, int prec, void* wimg, int wimg_ready,
                                 cudaStream_t s, void (*mark)(cudaStream_t), int mode = TFNO_FULLY_FUSED);
// natural-order mode tensors [planes][kx][ky] (spectrum API); inverse scaled by `scale`
cudaError_t launch_plane2d_fwd(const tfno_cfg* c, const float2* x, float2* modes, const float2* tw, cudaStream_t s);
cudaError_t launch_plane2d_inv(const tfno_cfg* c, const float2* modes, float2* y, float scale, const float2* tw,
                               cudaStream_t s);
}  // namespace tfno
