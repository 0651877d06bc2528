#include "plane2d.cuh"

namespace tfno {
bool plane2d_supported(const tfno_cfg*) { return false; }
cudaError_t launch_plane2d_layer(const tfno_cfg*, const float2*, const float2*, float2*, float2*, float2*,
                                 const float2*, int, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace tfno
