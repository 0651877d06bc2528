// Minimal reproductions of the two hand-off patterns compute-sanitizer racecheck
// flags in the layer kernels (profiles/r02/sanitizer/):
//   1. TMA bulk copy (cp.async.bulk, async proxy) into shared memory, completion
//      tracked by an mbarrier (expect_tx / complete_tx); consumers read the tile
//      after mbarrier.try_wait.parity -- the ring slots of plane_fwd2d / plane_fwd_g /
//      plane_invmix_g and the row slots of fused1d.
//   2. Generic stores to shared memory by producer warps, mbarrier.arrive (release)
//      by them, consumer warps read after mbarrier.try_wait (acquire) -- the A-chunk
//      and C-tile hand-offs of fused1d between its FFT and GEMM warps.
// Both are ordered by the PTX memory model (complete_tx / arrive have release
// semantics, try_wait acquire).  If racecheck reports hazards on THIS kernel, its
// reports on the same patterns in the layer kernels are the same false positive.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o racecheck_mbar_probe racecheck_mbar_probe.cu
//   compute-sanitizer --tool racecheck ./racecheck_mbar_probe
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const float* __restrict__ src, float* __restrict__ out, int rounds) {
  __shared__ __align__(128) float tile[2][1024];
  __shared__ __align__(8) uint64_t full[2], done[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&done[s])), "r"(blockDim.x / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float acc = 0.f;
  for (int r = 0; r < rounds; ++r) {
    const int s = r & 1;
    const uint32_t ph = (uint32_t)((r >> 1) & 1);
    if (tid == 0) {
      if (r >= 2) {  // slot reuse: every warp released it (pattern 2 in reverse)
        asm volatile("{\n\t.reg .pred p;\nW0_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W0_%=;\n}"
                     ::"r"(sa(&done[s])), "r"(ph ^ 1u) : "memory");
      }
      if (r & 2) {  // pattern 1: TMA bulk copy, completion on the mbarrier
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(4096) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];"
                     ::"r"(sa(tile[s])), "l"(src + 1024 * r), "r"(sa(&full[s])) : "memory");
      } else {  // pattern 2: generic stores, then a releasing arrive
        for (int i = 0; i < 1024; ++i) tile[s][i] = src[1024 * r + i];
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sa(&full[s])) : "memory");
      }
    }
    asm volatile("{\n\t.reg .pred p;\nW1_%=:\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t@!p bra W1_%=;\n}"
                 ::"r"(sa(&full[s])), "r"(ph) : "memory");
    for (int i = tid; i < 1024; i += blockDim.x) acc += tile[s][i];
    __syncwarp();
    if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&done[s])) : "memory");
  }
  out[blockIdx.x * blockDim.x + tid] = acc;
}

int main() {
  const int rounds = 8, threads = 128;
  float *src, *out;
  cudaMalloc(&src, sizeof(float) * 1024 * rounds);
  cudaMalloc(&out, sizeof(float) * threads);
  float h[1024 * rounds];
  for (int i = 0; i < 1024 * rounds; ++i) h[i] = 1.0f;
  cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice);
  probe<<<1, threads>>>(src, out, rounds);
  float o[threads];
  cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
  double tot = 0;
  for (int i = 0; i < threads; ++i) tot += o[i];
  printf("probe sum %.0f (expect %d) %s\n", tot, 1024 * rounds, cudaGetErrorString(cudaGetLastError()));
  return tot == 1024.0 * rounds ? 0 : 1;
}
