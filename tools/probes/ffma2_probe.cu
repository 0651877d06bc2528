// Throughput probe: scalar FFMA vs packed FFMA2 / FADD2 (sm_100a) — does the
// packed form double FP32 work per issue slot?  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
template <int MODE>
__global__ void k(float* out, int iters, float s) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
  unsigned long long p[8];
  for (int i = 0; i < 8; ++i) p[i] = f2u(make_float2(a[2 * i], a[2 * i + 1]));
  const unsigned long long ss = f2u(make_float2(s, s));
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 0.5f);
    } else if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[i]) : "l"(ss));
    } else if (MODE == 2) {
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(ss));
    } else {
      // FFMA2 with a broadcast operand: (a, a) * p + p
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float bx = a[i];
        asm volatile("{.reg .b64 t; mov.b64 t, {%1, %1}; fma.rn.f32x2 %0, t, %0, %2;}" : "+l"(p[i]) : "f"(bx), "l"(ss));
      }
    }
  }
  float r = 0.f;
  for (int i = 0; i < 16; ++i) r += a[i];
  for (int i = 0; i < 8; ++i) { float2 v = u2f(p[i]); r += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 20000;
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<148 * 8, 256>>>(out, iters, 0.999f);
      if (mode == 1) k<1><<<148 * 8, 256>>>(out, iters, 0.999f);
      if (mode == 2) k<2><<<148 * 8, 256>>>(out, iters, 0.999f);
      if (mode == 3) k<3><<<148 * 8, 256>>>(out, iters, 0.999f);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double flops = 148.0 * 8 * 256 * iters * 16 * (mode == 2 ? 1 : 2);
      if (rep) printf("%s: %.3f ms  %.1f TFLOP/s (fp32 lane-ops incl. FMA=2)\n",
                      mode == 0 ? "FFMA scalar" : mode == 1 ? "FFMA2 packed" : mode == 2 ? "FADD2 packed" : "FFMA2 bcast", ms, flops / ms / 1e9);
    }
  }
  return 0;
}
