// Latency-bound small 1D layers (BASELINE configs[0] = C1: 16 batch elements,
// 64 -> 64 channels, N = 128, keep 32): ONE kernel, no cluster, no
// cross-CTA hand-off.  CTA (b, g) owns output channels [8g, 8g + 8) of batch
// element b and recomputes the (cheap) truncated forward FFTs of all H input
// rows of b -- the 8 CTAs of one b re-read x[b] from L2 -- so every CTA runs
// load -> FFT -> mix -> padded iFFT -> store with only __syncthreads between
// the phases (reference semantics: pipeline.py:185-206 + 236-275, rank 1).
//
//   phase 1  16 row teams of 16 lanes: row = 16 lanes x 8 values (x[t + 16 j]),
//            DFT8, twiddle w_128^{t k1}, XOR-swizzled 8 x 16 transpose, DFT8 over
//            t' and a one-shuffle sum of the two half sequences -> the first
//            16*KP bins of the row into A[h][q] (bins q >= keep written as 0)
//   phase 2  C[g][q] = sum_h A[h][q] W[h][8g + g'] (h ascending, FP32 FMA)
//   phase 3  8 teams: zero-padded inverse of the CTA's 8 output rows, x 1/N,
//            streaming stores
// Only x (1 MiB at C1, read once from HBM), W and y touch global memory.
// Launched with programmatic dependent launch: the twiddle prologue of layer
// i+1 overlaps layer i.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace tfno {

namespace {

constexpr int kTN = 128;     // row length
constexpr int kTL = 16;      // lanes per row team
constexpr int kTTeams = 16;  // 256 threads
constexpr int kTNG = 8;      // output channels per CTA

// 8 x 16 tile [k1][t], column XOR-swizzled by 2*k1 (conflict-free row writes and
// (k1 = lane/2, t = lane%2 + 2t') reads) -- the fused 1D kernel's N = 128 layout
__device__ __forceinline__ int tsw(int r, int c) { return r * 16 + (c ^ (2 * r)); }

template <int KP>
__global__ void __launch_bounds__(256, 1)
    tiny1d_kernel(const float2* __restrict__ x, const float2* __restrict__ W, float2* __restrict__ y, int H, int N,
                  int keep, const float2* __restrict__ twg, float inv_scale) {
  constexpr int K2 = 2 * KP, KT = 8 * K2;  // stored bins per row: q = k1 + 8 k2 < KT
  extern __shared__ __align__(16) float2 sm[];
  float2* As = sm;                      // [H][KT]
  float2* Wt = As + (size_t)H * KT;     // [H][8]
  float2* Cs = Wt + (size_t)H * kTNG;   // [8][KT]
  float2* tr = Cs + kTNG * KT;          // [16 teams][128]
  float2* twN = tr + kTTeams * kTN;     // [k1][t] = w_128^{t k1}
  float2* twL = twN + kTN;              // w_16^k

  const int tid = threadIdx.x, team = tid / kTL, lane = tid % kTL;
  const unsigned tmask = 0xffffu << (16 * (team & 1));
  const int b = blockIdx.y, n0 = blockIdx.x * kTNG;
  for (int k = tid; k < kTL; k += 256) twL[k] = __ldg(&twg[(size_t)k * (TFNO_TW_MAX / kTL)]);
  for (int i = tid; i < kTN; i += 256) {
    const int k1 = i / kTL, t = i % kTL;
    twN[i] = __ldg(&twg[(size_t)((t * k1) % kTN) * (TFNO_TW_MAX / kTN)]);
  }
  pdl_wait();  // x / W are read, y written, only once the previous kernel has completed
  pdl_launch_dependents();

  // W columns of this CTA (zeros past N)
  for (int i = tid; i < H * kTNG; i += 256) {
    const int h = i / kTNG, g = i % kTNG;
    Wt[i] = (n0 + g < N) ? __ldg(&W[(int64_t)h * N + n0 + g]) : make_float2(0.f, 0.f);
  }
  float2* trr = tr + team * kTN;
  const int k1 = lane >> 1, hf = lane & 1;
  // ---- phase 1: truncated forward FFT of the rows h = team + 16 r, four rows in flight
  constexpr int RB = 4;
  for (int h0 = team; h0 < H; h0 += kTTeams * RB) {
    float2 v[RB][8];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int h = h0 + kTTeams * r;
      const float2* row = x + ((int64_t)b * H + h) * kTN;
#pragma unroll
      for (int j = 0; j < 8; ++j) v[r][j] = h < H ? __ldcs(row + lane + kTL * j) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int h = h0 + kTTeams * r;
      if (h >= H) break;  // uniform across the team
      float2 u[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) u[j] = v[r][j];
      dft8<-1>(u);
#pragma unroll
      for (int kk = 1; kk < 8; ++kk) u[kk] = cmul(u[kk], twN[kk * kTL + lane]);
      __syncwarp(tmask);  // the previous row's transpose reads are done
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) trr[tsw(kk, lane)] = u[kk];
      __syncwarp(tmask);
#pragma unroll
      for (int t2 = 0; t2 < 8; ++t2) u[t2] = trr[tsw(k1, hf + 2 * t2)];
      dft8<-1>(u);
#pragma unroll
      for (int k2 = 1; k2 < K2; ++k2)
        if (hf) u[k2] = cmul(u[k2], twL[k2]);
#pragma unroll
      for (int k2 = 0; k2 < K2; ++k2) {
        const float2 p = make_float2(__shfl_xor_sync(tmask, u[k2].x, 1), __shfl_xor_sync(tmask, u[k2].y, 1));
        u[k2] = cadd(u[k2], p);
      }
#pragma unroll
      for (int k2 = 0; k2 < K2; ++k2) {
        if ((k2 & 1) != hf) continue;
        const int q = k1 + 8 * k2;
        As[(size_t)h * KT + q] = q < keep ? u[k2] : make_float2(0.f, 0.f);
      }
    }
  }
  __syncthreads();
  // ---- phase 2: C[g][q] = sum_h A[h][q] W[h][g], h ascending
  for (int o = tid; o < kTNG * KT; o += 256) {
    const int g = o / KT, q = o % KT;
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int h = 0; h < H; ++h) cmac(acc, As[(size_t)h * KT + q], Wt[h * kTNG + g]);
    Cs[o] = acc;
  }
  __syncthreads();
  // ---- phase 3: zero-padded inverse of output rows n0 + team (teams 0..7)
  if (team < kTNG && n0 + team < N) {
    const float2* cr = Cs + team * KT;
    float2 z[8];
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) {
      const int q = k1 + 8 * k2;
      z[k2] = (k2 < K2 && q < keep) ? cr[q] : make_float2(0.f, 0.f);
      if (k2 < K2 && k2 && hf) z[k2] = cmul(z[k2], conjf2(twL[k2]));
    }
    dft8<1>(z);
#pragma unroll
    for (int t2 = 0; t2 < 8; ++t2) {
      const int t = hf + 2 * t2;
      trr[tsw(k1, t)] = k1 ? cmul(z[t2], conjf2(twN[k1 * kTL + t])) : z[t2];
    }
    __syncwarp(tmask);
#pragma unroll
    for (int r = 0; r < 8; ++r) z[r] = trr[tsw(r, lane)];
    dft8<1>(z);
    float2* dst = y + ((int64_t)b * N + n0 + team) * kTN;
#pragma unroll
    for (int j = 0; j < 8; ++j) __stcs(dst + lane + kTL * j, cscale(z[j], inv_scale));
  }
}

template <int KP>
size_t tiny_smem(int H) {
  constexpr int KT = 16 * KP;
  return sizeof(float2) * ((size_t)H * KT + (size_t)H * kTNG + kTNG * KT + kTTeams * kTN + kTN + kTL);
}

template <int KP>
cudaError_t launch_tiny_t(const float2* x, const float2* W, float2* y, int B, int H, int N, int keep,
                          const float2* tw, cudaStream_t s) {
  const size_t smem = tiny_smem<KP>(H);
  auto kern = tiny1d_kernel<KP>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)((N + kTNG - 1) / kTNG), (unsigned)B);
  e = launch_pdl1(kern, grid, dim3(256), smem, s, x, W, y, H, N, keep, tw, 1.0f / kTN);
  if (e != cudaSuccess) return e;
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace

bool tiny1d_supported(int n, int keep, int B, int H, int N) {
  if (n != kTN || keep < 1 || keep > 64 || H < 1 || N < 1 || B < 1 || B > 65535) return false;
  const int kp = (keep + 15) / 16;
  return sizeof(float2) * ((size_t)H * 16 * kp + (size_t)H * kTNG + kTNG * 16 * kp + kTTeams * kTN + kTN + kTL) <=
         200 * 1024;
}

cudaError_t launch_tiny1d(const float2* x, const float2* W, float2* y, int B, int H, int N, int keep,
                          const float2* tw, cudaStream_t s) {
  switch ((keep + 15) / 16) {
    case 1: return launch_tiny_t<1>(x, W, y, B, H, N, keep, tw, s);
    case 2: return launch_tiny_t<2>(x, W, y, B, H, N, keep, tw, s);
    case 3: return launch_tiny_t<3>(x, W, y, B, H, N, keep, tw, s);
    case 4: return launch_tiny_t<4>(x, W, y, B, H, N, keep, tw, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace tfno
