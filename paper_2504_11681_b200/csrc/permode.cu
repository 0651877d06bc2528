// Per-mode channel mix (extension beyond the reference):
//   C[b][n][q] = alpha * sum_h A[b][h][q] * W[h][n][q]      (einsum bhq,hnq->bnq)
// on the natural layouts the spectrum kernels produce and consume — A is the
// truncated spectrum [B][H][kx*ky], W the user's [H][N][kx][ky] weights, C the
// modes the padded inverse reads — so the per-mode layer needs no mode-major
// permute copies of A, W or C (paper_2504_11681_b200/permode.py).
//
// The mode index q is the fastest axis of all three tensors, so a warp's 32
// lanes own 32 consecutive modes: every global row access is one coalesced
// 256-byte segment and every shared-memory read is conflict-free.  A CTA owns
// a 32-mode x 16-batch x 16-channel tile (8 warps, each 8 b x 4 n accumulators
// per lane) and streams H in chunks of 4 through a 3-stage cp.async ring (no
// prefetch registers: two CTAs per SM).  Consecutive CTAs share one mode
// tile, so the A and W slices of the resident CTAs stay in L2 and HBM sees A,
// W and C about once; the kernel is bound by the FP32 pipe (scalar 4-FFMA MAC,
// like the mode CGEMM).

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace tfno {
namespace {

constexpr int PM_Q = 32, PM_BT = 16, PM_NT = 16, PM_HC = 4, PM_S = 3;
constexpr int PM_RA = PM_HC * PM_BT / 8, PM_RW = PM_HC * PM_NT / 8;  // rows per warp per stage (8 + 8)
constexpr int PM_STAGE = PM_HC * (PM_BT + PM_NT) * PM_Q;             // complex per stage (32 KiB)

// 8-byte cp.async, zero-filled when !ok (src_size 0)
__device__ __forceinline__ void cp_async8(float2* sdst, const float2* gsrc, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(gsrc), "r"(ok ? 8 : 0) : "memory");
}

// stage rows are interleaved over the 8 warps: warp w copies A rows (h = i / 2, b = 8 (i & 1) + w)
// and W rows (h = i / 2, n = 8 (i & 1) + w), i compile-time, so every address is a base pointer
// plus constant multiples of H*MQ / N*MQ / MQ
__global__ void __launch_bounds__(256, 2)
    permode_mix_kernel(const float2* __restrict__ A, const float2* __restrict__ W, float2* __restrict__ C,
                       int64_t B, int64_t H, int64_t N, int64_t MQ, float alpha, int ntn) {
  extern __shared__ __align__(16) float2 pm_smem[];  // PM_S x { As[HC][BT][32], Ws[HC][NT][32] }
  pdl_wait();
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n0 = (int64_t)(blockIdx.x % ntn) * PM_NT, b0 = (int64_t)(blockIdx.x / ntn) * PM_BT;
  const int64_t q = (int64_t)blockIdx.y * PM_Q + lane;
  const bool q_ok = q < MQ;
  const float2* Ab = A + ((b0 + warp) * H) * MQ + (q_ok ? q : 0);  // row (h, b0 + warp)
  const float2* Wb = W + (n0 + warp) * MQ + (q_ok ? q : 0);        // row (h, n0 + warp)
  const int64_t a_b8 = 8 * H * MQ, w_h = N * MQ, w_n8 = 8 * MQ;
  const bool b_ok0 = q_ok && b0 + warp < B, b_ok1 = q_ok && b0 + warp + 8 < B;
  const bool n_ok0 = q_ok && n0 + warp < N, n_ok1 = q_ok && n0 + warp + 8 < N;
  const int64_t nchunks = (H + PM_HC - 1) / PM_HC;
  auto issue = [&](int64_t c) {  // chunk c -> stage c % PM_S
    if (c < nchunks) {
      float2* As = pm_smem + (c % PM_S) * PM_STAGE;
      float2* Ws = As + PM_HC * PM_BT * PM_Q;
      const int64_t h0 = c * PM_HC;
#pragma unroll
      for (int i = 0; i < PM_RA; ++i) {
        const int64_t h = h0 + (i >> 1);
        const bool ok = h < H && ((i & 1) ? b_ok1 : b_ok0);
        cp_async8(&As[((i >> 1) * PM_BT + warp + 8 * (i & 1)) * PM_Q + lane],
                  ok ? Ab + (i & 1) * a_b8 + h * MQ : A, ok);
      }
#pragma unroll
      for (int i = 0; i < PM_RW; ++i) {
        const int64_t h = h0 + (i >> 1);
        const bool ok = h < H && ((i & 1) ? n_ok1 : n_ok0);
        cp_async8(&Ws[((i >> 1) * PM_NT + warp + 8 * (i & 1)) * PM_Q + lane],
                  ok ? Wb + h * w_h + (i & 1) * w_n8 : W, ok);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // (empty groups keep the count uniform)
  };
  // compute: warp = (b half, n quarter): 8 b x 4 n accumulators per lane
  const int bb = (warp >> 2) * 8, nb = (warp & 3) * 4;
  float2 acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < PM_S - 1; ++c) issue(c);
  for (int64_t c = 0; c < nchunks; ++c) {
    asm volatile("cp.async.wait_group %0;" ::"n"(PM_S - 2) : "memory");  // chunk c landed (this thread)
    __syncthreads();  // ... for every thread; and stage (c - 1) % S is free for chunk c + S - 1
    issue(c + PM_S - 1);
    const float2* As = pm_smem + (c % PM_S) * PM_STAGE;
    const float2* Ws = As + PM_HC * PM_BT * PM_Q;
#pragma unroll
    for (int hh = 0; hh < PM_HC; ++hh) {
      float2 av[8], wv[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) av[i] = As[(hh * PM_BT + bb + i) * PM_Q + lane];
#pragma unroll
      for (int j = 0; j < 4; ++j) wv[j] = Ws[(hh * PM_NT + nb + j) * PM_Q + lane];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) cmac_s(acc[i][j], av[i], wv[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (!q_ok) return;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t b = b0 + bb + i;
    if (b >= B) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + nb + j;
      if (n < N) C[(b * N + n) * MQ + q] = cscale(acc[i][j], alpha);
    }
  }
}

}  // namespace

cudaError_t launch_permode_mix(const float2* A, const float2* W, float2* C, int64_t B, int64_t H, int64_t N,
                               int64_t MQ, float alpha, cudaStream_t s) {
  const int64_t ntn = (N + PM_NT - 1) / PM_NT, ntb = (B + PM_BT - 1) / PM_BT, ntq = (MQ + PM_Q - 1) / PM_Q;
  if (ntn * ntb > INT32_MAX || ntq > 65535) return cudaErrorInvalidValue;
  constexpr size_t smem = (size_t)PM_S * PM_STAGE * sizeof(float2);  // 96 KiB: 2 CTAs per SM
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(permode_mix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured_dev = dev;
  }
  ++g_launches;
  return launch_pdl(permode_mix_kernel, dim3((unsigned)(ntn * ntb), (unsigned)ntq), dim3(256), smem, s, A, W, C, B,
                     H, N, MQ, alpha, (int)ntn);
}

}  // namespace tfno
