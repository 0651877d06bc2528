// Latency-bound small 1D layers (BASELINE configs[0] = C1: 16 batch elements,
// 64 -> 64 channels, N = 128, keep 32; and the batch-64 points of the C2
// sweep): ONE kernel, no cluster, no cross-CTA hand-off.  CTA (b, g) owns the
// NG output channels [NG g, NG g + NG) of batch element b and recomputes the
// (cheap) truncated forward FFTs of all H input rows of b -- the CTAs of one b
// re-read x[b] from L2 -- so every CTA runs load -> FFT -> mix -> padded iFFT
// -> store with only __syncthreads between the phases (reference semantics:
// pipeline.py:185-206 + 236-275, rank 1).  NG is the smallest of 8 / 32 / 64
// that keeps the grid within one wave of SMs.
//
//   phase 1  row teams of L lanes (L = 16 for N = 128 / 256, 32 for N = 1024),
//            V = N / L values per lane: the register FFTs of the fused 1D
//            kernel (wf_dft.cuh; N = 128: DFT8 + 8 x 16 transpose + DFT8 with a
//            one-shuffle sum) -> the first KT bins of each row into A[h][q]
//            (bins q >= keep written as 0)
//   phase 2  C[g][q] = sum_h A[h][q] W[h][NG g + g'] (h ascending, FP32 FMA)
//   phase 3  zero-padded inverse of the CTA's NG output rows, x 1/N, streaming stores
// Only x (read once from HBM, re-reads from L2), W and y touch global memory.
// Launched with programmatic dependent launch: the twiddle prologue of layer
// i+1 overlaps layer i.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"
#include "wf_dft.cuh"

namespace tfno {

namespace {

// 8 x 16 tile [k1][t] of the N = 128 rows, column XOR-swizzled by 2*k1
__device__ __forceinline__ int tsw8(int r, int c) { return r * 16 + (c ^ (2 * r)); }
// L x L tile, column XOR-swizzled by the row
template <int L>
__device__ __forceinline__ int tswl(int r, int c) { return r * L + (c ^ r); }

template <int NLEN>
struct TinyGeo {
  static constexpr int L = NLEN == 1024 ? 32 : 16;  // lanes per row team
  static constexpr int V = NLEN / L;                 // values per lane
  static constexpr int TEAMS = 256 / L;
  static constexpr int RB = NLEN == 1024 ? 1 : (NLEN == 256 ? 2 : 4);  // rows loaded ahead per team
  // stored bins per row: N = 128 keeps q = k1 + 8 k2 (k2 < 2 KP); else q = lane + L k2 (k2 < KP)
  template <int KP>
  __host__ __device__ static constexpr int kt() { return NLEN == 128 ? 16 * KP : L * KP; }
};

template <int NLEN, int KP, int NG>
__global__ void __launch_bounds__(256, 1)
    tiny1d_kernel(const float2* __restrict__ x, const float2* __restrict__ W, float2* __restrict__ y, int H, int N,
                  int keep, const float2* __restrict__ twg, float inv_scale) {
  using Gm = TinyGeo<NLEN>;
  constexpr int L = Gm::L, V = Gm::V, TEAMS = Gm::TEAMS, RB = Gm::RB, KT = Gm::template kt<KP>();
  extern __shared__ __align__(16) float2 sm[];
  float2* As = sm;                     // [H][KT]
  float2* Wt = As + (size_t)H * KT;    // [H][NG]
  float2* Cs = Wt + (size_t)H * NG;    // [NG][KT]
  float2* tr = Cs + NG * KT;           // [TEAMS][NLEN]
  float2* twN = tr + TEAMS * NLEN;     // [k1][t] = w_N^{t k1}, k1 < V, t < L
  float2* twL = twN + NLEN;            // w_L^k

  const int tid = threadIdx.x, team = tid / L, lane = tid % L;
  const unsigned tmask = L == 32 ? 0xffffffffu : (0xffffu << (16 * (team & 1)));
  const int b = blockIdx.y, n0 = blockIdx.x * NG;
  for (int k = tid; k < L; k += 256) twL[k] = __ldg(&twg[(size_t)k * (TFNO_TW_MAX / L)]);
  for (int i = tid; i < NLEN; i += 256) {
    const int k1 = i / L, t = i % L;
    twN[i] = __ldg(&twg[(size_t)((t * k1) % NLEN) * (TFNO_TW_MAX / NLEN)]);
  }
  __syncthreads();  // the twiddle tables are read by every team below
  pdl_wait();       // x / W are read, y written, only once the previous kernel has completed
  pdl_launch_dependents();

  for (int i = tid; i < H * NG; i += 256) {  // W columns of this CTA (zeros past N)
    const int h = i / NG, g = i % NG;
    Wt[i] = (n0 + g < N) ? __ldg(&W[(int64_t)h * N + n0 + g]) : make_float2(0.f, 0.f);
  }
  float2* trr = tr + team * NLEN;
  // ---- phase 1: truncated forward FFT of the rows h = team + TEAMS r, RB rows in flight
  for (int h0 = team; h0 < H; h0 += TEAMS * RB) {
    float2 v[RB][V];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int h = h0 + TEAMS * r;
      const float2* row = x + ((int64_t)b * H + h) * NLEN;
#pragma unroll
      for (int j = 0; j < V; ++j) v[r][j] = h < H ? __ldcs(row + lane + L * j) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int h = h0 + TEAMS * r;
      if (h >= H) break;  // uniform across the team
      float2* arow = As + (size_t)h * KT;
      if constexpr (NLEN == 128) {
        constexpr int K2 = 2 * KP;
        const int k1 = lane >> 1, hf = lane & 1;
        float2 u[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = v[r][j];
        dft8<-1>(u);
#pragma unroll
        for (int kk = 1; kk < 8; ++kk) u[kk] = cmul(u[kk], twN[kk * L + lane]);
        __syncwarp(tmask);  // the previous row's transpose reads are done
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) trr[tsw8(kk, lane)] = u[kk];
        __syncwarp(tmask);
#pragma unroll
        for (int t2 = 0; t2 < 8; ++t2) u[t2] = trr[tsw8(k1, hf + 2 * t2)];
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
          arow[q] = q < keep ? u[k2] : make_float2(0.f, 0.f);
        }
      } else {
        float2 u[L];
#pragma unroll
        for (int j = 0; j < L; ++j) u[j] = v[r][j];
        wf::dftL<L, -1>(u, twL);
#pragma unroll
        for (int k1 = 1; k1 < L; ++k1) u[k1] = cmul(u[k1], twN[k1 * L + lane]);
        __syncwarp(tmask);
#pragma unroll
        for (int k1 = 0; k1 < L; ++k1) trr[tswl<L>(k1, lane)] = u[k1];
        __syncwarp(tmask);
#pragma unroll
        for (int t = 0; t < L; ++t) u[t] = trr[tswl<L>(lane, t)];
        float2 o[KP];
        wf::dftL_first<L, KP>(u, o, twL);
#pragma unroll
        for (int k2 = 0; k2 < KP; ++k2) {
          const int q = lane + L * k2;
          arow[q] = q < keep ? o[k2] : make_float2(0.f, 0.f);
        }
      }
    }
  }
  __syncthreads();
  // ---- phase 2: C[g][q] = sum_h A[h][q] W[h][g], h ascending
  for (int o = tid; o < NG * KT; o += 256) {
    const int g = o / KT, q = o % KT;
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int h = 0; h < H; ++h) cmac(acc, As[(size_t)h * KT + q], Wt[h * NG + g]);
    Cs[o] = acc;
  }
  __syncthreads();
  // ---- phase 3: zero-padded inverse of output rows n0 + g (teams take rows g = team, team + TEAMS, ...)
  for (int g = team; g < NG && n0 + g < N; g += TEAMS) {
    const float2* cr = Cs + g * KT;
    float2* dst = y + ((int64_t)b * N + n0 + g) * NLEN;
    if constexpr (NLEN == 128) {
      constexpr int K2 = 2 * KP;
      const int k1 = lane >> 1, hf = lane & 1;
      float2 z[8];
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
        const int q = k1 + 8 * k2;
        z[k2] = (k2 < K2 && q < keep) ? cr[q] : make_float2(0.f, 0.f);
        if (k2 < K2 && k2 && hf) z[k2] = cmul(z[k2], conjf2(twL[k2]));
      }
      dft8<1>(z);
      __syncwarp(tmask);  // the previous row's transpose reads are done
#pragma unroll
      for (int t2 = 0; t2 < 8; ++t2) {
        const int t = hf + 2 * t2;
        trr[tsw8(k1, t)] = k1 ? cmul(z[t2], conjf2(twN[k1 * L + t])) : z[t2];
      }
      __syncwarp(tmask);
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) z[rr] = trr[tsw8(rr, lane)];
      dft8<1>(z);
#pragma unroll
      for (int j = 0; j < 8; ++j) __stcs(dst + lane + L * j, cscale(z[j], inv_scale));
    } else {
      float2 xk[KP];
#pragma unroll
      for (int k2 = 0; k2 < KP; ++k2) {
        const int q = lane + L * k2;
        xk[k2] = q < keep ? cr[q] : make_float2(0.f, 0.f);
      }
      float2 z[L];
      wf::idftL_padded<L, KP>(xk, z, twL);
#pragma unroll
      for (int t = 1; t < L; ++t) z[t] = cmul(z[t], conjf2(twN[t * L + lane]));
      __syncwarp(tmask);
#pragma unroll
      for (int t = 0; t < L; ++t) trr[tswl<L>(t, lane)] = z[t];
      __syncwarp(tmask);
#pragma unroll
      for (int k1 = 0; k1 < L; ++k1) z[k1] = trr[tswl<L>(lane, k1)];
      wf::dftL<L, 1>(z, twL);
#pragma unroll
      for (int j = 0; j < L; ++j) __stcs(dst + lane + L * j, cscale(z[j], inv_scale));
    }
  }
}

template <int NLEN, int KP, int NG>
size_t tiny_smem(int H) {
  using Gm = TinyGeo<NLEN>;
  constexpr int KT = Gm::template kt<KP>();
  return sizeof(float2) * ((size_t)H * KT + (size_t)H * NG + (size_t)NG * KT + (size_t)Gm::TEAMS * NLEN + NLEN + Gm::L);
}

template <int NLEN, int KP, int NG>
cudaError_t launch_tiny_t(const float2* x, const float2* W, float2* y, int B, int H, int N, int keep,
                          const float2* tw, cudaStream_t s) {
  const size_t smem = tiny_smem<NLEN, KP, NG>(H);
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  auto kern = tiny1d_kernel<NLEN, KP, NG>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)((N + NG - 1) / NG), (unsigned)B);
  e = launch_pdl1(kern, grid, dim3(256), smem, s, x, W, y, H, N, keep, tw, 1.0f / NLEN);
  if (e != cudaSuccess) return e;
  ++g_launches;
  return cudaGetLastError();
}

// KP: bins per lane group (N = 128: 16*KP stored bins; else L*KP); 3 rounds up to 4
int tiny_kp(int n, int keep) {
  const int per = n == 1024 ? 32 : 16;
  int kp = (keep + per - 1) / per;
  if (kp == 3) kp = 4;
  return kp;
}

// output channels per CTA: the smallest of 8 / 32 / 64 whose grid fits one wave
int tiny_ng(int B, int N, int sms) {
  for (int ng : {8, 32, 64})
    if ((int64_t)B * ((N + ng - 1) / ng) <= sms) return ng;
  return 0;
}

template <int NLEN, int NG>
cudaError_t dispatch_kp(int kp, const float2* x, const float2* W, float2* y, int B, int H, int N, int keep,
                        const float2* tw, cudaStream_t s) {
  switch (kp) {
    case 1: return launch_tiny_t<NLEN, 1, NG>(x, W, y, B, H, N, keep, tw, s);
    case 2: return launch_tiny_t<NLEN, 2, NG>(x, W, y, B, H, N, keep, tw, s);
    case 4: return launch_tiny_t<NLEN, 4, NG>(x, W, y, B, H, N, keep, tw, s);
    default: return cudaErrorNotSupported;
  }
}

template <int NLEN>
size_t tiny_bytes(int kp, int ng, int H) {
  const int KT = NLEN == 128 ? 16 * kp : TinyGeo<NLEN>::L * kp;
  return sizeof(float2) * ((size_t)H * KT + (size_t)H * ng + (size_t)ng * KT + (size_t)TinyGeo<NLEN>::TEAMS * NLEN +
                           NLEN + TinyGeo<NLEN>::L);
}

}  // namespace

int tiny1d_channels_per_cta(int B, int N) { return tiny_ng(B, N, device_sms()); }

bool tiny1d_supported(int n, int keep, int B, int H, int N) {
  if ((n != 128 && n != 256 && n != 1024) || keep < 1 || H < 1 || N < 1 || B < 1 || B > 65535) return false;
  const int kp = tiny_kp(n, keep);
  if (kp > 4) return false;
  const int ng = tiny_ng(B, N, device_sms());
  if (!ng) return false;
  const size_t bytes = n == 128 ? tiny_bytes<128>(kp, ng, H) : n == 256 ? tiny_bytes<256>(kp, ng, H)
                                                                        : tiny_bytes<1024>(kp, ng, H);
  return bytes <= 200 * 1024;
}

cudaError_t launch_tiny1d(const float2* x, const float2* W, float2* y, int n, int B, int H, int N, int keep,
                          const float2* tw, cudaStream_t s) {
  const int kp = tiny_kp(n, keep), ng = tiny_ng(B, N, device_sms());
#define TINY_NG(NL)                                                              \
  switch (ng) {                                                                  \
    case 8: return dispatch_kp<NL, 8>(kp, x, W, y, B, H, N, keep, tw, s);        \
    case 32: return dispatch_kp<NL, 32>(kp, x, W, y, B, H, N, keep, tw, s);      \
    case 64: return dispatch_kp<NL, 64>(kp, x, W, y, B, H, N, keep, tw, s);      \
    default: return cudaErrorNotSupported;                                       \
  }
  if (n == 128) { TINY_NG(128) }
  if (n == 256) { TINY_NG(256) }
  if (n == 1024) { TINY_NG(1024) }
#undef TINY_NG
  return cudaErrorNotSupported;
}

}  // namespace tfno
