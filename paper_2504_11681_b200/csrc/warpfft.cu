// Warp-synchronous register FFTs for contiguous rows of length N = L*L
// (L = 16: N = 256, half-warp per row; L = 32: N = 1024, one warp per row).
//
// Row index n = t + L*j (lane t holds its L values j in registers, loaded
// coalesced straight from HBM).  Forward, first `keep` bins (fft.py
// truncation semantics):
//   stage 1  Y_t[k1] = DFT_L over j of x[t + L j]   (in registers)
//            Y_t[k1] *= w_N^{t k1}                    (per-lane twiddles from a
//                                                      [k1][t] smem table: no conflicts)
//   transpose through a padded per-row smem tile (the only smem round trip)
//   stage 2  X[k1 + L k2] = DFT_L over t of Y_t[k1], lane k1 keeps k2 < ceil(keep/L)
// Inverse (zero-padded from src_len, x 1/N) mirrors it: lane k1 gathers its
// nonzero inputs X[k1 + L k2], padded DFT_L over k2 -> t, twiddle w_N^{+k1 t},
// transpose, DFT_L over k1 -> j, store y[t + L j].
// No CTA barriers: every row lives in one (half-)warp (__syncwarp only).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"
#include "warpfft.cuh"
#include "wf_dft.cuh"

namespace tfno {


__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}


// inverse: modes [P][src_len] (src stride) -> rows [P][N] (out stride), x scale
template <int L, int KP>
__global__ void __launch_bounds__(WfGeo<L>::NTH) warp_fft_inv_kernel(const float2* __restrict__ in,
                                                                   int64_t in_stride, float2* __restrict__ out,
                                                                   int64_t out_stride, int64_t P, int src_len,
                                                                   float scale, const float2* __restrict__ twg) {
  using G = WfGeo<L>;
  constexpr int N = G::N;
  extern __shared__ __align__(16) float2 sm[];
  float2* twL = sm;
  float2* twN = twL + L;
  float2* tr = twN + L * L;
  const int tid = threadIdx.x, lane = tid % L, rloc = tid / L;
  const unsigned tmask = L == 32 ? 0xffffffffu : (0xffffu << (16 * (rloc & 1)));
  for (int k = tid; k < L; k += G::NTH) twL[k] = __ldg(&twg[(size_t)k * (TFNO_TW_MAX / L)]);
  for (int i = tid; i < L * L; i += G::NTH) {
    const int k1 = i / L, t = i % L;
    twN[i] = __ldg(&twg[(size_t)((t * k1) % N) * (TFNO_TW_MAX / N)]);
  }
  __syncthreads();
  float2* trr = tr + rloc * L * G::TSTR;
  for (int64_t row = (int64_t)blockIdx.x * G::ROWS + rloc; row < P; row += (int64_t)gridDim.x * G::ROWS) {
    const float2* src = in + row * in_stride;
    // lane = k1: nonzero inputs X[k1 + L k2], k2 < KP
    float2 xk[KP];
#pragma unroll
    for (int k2 = 0; k2 < KP; ++k2) {
      const int k = lane + L * k2;
      xk[k2] = k < src_len ? __ldg(&src[k]) : make_float2(0.f, 0.f);
    }
    float2 z[L];
    wf::idftL_padded<L, KP>(xk, z, twL);   // z[t] = sum_k2 X[k1 + L k2] w_L^{+k2 t}
    // twiddle w_N^{+k1 t}; the table is symmetric (w^{t k1}), read [t][k1 = lane]: conflict-free
#pragma unroll
    for (int t = 1; t < L; ++t) z[t] = cmul(z[t], conjf2(twN[t * L + lane]));
    __syncwarp(tmask);
#pragma unroll
    for (int t = 0; t < L; ++t) trr[t * G::TSTR + lane] = z[t];
    __syncwarp(tmask);
    // lane = t: DFT_L over k1 -> j, y[t + L j]
#pragma unroll
    for (int k1 = 0; k1 < L; ++k1) z[k1] = trr[lane * G::TSTR + k1];
    wf::dftL<L, 1>(z, twL);
    float2* dst = out + row * out_stride;
#pragma unroll
    for (int j = 0; j < L; ++j) dst[lane + L * j] = cscale(z[j], scale);
  }
}

template <int L, int KP>
static cudaError_t launch_wf_inv(const float2* in, int64_t is, float2* out, int64_t os, int64_t P, int src_len,
                                 float scale, const float2* tw, cudaStream_t s) {
  using G = WfGeo<L>;
  const size_t smem = G::smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(warp_fft_inv_kernel<L, KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = (P + G::ROWS - 1) / G::ROWS;
  const int grid = (int)(blocks < (int64_t)sms * 8 ? blocks : (int64_t)sms * 8);
  warp_fft_inv_kernel<L, KP><<<grid, G::NTH, smem, s>>>(in, is, out, os, P, src_len, scale, tw);
  ++g_launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- fused 1D layer
// rows_fused on warp FFTs (K6 for N = L^2): per work item (row group g) the
// TEAMS row-teams FFT the H channel rows straight into the smem A panel
// As[h][q], a 256-thread register-tiled CGEMM forms C[q][n] against the
// CTA-resident W, C goes to smem (aliasing As) and the teams run the padded
// iFFT of every output channel row from smem to HBM.  Only x, W and y touch
// HBM (pipeline.py:185-206, 245-250 with the whole k-loop in one CTA).
template <int L>
struct WfFusedGeo {
  using G = WfGeo<L>;
  static constexpr int NTH = 256, TEAMS = NTH / L;
  static constexpr int TI = 4, TJ = 8;  // GEMM thread tile (q, n)
};

size_t warp_fused_smem_bytes(int n, int keep, int H, int NO) {
  const int L = n == 256 ? 16 : 32;
  const size_t panel = (size_t)keep * (H > NO ? H : NO);
  return sizeof(float2) * ((size_t)L + (size_t)L * L + (size_t)(256 / L) * L * (L + 1) + panel + (size_t)H * NO);
}

template <int L, int KP>
__global__ void __launch_bounds__(256, 1) warp_fused_kernel(FusedArgs a) {
  using G = WfGeo<L>;
  using F = WfFusedGeo<L>;
  constexpr int N = G::N, TEAMS = F::TEAMS, TI = F::TI, TJ = F::TJ;
  extern __shared__ __align__(16) float2 sm[];
  const int keep = a.keep, H = a.H, NO = a.N;
  float2* twL = sm;
  float2* twN = twL + L;
  float2* tr = twN + L * L;
  float2* P = tr + TEAMS * L * G::TSTR;                 // As[h][q] / Cs[n][q] (aliased)
  float2* Ws = P + (size_t)keep * (H > NO ? H : NO);    // W[h][n], CTA resident
  const int tid = threadIdx.x, lane = tid % L, team = tid / L;
  const unsigned tmask = L == 32 ? 0xffffffffu : (0xffffu << (16 * (team & 1)));  // this team's lanes
  for (int k = tid; k < L; k += F::NTH) twL[k] = __ldg(&a.twg[(size_t)k * (TFNO_TW_MAX / L)]);
  for (int i = tid; i < L * L; i += F::NTH) {
    const int k1 = i / L, t = i % L;
    twN[i] = __ldg(&a.twg[(size_t)((t * k1) % N) * (TFNO_TW_MAX / N)]);
  }
  for (int i = tid; i < H * NO; i += F::NTH) Ws[i] = __ldg(&a.W[i]);
  __syncthreads();
  float2* trr = tr + team * L * G::TSTR;
  // GEMM mapping: q = tm + MT*i (i < TI), n = tn + NTg*j (j < TJ)
  const int MT = (keep + TI - 1) / TI, NTg = (NO + TJ - 1) / TJ;
  const bool gthread = tid < MT * NTg;
  const int tm = tid % MT, tn = tid / MT;

  for (int64_t g = blockIdx.x; g < a.G; g += gridDim.x) {
    const int64_t bb = g / a.gx, pp = g % a.gx;
    const float2* xg = a.x + bb * a.x_sb + pp * a.x_sp;
    // ---- forward: rows h -> A panel
    for (int h = team; h < H; h += TEAMS) {
      const float2* src = xg + (int64_t)h * a.x_sh;
      float2 v[L];
#pragma unroll
      for (int j = 0; j < L; ++j) v[j] = __ldg(&src[lane + L * j]);
      wf::dftL<L, -1>(v, twL);
#pragma unroll
      for (int k1 = 1; k1 < L; ++k1) v[k1] = cmul(v[k1], twN[k1 * L + lane]);
      __syncwarp(tmask);
#pragma unroll
      for (int k1 = 0; k1 < L; ++k1) trr[k1 * G::TSTR + lane] = v[k1];
      __syncwarp(tmask);
#pragma unroll
      for (int t = 0; t < L; ++t) v[t] = trr[lane * G::TSTR + t];
      float2 o[KP];
      wf::dftL_first<L, KP>(v, o, twL);
      __syncwarp(tmask);
#pragma unroll
      for (int k2 = 0; k2 < KP; ++k2) {
        const int q = lane + L * k2;
        if (q < keep) P[(size_t)h * keep + q] = o[k2];
      }
    }
    __syncthreads();
    // ---- channel mix: C[q][n] = sum_h A[h][q] W[h][n]
    float2 acc[TI][TJ];
#pragma unroll
    for (int i = 0; i < TI; ++i)
#pragma unroll
      for (int j = 0; j < TJ; ++j) acc[i][j] = make_float2(0.f, 0.f);
    if (gthread) {
#pragma unroll 2
      for (int h = 0; h < H; ++h) {
        float2 av[TI], bv[TJ];
#pragma unroll
        for (int i = 0; i < TI; ++i) {
          const int q = tm + MT * i;
          av[i] = q < keep ? P[(size_t)h * keep + q] : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < TJ; ++j) {
          const int n = tn + NTg * j;
          bv[j] = n < NO ? Ws[h * NO + n] : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < TI; ++i)
#pragma unroll
          for (int j = 0; j < TJ; ++j) cmac(acc[i][j], av[i], bv[j]);
      }
    }
    __syncthreads();  // all A reads done before C overwrites the aliased panel
    if (gthread) {
#pragma unroll
      for (int j = 0; j < TJ; ++j) {
        const int n = tn + NTg * j;
#pragma unroll
        for (int i = 0; i < TI; ++i) {
          const int q = tm + MT * i;
          if (q < keep && n < NO) P[(size_t)n * keep + q] = acc[i][j];
        }
      }
    }
    __syncthreads();
    // ---- inverse: output rows n from the C tile
    float2* yg = a.y + bb * a.y_sb + pp * a.y_sp;
    for (int n = team; n < NO; n += TEAMS) {
      float2 xk[KP];
#pragma unroll
      for (int k2 = 0; k2 < KP; ++k2) {
        const int q = lane + L * k2;
        xk[k2] = q < keep ? P[(size_t)n * keep + q] : make_float2(0.f, 0.f);
      }
      float2 z[L];
      wf::idftL_padded<L, KP>(xk, z, twL);
#pragma unroll
      for (int t = 1; t < L; ++t) z[t] = cmul(z[t], conjf2(twN[t * L + lane]));
      __syncwarp(tmask);
#pragma unroll
      for (int t = 0; t < L; ++t) trr[t * G::TSTR + lane] = z[t];
      __syncwarp(tmask);
#pragma unroll
      for (int k1 = 0; k1 < L; ++k1) z[k1] = trr[lane * G::TSTR + k1];
      __syncwarp(tmask);
      wf::dftL<L, 1>(z, twL);
      float2* dst = yg + (int64_t)n * a.y_sn;
#pragma unroll
      for (int j = 0; j < L; ++j) dst[lane + L * j] = cscale(z[j], a.inv_scale);
    }
    __syncthreads();  // C reads done before the next item's A writes
  }
}

bool warp_fused_supported(int n, int keep, int H, int NO) {
  if (n != 256 && n != 1024) return false;
  const int L = n == 256 ? 16 : 32;
  const int kp = (keep + L - 1) / L;
  if (kp > 8 || kp > L / 2) return false;
  const int MT = (keep + 3) / 4, NTg = (NO + 7) / 8;
  if (MT * NTg > 256) return false;
  return warp_fused_smem_bytes(n, keep, H, NO) <= 220 * 1024;
}

template <int L, int KP>
static cudaError_t launch_wfused_t(const FusedArgs& a, cudaStream_t s) {
  const size_t smem = warp_fused_smem_bytes(L * L, a.keep, a.H, a.N);
  cudaError_t e =
      cudaFuncSetAttribute(warp_fused_kernel<L, KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)(a.G < sms ? a.G : sms);
  warp_fused_kernel<L, KP><<<grid, 256, smem, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_warp_fused(const FusedArgs& a, cudaStream_t s) {
  const int L = a.n == 256 ? 16 : 32;
  const int kp = (a.keep + L - 1) / L;
#define WFF_CASE(LL, KK) \
  if (L == LL && kp == KK) return launch_wfused_t<LL, KK>(a, s);
  WFF_CASE(16, 1) WFF_CASE(16, 2) WFF_CASE(16, 3) WFF_CASE(16, 4) WFF_CASE(16, 5) WFF_CASE(16, 6)
  WFF_CASE(16, 7) WFF_CASE(16, 8)
  WFF_CASE(32, 1) WFF_CASE(32, 2) WFF_CASE(32, 3) WFF_CASE(32, 4) WFF_CASE(32, 5) WFF_CASE(32, 6)
  WFF_CASE(32, 7) WFF_CASE(32, 8)
#undef WFF_CASE
  return cudaErrorNotSupported;
}

// ---------------------------------------------------------------- team FFTs, N = 1024*U
// A team of T = 32*U threads per row (U = 2: N = 2048, U = 4: N = 4096), 32
// register values per thread, n = t + T*j:
//   forward  stage 1: DFT32 over j (registers), twiddle w_N^{t k1}; transpose
//            [k1][t] through smem; stage 2: X[k1 + 32 k2] = sum_t w_T^{t k2} Y_t[k1]
//            with t = u + U*s: thread (k1, u) runs DFT32 over s, twiddles by
//            w_T^{u k2}, and the U partial sums of its k1 are reduced across the
//            U adjacent lanes with shuffles (first K2 = ceil(keep/32) outputs).
//   inverse  thread (k1, u): padded DFT32 over k2 of X[k1 + 32 k2] w_T^{+k2 u}
//            gives z[u + U s]; twiddle w_N^{+k1 t}; transpose [t][k1];
//            thread t: DFT32 over k1 -> y[t + T j].  No cross-lane reduction.
template <int U>
struct TfGeo {
  static constexpr int T = 32 * U, N = 32 * T, NTH = 512, TEAMS = NTH / T;
  static constexpr int LU = U == 4 ? 2 : 1;
  __host__ __device__ static constexpr size_t smem_bytes(int k2 = 0) {  // + inverse mode-row buffers (TEAMS x 2 x 32*K2)
    return sizeof(float2) * ((size_t)32 + (size_t)32 * T + (size_t)TEAMS * T * 32 + (size_t)T +
                             (size_t)TEAMS * 2 * 32 * k2);
  }
  // [t][k1] tile (row length 32, unpadded) with the column XOR-swizzled by a
  // 4-bit rotation of t: conflict-free both for 16 consecutive t at fixed k1
  // and for the (u, k1) lane pattern t = u + U*s of the stage-2 role.
  __device__ static __forceinline__ int swz(int t, int k1) {
    const int f = ((t & (U - 1)) << (4 - LU)) | ((t >> LU) & ((16 >> LU) - 1));
    return t * 32 + (k1 ^ f);
  }
};

template <int U, int K2>
__global__ void __launch_bounds__(512, 1) team_fft_fwd_kernel(const float2* __restrict__ in, int64_t in_stride,
                                                            float2* __restrict__ out, int64_t out_stride, int64_t P,
                                                            int keep, const float2* __restrict__ twg, int pfd) {
  using G = TfGeo<U>;
  constexpr int T = G::T, N = G::N;
  extern __shared__ __align__(16) float2 sm[];
  float2* tw32 = sm;                  // w_32^k
  float2* twN = tw32 + 32;            // w_N^{t k1} at G::swz(t, k1), k1 < 32, t < T
  float2* tr = twN + 32 * T;          // TEAMS x T x 32 (swizzled)
  float2* twT = tr + G::TEAMS * T * 32;  // w_T^k
  const int tid = threadIdx.x, team = tid / T, tt = tid % T;
  for (int k = tid; k < 32; k += G::NTH) tw32[k] = __ldg(&twg[(size_t)k * (TFNO_TW_MAX / 32)]);
  for (int k = tid; k < T; k += G::NTH) twT[k] = __ldg(&twg[(size_t)k * (TFNO_TW_MAX / T)]);
  for (int i = tid; i < 32 * T; i += G::NTH) {
    const int k1 = i / T, t = i % T;
    twN[G::swz(t, k1)] = __ldg(&twg[(size_t)(t * k1) * (TFNO_TW_MAX / N)]);
  }
  __syncthreads();
  float2* trr = tr + team * T * 32;
  const int k1s = tt / U, us = tt % U;  // stage-2 role
  for (int64_t row0 = (int64_t)blockIdx.x * G::TEAMS; row0 < P; row0 += (int64_t)gridDim.x * G::TEAMS) {
    const int64_t row = row0 + team;
    const bool live = row < P;
    float2 v[32];
    const float2* src = in + (live ? row : 0) * in_stride;
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = live ? __ldg(&src[tt + T * j]) : make_float2(0.f, 0.f);
    // pull the team's row pfd iterations ahead into L2 while this one computes
    // (one CTA per SM: without it HBM idles during each row's transform)
    if (pfd > 0 && tt == 0) {
      const int64_t step = (int64_t)gridDim.x * G::TEAMS;
      for (int d = (row0 == (int64_t)blockIdx.x * G::TEAMS) ? 1 : pfd; d <= pfd; ++d) {
        const int64_t nr = row + d * step;
        if (nr < P) l2_prefetch_bulk(in + nr * in_stride, N * sizeof(float2));
      }
    }
    wf::dftL<32, -1>(v, tw32);
#pragma unroll
    for (int k1 = 1; k1 < 32; ++k1) v[k1] = cmul(v[k1], twN[G::swz(tt, k1)]);
    named_bar_sync(1 + team, T);
#pragma unroll
    for (int k1 = 0; k1 < 32; ++k1) trr[G::swz(tt, k1)] = v[k1];  // [t][k1]
    named_bar_sync(1 + team, T);
    // thread (k1s, us): Y_{us + U s}[k1s] for s < 32
#pragma unroll
    for (int s2 = 0; s2 < 32; ++s2) v[s2] = trr[G::swz(us + U * s2, k1s)];
    wf::dftL<32, -1>(v, tw32);  // V_u[k2'] over s
    float2 o[K2];
#pragma unroll
    for (int k2 = 0; k2 < K2; ++k2) o[k2] = (us && k2) ? cmul(v[k2], twT[(us * k2) % T]) : v[k2];
    // sum over the U adjacent lanes (u)
#pragma unroll
    for (int m = 1; m < U; m <<= 1)
#pragma unroll
      for (int k2 = 0; k2 < K2; ++k2) {
        float2 p;
        p.x = __shfl_xor_sync(0xffffffffu, o[k2].x, m);
        p.y = __shfl_xor_sync(0xffffffffu, o[k2].y, m);
        o[k2] = cadd(o[k2], p);
      }
    if (live) {
      float2* dst = out + row * out_stride;
#pragma unroll
      for (int k2 = 0; k2 < K2; ++k2) {
        if (k2 % U != us) continue;  // lanes of a k1 group split the stores
        const int k = k1s + 32 * k2;
        if (k < keep) dst[k] = o[k2];
      }
    }
    named_bar_sync(1 + team, T);
  }
}

template <int U, int K2>
__global__ void __launch_bounds__(512, 1) team_fft_inv_kernel(const float2* __restrict__ in, int64_t in_stride,
                                                            float2* __restrict__ out, int64_t out_stride, int64_t P,
                                                            int src_len, float scale,
                                                            const float2* __restrict__ twg) {
  using G = TfGeo<U>;
  constexpr int T = G::T, N = G::N;
  extern __shared__ __align__(16) float2 sm[];
  float2* tw32 = sm;
  float2* twN = tw32 + 32;
  float2* tr = twN + 32 * T;
  float2* twT = tr + G::TEAMS * T * 32;
  const int tid = threadIdx.x, team = tid / T, tt = tid % T;
  for (int k = tid; k < 32; k += G::NTH) tw32[k] = __ldg(&twg[(size_t)k * (TFNO_TW_MAX / 32)]);
  for (int k = tid; k < T; k += G::NTH) twT[k] = __ldg(&twg[(size_t)k * (TFNO_TW_MAX / T)]);
  for (int i = tid; i < 32 * T; i += G::NTH) {
    const int k1 = i / T, t = i % T;
    twN[G::swz(t, k1)] = __ldg(&twg[(size_t)(t * k1) * (TFNO_TW_MAX / N)]);
  }
  __syncthreads();
  float2* trr = tr + team * T * 32;
  // cp.async double buffer of the mode rows when it fits in shared memory (PF)
  constexpr bool PF = G::smem_bytes(K2) <= 227 * 1024;
  float2* mbuf = twT + T + team * 2 * (32 * K2);  // this team's double-buffered mode rows
  const int k1s = tt / U, us = tt % U;
  // next row's nonzero modes: cp.async global -> shared one row ahead (the
  // per-row __ldg of the modes was the exposed latency: long-scoreboard stalls)
  const bool vec = (in_stride % 2 == 0) && (((uintptr_t)in & 15) == 0);
  auto prefetch = [&](int64_t r, int buf) {
    if constexpr (!PF) return;
    float2* d = mbuf + buf * (32 * K2);
    const float2* sr = in + r * in_stride;
    if (vec) {
      for (int e = 2 * tt; e < 32 * K2; e += 2 * T) {
        const int nb = e + 1 < src_len ? 16 : (e < src_len ? 8 : 0);
        const unsigned sd = (unsigned)__cvta_generic_to_shared(d + e);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sd), "l"(nb ? sr + e : sr), "r"(nb)
                     : "memory");
      }
    } else {
      for (int e = tt; e < 32 * K2; e += T) d[e] = e < src_len ? __ldg(&sr[e]) : make_float2(0.f, 0.f);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int it = 0;
  if (PF && (int64_t)blockIdx.x * G::TEAMS + team < P) prefetch((int64_t)blockIdx.x * G::TEAMS + team, 0);
  for (int64_t row0 = (int64_t)blockIdx.x * G::TEAMS; row0 < P; row0 += (int64_t)gridDim.x * G::TEAMS, ++it) {
    const int64_t row = row0 + team;
    const bool live = row < P;
    const int64_t nrow = row + (int64_t)gridDim.x * G::TEAMS;
    if constexpr (PF) {
      if (nrow < P) prefetch(nrow, (it + 1) & 1);
      else asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // this row's pieces landed
      named_bar_sync(1 + team, T);                           // ... everyone's
    }
    const float2* src = PF ? mbuf + (it & 1) * (32 * K2) : in + (live ? row : 0) * in_stride;
    // thread (k1s, us): inputs X[k1s + 32 k2] w_T^{+k2 us}, padded DFT32 over k2 -> s
    float2 z[32];
#pragma unroll
    for (int k2 = 0; k2 < 32; ++k2) {
      if (k2 < K2) {
        const int k = k1s + 32 * k2;
        float2 xv = (live && k < src_len) ? src[k] : make_float2(0.f, 0.f);
        z[k2] = (us && k2) ? cmul(xv, conjf2(twT[(us * k2) % T])) : xv;
      } else {
        z[k2] = make_float2(0.f, 0.f);
      }
    }
    wf::dftL<32, 1>(z, tw32);  // z[s] -> value at t = us + U s
    named_bar_sync(1 + team, T);
#pragma unroll
    for (int s2 = 0; s2 < 32; ++s2) {
      const int t = us + U * s2;
      trr[G::swz(t, k1s)] = cmul(z[s2], conjf2(twN[G::swz(t, k1s)]));  // w_N^{+k1 t}
    }
    named_bar_sync(1 + team, T);
    // thread t: DFT32 over k1 -> y[t + T j]
#pragma unroll
    for (int k1 = 0; k1 < 32; ++k1) z[k1] = trr[G::swz(tt, k1)];
    wf::dftL<32, 1>(z, tw32);
    if (live) {
      float2* dst = out + row * out_stride;
#pragma unroll
      for (int j = 0; j < 32; ++j) dst[tt + T * j] = cscale(z[j], scale);
    }
    named_bar_sync(1 + team, T);
  }
}

template <int U, int K2>
static cudaError_t launch_tf(int dir, const float2* in, int64_t is, float2* out, int64_t os, int64_t P, int keep,
                             int src_len, float scale, const float2* tw, cudaStream_t s) {
  using G = TfGeo<U>;
  const size_t smem = G::smem_bytes();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = (P + G::TEAMS - 1) / G::TEAMS;
  const int grid = (int)(blocks < (int64_t)sms ? blocks : (int64_t)sms);
  cudaError_t e;
  if (dir < 0) {
    e = cudaFuncSetAttribute(team_fft_fwd_kernel<U, K2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    static int pfd = -1;  // L2 prefetch distance in rows (TFNO_TEAM_PF; 0 = off)
    if (pfd < 0) {
      const char* env = getenv("TFNO_TEAM_PF");
      pfd = env ? atoi(env) : 1;
    }
    // bulk prefetch needs 16-byte aligned rows
    const int d = (((uintptr_t)in | (uintptr_t)(is * sizeof(float2))) & 15) ? 0 : pfd;
    team_fft_fwd_kernel<U, K2><<<grid, G::NTH, smem, s>>>(in, is, out, os, P, keep, tw, d);
  } else {
    const size_t smem_i = G::smem_bytes(K2) <= 227 * 1024 ? G::smem_bytes(K2) : smem;
    e = cudaFuncSetAttribute(team_fft_inv_kernel<U, K2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_i);
    if (e != cudaSuccess) return e;
    team_fft_inv_kernel<U, K2><<<grid, G::NTH, smem_i, s>>>(in, is, out, os, P, src_len, scale, tw);
  }
  ++g_launches;
  return cudaGetLastError();
}

// N = L^2 with keep (forward) / src_len (inverse) <= N/4: KP = ceil(k / L) <= L/4 <= 8
static int team_k2(int k) {  // K2 template bucket for the team kernels
  const int k2 = (k + 31) / 32;
  return k2 <= 4 ? 4 : k2 <= 8 ? 8 : k2 <= 16 ? 16 : 32;
}

bool warp_fft_supported(int n, int dir, int keep, int src_len) {
  if (n == 2048 || n == 4096) {
    if (dir < 0 && src_len != n) return false;
    if (dir > 0 && keep != n) return false;
    const int k = dir < 0 ? keep : src_len;
    return k >= 1 && (k + 31) / 32 <= 32;
  }
  if (n != 256 && n != 1024) return false;
  const int L = n == 256 ? 16 : 32;
  const int k = dir < 0 ? keep : src_len;
  if (dir < 0 && src_len != n) return false;
  if (dir > 0 && keep != n) return false;
  return k >= 1 && (k + L - 1) / L <= 8 && (k + L - 1) / L <= L / 2;
}

cudaError_t launch_warp_fft(int n, int dir, const float2* in, int64_t is, float2* out, int64_t os, int64_t P,
                            int keep, int src_len, float scale, const float2* tw, cudaStream_t s) {
  if (n == 2048 || n == 4096) {
    const int kb = team_k2(dir < 0 ? keep : src_len);
#define TF_CASE(UU, KK) \
  if (n == 1024 * UU && kb == KK) return launch_tf<UU, KK>(dir, in, is, out, os, P, keep, src_len, scale, tw, s);
    TF_CASE(2, 4) TF_CASE(2, 8) TF_CASE(2, 16) TF_CASE(2, 32) TF_CASE(4, 4) TF_CASE(4, 8) TF_CASE(4, 16)
    TF_CASE(4, 32)
#undef TF_CASE
    return cudaErrorNotSupported;
  }
  const int L = n == 256 ? 16 : 32;
  const int kp = ((dir < 0 ? keep : src_len) + L - 1) / L;
  if (dir < 0) return launch_warp_fft_fwd_rows(L, kp, in, is, out, os, P, keep, tw, s);  // warpfft_fwd.cu
#define WF_CASE(LL, KK) \
  if (L == LL && kp == KK) return launch_wf_inv<LL, KK>(in, is, out, os, P, src_len, scale, tw, s);
  WF_CASE(16, 1) WF_CASE(16, 2) WF_CASE(16, 3) WF_CASE(16, 4) WF_CASE(16, 5) WF_CASE(16, 6) WF_CASE(16, 7)
  WF_CASE(16, 8)
  WF_CASE(32, 1) WF_CASE(32, 2) WF_CASE(32, 3) WF_CASE(32, 4) WF_CASE(32, 5) WF_CASE(32, 6) WF_CASE(32, 7)
  WF_CASE(32, 8)
#undef WF_CASE
  return cudaErrorNotSupported;
}

}  // namespace tfno
