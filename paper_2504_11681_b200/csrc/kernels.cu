// General-shape kernels of the TurboFNO layer (any power-of-two length up to
// TFNO_TW_MAX, any keep/src_len, ragged H/N/B):
//
//   fft_pencils_kernel  K1/K2: batched truncating / zero-padded FFT over
//                       pencils with arbitrary (2-level) pencil strides and
//                       element stride: the rank-2 x-axis passes
//                       (pipeline.py:150-168, 277-292), the unfused y passes
//                       (pipeline.py:207-232, 236-275) and the standalone
//                       fft.execute / batched_execute API (fft.py:258-315).
//   cgemm_kernel        K3: strided-batched FP32 SIMT complex GEMM
//                       (cgemm.py:83-114), k ascending.
//   fused_rows_kernel   K4/K5/K6: the paper's fused kernel over rows
//                       (pipeline.py:185-206 k-loop, :245-250 epilogue):
//                       FFT of a k-chunk of channel rows straight into the
//                       shared-memory A panel, rank-k CGEMM update of a
//                       register accumulator, padded iFFT of the C tile from
//                       shared memory as the epilogue.  FUSE_FFT / FUSE_IFFT
//                       select the full or partial fusions.
//   pad_truncate_kernel staged baseline's truncate/pad copy passes
//                       (pipeline.py:162-166, 263-268).
#include <cuda_runtime.h>
#include <stdlib.h>

#include "fft_engine.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace tfno {

thread_local long long g_launches = 0;

int device_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

bool pdl_enabled(int level) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TFNO_PDL");
    v = e ? atoi(e) : 1;
  }
  return v >= level;
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

// ------------------------------------------------------------------------
// K1/K2: batched pencils
// ------------------------------------------------------------------------
struct GlobalPencilSrc {
  const float2* __restrict__ ptr;
  const int64_t* base;  // smem, per pencil in block
  int64_t es;
  int src_len, valid;
  __device__ __forceinline__ float2 load(int p, int e) const {
    if (e >= src_len || p >= valid) return make_float2(0.f, 0.f);
    return ptr[base[p] + (int64_t)e * es];
  }
};
struct GlobalPencilDst {
  float2* __restrict__ ptr;
  const int64_t* base;
  int64_t es;
  int valid;
  __device__ __forceinline__ void store(int p, int o, float2 v) const {
    if (p < valid) ptr[base[p] + (int64_t)o * es] = v;
  }
};

size_t fft_pencils_smem_bytes(int n, int PB, int pm) {
  return sizeof(float2) * (size_t)(n + 2 * smem_buf_elems(n, PB, pm)) + 2 * sizeof(int64_t) * PB;
}

template <int DIR>
__global__ void __launch_bounds__(256) fft_pencils_kernel(FftPencilArgs a) {
  extern __shared__ float4 smem_raw[];
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  const int be = smem_buf_elems(a.n, a.PB, a.pencil_major);
  float2* buf0 = tw + a.n;
  float2* buf1 = buf0 + be;
  int64_t* bin = reinterpret_cast<int64_t*>(buf1 + be);
  int64_t* bout = bin + a.PB;
  const int tid = threadIdx.x, nthr = blockDim.x;
  load_twiddles(tw, a.twg, a.n, tid, nthr);
  const RadixPlan rp = make_radix_plan(a.n);
  for (int64_t pb = (int64_t)blockIdx.x * a.PB; pb < a.P; pb += (int64_t)gridDim.x * a.PB) {
    for (int p = tid; p < a.PB; p += nthr) {
      int64_t pg = pb + p;
      if (pg < a.P) {
        bin[p] = (pg / a.im.P0) * a.im.s1 + (pg % a.im.P0) * a.im.s0;
        bout[p] = (pg / a.om.P0) * a.om.s1 + (pg % a.om.P0) * a.om.s0;
      }
    }
    __syncthreads();
    const int valid = (int)imin64(a.PB, a.P - pb);
    GlobalPencilSrc src{a.in, bin, a.im.es, a.src_len, valid};
    GlobalPencilDst dst{a.out, bout, a.om.es, valid};
    fft_block<DIR>(rp, a.PB, a.pencil_major, tid, nthr, tw, src, dst, buf0, buf1, a.keep, a.scale);
  }
}

cudaError_t launch_fft_pencils(const FftPencilArgs& a, int dir, cudaStream_t s) {
  size_t smem = fft_pencils_smem_bytes(a.n, a.PB, a.pencil_major);
  int64_t blocks = (a.P + a.PB - 1) / a.PB;
  int grid = (int)imin64(blocks, 148 * 16);
  if (grid < 1) grid = 1;
  cudaError_t e;
  if (dir < 0) {
    e = cudaFuncSetAttribute(fft_pencils_kernel<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fft_pencils_kernel<-1><<<grid, 256, smem, s>>>(a);
  } else {
    e = cudaFuncSetAttribute(fft_pencils_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fft_pencils_kernel<1><<<grid, 256, smem, s>>>(a);
  }
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------------
// K3: FP32 SIMT CGEMM, C[b] = alpha * A[b] (M x K) * W[b] (K x N)
// 64x64x8 block tile, 256 threads, 4x4 complex per thread (strided rows /
// cols so shared-memory reads are conflict-free / broadcast).
// ------------------------------------------------------------------------
namespace {
constexpr int GBM = 64, GBN = 64, GBK = 8;
}

__global__ void __launch_bounds__(256) cgemm_kernel(GemmArgs g) {
  __shared__ float2 As[GBK][GBM];
  __shared__ float2 Ws[GBK][GBN];
  const int tid = threadIdx.x;
  const int tm = tid % 16, tn = tid / 16;
  const int64_t m0 = (int64_t)blockIdx.x * GBM, n0 = (int64_t)blockIdx.y * GBN;
  const int64_t b = blockIdx.z;
  const float2* A = g.A + b * g.a_bs;
  const float2* W = g.W + b * g.w_bs;
  float2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
  for (int64_t k0 = 0; k0 < g.K; k0 += GBK) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      int i = tid + r * 256;
      int mm = i % GBM, kk = i / GBM;
      int64_t gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < g.M && gk < g.K) ? A[gm * g.a_ms + gk * g.a_ks] : make_float2(0.f, 0.f);
      int nn = i % GBN;
      int64_t gn = n0 + nn;
      Ws[kk][nn] = (gn < g.N && gk < g.K) ? W[gk * g.w_ks + gn * g.w_ns] : make_float2(0.f, 0.f);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      float2 av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][tm + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Ws[kk][tn + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) cmac_s(acc[i][j], av[i], bv[j]);
    }
    __syncthreads();
  }
  float2* C = g.C + b * g.c_bs;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t gm = m0 + tm + 16 * i;
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t gn = n0 + tn + 16 * j;
      if (gn < g.N) C[gm * g.c_ms + gn * g.c_ns] = cscale(acc[i][j], g.alpha);
    }
  }
}

// Mode-layout fast path: A[b][k][m] and C[b][n][m] m-contiguous, W[k][n]
// n-contiguous.  CTA tile 64 (m) x 128 (n) so the A panel is streamed from
// HBM once for N <= 128; BK = 16; 4 x 8 complex accumulators per thread
// (m = tm + 16 i, n = tn + 16 j: conflict-free / broadcast shared reads);
// next chunk prefetched into registers (float4) while the current one is
// consumed from shared memory (double buffer).
// TI x TJ = 8 x 8 (128 x 128 tile, BK = 8, one CTA of 200+ registers per
// SM) halves the shared-memory operand loads per FFMA for large M and N.
// PK: packed f32x2 form — the W chunk is staged as (wr, wi, -wi, wr) so one
// complex MAC is two FFMA2 with broadcast A operands (half the issue slots of
// the 4-FFMA form at the same FP32-pipe rate).
template <int TI, int TJ, bool PK = false>
__global__ void __launch_bounds__(256, (TI * TJ > 32 ? 1 : TI * TJ <= 16 ? 4 : 2)) cgemm_modes_kernel(GemmArgs g) {
  constexpr int FBM = 16 * TI, FBN = 16 * TJ, FBK = (TI * TJ > 32 || TI * TJ <= 16 || PK ? 8 : 16);
  __shared__ __align__(16) float2 As[2][FBK][FBM];
  __shared__ __align__(16) float2 Ws[2][FBK][FBN * (PK ? 2 : 1)];
  pdl_wait();  // PDL launch: A is the previous kernel's output
  pdl_launch_dependents();
  const int tid = threadIdx.x;
  const int tm = tid % 16, tn = tid / 16;
  const int64_t m0 = (int64_t)blockIdx.x * FBM, n0 = (int64_t)blockIdx.y * FBN;
  // fold > 1: the tile spans `fold` batch elements of M (< FBM) modes each
  const int64_t fold = g.fold > 1 ? g.fold : 1;
  const int64_t b = blockIdx.z * fold;
  const float2* __restrict__ A = g.A + b * g.a_bs;
  const float2* __restrict__ W = g.W + (fold > 1 ? 0 : b * g.w_bs);
  auto a_off = [&](int64_t gm) -> int64_t {  // tile-local m -> element offset (batch folded)
    return fold > 1 ? (gm / g.M) * g.a_bs + gm % g.M : gm;
  };
  auto m_ok = [&](int64_t gm) { return fold > 1 ? (gm / g.M < fold && b + gm / g.M < g.batch) : gm < g.M; };
  // loader mapping: A chunk = FBK x FBM complex = 512 float4 (2 / thread),
  //                 W chunk = FBK x FBN complex = 1024 float4 (4 / thread)
  constexpr int NA = FBK * FBM / 2 / 256, NW = FBK * FBN / 2 / 256;  // float4 per thread
  float4 ra[NA], rw[NW];
  auto load_chunk = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < NA; ++r) {
      const int i = tid + r * 256;
      const int kk = i / (FBM / 2), mm = (i % (FBM / 2)) * 2;
      const int64_t gk = k0 + kk, gm = m0 + mm;
      if (fold > 1) {  // M even: the pair (gm, gm+1) stays inside one batch element
        ra[r] = (gk < g.K && m_ok(gm)) ? __ldg(reinterpret_cast<const float4*>(A + gk * g.a_ks + a_off(gm)))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
      } else if (gk < g.K && gm + 1 < g.M) {
        ra[r] = __ldg(reinterpret_cast<const float4*>(A + gk * g.a_ks + gm));
      } else {
        float2 v0 = (gk < g.K && gm < g.M) ? A[gk * g.a_ks + gm] : make_float2(0.f, 0.f);
        ra[r] = make_float4(v0.x, v0.y, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int r = 0; r < NW; ++r) {
      const int i = tid + r * 256;
      const int kk = i / (FBN / 2), nn = (i % (FBN / 2)) * 2;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      if (gk < g.K && gn + 1 < g.N) {
        rw[r] = __ldg(reinterpret_cast<const float4*>(W + gk * g.w_ks + gn));
      } else {
        float2 v0 = (gk < g.K && gn < g.N) ? W[gk * g.w_ks + gn] : make_float2(0.f, 0.f);
        rw[r] = make_float4(v0.x, v0.y, 0.f, 0.f);
      }
    }
  };
  auto store_chunk = [&](int buf) {
#pragma unroll
    for (int r = 0; r < NA; ++r) {
      const int i = tid + r * 256;
      *reinterpret_cast<float4*>(&As[buf][i / (FBM / 2)][(i % (FBM / 2)) * 2]) = ra[r];
    }
#pragma unroll
    for (int r = 0; r < NW; ++r) {
      const int i = tid + r * 256;
      const float4 w = rw[r];
      if constexpr (PK) {  // (wr, wi, -wi, wr) per complex W element
        float4* d = reinterpret_cast<float4*>(&Ws[buf][i / (FBN / 2)][(i % (FBN / 2)) * 4]);
        d[0] = make_float4(w.x, w.y, -w.y, w.x);
        d[1] = make_float4(w.z, w.w, -w.w, w.z);
      } else {
        *reinterpret_cast<float4*>(&Ws[buf][i / (FBN / 2)][(i % (FBN / 2)) * 2]) = w;
      }
    }
  };
  float2 acc[TI][TJ];
#pragma unroll
  for (int i = 0; i < TI; ++i)
#pragma unroll
    for (int j = 0; j < TJ; ++j) acc[i][j] = make_float2(0.f, 0.f);
  load_chunk(0);
  store_chunk(0);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = 0; k0 < g.K; k0 += FBK) {
    const bool more = k0 + FBK < g.K;
    if (more) load_chunk(k0 + FBK);
#pragma unroll
    for (int kk = 0; kk < FBK; ++kk) {
      float2 av[TI], bv[TJ];
#pragma unroll
      for (int i = 0; i < TI; ++i) av[i] = As[buf][kk][tm + 16 * i];
      if constexpr (PK) {
        float4 bq[TJ];
#pragma unroll
        for (int j = 0; j < TJ; ++j) bq[j] = *reinterpret_cast<const float4*>(&Ws[buf][kk][2 * (tn + 16 * j)]);
#pragma unroll
        for (int i = 0; i < TI; ++i)
#pragma unroll
          for (int j = 0; j < TJ; ++j) {
            acc[i][j] = fma2(make_float2(av[i].x, av[i].x), make_float2(bq[j].x, bq[j].y), acc[i][j]);
            acc[i][j] = fma2(make_float2(av[i].y, av[i].y), make_float2(bq[j].z, bq[j].w), acc[i][j]);
          }
      } else {
#pragma unroll
      for (int j = 0; j < TJ; ++j) bv[j] = Ws[buf][kk][tn + 16 * j];
#pragma unroll
      for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < TJ; ++j) cmac_s(acc[i][j], av[i], bv[j]);
      }
    }
    if (more) {
      store_chunk(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  float2* C = g.C + b * g.c_bs;
#pragma unroll
  for (int j = 0; j < TJ; ++j) {
    const int64_t gn = n0 + tn + 16 * j;
    if (gn >= g.N) continue;
#pragma unroll
    for (int i = 0; i < TI; ++i) {
      const int64_t gm = m0 + tm + 16 * i;
      if (fold > 1) {
        if (m_ok(gm)) C[(gm / g.M) * g.c_bs + gn * g.c_ns + gm % g.M] = cscale(acc[i][j], g.alpha);
      } else if (gm < g.M) {
        C[gn * g.c_ns + gm] = cscale(acc[i][j], g.alpha);
      }
    }
  }
}

// Gauss / 3M variant of the mode CGEMM: a complex MAC in 3 real FFMAs
// instead of 4.  With s = ar + ai, d = wi - wr, u = wr + wi:
//   t1 += s*wr,  t2 += ar*d,  t3 += ai*u;   Re C = t1 - t3,  Im C = t1 + t2.
// Raw (ar, ai) / (wr, wi) chunks stream global -> shared with cp.async
// (3 stages, no prefetch registers); once a chunk has landed the CTA rewrites
// it as float4 (ar, ai, s) / (wr, d, u) into a double-buffered compute tile,
// so the inner loop is TI + TJ LDS.128 per 3*TI*TJ FFMA (4M: TI + TJ LDS.64
// per 4*TI*TJ).  Same FP32 arithmetic as cgemm.gemm_kloop up to rounding of
// the sums; tests/test_gpu_parity.py holds it to 1e-5 vs float64.
// Measured on B200 (N1024 H256 B1024): 1.70 ms vs 1.46 ms for the 4M 8x8 tile:
// 20% fewer instructions but 56% issue (short-scoreboard on the LDS.128
// operands with one 8-warp CTA per SM), so it stays opt-in
// (TFNO_CGEMM_ALGO=3); profiles/r01/cgemm_3m_vs_4m.txt.
// 16-byte cp.async; bytes < 16 copies the first `bytes` and zero-fills the rest
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gsrc), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int TI, int TJ>
struct G3 {
  static constexpr int FBM = 16 * TI, FBN = 16 * TJ, FBK = 16, NST = 3;
  // float4 units: raw stages hold complex pairs, compute tiles hold one complex + sum
  static constexpr int RAW = FBK * (FBM + FBN) / 2;
  static constexpr int TILE = FBK * (FBM + FBN);
  static constexpr size_t smem() { return sizeof(float4) * ((size_t)NST * RAW + 2 * (size_t)TILE); }
};
template <int TI, int TJ>
constexpr size_t cgemm3m_smem() {
  return G3<TI, TJ>::smem();
}

template <int TI, int TJ>
__global__ void __launch_bounds__(256, 1) cgemm3m_modes_kernel(GemmArgs g) {
  using Q = G3<TI, TJ>;
  constexpr int FBM = Q::FBM, FBN = Q::FBN, FBK = Q::FBK, NST = Q::NST;
  extern __shared__ __align__(16) float4 sm3[];
  float4* raw = sm3;                         // [NST][FBK*FBM/2 (A pairs) + FBK*FBN/2 (W pairs)]
  float4* tile = sm3 + NST * Q::RAW;         // [2][FBK*FBM (A) + FBK*FBN (W)]
  const int tid = threadIdx.x;
  const int tm = tid % 16, tn = tid / 16;
  const int64_t m0 = (int64_t)blockIdx.x * FBM, n0 = (int64_t)blockIdx.y * FBN;
  const int64_t fold = g.fold > 1 ? g.fold : 1;
  const int64_t b = blockIdx.z * fold;
  const float2* __restrict__ A = g.A + b * g.a_bs;
  const float2* __restrict__ W = g.W + (fold > 1 ? 0 : b * g.w_bs);
  auto a_off = [&](int64_t gm) -> int64_t { return fold > 1 ? (gm / g.M) * g.a_bs + gm % g.M : gm; };
  auto m_ok = [&](int64_t gm) { return fold > 1 ? (gm / g.M < fold && b + gm / g.M < g.batch) : gm < g.M; };
  constexpr int PA = FBK * FBM / 2, PW = FBK * FBN / 2;  // 16-byte pieces per chunk
  const int nch = (int)((g.K + FBK - 1) / FBK);
  auto issue = [&](int st, int64_t k0) {
    float4* ra = raw + st * Q::RAW;
    float4* rw = ra + PA;
#pragma unroll
    for (int i = tid; i < PA; i += 256) {
      const int kk = i / (FBM / 2), mm = (i % (FBM / 2)) * 2;
      const int64_t gk = k0 + kk, gm = m0 + mm;
      const int nb = gk >= g.K ? 0 : fold > 1 ? (m_ok(gm) ? 16 : 0) : (gm + 1 < g.M ? 16 : gm < g.M ? 8 : 0);
      cp_async16(ra + i, nb ? (const void*)(A + gk * g.a_ks + a_off(gm)) : (const void*)A, nb);
    }
#pragma unroll
    for (int i = tid; i < PW; i += 256) {
      const int kk = i / (FBN / 2), nn = (i % (FBN / 2)) * 2;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      const int nb = gk >= g.K ? 0 : (gn + 1 < g.N ? 16 : gn < g.N ? 8 : 0);
      cp_async16(rw + i, nb ? (const void*)(W + gk * g.w_ks + gn) : (const void*)W, nb);
    }
  };
  auto transform = [&](int st, int tb) {
    const float4* ra = raw + st * Q::RAW;
    const float4* rw = ra + PA;
    float4* ta = tile + tb * Q::TILE;
    float4* tw = ta + FBK * FBM;
#pragma unroll
    for (int i = tid; i < PA; i += 256) {
      const float4 v = ra[i];
      ta[2 * i] = make_float4(v.x, v.y, v.x + v.y, 0.f);
      ta[2 * i + 1] = make_float4(v.z, v.w, v.z + v.w, 0.f);
    }
#pragma unroll
    for (int i = tid; i < PW; i += 256) {
      const float4 v = rw[i];
      tw[2 * i] = make_float4(v.x, v.y - v.x, v.x + v.y, 0.f);
      tw[2 * i + 1] = make_float4(v.z, v.w - v.z, v.z + v.w, 0.f);
    }
  };
  float t1[TI][TJ], t2[TI][TJ], t3[TI][TJ];
#pragma unroll
  for (int i = 0; i < TI; ++i)
#pragma unroll
    for (int j = 0; j < TJ; ++j) t1[i][j] = t2[i][j] = t3[i][j] = 0.f;
  issue(0, 0);
  cp_async_commit();
  if (nch > 1) issue(1, FBK);
  cp_async_commit();
  cp_async_wait<1>();
  __syncthreads();
  transform(0, 0);
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    if (c + 2 < nch) issue((c + 2) % NST, (int64_t)(c + 2) * FBK);
    cp_async_commit();  // (possibly empty) group c + 2 keeps the wait counts uniform
    const float4* ta = tile + (c & 1) * Q::TILE;
    const float4* tw = ta + FBK * FBM;
#pragma unroll
    for (int kk = 0; kk < FBK; ++kk) {
      float4 av[TI], bv[TJ];
#pragma unroll
      for (int i = 0; i < TI; ++i) av[i] = ta[kk * FBM + tm + 16 * i];
#pragma unroll
      for (int j = 0; j < TJ; ++j) bv[j] = tw[kk * FBN + tn + 16 * j];
#pragma unroll
      for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < TJ; ++j) {
          t1[i][j] = fmaf(av[i].z, bv[j].x, t1[i][j]);
          t2[i][j] = fmaf(av[i].x, bv[j].y, t2[i][j]);
          t3[i][j] = fmaf(av[i].y, bv[j].z, t3[i][j]);
        }
    }
    if (c + 1 < nch) {
      cp_async_wait<1>();  // chunk c + 1 has landed (this thread's pieces)
      __syncthreads();     // ... everyone's, and everyone is done with tile (c + 1) & 1's old data
      transform((c + 1) % NST, (c + 1) & 1);
      __syncthreads();
    }
  }
  float2* C = g.C + b * g.c_bs;
#pragma unroll
  for (int j = 0; j < TJ; ++j) {
    const int64_t gn = n0 + tn + 16 * j;
    if (gn >= g.N) continue;
#pragma unroll
    for (int i = 0; i < TI; ++i) {
      const int64_t gm = m0 + tm + 16 * i;
      const float2 c = make_float2((t1[i][j] - t3[i][j]) * g.alpha, (t1[i][j] + t2[i][j]) * g.alpha);
      if (fold > 1) {
        if (m_ok(gm)) C[(gm / g.M) * g.c_bs + gn * g.c_ns + gm % g.M] = c;
      } else if (gm < g.M) {
        C[gn * g.c_ns + gm] = c;
      }
    }
  }
}

template <int TI, int TJ>
static void launch3m(dim3 grid, const GemmArgs& g, cudaStream_t s) {
  cudaFuncSetAttribute(cgemm3m_modes_kernel<TI, TJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)cgemm3m_smem<TI, TJ>());
  cgemm3m_modes_kernel<TI, TJ><<<grid, 256, cgemm3m_smem<TI, TJ>(), s>>>(g);
}

static bool gemm_packed() {  // TFNO_CGEMM_PACKED=0 selects the scalar 4-FFMA inner loop (A/B)
  const char* e = getenv("TFNO_CGEMM_PACKED");
  return e ? atoi(e) != 0 : true;
}

static int gemm_algo() {  // TFNO_CGEMM_ALGO: 4 = classic 4M product (default), 3 = Gauss 3M (read per call)
  const char* e = getenv("TFNO_CGEMM_ALGO");
  return e ? atoi(e) : 4;
}

static bool big_tiles() {  // TFNO_CGEMM_BIG=0 selects the 64 x 128 tile (A/B runs)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TFNO_CGEMM_BIG");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

static bool small_tiles() {  // TFNO_CGEMM_SMALL=1: 64 x 64 tiles for N <= 64 (more CTAs per wave; A/B)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TFNO_CGEMM_SMALL");
    v = e ? atoi(e) : 0;
  }
  return v != 0;
}

cudaError_t launch_cgemm(const GemmArgs& g, cudaStream_t s) {
  const bool fast = g.a_ms == 1 && g.c_ms == 1 && g.w_ns == 1 && (g.a_ks % 2 == 0) && (g.a_bs % 2 == 0) &&
                    (g.w_ks % 2 == 0) && (g.w_bs % 2 == 0) && g.N > 16 && g.M >= 64 &&
                    ((uintptr_t)g.A % 16 == 0) && ((uintptr_t)g.W % 16 == 0);
  // small M (1D modes): fold batch elements into the M tile; the tile shape
  // follows N (64 x 128 for N > 64, 128 x 64 otherwise: no idle columns)
  const bool wide = g.N > 64;
  const int64_t FBMf = wide ? 64 : 128;
  const bool foldable = g.a_ms == 1 && g.c_ms == 1 && g.w_ns == 1 && g.w_bs == 0 && g.M >= 2 && g.M < FBMf &&
                        (FBMf % g.M == 0) && (g.a_ks % 2 == 0) && (g.a_bs % 2 == 0) && (g.w_ks % 2 == 0) &&
                        ((uintptr_t)g.A % 16 == 0) && ((uintptr_t)g.W % 16 == 0) && g.N > 16;
  const bool g3 = gemm_algo() == 3;
  if (foldable) {
    GemmArgs f = g;
    f.fold = FBMf / g.M;
    dim3 grid(1u, (unsigned)((g.N + (wide ? 127 : 63)) / (wide ? 128 : 64)),
              (unsigned)((g.batch + f.fold - 1) / f.fold));
    if (g3)
      wide ? launch3m<4, 8>(grid, f, s) : launch3m<8, 4>(grid, f, s);
    else if (wide)
      launch_pdl(cgemm_modes_kernel<4, 8>, grid, dim3(256), 0, s, f);
    else
      launch_pdl(cgemm_modes_kernel<8, 4>, grid, dim3(256), 0, s, f);
  } else if (fast && g.N > 64 && g3) {
    dim3 grid((unsigned)((g.M + 63) / 64), (unsigned)((g.N + 127) / 128), (unsigned)g.batch);
    launch3m<4, 8>(grid, g, s);
  } else if (fast && g.M >= 128 && g3) {
    dim3 grid((unsigned)((g.M + 127) / 128), (unsigned)((g.N + 63) / 64), (unsigned)g.batch);
    launch3m<8, 4>(grid, g, s);
  } else if (fast && g.N > 64 && g.M >= 128 && big_tiles()) {
    dim3 grid((unsigned)((g.M + 127) / 128), (unsigned)((g.N + 127) / 128), (unsigned)g.batch);
    if (gemm_packed())
      launch_pdl(cgemm_modes_kernel<8, 8, true>, grid, dim3(256), 0, s, g);
    else
      launch_pdl(cgemm_modes_kernel<8, 8>, grid, dim3(256), 0, s, g);
  } else if (fast && g.N > 64) {
    dim3 grid((unsigned)((g.M + 63) / 64), (unsigned)((g.N + 127) / 128), (unsigned)g.batch);
    launch_pdl(cgemm_modes_kernel<4, 8>, grid, dim3(256), 0, s, g);  // packed form spills at 2 CTAs/SM
  } else if (fast && g.M >= 128 && g.N <= 64 && small_tiles()) {
    dim3 grid((unsigned)((g.M + 63) / 64), (unsigned)((g.N + 63) / 64), (unsigned)g.batch);
    launch_pdl(cgemm_modes_kernel<4, 4>, grid, dim3(256), 0, s, g);
  } else if (fast && g.M >= 128) {
    dim3 grid((unsigned)((g.M + 127) / 128), (unsigned)((g.N + 63) / 64), (unsigned)g.batch);
    launch_pdl(cgemm_modes_kernel<8, 4>, grid, dim3(256), 0, s, g);
  } else {
    dim3 grid((unsigned)((g.M + GBM - 1) / GBM), (unsigned)((g.N + GBN - 1) / GBN), (unsigned)g.batch);
    cgemm_kernel<<<grid, 256, 0, s>>>(g);
  }
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------------
// K4/K5/K6: fused rows kernel
// ------------------------------------------------------------------------
struct RowSrc {  // global rows, contiguous, full length
  const float2* __restrict__ base;
  int64_t sh;
  __device__ __forceinline__ float2 load(int p, int e) const { return base[(int64_t)p * sh + e]; }
};
struct PanelDst {  // A panel As[k][q]
  float2* as;
  int keep;
  __device__ __forceinline__ void store(int p, int o, float2 v) const { as[p * keep + o] = v; }
};
struct ColSrc {  // C tile columns Cs[j][q], zero beyond keep
  const float2* cs;
  int keep, c0;
  __device__ __forceinline__ float2 load(int p, int e) const {
    return e < keep ? cs[(c0 + p) * keep + e] : make_float2(0.f, 0.f);
  }
};
struct RowDst {  // global output rows
  float2* __restrict__ base;
  int64_t sn;
  int c0;
  __device__ __forceinline__ void store(int p, int o, float2 v) const { base[(int64_t)(c0 + p) * sn + o] = v; }
};

size_t fused_smem_bytes(const FusedArgs& a) {
  int PB = a.KC > a.EC ? a.KC : a.EC;
  size_t e = (size_t)a.n + 2 * (size_t)smem_buf_elems(a.n, PB, 0) + (size_t)a.KC * a.keep +
             (size_t)a.KC * a.NT + (size_t)a.NT * a.keep;
  return e * sizeof(float2);
}

template <bool FUSE_FFT, bool FUSE_IFFT>
__global__ void __launch_bounds__(256) fused_rows_kernel(FusedArgs a) {
  extern __shared__ float4 smem_raw[];
  const int n = a.n, keep = a.keep;
  const int PB = a.KC > a.EC ? a.KC : a.EC;
  const int be = smem_buf_elems(n, PB, 0);
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  float2* buf0 = tw + n;
  float2* buf1 = buf0 + be;
  float2* As = buf1 + be;
  float2* Ws = As + a.KC * keep;
  float2* Cs = Ws + a.KC * a.NT;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int64_t g = blockIdx.x;
  const int64_t bb = g / a.gx, pp = g % a.gx;
  const int n0 = blockIdx.y * a.NT;
  const int ntc = min(a.NT, a.N - n0);
  const int MT = (keep + 3) / 4, NTg = (a.NT + 3) / 4;
  const bool gemm_thread = tid < MT * NTg;
  const int tm = tid % MT, tn = tid / MT;
  if (FUSE_FFT || FUSE_IFFT) load_twiddles(tw, a.twg, n, tid, nthr);
  const RadixPlan rp = make_radix_plan(n);
  float2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
  __syncthreads();

  for (int kc = 0; kc < a.H; kc += a.KC) {
    const int kcn = min(a.KC, a.H - kc);
    for (int i = tid; i < a.KC * a.NT; i += nthr) {
      int k = i / a.NT, j = i % a.NT;
      Ws[i] = (k < kcn && j < ntc) ? a.W[(int64_t)(kc + k) * a.N + n0 + j] : make_float2(0.f, 0.f);
    }
    if (FUSE_FFT) {
      // rows of channels kc..kc+kcn -> FFT (keep) -> A panel in smem
      RowSrc src{a.x + bb * a.x_sb + pp * a.x_sp + (int64_t)kc * a.x_sh, a.x_sh};
      fft_block<-1>(rp, kcn, 0, tid, nthr, tw, src, PanelDst{As, keep}, buf0, buf1, keep, 1.0f);
      if (kcn < a.KC) {
        for (int i = tid; i < (a.KC - kcn) * keep; i += nthr) As[kcn * keep + i] = make_float2(0.f, 0.f);
        __syncthreads();
      }
    } else {
      const float2* Ab = a.A + bb * a.a_sb + pp * a.a_sp + (int64_t)kc * a.a_sh;
      for (int i = tid; i < a.KC * keep; i += nthr) {
        int k = i / keep, q = i % keep;
        As[i] = k < kcn ? Ab[(int64_t)k * a.a_sh + q] : make_float2(0.f, 0.f);
      }
      __syncthreads();
    }
    if (gemm_thread) {
      for (int k = 0; k < a.KC; ++k) {
        float2 av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          int q = tm + MT * i;
          av[i] = q < keep ? As[k * keep + q] : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          int c = tn + NTg * j;
          bv[j] = c < a.NT ? Ws[k * a.NT + c] : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) cmac(acc[i][j], av[i], bv[j]);
      }
    }
    __syncthreads();
  }

  if (FUSE_IFFT) {
    if (gemm_thread) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int q = tm + MT * i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          int c = tn + NTg * j;
          if (q < keep && c < a.NT) Cs[c * keep + q] = acc[i][j];
        }
      }
    }
    __syncthreads();
    float2* ybase = a.y + bb * a.y_sb + pp * a.y_sp + (int64_t)n0 * a.y_sn;
    for (int c0 = 0; c0 < ntc; c0 += a.EC) {
      int pb = min(a.EC, ntc - c0);
      fft_block<1>(rp, pb, 0, tid, nthr, tw, ColSrc{Cs, keep, c0}, RowDst{ybase, a.y_sn, c0}, buf0, buf1, n,
                   a.inv_scale);
    }
  } else {
    if (gemm_thread) {
      float2* cbase = a.C + bb * a.c_sb + pp * a.c_sp + (int64_t)n0 * a.c_sn;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int q = tm + MT * i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          int c = tn + NTg * j;
          if (q < keep && c < ntc) cbase[(int64_t)c * a.c_sn + q] = acc[i][j];
        }
      }
    }
  }
}

template <bool F, bool I>
static cudaError_t launch_fused_t(const FusedArgs& a, cudaStream_t s) {
  size_t smem = fused_smem_bytes(a);
  cudaError_t e =
      cudaFuncSetAttribute(fused_rows_kernel<F, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)a.G, (unsigned)((a.N + a.NT - 1) / a.NT));
  fused_rows_kernel<F, I><<<grid, 256, smem, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_fused(const FusedArgs& a, bool fuse_fft, bool fuse_ifft, cudaStream_t s) {
  if (fuse_fft && fuse_ifft) return launch_fused_t<true, true>(a, s);
  if (fuse_fft) return launch_fused_t<true, false>(a, s);
  if (fuse_ifft) return launch_fused_t<false, true>(a, s);
  return launch_fused_t<false, false>(a, s);
}

// ------------------------------------------------------------------------
// plane modulation: out = scale * in * w_TW^{-sign*(sx*x*(TW/dx) + sy*y*(TW/dy)) mod TW}
// (the master table holds exp(-2 pi i k / TW)); float4 = two complex per thread
__global__ void modulate_kernel(const float2* __restrict__ in, float2* __restrict__ out, int64_t total, int dx,
                                int dy, int sx, int sy, int sign, float scale, const float2* __restrict__ tw) {
  const int64_t per = (int64_t)dx * dy;
  const int ux = TFNO_TW_MAX / dx, uy = TFNO_TW_MAX / dy;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i % per);
    const int xx = r / dy, yy = r % dy;
    const int k = (int)(((int64_t)sx * xx * ux + (int64_t)sy * yy * uy) & (TFNO_TW_MAX - 1));
    float2 w = __ldg(&tw[k]);  // exp(-2 pi i k / TW)
    if (sign > 0) w.y = -w.y;  // exp(+2 pi i k / TW)
    out[i] = cscale(cmul(__ldg(&in[i]), w), scale);
  }
}

cudaError_t launch_modulate(const float2* in, float2* out, int64_t planes, int dx, int dy, int sx, int sy, int sign,
                            float scale, const float2* tw, cudaStream_t s) {
  const int64_t total = planes * dx * dy;
  if (total <= 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  modulate_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, out, total, dx, dy, sx, sy, sign, scale, tw);
  ++g_launches;
  return cudaGetLastError();
}

// out[i] = sum over b (ascending, fixed order: deterministic) of in[b][i] -- the batch
// reduction of per-batch-element partial products (grad_W of the backward pass)
__global__ void batch_sum_kernel(const float2* __restrict__ in, int64_t batch, int64_t n, float2* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float2 s = make_float2(0.f, 0.f);
    for (int64_t b = 0; b < batch; ++b) s = cadd(s, __ldg(&in[b * n + i]));
    out[i] = s;
  }
}

cudaError_t launch_batch_sum(const float2* in, int64_t batch, int64_t n, float2* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  batch_sum_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, batch, n, out);
  ++g_launches;
  return cudaGetLastError();
}

// staged baseline copy passes: dst[plane][x][y] = x<cx && y<cy ? scale*src : 0
// ------------------------------------------------------------------------
__global__ void pad_truncate_kernel(const float2* __restrict__ src, int64_t planes, int sx, int sy,
                                    int64_t s_plane, float2* __restrict__ dst, int dx2, int dy2,
                                    int64_t d_plane, int cx, int cy, float scale) {
  const int64_t per = (int64_t)dx2 * dy2;
  const int64_t total = planes * per;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t pl = i / per;
    int r = (int)(i % per);
    int xx = r / dy2, yy = r % dy2;
    float2 v = make_float2(0.f, 0.f);
    if (xx < cx && yy < cy && xx < sx && yy < sy) v = cscale(src[pl * s_plane + (int64_t)xx * sy + yy], scale);
    dst[pl * d_plane + (int64_t)xx * dy2 + yy] = v;
  }
}

cudaError_t launch_pad_truncate(const float2* src, int64_t planes, int sx, int sy, int64_t s_plane, float2* dst,
                                int dx2, int dy2, int64_t d_plane, int cx, int cy, float scale,
                                cudaStream_t s) {
  int64_t total = planes * dx2 * (int64_t)dy2;
  int grid = (int)imin64((total + 255) / 256, 148 * 32);
  if (grid < 1) grid = 1;
  pad_truncate_kernel<<<grid, 256, 0, s>>>(src, planes, sx, sy, s_plane, dst, dx2, dy2, d_plane, cx, cy, scale);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace tfno
