// tcgen05 (5th-gen tensor core) mode contraction for sm_100a:
//   C[b][n][m] = alpha * sum_h A[b][h][m] * W[h][n]      (complex64)
// the channel mix of the Fourier layer (pipeline.py:198-199, cgemm.py:83-95)
// for the TF32 / 3xTF32 precisions (BASELINE C5: "TF32/BF16 tcgen05 CGEMM
// variant vs FP32").
//
// Real embedding without re-layout: K' = 2h + c (c = re/im of A), N' = 2n + c',
//   W'[2h+c][2n+c'] = [[Wr, Wi], [-Wi, Wr]][c][c'],
// so D[m][2n+c'] = (Re, Im) of C[m][n] and an interleaved complex64 A row
// pair is exactly two K' rows.  Per CTA: M tile of 128 modes (TMEM lanes),
// D = 128 x N' fp32 in TMEM (N' = 2N <= 256 columns), K' streamed in chunks
// of 32 through a 2-stage shared-memory ring in the K-major SWIZZLE_NONE
// canonical layout (core matrix = 8 MN rows x 4 K fp32 = 128 B; SBO = 128 B
// between MN groups, LBO between K groups).  One elected thread issues
// tcgen05.mma.cta_group::1.kind::tf32 (M=128, N=N', K=8) x 4 per chunk
// (x3 for 3xTF32: hi*hi + hi*lo + lo*hi, lo = x - tf32(x)) and
// tcgen05.commit's to the stage's mbarrier; the next chunk's global loads are
// already in flight in registers.  Epilogue: tcgen05.ld 32x32b.x32 -> alpha
// -> coalesced complex stores.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.cuh"
#include "tcgen05.cuh"

namespace tfno {



constexpr int TC_BM = 128, TC_BK = 32;  // M tile (TMEM lanes), K' chunk

template <int NP>
struct TcGeo {
  static constexpr int A_TILE = TC_BM * TC_BK * 4;  // bytes of one A tile (hi or lo)
  static constexpr int B_TILE = NP * TC_BK * 4;
  // K-group stride inside a tile: MN-major groups of 8 K hold E/4 core matrices,
  // K-major groups of 4 K hold E/8 core matrices
  static constexpr int TMEM_COLS = NP <= 32 ? 32 : NP <= 64 ? 64 : NP <= 128 ? 128 : 256;
};

// W' image: for every output-channel block nb and K' chunk c, the B tile(s)
// exactly as they sit in shared memory (K-major canonical, hi then lo for
// 3xTF32).  Built once per call by wimg_kernel, then each CTA fetches a
// chunk with one cp.async.bulk instead of converting W element by element.
template <int NP, int PASSES>
__global__ void __launch_bounds__(256) wimg_kernel(GemmArgs g, uint8_t* img) {
  constexpr int B_LBO = (NP / 8) * 128, BT = TcGeo<NP>::B_TILE, CH = (PASSES > 1 ? 2 : 1) * BT;
  const int64_t N = g.N, K = g.K;
  const int nchunks = (int)((2 * K + TC_BK - 1) / TC_BK);
  const int nsplit = (int)((N + NP / 2 - 1) / (NP / 2));
  const int64_t items = (int64_t)nsplit * nchunks * (NP / 2) * (TC_BK / 4);  // (n, channel pair) items
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items; it += (int64_t)gridDim.x * blockDim.x) {
    const int nl = (int)(it % (NP / 2));
    const int hp = (int)((it / (NP / 2)) % (TC_BK / 4));
    const int64_t blk = it / ((NP / 2) * (TC_BK / 4));  // nb * nchunks + c
    const int c = (int)(blk % nchunks);
    const int64_t nb = blk / nchunks;
    const int64_t h = (int64_t)c * (TC_BK / 2) + 2 * hp, n = nb * (NP / 2) + nl;
    const float2 w0 = (n < N && h < K) ? g.W[h * g.w_ks + n] : make_float2(0.f, 0.f);
    const float2 w1 = (n < N && h + 1 < K) ? g.W[(h + 1) * g.w_ks + n] : make_float2(0.f, 0.f);
    const float4 re_row = make_float4(w0.x, -w0.y, w1.x, -w1.y);
    const float4 im_row = make_float4(w0.y, w0.x, w1.y, w1.x);
    uint8_t* base = img + blk * CH;
    const uint32_t o0 = cm_off(2 * nl, 4 * hp, B_LBO), o1 = cm_off(2 * nl + 1, 4 * hp, B_LBO);
    if (PASSES == 1) {
      *reinterpret_cast<float4*>(base + o0) = re_row;
      *reinterpret_cast<float4*>(base + o1) = im_row;
    } else {
      const float4 h0 = hi4(re_row), h1 = hi4(im_row);
      *reinterpret_cast<float4*>(base + o0) = h0;
      *reinterpret_cast<float4*>(base + o1) = h1;
      *reinterpret_cast<float4*>(base + BT + o0) = sub4(re_row, h0);
      *reinterpret_cast<float4*>(base + BT + o1) = sub4(im_row, h1);
    }
  }
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::saddr(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(tc::saddr(dst)),
      "l"(src), "r"(bytes), "r"(tc::saddr(bar))
      : "memory");
}

// W'-image variant: 256 threads stage A (two modes per 16-byte load), one
// thread TMA-copies the chunk's W' tile(s); stage = [A hi | A lo | B hi | B lo].
template <int NP, int PASSES>
__global__ void __launch_bounds__(256, 1) cgemm_tc_img_kernel(GemmArgs g) {
  using Gm = TcGeo<NP>;
  constexpr int A_LBO = (TC_BM / 8) * 128, B_LBO = (NP / 8) * 128;
  constexpr int AT = Gm::A_TILE, BT = Gm::B_TILE, NPASS = PASSES > 1 ? 2 : 1;
  constexpr int STAGE = NPASS * (AT + BT);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* stage_base = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * STAGE);  // [2] MMA done, [2] W' landed
  uint64_t* wbars = bars + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t M = g.M, N = g.N, K = g.K;
  const int mtiles = (int)((M + TC_BM - 1) / TC_BM);
  const int nsplit = (int)((N + NP / 2 - 1) / (NP / 2));
  const int64_t tiles = (int64_t)mtiles * nsplit * g.batch;
  const int nchunks = (int)((2 * K + TC_BK - 1) / TC_BK);
  const uint8_t* img = reinterpret_cast<const uint8_t*>(g.wimg);
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) tc::mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::saddr(tmem_slot)),
                 "n"(Gm::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t IDESC = tc::make_idesc(TC_BM, NP, true);
  // A item = (mode pair, channel pair): A[h][m..m+1], A[h+1][m..m+1] (two float4 loads)
  // -> K-major rows m and m+1 of (re_h, im_h, re_h+1, im_h+1)
  constexpr int AI = (TC_BM / 2) * (TC_BK / 4) / 256;  // 2 items per thread
  float4 ra[AI][2];
  const bool vec = (M % 2 == 0) && (g.a_ks % 2 == 0) && (g.a_bs % 2 == 0);
  auto load_chunk = [&](int64_t tile, int c) {
    const int64_t b = tile / ((int64_t)mtiles * nsplit);
    const int64_t m0 = (tile % mtiles) * TC_BM;
    const int64_t h0 = (int64_t)c * (TC_BK / 2);
    const float2* Ab = g.A + b * g.a_bs;
#pragma unroll
    for (int i = 0; i < AI; ++i) {
      const int idx = tid + i * 256;
      const int mp = idx % (TC_BM / 2), hp = idx / (TC_BM / 2);
      const int64_t m = m0 + 2 * mp, h = h0 + 2 * hp;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int64_t hh = h + r;
        if (hh < K && m + 1 < M && vec) {
          ra[i][r] = __ldg(reinterpret_cast<const float4*>(Ab + hh * g.a_ks + m));
        } else {
          const float2 u0 = (hh < K && m < M) ? __ldg(Ab + hh * g.a_ks + m) : make_float2(0.f, 0.f);
          const float2 u1 = (hh < K && m + 1 < M) ? __ldg(Ab + hh * g.a_ks + m + 1) : make_float2(0.f, 0.f);
          ra[i][r] = make_float4(u0.x, u0.y, u1.x, u1.y);
        }
      }
    }
  };
  auto store_chunk = [&](int st) {
    uint8_t* sA = stage_base + st * STAGE;
#pragma unroll
    for (int i = 0; i < AI; ++i) {
      const int idx = tid + i * 256;
      const int mp = idx % (TC_BM / 2), hp = idx / (TC_BM / 2);
      const float4 v0 = ra[i][0], v1 = ra[i][1];  // (re,im) of m, m+1 at h; at h+1
      const float4 r0 = make_float4(v0.x, v0.y, v1.x, v1.y), r1 = make_float4(v0.z, v0.w, v1.z, v1.w);
      const uint32_t o0 = cm_off(2 * mp, 4 * hp, A_LBO), o1 = cm_off(2 * mp + 1, 4 * hp, A_LBO);
      if (PASSES == 1) {
        *reinterpret_cast<float4*>(sA + o0) = r0;
        *reinterpret_cast<float4*>(sA + o1) = r1;
      } else {
        const float4 h0 = hi4(r0), h1 = hi4(r1);
        *reinterpret_cast<float4*>(sA + o0) = h0;
        *reinterpret_cast<float4*>(sA + o1) = h1;
        *reinterpret_cast<float4*>(sA + AT + o0) = sub4(r0, h0);
        *reinterpret_cast<float4*>(sA + AT + o1) = sub4(r1, h1);
      }
    }
  };
  int64_t gch = 0;
  int64_t tile = blockIdx.x;
  // W' tile(s) of a chunk straight from the image (L2-resident), one chunk ahead:
  // chunk j goes to stage j & 1 once the MMAs of chunk j - 2 have drained
  auto w_issue = [&](int64_t t, int c, int st) {
    const int64_t nbx = (t / mtiles) % nsplit;
    bulk_g2s(stage_base + st * STAGE + NPASS * AT, img + (nbx * nchunks + c) * (int64_t)(NPASS * BT), NPASS * BT,
             &wbars[st]);
  };
  if (tile < tiles) {
    load_chunk(tile, 0);
    if (tid == 0) w_issue(tile, 0, 0);
  }
  for (; tile < tiles; tile += gridDim.x) {
    const int64_t nb = (tile / mtiles) % nsplit;
    for (int c = 0; c < nchunks; ++c, ++gch) {
      const int st = (int)(gch & 1);
      if (gch >= 2) tc::mbar_wait(&bars[st], (uint32_t)(((gch - 2) >> 1) & 1));  // stage free
      store_chunk(st);
      if (c + 1 < nchunks)
        load_chunk(tile, c + 1);
      else if (tile + gridDim.x < tiles)
        load_chunk(tile + gridDim.x, 0);
      tc::fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tc::mbar_wait(&wbars[st], (uint32_t)((gch >> 1) & 1));
        tc::fence_after();
        const uint32_t a0 = tc::saddr(stage_base + st * STAGE);
        const uint32_t al = a0 + AT;
        const uint32_t b0 = a0 + NPASS * AT, bl = b0 + BT;
#pragma unroll
        for (int s = 0; s < TC_BK / 8; ++s) {
          const uint64_t ad = tc::make_desc(a0 + 2 * s * A_LBO, A_LBO, 128);
          const uint64_t bd = tc::make_desc(b0 + 2 * s * B_LBO, B_LBO, 128);
          tc::mma_tf32(tmem, ad, bd, IDESC, (c > 0 || s > 0) ? 1u : 0u);
          if (PASSES > 1) {
            const uint64_t adl = tc::make_desc(al + 2 * s * A_LBO, A_LBO, 128);
            const uint64_t bdl = tc::make_desc(bl + 2 * s * B_LBO, B_LBO, 128);
            tc::mma_tf32(tmem, ad, bdl, IDESC, 1u);
            tc::mma_tf32(tmem, adl, bd, IDESC, 1u);
          }
        }
        tc::commit(&bars[st]);
        // prefetch the next chunk's W' into the other stage once its MMAs (chunk gch - 1) drained
        const bool more = c + 1 < nchunks || tile + gridDim.x < tiles;
        if (more) {
          if (gch >= 1) tc::mbar_wait(&bars[st ^ 1], (uint32_t)(((gch - 1) >> 1) & 1));
          if (c + 1 < nchunks)
            w_issue(tile, c + 1, st ^ 1);
          else
            w_issue(tile + gridDim.x, 0, st ^ 1);
        }
      }
    }
    {
      const int64_t last = gch - 1;
      tc::mbar_wait(&bars[last & 1], (uint32_t)((last >> 1) & 1));
      tc::fence_after();
      const int64_t b = tile / ((int64_t)mtiles * nsplit);
      const int64_t n0 = nb * (NP / 2);
      const int lw = warp & 3;  // TMEM lane quarter of this warp
      const int64_t m = (tile % mtiles) * TC_BM + lw * 32 + lane;
      float2* Cb = g.C + b * g.c_bs;
      const int cbeg = (warp >> 2) * (NP / 2), cend = cbeg + NP / 2;
#pragma unroll 1
      for (int col = cbeg; col < cend; col += 32) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(lw * 32) << 16) + col, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int64_t n = n0 + col / 2 + q;
          if (m < M && n < N) Cb[n * g.c_ns + m] = make_float2(g.alpha * v[2 * q], g.alpha * v[2 * q + 1]);
        }
      }
      tc::fence_before();
      __syncthreads();
    }
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Gm::TMEM_COLS) : "memory");
}

template <int NP, int PASSES>
__global__ void __launch_bounds__(128, 1) cgemm_tc_kernel(GemmArgs g) {
  using Gm = TcGeo<NP>;
  constexpr int A_LBO = (TC_BM / 8) * 128, B_LBO = (NP / 8) * 128;
  constexpr int STAGE = (PASSES > 1 ? 2 : 1) * (Gm::A_TILE + Gm::B_TILE);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* stage_base = smem;  // 2 stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * STAGE);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t M = g.M, N = g.N, K = g.K;  // complex dims: modes, out channels, hidden
  const int mtiles = (int)((M + TC_BM - 1) / TC_BM);
  const int nsplit = (int)((N + NP / 2 - 1) / (NP / 2));    // output-channel blocks of NP/2
  const int64_t tiles = (int64_t)mtiles * nsplit * g.batch;
  const int nchunks = (int)((2 * K + TC_BK - 1) / TC_BK);  // K' = 2K real, 16 channels per chunk

  if (tid == 0) {
    tc::mbar_init(&bars[0], 1);
    tc::mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::saddr(tmem_slot)),
                 "n"(Gm::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t IDESC = tc::make_idesc(TC_BM, NP, true);

  // chunk = 16 channels = 8 channel pairs.  A item (m, pair): A[h][m], A[h+1][m]
  // -> one K-major row (re_h, im_h, re_h+1, im_h+1).  B item (n, pair):
  // W[h][n], W[h+1][n] -> rows n' = 2n (Wr, -Wi, ...) and 2n+1 (Wi, Wr, ...).
  constexpr int AI = TC_BM * 8 / 128;       // 8 A items per thread
  constexpr int BI = (NP / 2) * 8 / 128;    // B items per thread (NP/32)
  float4 ra[AI], rb[BI];

  auto load_chunk = [&](int64_t tile, int c) {
    const int64_t b = tile / ((int64_t)mtiles * nsplit);
    const int64_t m0 = (tile % mtiles) * TC_BM;
    const int64_t n0 = ((tile / mtiles) % nsplit) * (NP / 2);
    const int64_t h0 = (int64_t)c * (TC_BK / 2);
    const float2* Ab = g.A + b * g.a_bs;
#pragma unroll
    for (int i = 0; i < AI; ++i) {
      const int idx = tid + i * 128;
      const int ml = idx % TC_BM, hp = idx / TC_BM;
      const int64_t m = m0 + ml, h = h0 + 2 * hp;
      const float2 v0 = (m < M && h < K) ? __ldg(Ab + h * g.a_ks + m) : make_float2(0.f, 0.f);
      const float2 v1 = (m < M && h + 1 < K) ? __ldg(Ab + (h + 1) * g.a_ks + m) : make_float2(0.f, 0.f);
      ra[i] = make_float4(v0.x, v0.y, v1.x, v1.y);
    }
#pragma unroll
    for (int i = 0; i < BI; ++i) {
      const int idx = tid + i * 128;
      const int nl = idx % (NP / 2), hp = idx / (NP / 2);
      const int64_t h = h0 + 2 * hp, n = n0 + nl;
      const float2 w0 = (n < N && h < K) ? __ldg(g.W + h * g.w_ks + n) : make_float2(0.f, 0.f);
      const float2 w1 = (n < N && h + 1 < K) ? __ldg(g.W + (h + 1) * g.w_ks + n) : make_float2(0.f, 0.f);
      rb[i] = make_float4(w0.x, w0.y, w1.x, w1.y);
    }
  };
  auto store_chunk = [&](int st) {
    uint8_t* sA = stage_base + st * STAGE;
    uint8_t* sB = sA + Gm::A_TILE;
    uint8_t* sAl = sB + Gm::B_TILE;
    uint8_t* sBl = sAl + Gm::A_TILE;
#pragma unroll
    for (int i = 0; i < AI; ++i) {
      const int idx = tid + i * 128;
      const int ml = idx % TC_BM, hp = idx / TC_BM;
      const uint32_t o = cm_off(ml, 4 * hp, A_LBO);
      if (PASSES == 1) {
        *reinterpret_cast<float4*>(sA + o) = ra[i];
      } else {
        const float4 h = hi4(ra[i]);
        *reinterpret_cast<float4*>(sA + o) = h;
        *reinterpret_cast<float4*>(sAl + o) = sub4(ra[i], h);
      }
    }
#pragma unroll
    for (int i = 0; i < BI; ++i) {
      const int idx = tid + i * 128;
      const int nl = idx % (NP / 2), hp = idx / (NP / 2);
      const float4 w = rb[i];  // (Wr_h, Wi_h, Wr_h+1, Wi_h+1)
      const float4 re_row = make_float4(w.x, -w.y, w.z, -w.w);  // n' = 2n   (c' = 0)
      const float4 im_row = make_float4(w.y, w.x, w.w, w.z);    // n' = 2n+1 (c' = 1)
      const uint32_t o0 = cm_off(2 * nl, 4 * hp, B_LBO), o1 = cm_off(2 * nl + 1, 4 * hp, B_LBO);
      if (PASSES == 1) {
        *reinterpret_cast<float4*>(sB + o0) = re_row;
        *reinterpret_cast<float4*>(sB + o1) = im_row;
      } else {
        const float4 h0 = hi4(re_row), h1 = hi4(im_row);
        *reinterpret_cast<float4*>(sB + o0) = h0;
        *reinterpret_cast<float4*>(sB + o1) = h1;
        *reinterpret_cast<float4*>(sBl + o0) = sub4(re_row, h0);
        *reinterpret_cast<float4*>(sBl + o1) = sub4(im_row, h1);
      }
    }
  };

  int64_t gch = 0;  // global chunk counter (stage = gch & 1, parity = (gch >> 1) & 1)
  int64_t tile = blockIdx.x;
  if (tile < tiles) load_chunk(tile, 0);
  for (; tile < tiles; tile += gridDim.x) {
    for (int c = 0; c < nchunks; ++c, ++gch) {
      const int st = (int)(gch & 1);
      if (gch >= 2) tc::mbar_wait(&bars[st], (uint32_t)(((gch - 2) >> 1) & 1));  // stage free
      store_chunk(st);
      // next chunk (or the first chunk of the next tile) in flight during the MMAs
      if (c + 1 < nchunks)
        load_chunk(tile, c + 1);
      else if (tile + gridDim.x < tiles)
        load_chunk(tile + gridDim.x, 0);
      tc::fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after();
        const uint32_t a0 = tc::saddr(stage_base + st * STAGE);
        const uint32_t b0 = a0 + Gm::A_TILE;
        const uint32_t al = b0 + Gm::B_TILE, bl = al + Gm::A_TILE;
#pragma unroll
        for (int s = 0; s < TC_BK / 8; ++s) {  // K = 8 per MMA = 2 K groups
          const uint64_t ad = tc::make_desc(a0 + 2 * s * A_LBO, A_LBO, 128);
          const uint64_t bd = tc::make_desc(b0 + 2 * s * B_LBO, B_LBO, 128);
          tc::mma_tf32(tmem, ad, bd, IDESC, (c > 0 || s > 0) ? 1u : 0u);
          if (PASSES > 1) {
            const uint64_t adl = tc::make_desc(al + 2 * s * A_LBO, A_LBO, 128);
            const uint64_t bdl = tc::make_desc(bl + 2 * s * B_LBO, B_LBO, 128);
            tc::mma_tf32(tmem, ad, bdl, IDESC, 1u);
            tc::mma_tf32(tmem, adl, bd, IDESC, 1u);
          }
        }
        tc::commit(&bars[st]);
      }
    }
    // epilogue: wait for the tile's last MMA batch, TMEM -> registers -> C
    {
      const int64_t last = gch - 1;
      tc::mbar_wait(&bars[last & 1], (uint32_t)((last >> 1) & 1));
      tc::fence_after();
      const int64_t b = tile / ((int64_t)mtiles * nsplit);
      const int64_t n0 = ((tile / mtiles) % nsplit) * (NP / 2);
      const int64_t m = (tile % mtiles) * TC_BM + warp * 32 + lane;
      float2* Cb = g.C + b * g.c_bs;
#pragma unroll 1
      for (int col = 0; col < NP; col += 32) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + col, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int64_t n = n0 + col / 2 + q;
          if (m < M && n < N) Cb[n * g.c_ns + m] = make_float2(g.alpha * v[2 * q], g.alpha * v[2 * q + 1]);
        }
      }
      tc::fence_before();
      __syncthreads();  // TMEM reads done before the next tile's first MMA overwrites D
    }
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Gm::TMEM_COLS) : "memory");
}

// ---------------------------------------------------------------- BF16 variant
// Same structure; kind::f16 with bf16 operands: K = 16 per MMA, K-major core
// matrix = 8 rows x 8 bf16 (16 B), LBO between groups of 8 K.  A item (m, quad
// of 4 channels) = one 16-byte row (re/im of 4 channels); B item (n, quad)
// = rows 2n (Wr, -Wi, ...) and 2n+1 (Wi, Wr, ...).
__device__ __forceinline__ uint32_t cm_off16(int mn, int k, int lbo) {
  return (uint32_t)((k >> 3) * lbo + (mn >> 3) * 128 + (mn & 7) * 16 + (k & 7) * 2);
}

template <int NP>
__global__ void __launch_bounds__(128, 1) cgemm_tc_bf16_kernel(GemmArgs g) {
  using Gm = TcGeo<NP>;
  constexpr int A_TILE = TC_BM * TC_BK * 2, B_TILE = NP * TC_BK * 2;
  constexpr int A_LBO = (TC_BM / 8) * 128, B_LBO = (NP / 8) * 128;
  constexpr int STAGE = A_TILE + B_TILE;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* stage_base = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * STAGE);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t M = g.M, N = g.N, K = g.K;
  const int mtiles = (int)((M + TC_BM - 1) / TC_BM);
  const int nsplit = (int)((N + NP / 2 - 1) / (NP / 2));
  const int64_t tiles = (int64_t)mtiles * nsplit * g.batch;
  const int nchunks = (int)((2 * K + TC_BK - 1) / TC_BK);
  if (tid == 0) {
    tc::mbar_init(&bars[0], 1);
    tc::mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::saddr(tmem_slot)),
                 "n"(Gm::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t IDESC = tc::make_idesc_bf16(TC_BM, NP);
  constexpr int AI = TC_BM * 4 / 128, BI = (NP / 2) * 4 / 128;  // items per thread
  uint4 ra[AI], rb0[BI], rb1[BI];

  auto load_chunk = [&](int64_t tile, int c) {
    const int64_t b = tile / ((int64_t)mtiles * nsplit);
    const int64_t m0 = (tile % mtiles) * TC_BM;
    const int64_t n0 = ((tile / mtiles) % nsplit) * (NP / 2);
    const int64_t h0 = (int64_t)c * (TC_BK / 2);
    const float2* Ab = g.A + b * g.a_bs;
#pragma unroll
    for (int i = 0; i < AI; ++i) {
      const int idx = tid + i * 128;
      const int ml = idx % TC_BM, hq = idx / TC_BM;
      const int64_t m = m0 + ml, h = h0 + 4 * hq;
      float2 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = (m < M && h + q < K) ? __ldg(Ab + (h + q) * g.a_ks + m) : make_float2(0.f, 0.f);
      ra[i] = make_uint4(tc::pack_bf16(v[0].x, v[0].y), tc::pack_bf16(v[1].x, v[1].y), tc::pack_bf16(v[2].x, v[2].y),
                         tc::pack_bf16(v[3].x, v[3].y));
    }
#pragma unroll
    for (int i = 0; i < BI; ++i) {
      const int idx = tid + i * 128;
      const int nl = idx % (NP / 2), hq = idx / (NP / 2);
      const int64_t h = h0 + 4 * hq, n = n0 + nl;
      float2 w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = (n < N && h + q < K) ? __ldg(g.W + (h + q) * g.w_ks + n) : make_float2(0.f, 0.f);
      rb0[i] = make_uint4(tc::pack_bf16(w[0].x, -w[0].y), tc::pack_bf16(w[1].x, -w[1].y),
                          tc::pack_bf16(w[2].x, -w[2].y), tc::pack_bf16(w[3].x, -w[3].y));
      rb1[i] = make_uint4(tc::pack_bf16(w[0].y, w[0].x), tc::pack_bf16(w[1].y, w[1].x),
                          tc::pack_bf16(w[2].y, w[2].x), tc::pack_bf16(w[3].y, w[3].x));
    }
  };
  auto store_chunk = [&](int st) {
    uint8_t* sA = stage_base + st * STAGE;
    uint8_t* sB = sA + A_TILE;
#pragma unroll
    for (int i = 0; i < AI; ++i) {
      const int idx = tid + i * 128;
      const int ml = idx % TC_BM, hq = idx / TC_BM;
      *reinterpret_cast<uint4*>(sA + cm_off16(ml, 8 * hq, A_LBO)) = ra[i];
    }
#pragma unroll
    for (int i = 0; i < BI; ++i) {
      const int idx = tid + i * 128;
      const int nl = idx % (NP / 2), hq = idx / (NP / 2);
      *reinterpret_cast<uint4*>(sB + cm_off16(2 * nl, 8 * hq, B_LBO)) = rb0[i];
      *reinterpret_cast<uint4*>(sB + cm_off16(2 * nl + 1, 8 * hq, B_LBO)) = rb1[i];
    }
  };

  int64_t gch = 0;
  int64_t tile = blockIdx.x;
  if (tile < tiles) load_chunk(tile, 0);
  for (; tile < tiles; tile += gridDim.x) {
    for (int c = 0; c < nchunks; ++c, ++gch) {
      const int st = (int)(gch & 1);
      if (gch >= 2) tc::mbar_wait(&bars[st], (uint32_t)(((gch - 2) >> 1) & 1));
      store_chunk(st);
      if (c + 1 < nchunks)
        load_chunk(tile, c + 1);
      else if (tile + gridDim.x < tiles)
        load_chunk(tile + gridDim.x, 0);
      tc::fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after();
        const uint32_t a0 = tc::saddr(stage_base + st * STAGE), b0 = a0 + A_TILE;
#pragma unroll
        for (int s = 0; s < TC_BK / 16; ++s) {  // K = 16 per MMA = 2 K groups of 8
          const uint64_t ad = tc::make_desc(a0 + 2 * s * A_LBO, A_LBO, 128);
          const uint64_t bd = tc::make_desc(b0 + 2 * s * B_LBO, B_LBO, 128);
          tc::mma_bf16(tmem, ad, bd, IDESC, (c > 0 || s > 0) ? 1u : 0u);
        }
        tc::commit(&bars[st]);
      }
    }
    {
      const int64_t last = gch - 1;
      tc::mbar_wait(&bars[last & 1], (uint32_t)((last >> 1) & 1));
      tc::fence_after();
      const int64_t b = tile / ((int64_t)mtiles * nsplit);
      const int64_t n0 = ((tile / mtiles) % nsplit) * (NP / 2);
      const int64_t m = (tile % mtiles) * TC_BM + warp * 32 + lane;
      float2* Cb = g.C + b * g.c_bs;
#pragma unroll 1
      for (int col = 0; col < NP; col += 32) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + col, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int64_t n = n0 + col / 2 + q;
          if (m < M && n < N) Cb[n * g.c_ns + m] = make_float2(g.alpha * v[2 * q], g.alpha * v[2 * q + 1]);
        }
      }
      tc::fence_before();
      __syncthreads();
    }
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Gm::TMEM_COLS) : "memory");
}

// BF16 W' image: per (output-channel block, K' chunk) the B tile exactly as it
// sits in shared memory (K-major, core matrix 8 rows x 8 bf16): rows 2n =
// (Wr, -Wi) and 2n+1 = (Wi, Wr) per channel.  Built once (per call, or once
// per weight tensor by tfno_prepare_weights).
template <int NP>
__global__ void __launch_bounds__(256) wimg_bf16_kernel(GemmArgs g, uint8_t* img) {
  constexpr int B_LBO = (NP / 8) * 128, BT = NP * TC_BK * 2;
  const int64_t N = g.N, K = g.K;
  const int nchunks = (int)((2 * K + TC_BK - 1) / TC_BK);
  const int nsplit = (int)((N + NP / 2 - 1) / (NP / 2));
  const int64_t items = (int64_t)nsplit * nchunks * (NP / 2) * (TC_BK / 8);  // (n, channel quad)
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items; it += (int64_t)gridDim.x * blockDim.x) {
    const int nl = (int)(it % (NP / 2));
    const int hq = (int)((it / (NP / 2)) % (TC_BK / 8));
    const int64_t blk = it / ((NP / 2) * (TC_BK / 8));
    const int c = (int)(blk % nchunks);
    const int64_t nb = blk / nchunks;
    const int64_t h = (int64_t)c * (TC_BK / 2) + 4 * hq, n = nb * (NP / 2) + nl;
    float2 w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = (n < N && h + q < K) ? g.W[(h + q) * g.w_ks + n] : make_float2(0.f, 0.f);
    uint8_t* base = img + blk * BT;
    *reinterpret_cast<uint4*>(base + cm_off16(2 * nl, 8 * hq, B_LBO)) =
        make_uint4(tc::pack_bf16(w[0].x, -w[0].y), tc::pack_bf16(w[1].x, -w[1].y), tc::pack_bf16(w[2].x, -w[2].y),
                   tc::pack_bf16(w[3].x, -w[3].y));
    *reinterpret_cast<uint4*>(base + cm_off16(2 * nl + 1, 8 * hq, B_LBO)) =
        make_uint4(tc::pack_bf16(w[0].y, w[0].x), tc::pack_bf16(w[1].y, w[1].x), tc::pack_bf16(w[2].y, w[2].x),
                   tc::pack_bf16(w[3].y, w[3].x));
  }
}

// BF16 contraction on the W' image: 256 threads stage A with 16-byte loads
// (mode pair x channel quad per thread), one thread bulk-copies the chunk's
// W' tile one chunk ahead; kind::f16 MMAs (K = 16) into the TMEM accumulator.
template <int NP>
__global__ void __launch_bounds__(256, 1) cgemm_tc_bf16_img_kernel(GemmArgs g) {
  using Gm = TcGeo<NP>;
  constexpr int AT = TC_BM * TC_BK * 2, BT = NP * TC_BK * 2;
  constexpr int A_LBO = (TC_BM / 8) * 128, B_LBO = (NP / 8) * 128;
  constexpr int STAGE = AT + BT;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* stage_base = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * STAGE);  // [2] MMA done, [2] W' landed
  uint64_t* wbars = bars + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t M = g.M, N = g.N, K = g.K;
  const int mtiles = (int)((M + TC_BM - 1) / TC_BM);
  const int nsplit = (int)((N + NP / 2 - 1) / (NP / 2));
  const int64_t tiles = (int64_t)mtiles * nsplit * g.batch;
  const int nchunks = (int)((2 * K + TC_BK - 1) / TC_BK);
  const uint8_t* img = reinterpret_cast<const uint8_t*>(g.wimg);
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) tc::mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::saddr(tmem_slot)),
                 "n"(Gm::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t IDESC = tc::make_idesc_bf16(TC_BM, NP);
  // item = (mode pair mp < 64, channel quad hq < 4): 4 float4 loads -> rows m, m+1
  float4 ra[4];
  const bool vec = (M % 2 == 0) && (g.a_ks % 2 == 0) && (g.a_bs % 2 == 0);
  const int mp = tid % (TC_BM / 2), hq = tid / (TC_BM / 2);
  auto load_chunk = [&](int64_t t, int c) {
    const int64_t b = t / ((int64_t)mtiles * nsplit);
    const int64_t m = (t % mtiles) * TC_BM + 2 * mp;
    const int64_t h = (int64_t)c * (TC_BK / 2) + 4 * hq;
    const float2* Ab = g.A + b * g.a_bs;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t hh = h + q;
      if (hh < K && m + 1 < M && vec) {
        ra[q] = __ldg(reinterpret_cast<const float4*>(Ab + hh * g.a_ks + m));
      } else {
        const float2 u0 = (hh < K && m < M) ? __ldg(Ab + hh * g.a_ks + m) : make_float2(0.f, 0.f);
        const float2 u1 = (hh < K && m + 1 < M) ? __ldg(Ab + hh * g.a_ks + m + 1) : make_float2(0.f, 0.f);
        ra[q] = make_float4(u0.x, u0.y, u1.x, u1.y);
      }
    }
  };
  auto store_chunk = [&](int st) {
    uint8_t* sA = stage_base + st * STAGE;
    *reinterpret_cast<uint4*>(sA + cm_off16(2 * mp, 8 * hq, A_LBO)) =
        make_uint4(tc::pack_bf16(ra[0].x, ra[0].y), tc::pack_bf16(ra[1].x, ra[1].y), tc::pack_bf16(ra[2].x, ra[2].y),
                   tc::pack_bf16(ra[3].x, ra[3].y));
    *reinterpret_cast<uint4*>(sA + cm_off16(2 * mp + 1, 8 * hq, A_LBO)) =
        make_uint4(tc::pack_bf16(ra[0].z, ra[0].w), tc::pack_bf16(ra[1].z, ra[1].w), tc::pack_bf16(ra[2].z, ra[2].w),
                   tc::pack_bf16(ra[3].z, ra[3].w));
  };
  auto w_issue = [&](int64_t t, int c, int st) {
    const int64_t nbx = (t / mtiles) % nsplit;
    bulk_g2s(stage_base + st * STAGE + AT, img + (nbx * nchunks + c) * (int64_t)BT, BT, &wbars[st]);
  };
  int64_t gch = 0;
  int64_t tile = blockIdx.x;
  if (tile < tiles) {
    load_chunk(tile, 0);
    if (tid == 0) w_issue(tile, 0, 0);
  }
  for (; tile < tiles; tile += gridDim.x) {
    const int64_t nb = (tile / mtiles) % nsplit;
    for (int c = 0; c < nchunks; ++c, ++gch) {
      const int st = (int)(gch & 1);
      if (gch >= 2) tc::mbar_wait(&bars[st], (uint32_t)(((gch - 2) >> 1) & 1));  // stage free
      store_chunk(st);
      if (c + 1 < nchunks)
        load_chunk(tile, c + 1);
      else if (tile + gridDim.x < tiles)
        load_chunk(tile + gridDim.x, 0);
      tc::fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tc::mbar_wait(&wbars[st], (uint32_t)((gch >> 1) & 1));
        tc::fence_after();
        const uint32_t a0 = tc::saddr(stage_base + st * STAGE), b0 = a0 + AT;
#pragma unroll
        for (int s = 0; s < TC_BK / 16; ++s) {  // K = 16 per MMA = 2 K groups of 8
          const uint64_t ad = tc::make_desc(a0 + 2 * s * A_LBO, A_LBO, 128);
          const uint64_t bd = tc::make_desc(b0 + 2 * s * B_LBO, B_LBO, 128);
          tc::mma_bf16(tmem, ad, bd, IDESC, (c > 0 || s > 0) ? 1u : 0u);
        }
        tc::commit(&bars[st]);
        const bool more = c + 1 < nchunks || tile + gridDim.x < tiles;
        if (more) {
          if (gch >= 1) tc::mbar_wait(&bars[st ^ 1], (uint32_t)(((gch - 1) >> 1) & 1));
          if (c + 1 < nchunks)
            w_issue(tile, c + 1, st ^ 1);
          else
            w_issue(tile + gridDim.x, 0, st ^ 1);
        }
      }
    }
    {
      const int64_t last = gch - 1;
      tc::mbar_wait(&bars[last & 1], (uint32_t)((last >> 1) & 1));
      tc::fence_after();
      const int64_t b = tile / ((int64_t)mtiles * nsplit);
      const int64_t n0 = nb * (NP / 2);
      const int lw = warp & 3;
      const int64_t m = (tile % mtiles) * TC_BM + lw * 32 + lane;
      float2* Cb = g.C + b * g.c_bs;
      const int cbeg = (warp >> 2) * (NP / 2), cend = cbeg + NP / 2;
#pragma unroll 1
      for (int col = cbeg; col < cend; col += 32) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(lw * 32) << 16) + col, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int64_t n = n0 + col / 2 + q;
          if (m < M && n < N) Cb[n * g.c_ns + m] = make_float2(g.alpha * v[2 * q], g.alpha * v[2 * q + 1]);
        }
      }
      tc::fence_before();
      __syncthreads();
    }
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Gm::TMEM_COLS) : "memory");
}

template <int NP>
static cudaError_t launch_tc_bf16_t(const GemmArgs& g, cudaStream_t s) {
  const size_t smem = 2 * (TC_BM * TC_BK * 2 + NP * TC_BK * 2) + 64;
  cudaError_t e =
      cudaFuncSetAttribute(cgemm_tc_bf16_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = ((g.M + TC_BM - 1) / TC_BM) * ((g.N + NP / 2 - 1) / (NP / 2)) * g.batch;
  const int grid = (int)(tiles < sms ? tiles : sms);
  cgemm_tc_bf16_kernel<NP><<<grid, 128, smem, s>>>(g);
  ++g_launches;
  return cudaGetLastError();
}

template <int NP, int PASSES>
static cudaError_t launch_tc_t(const GemmArgs& g, cudaStream_t s) {
  constexpr int STAGE = (PASSES > 1 ? 2 : 1) * (TcGeo<NP>::A_TILE + TcGeo<NP>::B_TILE);
  const size_t smem = 2 * STAGE + 64;
  cudaError_t e =
      cudaFuncSetAttribute(cgemm_tc_kernel<NP, PASSES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int sms = device_sms();
  const int64_t tiles = ((g.M + TC_BM - 1) / TC_BM) * ((g.N + NP / 2 - 1) / (NP / 2)) * g.batch;
  const int grid = (int)(tiles < sms ? tiles : sms);
  cgemm_tc_kernel<NP, PASSES><<<grid, 128, smem, s>>>(g);
  ++g_launches;
  return cudaGetLastError();
}

template <int NP>
static size_t wimg_bytes_np(int64_t N, int64_t K, int passes) {
  const int64_t nchunks = (2 * K + TC_BK - 1) / TC_BK, nsplit = (N + NP / 2 - 1) / (NP / 2);
  return (size_t)(nsplit * nchunks * (passes > 1 ? 2 : 1) * TcGeo<NP>::B_TILE);
}

template <int NP>
static size_t wimg_bf16_bytes_np(int64_t N, int64_t K) {
  const int64_t nchunks = (2 * K + TC_BK - 1) / TC_BK, nsplit = (N + NP / 2 - 1) / (NP / 2);
  return (size_t)(nsplit * nchunks * NP * TC_BK * 2);
}

size_t cgemm_tc_wimg_bytes(int64_t N, int64_t K, int prec) {
  const int np = (int)(2 * N);
  if (prec == 2)  // BF16
    return np <= 64 ? wimg_bf16_bytes_np<64>(N, K) : np <= 128 ? wimg_bf16_bytes_np<128>(N, K)
                                                              : wimg_bf16_bytes_np<256>(N, K);
  if (prec != 1 && prec != 3) return 0;  // TF32 / 3xTF32
  const int passes = prec == 1 ? 1 : 3;
  return np <= 64 ? wimg_bytes_np<64>(N, K, passes) : np <= 128 ? wimg_bytes_np<128>(N, K, passes)
                                                                 : wimg_bytes_np<256>(N, K, passes);
}

// W' image builders (also the body of tfno_prepare_weights)
template <int NP, int PASSES>
static cudaError_t build_wimg_t(const GemmArgs& g, void* img, cudaStream_t s) {
  const int sms = device_sms();
  const int64_t nchunks = (2 * g.K + TC_BK - 1) / TC_BK, nsplit = (g.N + NP / 2 - 1) / (NP / 2);
  const int64_t items = nsplit * nchunks * (NP / 2) * (TC_BK / (PASSES == 0 ? 8 : 4));
  const int grid = (int)((items + 255) / 256 < 4 * sms ? (items + 255) / 256 : 4 * sms);
  if (PASSES == 0)
    wimg_bf16_kernel<NP><<<grid, 256, 0, s>>>(g, reinterpret_cast<uint8_t*>(img));
  else
    wimg_kernel<NP, (PASSES == 0 ? 1 : PASSES)><<<grid, 256, 0, s>>>(g, reinterpret_cast<uint8_t*>(img));
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t build_cgemm_wimg(const GemmArgs& g, int prec, void* img, cudaStream_t s) {
  if (!cgemm_tc_supported(g) || (prec != 1 && prec != 2 && prec != 3) || !img || ((uintptr_t)img & 15))
    return cudaErrorNotSupported;
  const int np = (int)(2 * g.N);
  const int passes = prec == 2 ? 0 : prec == 1 ? 1 : 3;
#define TFNO_WB(NPV)                                              \
  if (passes == 0) return build_wimg_t<NPV, 0>(g, img, s);       \
  if (passes == 1) return build_wimg_t<NPV, 1>(g, img, s);       \
  return build_wimg_t<NPV, 3>(g, img, s);
  if (np <= 64) { TFNO_WB(64) }
  if (np <= 128) { TFNO_WB(128) }
  TFNO_WB(256)
#undef TFNO_WB
}

// contraction on a W' image in g.wimg: built here first unless g.wimg_ready
// (tfno_prepare_weights built it once for this weight tensor).  PASSES 0 = BF16.
template <int NP, int PASSES>
static cudaError_t launch_tc_img_t(const GemmArgs& g, cudaStream_t s) {
  constexpr int STAGE = PASSES == 0 ? TC_BM * TC_BK * 2 + NP * TC_BK * 2
                                    : (PASSES > 1 ? 2 : 1) * (TcGeo<NP>::A_TILE + TcGeo<NP>::B_TILE);
  const size_t smem = 2 * STAGE + 128;
  const int sms = device_sms();
  cudaError_t e;
  if (!g.wimg_ready && (e = build_wimg_t<NP, PASSES>(g, g.wimg, s)) != cudaSuccess) return e;
  auto kern = PASSES == 0 ? cgemm_tc_bf16_img_kernel<NP> : cgemm_tc_img_kernel<NP, (PASSES == 0 ? 1 : PASSES)>;
  if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
    return e;
  const int64_t tiles = ((g.M + TC_BM - 1) / TC_BM) * ((g.N + NP / 2 - 1) / (NP / 2)) * g.batch;
  const int grid = (int)(tiles < sms ? tiles : sms);
  kern<<<grid, 256, smem, s>>>(g);
  ++g_launches;
  return cudaGetLastError();
}

bool cgemm_tc_supported(const GemmArgs& g) {
  return g.a_ms == 1 && g.c_ms == 1 && g.w_ns == 1 && g.w_bs == 0 && g.N >= 1;
}

cudaError_t launch_cgemm_tc(const GemmArgs& g, int passes, cudaStream_t s) {
  if (!cgemm_tc_supported(g)) return cudaErrorNotSupported;
  const int np = (int)(2 * g.N);
  if (passes == 0 && g.wimg && (uintptr_t)g.wimg % 16 == 0) {  // BF16 on the W' image
    if (np <= 64) return launch_tc_img_t<64, 0>(g, s);
    if (np <= 128) return launch_tc_img_t<128, 0>(g, s);
    return launch_tc_img_t<256, 0>(g, s);
  }
  if (passes == 0) {  // BF16 operands, W' converted per CTA
    if (np <= 64) return launch_tc_bf16_t<64>(g, s);
    if (np <= 128) return launch_tc_bf16_t<128>(g, s);
    return launch_tc_bf16_t<256>(g, s);
  }
  if (g.wimg && (uintptr_t)g.wimg % 16 == 0) {  // W' image in caller scratch
    if (passes == 1) {
      if (np <= 64) return launch_tc_img_t<64, 1>(g, s);
      if (np <= 128) return launch_tc_img_t<128, 1>(g, s);
      return launch_tc_img_t<256, 1>(g, s);
    }
    if (np <= 64) return launch_tc_img_t<64, 3>(g, s);
    if (np <= 128) return launch_tc_img_t<128, 3>(g, s);
    return launch_tc_img_t<256, 3>(g, s);
  }
  if (passes == 1) {
    if (np <= 64) return launch_tc_t<64, 1>(g, s);
    if (np <= 128) return launch_tc_t<128, 1>(g, s);
    return launch_tc_t<256, 1>(g, s);
  }
  if (np <= 64) return launch_tc_t<64, 3>(g, s);
  if (np <= 128) return launch_tc_t<128, 3>(g, s);
  return launch_tc_t<256, 3>(g, s);
}

}  // namespace tfno
