// CTA-cooperative mixed-radix (8/4/2) Stockham FFT engine with built-in
// truncation (keep) and input pruning (src_len).
//
// Semantics follow the reference transform (fnofuse/fft.py:1-21, 212-239):
// natural-order, unnormalised forward, inverse scaled by 1/n, only the first
// `keep` bins are produced and inputs at index >= src_len are structural
// zeros.  Our radix/order differs from the reference's radix-2 stages; parity
// is tolerance-based.
//
// Pass (radix R, sub-length L): butterfly k in [0, n/R), j = k mod L, inputs
// in[k + m n/R] * w_{LR}^{j m}, R-point DFT, outputs out[(k-j)R + j + m L].
// The last pass has L = n/R, so out index = j + m L and indices >= keep are
// never stored.  The first pass reads straight from the caller's source
// functor (global memory or a shared-memory panel) and applies src_len
// masking there; the last pass writes straight into the destination functor.
#pragma once
#include "common.cuh"

namespace tfno {

struct RadixPlan {
  int n, nr;
  int r[8];
};

__host__ __device__ inline RadixPlan make_radix_plan(int n) {
  RadixPlan p;
  p.n = n;
  p.nr = 0;
  int rem = n;
  // small radix first (its pass has L = 1: no twiddles)
  int lg = ilog2(n);
  int rest = lg % 3;
  if (rest == 1 && lg >= 1) {
    p.r[p.nr++] = 2;
    rem >>= 1;
  } else if (rest == 2) {
    p.r[p.nr++] = 4;
    rem >>= 2;
  }
  while (rem > 1) {
    p.r[p.nr++] = 8;
    rem >>= 3;
  }
  if (p.nr == 0) p.r[p.nr++] = 1;  // n == 1
  return p;
}

// shared-memory pencil buffer: element (p, e) of a PB x n block
struct SmemBuf {
  float2* base;
  int n, PB, pencil_major;
  __device__ __forceinline__ int idx(int p, int e) const {
    return pencil_major ? e * PB + p : p * (n + (n >= 32 ? 1 : 0)) + e;
  }
  __device__ __forceinline__ float2 load(int p, int e) const { return base[idx(p, e)]; }
  __device__ __forceinline__ void store(int p, int e, float2 v) const { base[idx(p, e)] = v; }
};

__host__ __device__ inline int smem_buf_elems(int n, int PB, int pencil_major) {
  return pencil_major ? n * PB : PB * (n + (n >= 32 ? 1 : 0));
}

// One radix-R pass.  Src: float2 load(int p, int e) (e < n; handles src_len);
// Dst: void store(int p, int o, float2 v).  tw: shared table w_n^k, k < n.
template <int R, int DIR, class Src, class Dst>
__device__ __forceinline__ void fft_pass(int n, int L, int PB, int pencil_major, int tid, int nthr,
                                         const float2* __restrict__ tw, const Src& src, const Dst& dst,
                                         bool last, int keep, float scale) {
  const int nb = n / R;
  const int total = PB * nb;
  const int twstep = n / (L * R);
  for (int idx = tid; idx < total; idx += nthr) {
    int p, k;
    if (pencil_major) {
      p = idx % PB;
      k = idx / PB;
    } else {
      k = idx % nb;
      p = idx / nb;
    }
    const int j = k & (L - 1);
    float2 v[R];
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = src.load(p, k + m * nb);
    if (L > 1) {
#pragma unroll
      for (int m = 1; m < R; ++m) v[m] = cmul(v[m], tw_dir<DIR>(tw[j * m * twstep]));
    }
    dft<R, DIR>(v);
    if (last) {
#pragma unroll
      for (int m = 0; m < R; ++m) {
        int o = j + m * L;
        if (o < keep) dst.store(p, o, scale == 1.0f ? v[m] : cscale(v[m], scale));
      }
    } else {
      const int base = (k - j) * R + j;
#pragma unroll
      for (int m = 0; m < R; ++m) dst.store(p, base + m * L, v[m]);
    }
  }
}

template <int DIR, class Src, class Dst>
__device__ __forceinline__ void fft_pass_r(int R, int n, int L, int PB, int pm, int tid, int nthr,
                                           const float2* tw, const Src& src, const Dst& dst, bool last,
                                           int keep, float scale) {
  switch (R) {
    case 8: fft_pass<8, DIR>(n, L, PB, pm, tid, nthr, tw, src, dst, last, keep, scale); break;
    case 4: fft_pass<4, DIR>(n, L, PB, pm, tid, nthr, tw, src, dst, last, keep, scale); break;
    case 2: fft_pass<2, DIR>(n, L, PB, pm, tid, nthr, tw, src, dst, last, keep, scale); break;
    default: fft_pass<1, DIR>(n, L, PB, pm, tid, nthr, tw, src, dst, last, keep, scale); break;
  }
}

struct SmemSrc {
  SmemBuf b;
  __device__ __forceinline__ float2 load(int p, int e) const { return b.load(p, e); }
};
struct SmemDst {
  SmemBuf b;
  __device__ __forceinline__ void store(int p, int e, float2 v) const { b.store(p, e, v); }
};

// Full transform of PB pencils: src -> (buf0/buf1 ping-pong) -> dst.
// Must be called by all nthr threads of the CTA (contains __syncthreads).
// On return, dst has been written; a trailing __syncthreads is included.
template <int DIR, class Src, class Dst>
__device__ void fft_block(const RadixPlan& rp, int PB, int pencil_major, int tid, int nthr,
                          const float2* tw, const Src& src, const Dst& dst, float2* buf0, float2* buf1,
                          int keep, float scale) {
  const int n = rp.n;
  SmemBuf b0{buf0, n, PB, pencil_major}, b1{buf1, n, PB, pencil_major};
  if (rp.nr == 1) {
    fft_pass_r<DIR>(rp.r[0], n, 1, PB, pencil_major, tid, nthr, tw, src, dst, true, keep, scale);
    __syncthreads();
    return;
  }
  int L = 1;
  fft_pass_r<DIR>(rp.r[0], n, L, PB, pencil_major, tid, nthr, tw, src, SmemDst{b0}, false, keep, scale);
  __syncthreads();
  L *= rp.r[0];
  bool in0 = true;
  for (int i = 1; i < rp.nr - 1; ++i) {
    if (in0)
      fft_pass_r<DIR>(rp.r[i], n, L, PB, pencil_major, tid, nthr, tw, SmemSrc{b0}, SmemDst{b1}, false, keep, scale);
    else
      fft_pass_r<DIR>(rp.r[i], n, L, PB, pencil_major, tid, nthr, tw, SmemSrc{b1}, SmemDst{b0}, false, keep, scale);
    __syncthreads();
    L *= rp.r[i];
    in0 = !in0;
  }
  if (in0)
    fft_pass_r<DIR>(rp.r[rp.nr - 1], n, L, PB, pencil_major, tid, nthr, tw, SmemSrc{b0}, dst, true, keep, scale);
  else
    fft_pass_r<DIR>(rp.r[rp.nr - 1], n, L, PB, pencil_major, tid, nthr, tw, SmemSrc{b1}, dst, true, keep, scale);
  __syncthreads();
}

// copy w_n^k (k < n) from the global master table (w_{TW_MAX}^k) into smem
__device__ __forceinline__ void load_twiddles(float2* tw_s, const float2* __restrict__ tw_g, int n, int tid,
                                              int nthr) {
  const int stride = TFNO_TW_MAX / n;
  for (int k = tid; k < n; k += nthr) tw_s[k] = __ldg(&tw_g[(size_t)k * stride]);
}

}  // namespace tfno
