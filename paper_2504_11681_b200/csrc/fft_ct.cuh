// Compile-time-specialised CTA FFT engine (length N a template parameter).
//
// Same semantics as fft_engine.cuh (natural-order Stockham, truncation to
// `keep`, structural zeros beyond `src_len`, reference fft.py:1-21), but
// every radix / stride / mask is a constant:
//   * radix plan N = R0 * 8^k, R0 in {1,2,4} first (its pass has no twiddles);
//   * per-pass twiddle tables laid out [m][j] (j = k mod L fastest) so a warp
//     reads consecutive entries: no bank conflicts;
//   * element-major padded layout e + (e >> 3): the stride-R writes of the
//     early passes and the stride-N/R reads are conflict-free;
//   * last pass pruned: butterflies whose outputs are all >= keep are skipped
//     and, when keep <= L, only the m = 0 output (a twiddled sum) is formed;
//   * first pass pruned for zero-padded inputs (src_len <= N/R0: every output
//     of the butterfly equals its single nonzero input).
#pragma once
#include "common.cuh"

namespace tfno {
namespace ct {

__host__ __device__ constexpr int clog2(int n) { return n <= 1 ? 0 : 1 + clog2(n / 2); }

template <int N>
struct Plan {
  static constexpr int LOGN = clog2(N);
  static constexpr int R0 = (LOGN % 3 == 1) ? 2 : (LOGN % 3 == 2) ? 4 : (N == 1 ? 1 : 8);
  static constexpr int NP = (N == 1) ? 1 : 1 + (LOGN - clog2(R0)) / 3;  // passes
  __host__ __device__ static constexpr int radix(int i) { return i == 0 ? R0 : 8; }
  __host__ __device__ static constexpr int sublen(int i) { return i == 0 ? 1 : R0 * (1 << (3 * (i - 1))); }  // L_i
  // twiddle table offset of pass i (entries m*L + j, m < R, j < L), pass 0 has none
  __host__ __device__ static constexpr int twoff(int i) { return i <= 1 ? 0 : twoff(i - 1) + radix(i - 1) * sublen(i - 1); }
  static constexpr int TWN = twoff(NP);  // total entries
  static constexpr int PSTRIDE = N + N / 8 + 2;  // padded pencil stride (complex)
};

__device__ __forceinline__ int pad(int e) { return e + (e >> 3); }

// Fill the per-pass tables (forward sign) from the master table w_{TW_MAX}^k.
template <int N, int NTH>
__device__ __forceinline__ void build_twiddles(float2* twp, const float2* __restrict__ twg, int tid) {
  using P = Plan<N>;
#pragma unroll
  for (int i = 1; i < P::NP; ++i) {
    constexpr int dummy = 0;
    (void)dummy;
    const int R = P::radix(i), L = P::sublen(i), off = P::twoff(i);
    for (int idx = tid; idx < R * L; idx += NTH) {
      const int m = idx / L, j = idx % L;
      const int e = j * m * (N / (R * L));  // w_{RL}^{jm} = w_N^{jm N/(RL)}
      twp[off + idx] = __ldg(&twg[(size_t)e * (TFNO_TW_MAX / N)]);
    }
  }
}

template <int R, int DIR>
__device__ __forceinline__ void dftR(float2* v) {
  dft<R, DIR>(v);
}

// One pass over PB pencils (p < PB).  Src: float2 load(int p, int e);
// Dst: void store(int p, int o, float2 v).  FIRST: src_len pruning;
// LAST: keep pruning + scale.
template <int N, int I, int DIR, int NTH, bool FIRST, bool LAST, class Src, class Dst>
__device__ __forceinline__ void pass(int PB, int tid, const float2* __restrict__ twp, const Src& src, const Dst& dst,
                                     int keep, int src_len, float scale) {
  using P = Plan<N>;
  constexpr int R = P::radix(I), L = P::sublen(I), NB = N / R, LNB = clog2(NB);
  const float2* tw = twp + P::twoff(I);
  const int total = PB * NB;
  for (int idx = tid; idx < total; idx += NTH) {
    const int p = idx >> LNB, k = idx & (NB - 1);
    const int j = k & (L - 1);
    if (LAST && keep <= L && j >= keep) continue;  // every output of this butterfly is dropped
    float2 v[R];
    if (FIRST && src_len <= NB) {
      // zero-padded input: only m = 0 can be nonzero -> all R outputs equal it
      const float2 x0 = k < src_len ? src.load(p, k) : make_float2(0.f, 0.f);
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = x0;
    } else {
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int e = k + m * NB;
        v[m] = (FIRST && e >= src_len) ? make_float2(0.f, 0.f) : src.load(p, e);
      }
      if (L > 1) {
#pragma unroll
        for (int m = 1; m < R; ++m) v[m] = cmul(v[m], tw_dir<DIR>(tw[m * L + j]));
      }
      if (LAST && keep <= L) {
        float2 s = v[0];
#pragma unroll
        for (int m = 1; m < R; ++m) s = cadd(s, v[m]);
        dst.store(p, j, cscale(s, scale));
        continue;
      }
      dftR<R, DIR>(v);
    }
    if (LAST) {
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int o = j + m * L;
        if (o < keep) dst.store(p, o, cscale(v[m], scale));
      }
    } else {
      const int base = (k - j) * R + j;
#pragma unroll
      for (int m = 0; m < R; ++m) dst.store(p, base + m * L, v[m]);
    }
  }
}

struct PadBuf {  // padded element-major pencil block in shared memory
  float2* b;
  int stride;
  __device__ __forceinline__ float2 load(int p, int e) const { return b[p * stride + pad(e)]; }
  __device__ __forceinline__ void store(int p, int e, float2 v) const { b[p * stride + pad(e)] = v; }
};

template <int N, int I, int DIR, int NTH, class Src, class Dst>
__device__ __forceinline__ void run_from(int PB, int tid, const float2* twp, const Src& src, const Dst& dst,
                                         float2* b0, float2* b1, int keep, int src_len, float scale) {
  using P = Plan<N>;
  if constexpr (I == P::NP - 1) {
    pass<N, I, DIR, NTH, I == 0, true>(PB, tid, twp, src, dst, keep, src_len, scale);
    __syncthreads();
  } else {
    const PadBuf o{b0, P::PSTRIDE};
    pass<N, I, DIR, NTH, I == 0, false>(PB, tid, twp, src, o, keep, src_len, scale);
    __syncthreads();
    run_from<N, I + 1, DIR, NTH>(PB, tid, twp, o, dst, b1, b0, keep, src_len, scale);
  }
}

// Whole transform of PB pencils, src -> dst, ping-ponging b0/b1 (each PB x
// PSTRIDE).  All NTH threads must call; ends with __syncthreads.
template <int N, int DIR, int NTH, class Src, class Dst>
__device__ __forceinline__ void transform(int PB, int tid, const float2* twp, const Src& src, const Dst& dst,
                                          float2* b0, float2* b1, int keep, int src_len, float scale) {
  run_from<N, 0, DIR, NTH>(PB, tid, twp, src, dst, b0, b1, keep, src_len, scale);
}

}  // namespace ct
}  // namespace tfno
