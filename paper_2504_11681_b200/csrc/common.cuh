// Shared device helpers for the TurboFNO B200 kernels (sm_100a).
//
// Element type everywhere is complex64 = float2 (re, im), matching the
// reference's COMPLEX_DTYPE (fnofuse/core.py:17-19).  Twiddles come from one
// table of omega_{TW_MAX}^k built in double precision on the host and rounded
// to fp32 (the reference builds its per-stage twiddles the same way,
// fnofuse/fft.py:114-124).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define TFNO_TW_LOG2 13
#define TFNO_TW_MAX (1 << TFNO_TW_LOG2)   // largest supported transform length

namespace tfno {

// ---- complex arithmetic --------------------------------------------------
// Blackwell issues packed FP32 (FADD2 / FMUL2 / FFMA2 on a register pair, with
// broadcast (.F32), swap (.LO_HI) and negation operand modifiers).  A packed
// instruction takes two FP32-pipe cycles but ONE issue slot, and the FFT /
// CGEMM kernels here are issue-bound (ncu: ~60% issue, 66% FP instructions),
// so the complex primitives are written on f32x2 (tools/probes/ffma2_probe.cu
// measured FFMA2 at the FFMA FLOP rate).  -DTFNO_SCALAR_COMPLEX restores the
// scalar forms for A/B.  Results are IEEE FP32 either way; only the operation
// grouping inside cmul/cmac differs (which product is rounded before the FMA).
#ifndef TFNO_SCALAR_COMPLEX
typedef unsigned long long tfno_pair;
__device__ __forceinline__ tfno_pair pk2(float2 v) {
  tfno_pair r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
__device__ __forceinline__ float2 upk2(tfno_pair v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  tfno_pair r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  tfno_pair r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  tfno_pair r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(r);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  tfno_pair r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
  return upk2(r);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return add2(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return sub2(a, b); }
// a * b: (a.x, a.x) * (b.x, b.y) + (a.y, a.y) * (-b.y, b.x)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return fma2(make_float2(a.y, a.y), make_float2(-b.y, b.x), mul2(make_float2(a.x, a.x), b));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return mul2(a, make_float2(s, s)); }
// acc += a * b (2 FFMA2 + the (-b.y, b.x) companion, shared across uses of b)
__device__ __forceinline__ void cmac(float2& acc, float2 a, float2 b) {
  acc = fma2(make_float2(a.x, a.x), b, acc);
  acc = fma2(make_float2(a.y, a.y), make_float2(-b.y, b.x), acc);
}
#else
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// acc += a * b (4 FFMA)
__device__ __forceinline__ void cmac(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}
#endif
// scalar 4-FFMA complex MAC: the SIMT mode CGEMMs are FMA-pipe-bound, where the
// packed form measured slower (C4 contraction 1.46 -> 1.54 ms)
__device__ __forceinline__ void cmac_s(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }
// loop-invariant twiddle with its companion (-b.y, b.x) precomputed: a * b is one
// FMUL2 + one FFMA2 (built per use, the companion costs a MOV + an FADD)
struct twp {
  float2 b, c;
};
__device__ __forceinline__ twp make_twp(float2 b) { return twp{b, make_float2(-b.y, b.x)}; }
__device__ __forceinline__ float2 cmul_p(float2 a, const twp& t) {
#ifndef TFNO_SCALAR_COMPLEX
  return fma2(make_float2(a.y, a.y), t.c, mul2(make_float2(a.x, a.x), t.b));
#else
  return cmul(a, t.b);
#endif
}
// a * (wr + i wi) for a compile-time constant: swap(a) * (-wi, wi) + a * wr
// (the swap is an operand modifier, wr a broadcast immediate)
__device__ __forceinline__ float2 cmul_k(float2 a, float wr, float wi) {
#ifndef TFNO_SCALAR_COMPLEX
  return fma2(make_float2(a.y, a.x), make_float2(-wi, wi), mul2(a, make_float2(wr, wr)));
#else
  return cmul(a, make_float2(wr, wi));
#endif
}
// multiply by -i (forward, DIR = -1) or +i (inverse, DIR = +1)
template <int DIR>
__device__ __forceinline__ float2 mul_dir_i(float2 a) {
  return DIR < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
}
// x +/- (DIR i) y: one packed FMA with the swapped y and a (+1, -1) sign pair
template <int DIR>
__device__ __forceinline__ float2 cadd_dir_i(float2 x, float2 y) {
#ifndef TFNO_SCALAR_COMPLEX
  return fma2(make_float2(y.y, y.x), DIR < 0 ? make_float2(1.f, -1.f) : make_float2(-1.f, 1.f), x);
#else
  return cadd(x, mul_dir_i<DIR>(y));
#endif
}
template <int DIR>
__device__ __forceinline__ float2 csub_dir_i(float2 x, float2 y) {
#ifndef TFNO_SCALAR_COMPLEX
  return fma2(make_float2(y.y, y.x), DIR < 0 ? make_float2(-1.f, 1.f) : make_float2(1.f, -1.f), x);
#else
  return csub(x, mul_dir_i<DIR>(y));
#endif
}

// twiddle omega_n^k for direction DIR from the forward table of length n
// (tw[k] = exp(-2 pi i k / n)); the inverse is the conjugate.
template <int DIR>
__device__ __forceinline__ float2 tw_dir(float2 t) { return DIR < 0 ? t : conjf2(t); }

// ---- in-register DFTs, natural-order output, y_m = sum_k x_k w_R^{DIR*m*k} ----
template <int DIR>
__device__ __forceinline__ void dft2(float2& a, float2& b) {
  float2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <int DIR>
__device__ __forceinline__ void dft4(float2& x0, float2& x1, float2& x2, float2& x3) {
  const float2 t0 = cadd(x0, x2), t1 = csub(x0, x2);
  const float2 t2 = cadd(x1, x3), d = csub(x1, x3);
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd_dir_i<DIR>(t1, d);  // t1 + (DIR i) d
  x3 = csub_dir_i<DIR>(t1, d);
}

template <int DIR>
__device__ __forceinline__ void dft8(float2* v) {
  const float r = 0.70710678118654752440f;
  float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  float2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<DIR>(e0, e1, e2, e3);
  dft4<DIR>(o0, o1, o2, o3);
  // o1 *= w8^1 = (1 + DIR i)/sqrt2, o3 *= w8^3 = (-1 + DIR i)/sqrt2, o2 *= w8^2 = DIR i
  const float2 t1 = cscale(cadd_dir_i<DIR>(o1, o1), r);
  const float2 t3 = cscale(csub(mul_dir_i<DIR>(o3), o3), r);
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, t1);
  v[5] = csub(e1, t1);
  v[2] = cadd_dir_i<DIR>(e2, o2);
  v[6] = csub_dir_i<DIR>(e2, o2);
  v[3] = cadd(e3, t3);
  v[7] = csub(e3, t3);
}

// 16-point DFT, natural order in and out: n = n1 + 4 n2, k = k1 + 4 k2 --
// four radix-4 DFTs over n2, twiddles w16^{n1 k1}, four radix-4 DFTs over n1
// (the final 4x4 transpose is register renaming).
template <int DIR>
__device__ __forceinline__ void dft16(float2* v) {
  const float c1 = 0.92387953251128675613f, s1 = 0.38268343236508977173f, r2 = 0.70710678118654752440f;
  const float d = (float)DIR;
#pragma unroll
  for (int n1 = 0; n1 < 4; ++n1) dft4<DIR>(v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]);
  // Y[n1][k1] now at v[n1 + 4 k1]; twiddle w16^{n1 k1}
  v[1 + 4] = cmul_k(v[1 + 4], c1, d * s1);     // w^1
  v[1 + 8] = cmul_k(v[1 + 8], r2, d * r2);     // w^2
  v[1 + 12] = cmul_k(v[1 + 12], s1, d * c1);   // w^3
  v[2 + 4] = cmul_k(v[2 + 4], r2, d * r2);     // w^2
  v[2 + 8] = mul_dir_i<DIR>(v[2 + 8]);                    // w^4 = DIR i
  v[2 + 12] = cmul_k(v[2 + 12], -r2, d * r2);  // w^6
  v[3 + 4] = cmul_k(v[3 + 4], s1, d * c1);     // w^3
  v[3 + 8] = cmul_k(v[3 + 8], -r2, d * r2);    // w^6
  v[3 + 12] = cmul_k(v[3 + 12], -c1, -d * s1); // w^9
  float2 o[16];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    float2 y0 = v[0 + 4 * k1], y1 = v[1 + 4 * k1], y2 = v[2 + 4 * k1], y3 = v[3 + 4 * k1];
    dft4<DIR>(y0, y1, y2, y3);
    o[k1] = y0;
    o[k1 + 4] = y1;
    o[k1 + 8] = y2;
    o[k1 + 12] = y3;
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = o[k];
}

// ---- input-pruned DFTs: inputs n >= NIN are known zeros (no adds of zeros;
// unused outputs are removed by the compiler anyway)
template <int DIR, int NIN>
__device__ __forceinline__ void dft4_in(float2& x0, float2& x1, float2& x2, float2& x3) {
  if constexpr (NIN >= 4) {
    dft4<DIR>(x0, x1, x2, x3);
  } else if constexpr (NIN == 3) {
    const float2 t0 = cadd(x0, x2), t1 = csub(x0, x2);
    x0 = cadd(t0, x1);
    x2 = csub(t0, x1);
    const float2 a = cadd_dir_i<DIR>(t1, x1), b = csub_dir_i<DIR>(t1, x1);
    x1 = a;
    x3 = b;
  } else if constexpr (NIN == 2) {
    const float2 a = x0, b = x1;
    x0 = cadd(a, b);
    x2 = csub(a, b);
    x1 = cadd_dir_i<DIR>(a, b);
    x3 = csub_dir_i<DIR>(a, b);
  } else if constexpr (NIN == 1) {
    x1 = x0;
    x2 = x0;
    x3 = x0;
  } else {
    x0 = x1 = x2 = x3 = make_float2(0.f, 0.f);
  }
}

template <int DIR, int NIN>
__device__ __forceinline__ void dft8_in(float2* v) {
  if constexpr (NIN >= 8) {
    dft8<DIR>(v);
  } else {
    constexpr int NE = (NIN + 1) / 2, NO = NIN / 2;
    const float r = 0.70710678118654752440f;
    float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    float2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4_in<DIR, NE>(e0, e1, e2, e3);
    if constexpr (NO == 0) {
      v[0] = v[4] = e0;
      v[1] = v[5] = e1;
      v[2] = v[6] = e2;
      v[3] = v[7] = e3;
    } else {
      dft4_in<DIR, NO>(o0, o1, o2, o3);
      const float2 t1 = cscale(cadd_dir_i<DIR>(o1, o1), r);
      const float2 t3 = cscale(csub(mul_dir_i<DIR>(o3), o3), r);
      v[0] = cadd(e0, o0);
      v[4] = csub(e0, o0);
      v[1] = cadd(e1, t1);
      v[5] = csub(e1, t1);
      v[2] = cadd_dir_i<DIR>(e2, o2);
      v[6] = csub_dir_i<DIR>(e2, o2);
      v[3] = cadd(e3, t3);
      v[7] = csub(e3, t3);
    }
  }
}

template <int DIR, int NIN>
__device__ __forceinline__ void dft16_in(float2* v) {
  if constexpr (NIN >= 16) {
    dft16<DIR>(v);
  } else {
    const float c1 = 0.92387953251128675613f, s1 = 0.38268343236508977173f, r2 = 0.70710678118654752440f;
    const float d = (float)DIR;
    // step 1: radix 4 over n2 for each n1 (inputs n1 + 4 n2 < NIN)
    dft4_in<DIR, (NIN + 3) / 4>(v[0], v[4], v[8], v[12]);
    dft4_in<DIR, (NIN + 2) / 4>(v[1], v[5], v[9], v[13]);
    dft4_in<DIR, (NIN + 1) / 4>(v[2], v[6], v[10], v[14]);
    dft4_in<DIR, NIN / 4>(v[3], v[7], v[11], v[15]);
    constexpr int N1 = NIN < 4 ? NIN : 4;  // nonzero n1 rows
    if constexpr (N1 > 1) {
      v[1 + 4] = cmul_k(v[1 + 4], c1, d * s1);
      v[1 + 8] = cmul_k(v[1 + 8], r2, d * r2);
      v[1 + 12] = cmul_k(v[1 + 12], s1, d * c1);
    }
    if constexpr (N1 > 2) {
      v[2 + 4] = cmul_k(v[2 + 4], r2, d * r2);
      v[2 + 8] = mul_dir_i<DIR>(v[2 + 8]);
      v[2 + 12] = cmul_k(v[2 + 12], -r2, d * r2);
    }
    if constexpr (N1 > 3) {
      v[3 + 4] = cmul_k(v[3 + 4], s1, d * c1);
      v[3 + 8] = cmul_k(v[3 + 8], -r2, d * r2);
      v[3 + 12] = cmul_k(v[3 + 12], -c1, -d * s1);
    }
    float2 o[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      float2 y0 = v[0 + 4 * k1], y1 = v[1 + 4 * k1], y2 = v[2 + 4 * k1], y3 = v[3 + 4 * k1];
      dft4_in<DIR, N1>(y0, y1, y2, y3);
      o[k1] = y0;
      o[k1 + 4] = y1;
      o[k1 + 8] = y2;
      o[k1 + 12] = y3;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = o[k];
  }
}

// V-point DFT with the inputs n >= NIN known to be zero
template <int V, int DIR, int NIN>
__device__ __forceinline__ void dft_in(float2* v) {
  if constexpr (V == 16)
    dft16_in<DIR, NIN>(v);
  else {
    static_assert(V == 8, "dft_in: V in {8, 16}");
    dft8_in<DIR, NIN>(v);
  }
}

template <int R, int DIR>
__device__ __forceinline__ void dft(float2* v) {
  if constexpr (R == 2) {
    dft2<DIR>(v[0], v[1]);
  } else if constexpr (R == 4) {
    dft4<DIR>(v[0], v[1], v[2], v[3]);
  } else if constexpr (R == 8) {
    dft8<DIR>(v);
  } else if constexpr (R == 16) {
    dft16<DIR>(v);
  } else if constexpr (R == 1) {
  }
}

__host__ __device__ __forceinline__ int ilog2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

}  // namespace tfno
