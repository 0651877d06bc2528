// Per-plane 2D Fourier-layer kernels for sm_100a (rank-2 fully_fused fast path).
//
// The reference runs rank 2 as x-FFT (own pass) -> fused y-FFT/CGEMM/y-iFFT
// -> x-iFFT (own pass) (pipeline.py:149-292), which streams the truncated
// stage-1 spectrum and the pre-x-iFFT output through HBM (2.5x the
// input+output bytes at keep/dim = 1/8).  Here each persistent CTA owns whole
// (b, channel) planes:
//
//   plane_fwd2d   x[b,h] (dx*dy) -> A[b,h,kx,ky]: every row streams into a
//                 shared-memory ring with TMA bulk copies (cp.async.bulk +
//                 mbarrier); a team of dy/8 threads does the truncated row
//                 FFT (radix-8 in registers, smem transpose, radix-8 +
//                 warp-shuffle transposed reduction) into the class buffer;
//                 the x direction is a four-step transform: rows x = x0 + R*x1
//                 (R = dx/kx) form class x0, whose kx-point column FFT is
//                 twiddled by w_dx^{p*x0} and accumulated in registers.
//   cgemm         C[b,n,p,q] = sum_h A[b,h,p,q] W[h,n] / (dx*dy)  (kernels.cu)
//   plane_inv2d   C[b,n] (kx*ky) -> y[b,n] (dx*dy): per class x0, twiddle +
//                 kx-point column iFFT gives rows x0 + R*x1 at ky bins; each
//                 row's padded iFFT (radix-8, smem transpose, radix-8) is
//                 written to a smem staging ring and TMA bulk-stored.
//
// Only x, y and the two mode tensors (kx*ky/(dx*dy) = 1/64 of a plane for
// C3/C4) touch HBM.  Math: SURVEY.md Appendix A; row FFT decomposition
// X[r+8t] = sum_a w_M^{ta} sum_c w_8^{tc} w_N^{r(a+Ac)} Z[a+Ac, r],
// Z[y1, r] = sum_{y2} w_8^{r y2} x[y1 + M y2], M = N/8, A = M/8.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"
#include "plane2d.cuh"
#include "ptx.cuh"

namespace tfno {

// ---------------------------------------------------------------- geometry
template <int DX_, int KX_, int NY_, int KY_, int NTH_, int RPT_ = 1>
struct PlaneGeo {
  static constexpr int DX = DX_, KX = KX_, NY = NY_, KY = KY_, NTH = NTH_;
  static constexpr int RPT = RPT_;  // rows per thread team per iteration (forward ILP)
  static constexpr int M = NY / 8;  // threads per row team
  static constexpr int A = M / 8;
  static constexpr int T = (KY + 7) / 8;
  static constexpr int LOGA = (A >= 16 ? 4 : A >= 8 ? 3 : A >= 4 ? 2 : A >= 2 ? 1 : 0);
  static constexpr int LOGT = (T >= 8 ? 3 : T >= 4 ? 2 : T >= 2 ? 1 : 0);
  static constexpr int TEAMS = NTH / M;  // thread teams
  static constexpr int ROWS = TEAMS * RPT;  // rows per iteration
  static constexpr int R = DX / KX;      // four-step classes along x
  static constexpr int KA = KX / 8;      // kx = 8 * KA
  static constexpr int IPC = KX / ROWS;  // iterations per class
  static constexpr int PAD = ((-7 * A) % 16 + 16) % 16;
  static constexpr int RT = T + 2;                 // reduction buffer: padded t-stride
  // per-r stride, == T (mod 16 complex): the reduction reads (lane = rq*T + tq) then cover 32
  // consecutive complex values modulo the 32 banks (256²/32: 4-way -> conflict-free); 512²/64 unchanged
#ifdef TFNO_PLANE_RS_OLD
  static constexpr int RS = A * RT + 8;
#else
  static constexpr int RS = A * RT + (((T - A * RT) % 16) + 16) % 16;
#endif
  static constexpr int TS = M + PAD;  // transposed-row stride (== A mod 16: conflict-free reads)
  static constexpr int TASKS2 = (8 * KY + NTH - 1) / NTH;
  static_assert(A >= 1 && (1 << LOGA) == A, "A power of two");
  static_assert((1 << LOGT) == T && T <= A && T <= 8, "ky <= 8*min(8, dy/64)");
  static_assert(8 * T == KY, "ky multiple of 8");
  static_assert(KX % 8 == 0 && KA <= 8 && KX % ROWS == 0 && DX % KX == 0, "kx shape");
  static_assert(NTH % M == 0 && (M % 32 == 0 || 32 % M == 0), "team shape");
};

template <int KA, int DIR>
__device__ __forceinline__ void dft_small(float2* v) {
  dft<KA, DIR>(v);
}

// row-team barrier: a team is M = dy/8 threads (one warp or less -> __syncwarp)
template <int M>
__device__ __forceinline__ void team_sync(int team) {
  if constexpr (M <= 32)
    __syncwarp();
  else
    named_bar(1 + team, M);
}
constexpr int kComputeBar = 15;

// ============================================================== forward
// Warp-specialised: warp NTH/32 is the TMA producer (ring of S slots, full /
// empty mbarriers); the NTH compute threads form row teams that synchronise
// only inside the team, plus one compute-wide barrier per class (column pass).
// SKEW: the class tail is software-pipelined over three class buffers — in the
// iteration that runs the rows of class c, threads [NTH - KA*KY, NTH) run the
// column pass 1 of class c-1 and threads [0, 8*KY) the pass 2 + accumulation of
// class c-2, then ONE compute-wide barrier (instead of three per class with 3/4
// or 1/2 of the threads idle between them).  Same operations in the same order:
// bitwise-identical modes.
template <class G>
__host__ __device__ constexpr bool fwd_skew_ok() { return 8 * G::KY + (G::KX / 8) * G::KY <= G::NTH; }

template <class G, int S, bool NATURAL, bool DLD, bool SKEW = false>
__global__ void __launch_bounds__(G::NTH + 32, 1)
    plane_fwd2d_kernel(const float2* __restrict__ x, float2* __restrict__ Aout, int64_t planes,
                       const float2* __restrict__ twg) {
  constexpr int NY = G::NY, M = G::M, A = G::A, T = G::T, TEAMS = G::TEAMS, R = G::R, KA = G::KA;
  constexpr int KX = G::KX, KY = G::KY, DX = G::DX, IPC = G::IPC, TS = G::TS, NTH = G::NTH;
  constexpr int RT = G::RT, RS = G::RS, RPT = G::RPT, ROWS = G::ROWS;
  static_assert(RPT == 1 || !DLD, "direct loads only with one row per team");
  static_assert(!SKEW || fwd_skew_ok<G>(), "skewed tail: disjoint pass-1 / pass-2 thread ranges");
  extern __shared__ __align__(128) uint8_t smem[];
  float2* ring = reinterpret_cast<float2*>(smem);
  float2* tr = ring + (DLD ? 0 : S * ROWS * NY);  // DLD: rows go straight to registers (no ring)
  float2* red = tr + ROWS * 8 * TS;
  float2* const Tc0 = red + ROWS * 8 * RS;
  // SKEW: the row twiddle table (read into registers once, before any row) aliases
  // class buffer 2, first written by the rows of class 2, two barriers later
  static_assert(!SKEW || NY <= KX * KY, "twy alias");
  float2* twy = SKEW ? Tc0 + 2 * KX * KY : Tc0 + KX * KY;
  float2* twx = SKEW ? Tc0 + 3 * KX * KY : twy + NY;
  uint64_t* full = reinterpret_cast<uint64_t*>(twx + DX);
  uint64_t* empty = full + S;

  const int tid = threadIdx.x;
  const int64_t nmine = planes > blockIdx.x ? (planes - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t NIT = nmine * R * IPC;
  const int64_t NCL = nmine * R;  // classes of this CTA

  for (int k = tid; k < NY; k += blockDim.x) twy[k] = __ldg(&twg[(size_t)k * (TFNO_TW_MAX / NY)]);
  for (int k = tid; k < DX; k += blockDim.x) twx[k] = __ldg(&twg[(size_t)k * (TFNO_TW_MAX / DX)]);
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NTH / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();  // x is read (A written) only once the previous kernel has completed
  pdl_launch_dependents();

  if (tid >= NTH) {
    // ---------------- producer warp: stream the plane rows, class by class
    if (!DLD && tid == NTH) {
      const uint64_t pol = policy_evict_first();
      // nested (plane, class, iteration) loops with the ring slot / phase kept
      // incrementally: no 64-bit divisions on the issue path
      int slot = 0, cnt = 0;
      uint32_t phase = 0;
      for (int64_t kp = 0; kp < nmine; ++kp) {
        const float2* src = x + (blockIdx.x + kp * gridDim.x) * (int64_t)DX * NY;
        for (int x0 = 0; x0 < R; ++x0) {
          for (int j = 0; j < IPC; ++j, ++cnt) {
            if (cnt >= S) mbar_wait(&empty[slot], phase ^ 1u);
            float2* dst = ring + slot * ROWS * NY;
            mbar_expect_tx(&full[slot], ROWS * NY * 8);
#pragma unroll 1
            for (int tm = 0; tm < ROWS; ++tm) {
              const int row = x0 + R * (j * ROWS + tm);
              tma_load_1d(dst + tm * NY, src + (int64_t)row * NY, NY * 8, &full[slot], pol);
            }
            if (++slot == S) {
              slot = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
    return;
  }

  // ---------------- compute threads
  const int team = tid / M, tt = tid % M;
  const int a_ = tt % A, r_ = tt / A;
  // row tm = team + TEAMS * r2 of the iteration (r2 < RPT): its transpose / reduction buffers
  auto trt = [&](int r2) { return tr + (team + TEAMS * r2) * 8 * TS; };
  auto redt = [&](int r2) { return red + (team + TEAMS * r2) * 8 * RS; };
  // per-thread constant twiddles (a strided table walk is an 8-way bank conflict)
  float2 tw1[8], tw2[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) tw1[r] = twy[r * tt];
#pragma unroll
  for (int t = 0; t < 8; ++t) tw2[t] = twy[(8 * t * a_) % NY];
  // reduction reader role: output storage column q' = tt = t' + T*r'; its
  // twiddles w_M^{tq*a} are applied inside the sum (complex FMAs)
  const int tq = tt % T, rq = tt / T;
  float2 tw3[A];
#pragma unroll
  for (int a = 0; a < A; ++a) tw3[a] = twy[(8 * tq * a) % NY];

  float2 acc[G::TASKS2][KA];
#pragma unroll
  for (int a = 0; a < G::TASKS2; ++a)
#pragma unroll
    for (int u = 0; u < KA; ++u) acc[a][u] = make_float2(0.f, 0.f);

  // DLD: this thread's 8 inputs of the next iteration's row, loaded one iteration ahead
  auto row_ptr = [&](int64_t it2) {
    const int64_t pl = blockIdx.x + (it2 / (R * IPC)) * gridDim.x;
    const int xx0 = (int)((it2 / IPC) % R), jj = (int)(it2 % IPC);
    return x + pl * (int64_t)DX * NY + (int64_t)(xx0 + R * (jj * TEAMS + team)) * NY;
  };
  float2 nxt[8];
  if (DLD && NIT > 0) {
    const float2* rp = row_ptr(0);
#pragma unroll
    for (int y2 = 0; y2 < 8; ++y2) nxt[y2] = __ldcs(rp + tt + M * y2);
  }
  // nested (plane, class, row-group) loops, ring slot / phase kept incrementally
  // (no 64-bit index divisions): C4 forward 6.98 -> 6.67 ms on one box
  // SKEW: pass 1 of class c-1 (threads [NTH - KA*KY, NTH)) and pass 2 of class c-2
  // (threads [0, 8*KY)) on their own class buffers, then the one barrier per class
  auto skew_tail = [&](int64_t c) {
    if (c >= 1 && c - 1 < NCL) {
      const int tau = tid - (NTH - KA * KY);
      if (tau >= 0) {
        float2* T1 = Tc0 + (int)((c - 1) % 3) * (KX * KY);
        const int q = tau % KY, i = tau / KY;
        float2 v[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) v[m] = T1[(i + KA * m) * KY + q];
        dft8<-1>(v);
#pragma unroll
        for (int s2 = 1; s2 < 8; ++s2) v[s2] = cmul(v[s2], twx[i * s2 * R]);
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) T1[(s2 * KA + i) * KY + q] = v[s2];
      }
    }
    if (c >= 2 && c - 2 < NCL && tid < 8 * KY) {
      const int64_t c2 = c - 2;
      const int x0c = (int)(c2 % R);
      const float2* T2 = Tc0 + (int)(c2 % 3) * (KX * KY);
      const int q = tid % KY, s2 = tid / KY;
      float2 w[KA];
#pragma unroll
      for (int i = 0; i < KA; ++i) w[i] = T2[(s2 * KA + i) * KY + q];
      dft_small<KA, -1>(w);
#pragma unroll
      for (int u = 0; u < KA; ++u) cmac(acc[0][u], w[u], twx[(s2 + 8 * u) * x0c]);
      if (x0c == R - 1) {
        float2* dst = Aout + (blockIdx.x + (c2 / R) * gridDim.x) * (int64_t)KX * KY;
        const int qo = NATURAL ? (q / T) + 8 * (q % T) : q;
#pragma unroll
        for (int u = 0; u < KA; ++u) {
          dst[(s2 + 8 * u) * KY + qo] = acc[0][u];
          acc[0][u] = make_float2(0.f, 0.f);
        }
      }
    }
    named_bar(kComputeBar, NTH);
  };

  int it = 0, slot = 0;
  uint32_t phase = 0;
  int64_t cl = 0;  // class counter (SKEW)
  for (int64_t kp = 0; kp < nmine; ++kp) {
  const int64_t pl = blockIdx.x + kp * gridDim.x;
#pragma unroll 1
  for (int x0 = 0; x0 < R; ++x0, ++cl) {
  float2* const Tc = SKEW ? Tc0 + (int)(cl % 3) * (KX * KY) : Tc0;
#pragma unroll 1
  for (int j = 0; j < IPC; ++j, ++it) {
    if (!DLD) mbar_wait(&full[slot], phase);
    // ---- row stage 1: radix-8 over y2, twiddle w_N^{r*y1}, transpose
    // (RPT independent rows per thread, interleaved for ILP)
    {
      float2 v[RPT][8];
      if (DLD) {
#pragma unroll
        for (int y2 = 0; y2 < 8; ++y2) v[0][y2] = nxt[y2];
        if (it + 1 < NIT) {
          const float2* rp = row_ptr((int64_t)it + 1);
#pragma unroll
          for (int y2 = 0; y2 < 8; ++y2) nxt[y2] = __ldcs(rp + tt + M * y2);
        }
      } else {
#pragma unroll
        for (int r2 = 0; r2 < RPT; ++r2) {
          const float2* row = ring + slot * ROWS * NY + (team + TEAMS * r2) * NY;
#pragma unroll
          for (int y2 = 0; y2 < 8; ++y2) v[r2][y2] = row[tt + M * y2];
        }
      }
#pragma unroll
      for (int r2 = 0; r2 < RPT; ++r2) dft8<-1>(v[r2]);
      if (!DLD) {
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[slot]);  // this warp is done with the slot
      }
#pragma unroll
      for (int r2 = 0; r2 < RPT; ++r2) {
#pragma unroll
        for (int r = 1; r < 8; ++r) v[r2][r] = cmul(v[r2][r], tw1[r]);
        float2* tb = trt(r2);
#pragma unroll
        for (int r = 0; r < 8; ++r) tb[r * TS + tt] = v[r2][r];
      }
    }
    team_sync<M>(team);
    // ---- row stage 2: radix-8 over c, twiddle w_M^{t*a} -> reduction buffer
    {
      float2 u[RPT][8];
#pragma unroll
      for (int r2 = 0; r2 < RPT; ++r2) {
        const float2* tb = trt(r2);
#pragma unroll
        for (int c = 0; c < 8; ++c) u[r2][c] = tb[r_ * TS + a_ + A * c];
      }
#pragma unroll
      for (int r2 = 0; r2 < RPT; ++r2) {
        dft8<-1>(u[r2]);  // twiddle w_M^{t a} deferred to the reduction (FMA-fused)
        float2* dst = redt(r2) + r_ * RS + a_ * RT;
        if constexpr (T % 2 == 0) {
#pragma unroll
          for (int t = 0; t < T; t += 2)
            *reinterpret_cast<float4*>(dst + t) = make_float4(u[r2][t].x, u[r2][t].y, u[r2][t + 1].x, u[r2][t + 1].y);
        } else {
#pragma unroll
          for (int t = 0; t < T; ++t) dst[t] = u[r2][t];
        }
      }
    }
    team_sync<M>(team);
    // ---- sum over a: X[r + 8t] for the thread's storage column q' = tt
    if (tt < KY) {
      float2 part[RPT][A];
#pragma unroll
      for (int r2 = 0; r2 < RPT; ++r2) {
        const float2* rb = redt(r2);
#pragma unroll
        for (int a = 0; a < A; ++a) part[r2][a] = rb[rq * RS + a * RT + tq];
      }
#pragma unroll
      for (int r2 = 0; r2 < RPT; ++r2) {
        // sum_a w_M^{tq a} part[a]: two interleaved FMA chains, then one add
        float2 s0 = part[r2][0], s1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int a = 1; a < A; ++a) {
          if (a & 1)
            cmac(s1, part[r2][a], tw3[a]);
          else
            cmac(s0, part[r2][a], tw3[a]);
        }
        const int x1 = j * ROWS + team + TEAMS * r2;
        Tc[x1 * KY + tt] = cadd(s0, s1);
      }
    }
    if (++slot == S) {
      slot = 0;
      phase ^= 1u;
    }
  }  // j: rows of class x0
    if constexpr (SKEW) {
      skew_tail(cl);
    } else {
      named_bar(kComputeBar, NTH);
      // ---- class x0 complete: kx-point column FFT, pass 1 (radix 8 over m)
      for (int tau = tid; tau < KA * KY; tau += NTH) {
        const int q = tau % KY, i = tau / KY;
        float2 v[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) v[m] = Tc[(i + KA * m) * KY + q];
        dft8<-1>(v);
#pragma unroll
        for (int s2 = 1; s2 < 8; ++s2) v[s2] = cmul(v[s2], twx[i * s2 * R]);
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) Tc[(s2 * KA + i) * KY + q] = v[s2];
      }
      named_bar(kComputeBar, NTH);
      // pass 2 (radix KA over i) + four-step twiddle w_dx^{p*x0}, accumulate
#pragma unroll
      for (int jj = 0; jj < G::TASKS2; ++jj) {
        const int tau = tid + jj * NTH;
        if (tau < 8 * KY) {
          const int q = tau % KY, s2 = tau / KY;
          float2 w[KA];
#pragma unroll
          for (int i = 0; i < KA; ++i) w[i] = Tc[(s2 * KA + i) * KY + q];
          dft_small<KA, -1>(w);
#pragma unroll
          for (int u = 0; u < KA; ++u) cmac(acc[jj][u], w[u], twx[(s2 + 8 * u) * x0]);
        }
      }
      named_bar(kComputeBar, NTH);
      if (x0 == R - 1) {
        // mode tensor in storage order (q' = t + T*r); the mode GEMM is
        // order-agnostic and the inverse reads the same order back
        float2* dst = Aout + pl * (int64_t)KX * KY;
#pragma unroll
        for (int jj = 0; jj < G::TASKS2; ++jj) {
          const int tau = tid + jj * NTH;
          if (tau < 8 * KY) {
            const int q = tau % KY, s2 = tau / KY;
            const int qo = NATURAL ? (q / T) + 8 * (q % T) : q;
#pragma unroll
            for (int u = 0; u < KA; ++u) {
              dst[(s2 + 8 * u) * KY + qo] = acc[jj][u];
              acc[jj][u] = make_float2(0.f, 0.f);
            }
          }
        }
      }
    }
  }  // x0
  }  // planes
  if constexpr (SKEW) {  // drain: the last two classes' column passes
    skew_tail(NCL);
    skew_tail(NCL + 1);
  }
}

// ============================================================== inverse
// Row teams run decoupled (team barriers only); each team's elected thread
// TMA-stores its own finished rows from a per-team staging ring.
// SKEW: the class head is software-pipelined like the forward's tail — while the
// rows of class c are written, the column pass 2 of class c+1 and pass 1 of class
// c+2 run on their own class buffers (three), the mode tile is double-buffered
// (the next plane's tile lands while this plane's last classes run), one
// compute-wide barrier per class instead of three.  Same operations, same order.
template <class G, int SO, bool NATURAL, bool DST, bool SKEW = false>
__global__ void __launch_bounds__(G::NTH, 1)
    plane_inv2d_kernel(const float2* __restrict__ Cin, float2* __restrict__ y, int64_t planes,
                       const float2* __restrict__ twg, float scale) {
  constexpr int NY = G::NY, M = G::M, A = G::A, T = G::T, TEAMS = G::TEAMS, R = G::R, KA = G::KA;
  constexpr int KX = G::KX, KY = G::KY, DX = G::DX, IPC = G::IPC, TS = G::TS, NTH = G::NTH;
  extern __shared__ __align__(128) uint8_t smem[];
  float2* ost = reinterpret_cast<float2*>(smem);  // TEAMS x SO x NY (TMA store sources; unused if DST)
  float2* cin = ost + (DST ? 0 : TEAMS * SO * NY);  // KX*KY (TMA load target; SKEW: two)
  float2* Gb = cin + (SKEW ? 2 : 1) * KX * KY;      // KX*KY (SKEW: three class buffers)
  float2* tr = Gb + (SKEW ? 3 : 1) * KX * KY;
  float2* twy = tr + TEAMS * 8 * TS;
  float2* twx = twy + NY;
  uint64_t* bar = reinterpret_cast<uint64_t*>(twx + DX);  // SKEW: two (one per mode-tile buffer)

  const int tid = threadIdx.x;
  const int team = tid / M, tt = tid % M;
  const int64_t nmine = planes > blockIdx.x ? (planes - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  for (int k = tid; k < NY; k += NTH) twy[k] = conjf2(__ldg(&twg[(size_t)k * (TFNO_TW_MAX / NY)]));
  for (int k = tid; k < DX; k += NTH) twx[k] = cscale(conjf2(__ldg(&twg[(size_t)k * (TFNO_TW_MAX / DX)])), scale);
  if (tid == 0) {
    mbar_init(bar, 1);
    if (SKEW) mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();
  const uint64_t pol = policy_evict_first();
  auto issue = [&](int64_t k) {
    const int64_t pl = blockIdx.x + k * gridDim.x;
    const int b = SKEW ? (int)(k & 1) : 0;
    mbar_expect_tx(bar + b, KX * KY * 8);
    tma_load_1d(cin + b * (KX * KY), Cin + pl * (int64_t)KX * KY, KX * KY * 8, bar + b, pol);
  };
  if (tid == 0 && nmine > 0) issue(0);
  if (SKEW && tid == 0 && nmine > 1) issue(1);

  float2* trt = tr + team * 8 * TS;
  float2* ostt = ost + team * SO * NY;
  const int a_ = tt % A, r_ = tt / A;
  const bool elected = (tt == 0);
  float2 tw1[8], tw2[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) tw1[r] = twy[r * tt];
#pragma unroll
  for (int t = 0; t < 8; ++t) tw2[t] = twy[(8 * t * a_) % NY];
  int oslot = 0;  // team-local staging-ring slot (row iteration mod SO, kept incrementally)
  if constexpr (SKEW) {
    const int64_t NCL = nmine * R;
    // rows of class c (team-decoupled), from class buffer Gc
    auto rows_of = [&](int64_t cl) {
      const float2* Gc = Gb + (int)(cl % 3) * (KX * KY);
      const int x0 = (int)(cl % R);
      float2* yp = y + (blockIdx.x + (cl / R) * gridDim.x) * (int64_t)DX * NY;
      for (int j = 0; j < IPC; ++j, oslot = (oslot + 1 == SO ? 0 : oslot + 1)) {
        const int x1 = j * TEAMS + team;
        // ---- row stage A: twiddle w_M^{+t a}, radix 8 over t (t < T nonzero)
        {
          float2 u[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            if (t < T) {
              float2 g = Gc[x1 * KY + t + T * r_];  // storage column q' = t + T*r
              u[t] = t ? cmul(g, tw2[t]) : g;
            } else {
              u[t] = make_float2(0.f, 0.f);
            }
          }
          dft8<1>(u);
#pragma unroll
          for (int c = 0; c < 8; ++c) trt[r_ * TS + a_ + A * c] = u[c];
        }
        const int slot = oslot;
        if (!DST && elected) bulk_wait_read<SO - 1>();  // staging slot free again
        team_sync<M>(team);
        // ---- row stage B: twiddle w_N^{+r y1}, radix 8 over r -> staging row
        {
          float2 v[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) v[r] = trt[r * TS + tt];
#pragma unroll
          for (int r = 1; r < 8; ++r) v[r] = cmul(v[r], tw1[r]);
          dft8<1>(v);
          if (DST) {  // coalesced streaming stores straight from registers (no smem staging)
            float2* orow = yp + (int64_t)(x0 + R * x1) * NY;
#pragma unroll
            for (int y2 = 0; y2 < 8; ++y2) __stcs(orow + tt + M * y2, v[y2]);
          } else {
            float2* o = ostt + slot * NY;
#pragma unroll
            for (int y2 = 0; y2 < 8; ++y2) o[tt + M * y2] = v[y2];
          }
        }
        if (!DST) fence_proxy_async();
        team_sync<M>(team);
        if (!DST && elected) {
          const int row = x0 + R * x1;
          tma_store_1d(yp + (int64_t)row * NY, ostt + slot * NY, NY * 8, pol);
          bulk_commit();
        }
      }
    };
    auto pass1_of = [&](int64_t c) {  // twiddle w_dx^{+p x0} (x output scale), radix KA over u
      const int64_t k = c / R;
      const int x0 = (int)(c % R);
      if (x0 == 0) mbar_wait(bar + (k & 1), (uint32_t)((k >> 1) & 1));
      const float2* ci = cin + (int)(k & 1) * (KX * KY);
      float2* G1 = Gb + (int)(c % 3) * (KX * KY);
      for (int tau = tid; tau < 8 * KY; tau += NTH) {
        const int q = tau % KY, s2 = tau / KY;
        float2 w[KA];
        const int qi = NATURAL ? (q / T) + 8 * (q % T) : q;
#pragma unroll
        for (int u = 0; u < KA; ++u) {
          const int p = s2 + 8 * u;
          w[u] = cmul(ci[p * KY + qi], twx[p * x0]);
        }
        dft_small<KA, 1>(w);
#pragma unroll
        for (int i = 1; i < KA; ++i) w[i] = cmul(w[i], twy[s2 * i * (NY / KX)]);
#pragma unroll
        for (int i = 0; i < KA; ++i) G1[(s2 * KA + i) * KY + q] = w[i];
      }
    };
    auto pass2_of = [&](int64_t c) {  // radix 8 over s -> rows x1 = i + KA*m (in place per task)
      float2* G2 = Gb + (int)(c % 3) * (KX * KY);
      for (int tau = tid; tau < KA * KY; tau += NTH) {
        const int q = tau % KY, i = tau / KY;
        float2 v[8];
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) v[s2] = G2[(s2 * KA + i) * KY + q];
        dft8<1>(v);
#pragma unroll
        for (int m = 0; m < 8; ++m) G2[(i + KA * m) * KY + q] = v[m];
      }
    };
    // after the barrier that completes pass 1 of class c: the last class of plane k
    // frees mode-tile buffer k&1 for plane k+2
    auto refill = [&](int64_t c) {
      if (tid == 0 && c >= 0 && c < NCL && (int)(c % R) == R - 1 && c / R + 2 < nmine) issue(c / R + 2);
    };
    if (NCL > 0) pass1_of(0);
    named_bar(kComputeBar, NTH);
    refill(0);
    if (NCL > 0) pass2_of(0);
    if (NCL > 1) pass1_of(1);
    named_bar(kComputeBar, NTH);
    refill(1);
#pragma unroll 1
    for (int64_t c = 0; c < NCL; ++c) {
      rows_of(c);
      if (c + 1 < NCL) pass2_of(c + 1);
      if (c + 2 < NCL) pass1_of(c + 2);
      named_bar(kComputeBar, NTH);
      refill(c + 2);
    }
  } else {
    for (int64_t k = 0; k < nmine; ++k) {
      mbar_wait(bar, (uint32_t)(k & 1));
      const int64_t pl = blockIdx.x + k * gridDim.x;
      float2* yp = y + pl * (int64_t)DX * NY;
      for (int x0 = 0; x0 < R; ++x0) {
        named_bar(kComputeBar, NTH);  // previous class's rows are done with Gb
        // ---- column iFFT, pass 1: twiddle w_dx^{+p x0}, radix KA over u
        for (int tau = tid; tau < 8 * KY; tau += NTH) {
          const int q = tau % KY, s2 = tau / KY;
          float2 w[KA];
          const int qi = NATURAL ? (q / T) + 8 * (q % T) : q;
  #pragma unroll
          for (int u = 0; u < KA; ++u) {
            const int p = s2 + 8 * u;
            w[u] = cmul(cin[p * KY + qi], twx[p * x0]);  // twx carries the output scale
          }
          dft_small<KA, 1>(w);
  #pragma unroll
          for (int i = 1; i < KA; ++i) w[i] = cmul(w[i], twy[s2 * i * (NY / KX)]);
  #pragma unroll
          for (int i = 0; i < KA; ++i) Gb[(s2 * KA + i) * KY + q] = w[i];
        }
        named_bar(kComputeBar, NTH);
        if (x0 == R - 1 && tid == 0 && k + 1 < nmine) issue(k + 1);  // cin fully consumed
        // pass 2: radix 8 over s -> rows x1 = i + KA*m (in place per task)
        for (int tau = tid; tau < KA * KY; tau += NTH) {
          const int q = tau % KY, i = tau / KY;
          float2 v[8];
  #pragma unroll
          for (int s2 = 0; s2 < 8; ++s2) v[s2] = Gb[(s2 * KA + i) * KY + q];
          dft8<1>(v);
  #pragma unroll
          for (int m = 0; m < 8; ++m) Gb[(i + KA * m) * KY + q] = v[m];
        }
        named_bar(kComputeBar, NTH);
        for (int j = 0; j < IPC; ++j, oslot = (oslot + 1 == SO ? 0 : oslot + 1)) {
          const int x1 = j * TEAMS + team;
          // ---- row stage A: twiddle w_M^{+t a}, radix 8 over t (t < T nonzero)
          {
            float2 u[8];
  #pragma unroll
            for (int t = 0; t < 8; ++t) {
              if (t < T) {
                float2 g = Gb[x1 * KY + t + T * r_];  // storage column q' = t + T*r
                u[t] = t ? cmul(g, tw2[t]) : g;
              } else {
                u[t] = make_float2(0.f, 0.f);
              }
            }
            dft8<1>(u);
  #pragma unroll
            for (int c = 0; c < 8; ++c) trt[r_ * TS + a_ + A * c] = u[c];
          }
          const int slot = oslot;
          if (!DST && elected) bulk_wait_read<SO - 1>();  // staging slot free again
          team_sync<M>(team);
          // ---- row stage B: twiddle w_N^{+r y1}, radix 8 over r -> staging row
          {
            float2 v[8];
  #pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = trt[r * TS + tt];
  #pragma unroll
            for (int r = 1; r < 8; ++r) v[r] = cmul(v[r], tw1[r]);
            dft8<1>(v);
            if (DST) {  // coalesced streaming stores straight from registers (no smem staging)
              float2* orow = yp + (int64_t)(x0 + R * x1) * NY;
  #pragma unroll
              for (int y2 = 0; y2 < 8; ++y2) __stcs(orow + tt + M * y2, v[y2]);
            } else {
              float2* o = ostt + slot * NY;
  #pragma unroll
              for (int y2 = 0; y2 < 8; ++y2) o[tt + M * y2] = v[y2];
            }
          }
          if (!DST) fence_proxy_async();
          team_sync<M>(team);
          if (!DST && elected) {
            const int row = x0 + R * x1;
            tma_store_1d(yp + (int64_t)row * NY, ostt + slot * NY, NY * 8, pol);
            bulk_commit();
          }
        }
      }
    }
  }
  if (!DST && elected) bulk_wait_all();
}

// ---------------------------------------------------------------- dispatch
template <class G>
constexpr size_t fwd_smem(int S, bool dld = false, bool skew = false) {
  return sizeof(float2) * ((size_t)(dld ? 0 : S) * G::ROWS * G::NY + G::ROWS * 8 * (G::TS + G::RS) +
                           (skew ? 3 * G::KX * G::KY : G::KX * G::KY + G::NY) + G::DX) +
         16 * S + 64;
}
template <class G>
constexpr size_t inv_smem(int SO, bool dst = false, bool skew = false) {
  return sizeof(float2) * ((skew ? 5 : 2) * (size_t)G::KX * G::KY + G::TEAMS * 8 * G::TS +
                           (size_t)(dst ? 0 : SO) * G::TEAMS * G::NY + G::NY + G::DX) +
         16 + 64;
}

// HBM-side data paths per geometry (bit0 = inverse stores rows straight from
// registers with st.global.cs, else smem staging + TMA bulk store; bit1 =
// forward loads rows straight into registers one iteration ahead, else TMA
// ring + producer warp).  Defaults are the measured winners per geometry
// (profiles/r01/plane_variants.txt); TFNO_PLANE_VARIANT overrides for A/B runs.
template <class G>
constexpr int plane_variant_default() {
  return (G::KX == 16 && G::DX == 256) ? 3 : 1;  // re-measured with packed f32x2 math (profiles/r01/plane_variants.txt)
}
template <class G>
static int plane_variant() {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("TFNO_PLANE_VARIANT");
    env = e ? atoi(e) : -1;
  }
  return env >= 0 ? env : plane_variant_default<G>();
}

static int num_sms() { return device_sms(); }

static int plane_skew_env() {  // TFNO_PLANE_SKEW=0/1 overrides the per-geometry default (A/B)
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("TFNO_PLANE_SKEW");
    v = e ? atoi(e) : -1;
  }
  return v;
}
// measured same box, alternating (profiles/r02/skew_ab.txt): C5 plane (256^2 keep 16) forward
// 1.567 -> 1.537 ms with the pipelined tail; C3 plane (keep 32) 0.2175 -> 0.2339 ms (slower: kept off)
template <class G>
constexpr bool fwd_skew_default() { return G::KX == 16 && G::DX == 256; }

template <class G, int S, bool NAT, bool DLD, bool SKEW>
static cudaError_t launch_fwd_k(const float2* x, float2* A, int64_t planes, const float2* tw, cudaStream_t st) {
  const int sms = num_sms();
  size_t smem = fwd_smem<G>(S, DLD, SKEW);
  int grid = (int)(planes < sms ? planes : sms);
  if (grid < 1) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(plane_fwd2d_kernel<G, S, NAT, DLD, SKEW>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(plane_fwd2d_kernel<G, S, NAT, DLD, SKEW>, dim3(grid), dim3(G::NTH + 32), smem, st, x, A, planes, tw);
  if (e != cudaSuccess) return e;
  ++g_launches;
  return cudaGetLastError();
}

template <class G, int S, bool NAT, bool DLD>
static cudaError_t launch_fwd_v(const float2* x, float2* A, int64_t planes, const float2* tw, cudaStream_t st) {
  if constexpr (fwd_skew_ok<G>()) {
    const int e = plane_skew_env();
    if (e > 0 || (e < 0 && fwd_skew_default<G>())) return launch_fwd_k<G, S, NAT, DLD, true>(x, A, planes, tw, st);
  }
  return launch_fwd_k<G, S, NAT, DLD, false>(x, A, planes, tw, st);
}

template <class G, int S>
static cudaError_t launch_fwd(const float2* x, float2* A, int64_t planes, const float2* tw, bool natural,
                              cudaStream_t st) {
  if constexpr (G::RPT > 1) {  // interleaved rows come from the TMA ring only
    return natural ? launch_fwd_v<G, S, true, false>(x, A, planes, tw, st)
                   : launch_fwd_v<G, S, false, false>(x, A, planes, tw, st);
  } else {
    const bool dld = (plane_variant<G>() & 2) != 0;
    if (natural)
      return dld ? launch_fwd_v<G, S, true, true>(x, A, planes, tw, st) : launch_fwd_v<G, S, true, false>(x, A, planes, tw, st);
    return dld ? launch_fwd_v<G, S, false, true>(x, A, planes, tw, st) : launch_fwd_v<G, S, false, false>(x, A, planes, tw, st);
  }
}

template <class G, int SO, bool NAT, bool DST, bool SKEW>
static cudaError_t launch_inv_k(const float2* Cm, float2* y, int64_t planes, const float2* tw, float scale,
                                cudaStream_t st) {
  const int sms = num_sms();
  size_t smem = inv_smem<G>(SO, DST, SKEW);
  int grid = (int)(planes < sms ? planes : sms);
  if (grid < 1) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(plane_inv2d_kernel<G, SO, NAT, DST, SKEW>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(plane_inv2d_kernel<G, SO, NAT, DST, SKEW>, dim3(grid), dim3(G::NTH), smem, st, Cm, y, planes, tw, scale);
  if (e != cudaSuccess) return e;
  ++g_launches;
  return cudaGetLastError();
}

// TFNO_PLANE_ISKEW=1 selects the pipelined class head (opt-in A/B): parity-green and bitwise
// equal, but measured slower (profiles/r02/iskew_ab.txt: C3 inverse 0.1864 -> 0.190 ms, C5 plane
// inverse 1.492 -> 1.686 ms) — the lock-stepped row teams write more evenly than drifting ones
static int plane_iskew_env() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("TFNO_PLANE_ISKEW");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <class G, int SO, bool NAT, bool DST>
static cudaError_t launch_inv_v(const float2* Cm, float2* y, int64_t planes, const float2* tw, float scale,
                                cudaStream_t st) {
  if constexpr (inv_smem<G>(SO, DST, true) <= 227 * 1024) {
    if (plane_iskew_env() != 0) return launch_inv_k<G, SO, NAT, DST, true>(Cm, y, planes, tw, scale, st);
  }
  return launch_inv_k<G, SO, NAT, DST, false>(Cm, y, planes, tw, scale, st);
}

template <class G, int SO>
static cudaError_t launch_inv(const float2* Cm, float2* y, int64_t planes, const float2* tw, float scale, bool natural,
                              cudaStream_t st) {
  const bool dst = (plane_variant<G>() & 1) != 0;
  if (natural)
    return dst ? launch_inv_v<G, SO, true, true>(Cm, y, planes, tw, scale, st)
               : launch_inv_v<G, SO, true, false>(Cm, y, planes, tw, scale, st);
  return dst ? launch_inv_v<G, SO, false, true>(Cm, y, planes, tw, scale, st)
             : launch_inv_v<G, SO, false, false>(Cm, y, planes, tw, scale, st);
}

using G512 = PlaneGeo<512, 64, 512, 64, 512>;
// forward of the 512 geometry: 4 teams x 2 interleaved rows (ILP against the
// shared-memory latency that bounds the packed-math forward), same smem
using G512f = PlaneGeo<512, 64, 512, 64, 256, 2>;
static bool fwd_rpt2() {  // TFNO_PLANE_RPT=1 selects the 8-team / 1-row forward (A/B)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TFNO_PLANE_RPT");
    v = e ? atoi(e) : 2;
  }
  return v != 1;
}
using G256a = PlaneGeo<256, 32, 256, 32, 512>;
using G256b = PlaneGeo<256, 16, 256, 16, 512>;
// half-thread inverses (fewer teams -> fewer idle threads in the column passes
// between the class barriers); A/B with TFNO_PLANE_INV_HALF=0/1
using G256b8 = PlaneGeo<256, 16, 256, 16, 256>;
using G256a8 = PlaneGeo<256, 32, 256, 32, 256>;
using G512i = PlaneGeo<512, 64, 512, 64, 256>;
static int inv_half_env() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("TFNO_PLANE_INV_HALF");
    v = e ? atoi(e) : -1;
  }
  return v;
}
// measured (profiles/r01/plane_variants.txt): C5 1.753 -> 1.493 ms, C3 0.202 -> 0.187 ms,
// C4 5.62 -> 7.44 ms (worse: 512 geometry keeps 8 teams)
static bool inv256b_8() { return inv_half_env() != 0; }
static bool inv256a_8() { return inv_half_env() != 0; }
static bool inv512_half() { return inv_half_env() == 2; }
using G128 = PlaneGeo<128, 16, 128, 16, 256>;

static_assert(fwd_smem<G512>(3) <= 227 * 1024, "smem");
static_assert(fwd_smem<G256a>(4, false, true) <= 227 * 1024 && fwd_smem<G256b>(4, false, true) <= 227 * 1024 &&
                  fwd_smem<G128>(4, false, true) <= 227 * 1024, "smem (skewed tail)");
static_assert(fwd_smem<G512f>(3) <= 227 * 1024, "smem");
static_assert(inv_smem<G512>(3) <= 227 * 1024, "smem");

// the four hand-tuned geometries (C3 / C4 / C5 plane shapes + 128^2 keep 16)
static bool plane2d_tuned(const tfno_cfg* c) {
  if (c->rank != 2 || c->batch * (int64_t)c->hidden_dim > (1LL << 40)) return false;
  const int dx = c->dim_x, dy = c->dim_y, kx = c->keep_x, ky = c->keep_y;
  return (dx == 512 && dy == 512 && kx == 64 && ky == 64) || (dx == 256 && dy == 256 && kx == 32 && ky == 32) ||
         (dx == 256 && dy == 256 && kx == 16 && ky == 16) || (dx == 128 && dy == 128 && kx == 16 && ky == 16);
}

// generic per-plane kernels (plane_g.cuh): padded keep KP (power of two, 8..128)
int plane_g_kp(const tfno_cfg* c) {
  if (c->rank != 2 || (int64_t)c->batch * c->hidden_dim > (1LL << 40) ||
      (int64_t)c->batch * c->output_dim > (1LL << 40))
    return 0;
  const int dx = c->dim_x, dy = c->dim_y;
  if (dy < 64 || dy > 1024 || (dy & (dy - 1)) || dx > 1024 || (dx & (dx - 1))) return 0;
  const int k = c->keep_x > c->keep_y ? c->keep_x : c->keep_y;
  int kp = 8;
  while (kp < k) kp <<= 1;
  if (kp > 128 || kp > dy || kp > dx) return 0;
  return kp;
}

static int plane_generic_env() {  // TFNO_PLANE_GENERIC=0..3 (bit 0 forward, bit 1 inverse) for A/B
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("TFNO_PLANE_GENERIC");
    v = e ? atoi(e) : -1;
  }
  return v;
}
static int plane_mix(const tfno_cfg* c);

bool plane2d_supported(const tfno_cfg* c) { return plane2d_tuned(c) || plane_g_kp(c) > 0; }

int64_t plane2d_modes(const tfno_cfg* c) {
  if (plane2d_tuned(c)) return (int64_t)c->keep_x * c->keep_y;  // == KP^2 there
  const int kp = plane_g_kp(c);
  return (int64_t)kp * kp;
}

bool plane2d_spectrum_ok(const tfno_cfg* c) {
  if (plane2d_tuned(c)) return true;
  const int kp = plane_g_kp(c);
  return kp > 0 && c->keep_x == kp && c->keep_y == kp;
}

cudaError_t plane_g_run_64(int, int, const float2*, float2*, int64_t, int, int, int, const float2*, float, cudaStream_t);
cudaError_t plane_g_run_128(int, int, const float2*, float2*, int64_t, int, int, int, const float2*, float, cudaStream_t);
cudaError_t plane_g_run_256(int, int, const float2*, float2*, int64_t, int, int, int, const float2*, float, cudaStream_t);
cudaError_t plane_g_run_512(int, int, const float2*, float2*, int64_t, int, int, int, const float2*, float, cudaStream_t);
cudaError_t plane_g_run_1024(int, int, const float2*, float2*, int64_t, int, int, int, const float2*, float, cudaStream_t);

size_t plane_g_invmix_smem_64(int, int, int, int);
size_t plane_g_invmix_smem_128(int, int, int, int);
size_t plane_g_invmix_smem_256(int, int, int, int);
size_t plane_g_invmix_smem_512(int, int, int, int);
size_t plane_g_invmix_smem_1024(int, int, int, int);
cudaError_t plane_g_invmix_run_64(int, const float2*, const float2*, float2*, float2*, int, int, int, int,
                                  const float2*, float, int, cudaStream_t);
cudaError_t plane_g_invmix_run_128(int, const float2*, const float2*, float2*, float2*, int, int, int, int,
                                  const float2*, float, int, cudaStream_t);
cudaError_t plane_g_invmix_run_256(int, const float2*, const float2*, float2*, float2*, int, int, int, int,
                                  const float2*, float, int, cudaStream_t);
cudaError_t plane_g_invmix_run_512(int, const float2*, const float2*, float2*, float2*, int, int, int, int,
                                  const float2*, float, int, cudaStream_t);
cudaError_t plane_g_invmix_run_1024(int, const float2*, const float2*, float2*, float2*, int, int, int, int,
                                  const float2*, float, int, cudaStream_t);

static size_t plane_g_invmix_smem(const tfno_cfg* c, int prec) {
  const int kp = plane_g_kp(c);
  if (!kp || c->hidden_dim > 4096) return 0;
  const int H = c->hidden_dim, dx = c->dim_x;
  switch (c->dim_y) {
    case 64: return plane_g_invmix_smem_64(kp, H, dx, prec);
    case 128: return plane_g_invmix_smem_128(kp, H, dx, prec);
    case 256: return plane_g_invmix_smem_256(kp, H, dx, prec);
    case 512: return plane_g_invmix_smem_512(kp, H, dx, prec);
    case 1024: return plane_g_invmix_smem_1024(kp, H, dx, prec);
    default: return 0;
  }
}

static cudaError_t plane_g_invmix_run(const tfno_cfg* c, const float2* A, const float2* w, float2* Cs, float2* y,
                                      const float2* tw, float alpha, int prec, cudaStream_t st) {
  const int kp = plane_g_kp(c);
  const int B = c->batch, H = c->hidden_dim, N = c->output_dim, dx = c->dim_x;
  switch (c->dim_y) {
    case 64: return plane_g_invmix_run_64(kp, A, w, Cs, y, B, H, N, dx, tw, alpha, prec, st);
    case 128: return plane_g_invmix_run_128(kp, A, w, Cs, y, B, H, N, dx, tw, alpha, prec, st);
    case 256: return plane_g_invmix_run_256(kp, A, w, Cs, y, B, H, N, dx, tw, alpha, prec, st);
    case 512: return plane_g_invmix_run_512(kp, A, w, Cs, y, B, H, N, dx, tw, alpha, prec, st);
    case 1024: return plane_g_invmix_run_1024(kp, A, w, Cs, y, B, H, N, dx, tw, alpha, prec, st);
    default: return cudaErrorNotSupported;
  }
}

constexpr int kMixGNHost = 8;  // == kMixGN in plane_g.cu (output channels per fused-mix task)
static int plane_fusedmix_env() {  // TFNO_PLANE_FUSEDMIX=0/1 overrides the per-geometry default (A/B)
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("TFNO_PLANE_FUSEDMIX");
    v = e ? atoi(e) : -1;
  }
  return v;
}

bool plane2d_fusedmix(const tfno_cfg* c, int prec, int mode) {
  // FP32: SIMT mix warps; TF32 / 3xTF32: tcgen05 mix (BF16 keeps the standalone kind::f16 contraction)
  if ((prec != TFNO_FP32 && prec != TFNO_TF32 && prec != TFNO_TF32X3) || !plane2d_supported(c)) return false;
  if ((int64_t)c->batch * ((c->output_dim + 7) / 8) > (1LL << 40)) return false;
  const int env = plane_fusedmix_env();
  if (env == 0 || plane_g_invmix_smem(c, prec) == 0) return false;
  if (env == 1) return true;
  // fused_gemm_ifft asks for exactly this fusion (channel mix + inverse in one kernel)
  if (mode == TFNO_FUSED_GEMM_IFFT) return prec == TFNO_FP32;
  // the tcgen05 mix inside the inverse is opt-in (TFNO_PLANE_FUSEDMIX=1): its A staging
  // (global -> registers -> canonical K-major tiles, one K step per chunk) keeps too few
  // loads in flight -- measured (profiles/r02/tcmix_ab.txt) C4 3xTF32 mix + inverse 8.08 ms
  // vs 0.46 ms standalone tcgen05 CGEMM (W' image) + 5.91 ms inverse
  if (prec != TFNO_FP32) return false;
  // default: where the standalone contraction is a large share of the layer and
  // every CTA has enough tasks to hide the first task's mix (the prologue) --
  // measured (profiles/r02/fusedmix_ab*.txt): C4 (H = N = 128, 13.8 tasks per
  // CTA) 7.81 -> 7.43 ms for mix + inverse; C3 / C5 (H = N = 64, <= 1.7 tasks
  // per CTA at C3) lose 0.22 -> 0.31 ms / 1.56 -> 1.91 ms
  const int64_t tasks = (int64_t)c->batch * ((c->output_dim + kMixGNHost - 1) / kMixGNHost);
  return (int64_t)c->hidden_dim * c->output_dim >= 128 * 128 && tasks >= 8LL * device_sms();
}

int64_t plane2d_c_elems(const tfno_cfg* c, int prec, int mode) {
  const int64_t mq = plane2d_modes(c);
  if (plane2d_fusedmix(c, prec, mode)) return (int64_t)device_sms() * 2 * kMixGNHost * mq;
  return (int64_t)c->batch * c->output_dim * mq;
}

static cudaError_t plane_g_run(const tfno_cfg* c, int dir, const float2* in, float2* out, int64_t planes,
                               const float2* tw, float scale, cudaStream_t st) {
  const int kp = plane_g_kp(c);
  if (!kp) return cudaErrorNotSupported;
  const int dx = c->dim_x, kx = c->keep_x, ky = c->keep_y;
  switch (c->dim_y) {
    case 64: return plane_g_run_64(kp, dir, in, out, planes, dx, kx, ky, tw, scale, st);
    case 128: return plane_g_run_128(kp, dir, in, out, planes, dx, kx, ky, tw, scale, st);
    case 256: return plane_g_run_256(kp, dir, in, out, planes, dx, kx, ky, tw, scale, st);
    case 512: return plane_g_run_512(kp, dir, in, out, planes, dx, kx, ky, tw, scale, st);
    case 1024: return plane_g_run_1024(kp, dir, in, out, planes, dx, kx, ky, tw, scale, st);
    default: return cudaErrorNotSupported;
  }
}

// tuned kernels of the four hand-tuned geometries (storage order q' unless natural)
static cudaError_t tuned_fwd(const tfno_cfg* c, const float2* x, float2* A, int64_t P, const float2* tw, bool nat,
                             cudaStream_t st) {
  const int dx = c->dim_x, kx = c->keep_x;
  if (dx == 512) return fwd_rpt2() ? launch_fwd<G512f, 3>(x, A, P, tw, nat, st) : launch_fwd<G512, 3>(x, A, P, tw, nat, st);
  if (dx == 256 && kx == 32) return launch_fwd<G256a, 4>(x, A, P, tw, nat, st);
  if (dx == 256 && kx == 16) return launch_fwd<G256b, 4>(x, A, P, tw, nat, st);
  if (dx == 128) return launch_fwd<G128, 4>(x, A, P, tw, nat, st);
  return cudaErrorNotSupported;
}
static cudaError_t tuned_inv(const tfno_cfg* c, const float2* Cm, float2* y, int64_t P, const float2* tw, float scale,
                             bool nat, cudaStream_t st) {
  const int dx = c->dim_x, kx = c->keep_x;
  if (dx == 512) return inv512_half() ? launch_inv<G512i, 3>(Cm, y, P, tw, scale, nat, st)
                                      : launch_inv<G512, 3>(Cm, y, P, tw, scale, nat, st);
  if (dx == 256 && kx == 32) return inv256a_8() ? launch_inv<G256a8, 2>(Cm, y, P, tw, scale, nat, st)
                                                : launch_inv<G256a, 2>(Cm, y, P, tw, scale, nat, st);
  if (dx == 256 && kx == 16) return inv256b_8() ? launch_inv<G256b8, 2>(Cm, y, P, tw, scale, nat, st)
                                                : launch_inv<G256b, 2>(Cm, y, P, tw, scale, nat, st);
  if (dx == 128) return launch_inv<G128, 2>(Cm, y, P, tw, scale, nat, st);
  return cudaErrorNotSupported;
}

// which kernels run the generic code (bit 0 forward, bit 1 inverse): always
// both outside the tuned geometries; there the measured winner per kernel
// (profiles/r02/plane_mix.txt), TFNO_PLANE_GENERIC=0..3 overrides for A/B
static int plane_mix(const tfno_cfg* c) {
  if (!plane2d_tuned(c)) return 3;
  const int env = plane_generic_env();
  if (env >= 0) return env & 3;
  // measured, same box (profiles/r02/ab_r1.txt, mix_c5.txt): at 512^2 / 64 both generic kernels
  // (C4 13.80-13.89 ms vs 14.12-14.13 tuned and 14.11-14.18 for generic forward + tuned inverse, whose
  // natural-order tile reads conflict); the tuned pair elsewhere (C3 0.460 vs 0.474-0.484, C5L 3.14 vs 3.18-3.60)
  return c->dim_x == 512 && c->dim_y == 512 && c->keep_x == 64 ? 3 : 0;
}

cudaError_t launch_plane2d_fwd(const tfno_cfg* c, const float2* x, float2* modes, const float2* tw,
                               cudaStream_t st) {
  const int64_t P = (int64_t)c->batch * c->hidden_dim;
  if (plane_mix(c) & 1) return plane_g_run(c, -1, x, modes, P, tw, 1.0f, st);
  return tuned_fwd(c, x, modes, P, tw, true, st);
}

cudaError_t launch_plane2d_inv(const tfno_cfg* c, const float2* modes, float2* y, float scale, const float2* tw,
                               cudaStream_t st) {
  const int64_t P = (int64_t)c->batch * c->output_dim;
  if (plane_mix(c) & 2) return plane_g_run(c, 1, modes, y, P, tw, scale, st);
  return tuned_inv(c, modes, y, P, tw, scale, true, st);
}

cudaError_t launch_plane2d_layer(const tfno_cfg* c, const float2* x, const float2* w, float2* y, float2* A,
                                 float2* Cm, const float2* tw, int prec, void* wimg, int wimg_ready,
                                 cudaStream_t st, void (*mark)(cudaStream_t), int mode) {
  const int64_t B = c->batch, H = c->hidden_dim, N = c->output_dim;
  const int mix = plane_mix(c);
  if (plane2d_fusedmix(c, prec, mode)) {
    // forward in the natural mode order the generic inverse reads, then the
    // channel mix + inverse in one kernel (C stays in the per-CTA L2 ring Cm)
    cudaError_t e = (mix & 1) ? plane_g_run(c, -1, x, A, B * H, tw, 1.0f, st) : tuned_fwd(c, x, A, B * H, tw, true, st);
    if (e != cudaSuccess) return e;
    if (mark) mark(st);
    if ((e = plane_g_invmix_run(c, A, w, Cm, y, tw, (float)(1.0 / ((double)c->dim_x * c->dim_y)), prec, st)) !=
        cudaSuccess)
      return e;
    if (mark) mark(st);
    return cudaSuccess;
  }
  const bool nat = mix != 0;  // the generic kernels use the natural mode order; the tuned pair its own
  cudaError_t e = (mix & 1) ? plane_g_run(c, -1, x, A, B * H, tw, 1.0f, st) : tuned_fwd(c, x, A, B * H, tw, nat, st);
  if (e != cudaSuccess) return e;
  if (mark) mark(st);
  // channel mixing over modes, 1/(dx*dy) folded into alpha (the mix is order-agnostic)
  const int64_t MQ = plane2d_modes(c);
  GemmArgs ga{MQ, N, H, B, A, 1, MQ, H * MQ, w, N, 1, 0, Cm, 1, MQ, N * MQ,
              (float)(1.0 / ((double)c->dim_x * c->dim_y))};
  ga.wimg = wimg;
  ga.wimg_ready = wimg_ready;
  if ((e = launch_cgemm_prec(ga, prec, st)) != cudaSuccess) return e;
  if (mark) mark(st);
  e = (mix & 2) ? plane_g_run(c, 1, Cm, y, B * N, tw, 1.0f, st) : tuned_inv(c, Cm, y, B * N, tw, 1.0f, nat, st);
  if (e != cudaSuccess) return e;
  if (mark) mark(st);
  return cudaSuccess;
}

}  // namespace tfno
