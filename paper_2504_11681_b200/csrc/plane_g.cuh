// Generic per-plane 2D Fourier-layer kernels (rank-2 fully_fused path) for any
// power-of-two plane dy in {64 ... 1024}, dx in [KP, 1024], and any keep up to
// 128 per axis (padded to KP = a power of two >= max(kx, ky, 8); the bins
// p >= kx or q >= ky are written as exact zeros, so the channel mix and the
// padded inverse see precisely the reference's first-keep spectrum).
//
// Same plane-per-CTA structure as plane2d.cu, with a row FFT that moves less
// through shared memory.  A row of DY = V*M points (V = 16 for DY >= 256,
// else 8) is held by a team of M threads, V points each:
//   stage 1  V-point DFT in registers over y2 (x[tt + M*y2]), twiddle
//            w_DY^{r*tt}, ONE transpose through shared memory;
//   stage 2  thread (r, a) (A = M/V lanes per sequence) takes the V values
//            tt = a + A*c, V-point DFT over c, twiddle w_M^{k*a}; the sum over
//            a is a reduce-scatter across the A lanes with warp shuffles
//            (A <= 4), so only the kept bins q = r + V*k < KY leave registers.
// The reference does the same math as x-FFT | y-FFT (pipeline.py:149-206);
// SURVEY.md Appendix A.  x direction: four-step classes x = x0 + R*x1
// (R = dx/KP) exactly as in plane2d.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"
#include "tcgen05.cuh"

namespace tfno {

template <int DY_, int KXP_, int KYP_, int NTH_>
struct PG {
  static constexpr int DY = DY_, KXP = KXP_, KYP = KYP_, NTH = NTH_;
  static constexpr int V = DY >= 256 ? 16 : 8;  // points per thread in the row FFT
  static constexpr int M = DY / V;              // threads per row team
  static constexpr int A = M / V;               // lanes per sequence in stage 2
  static constexpr int T = KYP >= V ? KYP / V : 1;  // kept bins per sequence
  static constexpr int RN = KYP >= V ? V : KYP;     // sequences with kept bins
  static constexpr int TEAMS = NTH / M;
  static constexpr int KA = KXP / 8;  // column FFT: radix 8 x radix KA
  static constexpr int IPC = KXP / TEAMS;  // row iterations per class
  static constexpr int TS = M + A;         // transpose stride: == A (mod 16) -> conflict-free
  static constexpr int TB = TEAMS * V * TS;
  static constexpr int TASKS2 = (8 * KYP + NTH - 1) / NTH;
  static constexpr int F = T >= A ? T / A : 1;  // kept bins per lane after the reduce
  // transpose buffers: a team of <= 32 threads syncs with __syncwarp, so one
  // buffer + a second (free) team sync; 2-warp teams double-buffer instead
  static constexpr int NTB = M <= 32 ? 1 : 2;
  static_assert(A >= 1 && M == A * V, "row geometry");
  static_assert(NTH % M == 0 && TEAMS >= 1 && KXP % TEAMS == 0, "teams");
  static_assert(KXP >= 8 && KA <= 16 && KYP <= DY && KYP >= 1, "keep");
  static_assert(M <= 32 || M % 32 == 0, "team shape");
};

template <int M>
__device__ __forceinline__ void gteam_sync(int team) {
  if constexpr (M <= 32)
    __syncwarp();
  else
    named_bar(1 + team, M);
}
constexpr int kGComputeBar = 15;

// reduce-scatter of CNT values over the lane bits S, S/2, ..., 1: the lane
// with bit S set keeps the upper half; `off` = first kept index
template <int CNT, int S>
__device__ __forceinline__ void lane_reduce(float2* v, int a, int& off) {
  if constexpr (S >= 1) {
    const bool hi = (a & S) != 0;
    if constexpr (CNT >= 2) {
      constexpr int H = CNT / 2;
#pragma unroll
      for (int i = 0; i < H; ++i) {
        const float2 send = hi ? v[i] : v[i + H];
        const float2 keep = hi ? v[i + H] : v[i];
        v[i] = cadd(keep, shfl_xor2(send, S));
      }
      if (hi) off += H;
      lane_reduce<H, S / 2>(v, a, off);
    } else {
      v[0] = cadd(v[0], shfl_xor2(v[0], S));
      lane_reduce<1, S / 2>(v, a, off);
    }
  }
}

// ============================================================== forward
// x[plane] (dx*DY) -> A[plane][KXP][KYP] (natural order, masked to kx x ky)
// ACCG: large keeps accumulate the classes in the output tile (L2); else the
// per-thread accumulators live in shared memory (ACCS) or registers
template <class G, int S, bool ACCG, bool ACCS>
__global__ void __launch_bounds__(G::NTH + 32, 1)
    plane_fwd_g(const float2* __restrict__ x, float2* __restrict__ Aout, int64_t planes, int dx, int kx, int ky,
                const float2* __restrict__ twg) {
  constexpr int DY = G::DY, V = G::V, M = G::M, A = G::A, T = G::T, RN = G::RN, TEAMS = G::TEAMS;
  constexpr int KXP = G::KXP, KYP = G::KYP, KA = G::KA, IPC = G::IPC, TS = G::TS, NTH = G::NTH, F = G::F;
  extern __shared__ __align__(128) uint8_t smem[];
  float2* ring = reinterpret_cast<float2*>(smem);  // S x TEAMS x DY
  float2* tb = ring + S * TEAMS * DY;              // NTB x TB transpose buffers
  float2* Tc = tb + G::NTB * G::TB;                // KXP x KYP class buffer
  float2* accs = Tc + KXP * KYP;                   // ACCS: TASKS2 x KA x NTH accumulators
  // w_DY^k with its FFMA2 companion (-w.y, w.x): the hoisted row twiddles load both halves
  // from shared memory, so ptxas keeps the companions resident instead of rebuilding each one
  // (MOV + negating FADD) before every use (~10% of this kernel's instructions)
  float4* twy = reinterpret_cast<float4*>(accs + (ACCS ? G::TASKS2 * KA * NTH : 0));
  float2* twk = reinterpret_cast<float2*>(twy + DY);  // w_KXP^k
  float2* twx = twk + KXP;                         // w_dx^k
  uint64_t* full = reinterpret_cast<uint64_t*>(twx + dx);
  uint64_t* empty = full + S;

  const int tid = threadIdx.x;
  const int R = dx / KXP;
  const int64_t nmine = planes > blockIdx.x ? (planes - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  for (int k = tid; k < DY; k += blockDim.x) {
    const float2 w = __ldg(&twg[(size_t)k * (TFNO_TW_MAX / DY)]);
    twy[k] = make_float4(w.x, w.y, -w.y, w.x);
  }
  for (int k = tid; k < KXP; k += blockDim.x) twk[k] = __ldg(&twg[(size_t)k * (TFNO_TW_MAX / KXP)]);
  for (int k = tid; k < dx; k += blockDim.x) twx[k] = __ldg(&twg[(size_t)k * (TFNO_TW_MAX / dx)]);
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
    // ---------------- producer warp: TEAMS rows per ring slot, class by class
    if (tid == NTH) {
      const uint64_t pol = policy_evict_first();
      int slot = 0, cnt = 0;
      uint32_t phase = 0;
      for (int64_t kp = 0; kp < nmine; ++kp) {
        const float2* src = x + (blockIdx.x + kp * gridDim.x) * (int64_t)dx * DY;
        for (int x0 = 0; x0 < R; ++x0) {
          for (int j = 0; j < IPC; ++j, ++cnt) {
            if (cnt >= S) mbar_wait(&empty[slot], phase ^ 1u);
            float2* dst = ring + slot * TEAMS * DY;
            mbar_expect_tx(&full[slot], TEAMS * DY * 8);
#pragma unroll 1
            for (int tm = 0; tm < TEAMS; ++tm)
              tma_load_1d(dst + tm * DY, src + (int64_t)(x0 + R * (j * TEAMS + tm)) * DY, DY * 8, &full[slot], pol);
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
  const int r_ = tt / A, a_ = tt % A;
  auto twp_at = [&](int k) {
    const float4 t = twy[k];
#ifdef TFNO_TWP_REBUILD  // A/B: companions rebuilt from w (ptxas rematerialises them per use)
    return make_twp(make_float2(t.x, t.y));
#else
    return twp{make_float2(t.x, t.y), make_float2(t.z, t.w)};
#endif
  };
  twp tw1[V];
#pragma unroll
  for (int r = 0; r < V; ++r) tw1[r] = twp_at(r * tt);
  twp tw3[T];
#pragma unroll
  for (int k = 0; k < T; ++k) tw3[k] = twp_at((V * k * a_) % DY);
  // stage-2 output validity: lanes holding a kept bin after the reduce
  const bool st_ok = (r_ < RN) && (T >= A || (a_ % (A / (T < A ? T : A))) == 0);

  constexpr bool ACCR = !ACCG && !ACCS;  // register accumulators
  float2 acc[ACCR ? G::TASKS2 : 1][ACCR ? KA : 1];
  if constexpr (ACCR) {
#pragma unroll
    for (int a = 0; a < G::TASKS2; ++a)
#pragma unroll
      for (int u = 0; u < KA; ++u) acc[a][u] = make_float2(0.f, 0.f);
  }

  int slot = 0, buf = 0;
  uint32_t phase = 0;
  for (int64_t kp = 0; kp < nmine; ++kp) {
    const int64_t pl = blockIdx.x + kp * gridDim.x;
    float2* dstA = Aout + pl * (int64_t)KXP * KYP;
#pragma unroll 1
    for (int x0 = 0; x0 < R; ++x0) {
#pragma unroll 1
      for (int j = 0; j < IPC; ++j) {
        mbar_wait(&full[slot], phase);
        float2* tbt = tb + buf * G::TB + team * V * TS;
        if (G::NTB == 1 && j > 0) gteam_sync<M>(team);  // previous row's stage 2 is done with tbt
        // ---- stage 1: V-point DFT over y2, twiddle w_DY^{r tt}, transpose
        {
          float2 v[V];
          const float2* row = ring + slot * TEAMS * DY + team * DY;
#pragma unroll
          for (int y2 = 0; y2 < V; ++y2) v[y2] = row[tt + M * y2];
          __syncwarp();
          if ((tid & 31) == 0) mbar_arrive(&empty[slot]);
          dft<V, -1>(v);
#pragma unroll
          for (int r = 1; r < V; ++r) v[r] = cmul_p(v[r], tw1[r]);
#pragma unroll
          for (int r = 0; r < RN; ++r) tbt[r * TS + tt] = v[r];
        }
        gteam_sync<M>(team);
        // ---- stage 2: V-point DFT over c, twiddle w_M^{k a}, reduce over the A lanes
        {
          float2 u[V];
#pragma unroll
          for (int c = 0; c < V; ++c) u[c] = tbt[(r_ < RN ? r_ : 0) * TS + a_ + A * c];
          float2 vals[T];
          if constexpr (T == 1) {
            float2 s0 = u[0], s1 = u[1];
#pragma unroll
            for (int c = 2; c < V; c += 2) {
              s0 = cadd(s0, u[c]);
              s1 = cadd(s1, u[c + 1]);
            }
            vals[0] = cadd(s0, s1);
          } else {
            dft<V, -1>(u);
#pragma unroll
            for (int k = 0; k < T; ++k) vals[k] = (A > 1 && k > 0) ? cmul_p(u[k % V], tw3[k]) : u[k % V];
          }
          int off = 0;
          lane_reduce<T, A / 2>(vals, a_, off);
          if (st_ok) {
            const int x1 = j * TEAMS + team;
#pragma unroll
            for (int i = 0; i < F; ++i) Tc[x1 * KYP + r_ + V * (off + i)] = vals[i];
          }
        }
        if (G::NTB == 2) buf ^= 1;
        if (++slot == S) {
          slot = 0;
          phase ^= 1u;
        }
      }  // j: rows of class x0
      named_bar(kGComputeBar, NTH);
      // ---- class x0 complete: KXP-point column FFT, pass 1 (radix 8 over m)
      for (int tau = tid; tau < KA * KYP; tau += NTH) {
        const int q = tau % KYP, i = tau / KYP;
        float2 v[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) v[m] = Tc[(i + KA * m) * KYP + q];
        dft8<-1>(v);
        if (KA > 1) {
#pragma unroll
          for (int s2 = 1; s2 < 8; ++s2) v[s2] = cmul(v[s2], twk[i * s2]);
        }
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) Tc[(s2 * KA + i) * KYP + q] = v[s2];
      }
      named_bar(kGComputeBar, NTH);
      // pass 2 (radix KA over i) + four-step twiddle w_dx^{p x0}, accumulate
#pragma unroll
      for (int jj = 0; jj < G::TASKS2; ++jj) {
        const int tau = tid + jj * NTH;
        if (tau < 8 * KYP) {
          const int q = tau % KYP, s2 = tau / KYP;
          float2 w[KA];
#pragma unroll
          for (int i = 0; i < KA; ++i) w[i] = Tc[(s2 * KA + i) * KYP + q];
          dft<KA, -1>(w);
          if constexpr (ACCG) {
            // large keeps: accumulate the classes in the (L2-resident) output tile
#pragma unroll
            for (int u = 0; u < KA; ++u) {
              const int p = s2 + 8 * u;
              float2* d = dstA + p * KYP + q;
              if (p >= kx || q >= ky) {
                if (x0 == 0) *d = make_float2(0.f, 0.f);
              } else if (x0 == 0) {
                *d = w[u];
              } else {
                float2 o = *d;
                cmac(o, w[u], twx[p * x0]);
                *d = o;
              }
            }
          } else if constexpr (ACCS) {
#pragma unroll
            for (int u = 0; u < KA; ++u) {
              float2* ap = accs + (jj * KA + u) * NTH + tid;
              float2 o = x0 == 0 ? make_float2(0.f, 0.f) : *ap;
              cmac(o, w[u], twx[(s2 + 8 * u) * x0]);
              if (x0 == R - 1) {
                const int p = s2 + 8 * u;
                dstA[p * KYP + q] = (p < kx && q < ky) ? o : make_float2(0.f, 0.f);
              } else {
                *ap = o;
              }
            }
          } else {
#pragma unroll
            for (int u = 0; u < KA; ++u) cmac(acc[jj][u], w[u], twx[(s2 + 8 * u) * x0]);
          }
        }
      }
      named_bar(kGComputeBar, NTH);
      if constexpr (ACCR) {
        if (x0 == R - 1) {
#pragma unroll
          for (int jj = 0; jj < G::TASKS2; ++jj) {
            const int tau = tid + jj * NTH;
            if (tau < 8 * KYP) {
              const int q = tau % KYP, s2 = tau / KYP;
#pragma unroll
              for (int u = 0; u < KA; ++u) {
                const int p = s2 + 8 * u;
                dstA[p * KYP + q] = (p < kx && q < ky) ? acc[jj][u] : make_float2(0.f, 0.f);
                acc[jj][u] = make_float2(0.f, 0.f);
              }
            }
          }
        }
      }
    }  // x0
  }  // planes
}

// ============================================================== inverse
// C[plane][KXP][KYP] -> y[plane] (dx*DY), scaled by `scale`.  CING: the mode
// tile is read from global (L2) per class instead of being staged in smem.
template <class G, bool CING>
__global__ void __launch_bounds__(G::NTH, 1)
    plane_inv_g(const float2* __restrict__ Cin, float2* __restrict__ y, int64_t planes, int dx,
                const float2* __restrict__ twg, float scale) {
  constexpr int DY = G::DY, V = G::V, M = G::M, A = G::A, T = G::T, RN = G::RN, TEAMS = G::TEAMS;
  constexpr int KXP = G::KXP, KYP = G::KYP, KA = G::KA, IPC = G::IPC, TS = G::TS, NTH = G::NTH;
  extern __shared__ __align__(128) uint8_t smem[];
  float2* cin = reinterpret_cast<float2*>(smem);  // KXP x KYP (TMA target; unused if CING)
  float2* Gb = cin + (CING ? 0 : KXP * KYP);      // KXP x KYP
  float2* tb = Gb + KXP * KYP;                    // NTB x TB
  float2* twy = tb + G::NTB * G::TB;              // conj w_DY^k
  float2* twk = twy + DY;                         // conj w_KXP^k
  float2* twx = twk + KXP;                        // scale * conj w_dx^k
  uint64_t* bar = reinterpret_cast<uint64_t*>(twx + dx);

  const int tid = threadIdx.x;
  const int R = dx / KXP;
  const int team = tid / M, tt = tid % M;
  const int r_ = tt / A, a_ = tt % A;
  const int64_t nmine = planes > blockIdx.x ? (planes - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  for (int k = tid; k < DY; k += NTH) twy[k] = conjf2(__ldg(&twg[(size_t)k * (TFNO_TW_MAX / DY)]));
  for (int k = tid; k < KXP; k += NTH) twk[k] = conjf2(__ldg(&twg[(size_t)k * (TFNO_TW_MAX / KXP)]));
  for (int k = tid; k < dx; k += NTH) twx[k] = cscale(conjf2(__ldg(&twg[(size_t)k * (TFNO_TW_MAX / dx)])), scale);
  if (!CING && tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();
  const uint64_t pol = policy_evict_first();
  auto issue = [&](int64_t k) {
    const int64_t pl = blockIdx.x + k * gridDim.x;
    mbar_expect_tx(bar, KXP * KYP * 8);
    tma_load_1d(cin, Cin + pl * (int64_t)KXP * KYP, KXP * KYP * 8, bar, pol);
  };
  if (!CING && tid == 0 && nmine > 0) issue(0);

  twp tw1[V], tw3[T];
#pragma unroll
  for (int r = 0; r < V; ++r) tw1[r] = make_twp(twy[r * tt]);
#pragma unroll
  for (int k = 0; k < T; ++k) tw3[k] = make_twp(twy[(V * k * a_) % DY]);
  int buf = 0;
  for (int64_t k = 0; k < nmine; ++k) {
    const int64_t pl = blockIdx.x + k * gridDim.x;
    const float2* src = CING ? Cin + pl * (int64_t)KXP * KYP : cin;
    if (!CING) mbar_wait(bar, (uint32_t)(k & 1));
    float2* yp = y + pl * (int64_t)dx * DY;
    for (int x0 = 0; x0 < R; ++x0) {
      named_bar(kGComputeBar, NTH);  // previous class's rows are done with Gb
      // ---- column iFFT, pass 1: twiddle w_dx^{+p x0} (carries the scale), radix KA over u
      for (int tau = tid; tau < 8 * KYP; tau += NTH) {
        const int q = tau % KYP, s2 = tau / KYP;
        float2 w[KA];
#pragma unroll
        for (int u = 0; u < KA; ++u) {
          const int p = s2 + 8 * u;
          const float2 cv = CING ? __ldg(&src[p * KYP + q]) : src[p * KYP + q];
          w[u] = cmul(cv, twx[p * x0]);
        }
        dft<KA, 1>(w);
#pragma unroll
        for (int i = 1; i < KA; ++i) w[i] = cmul(w[i], twk[s2 * i]);
#pragma unroll
        for (int i = 0; i < KA; ++i) Gb[(s2 * KA + i) * KYP + q] = w[i];
      }
      named_bar(kGComputeBar, NTH);
      if (!CING && x0 == R - 1 && tid == 0 && k + 1 < nmine) issue(k + 1);  // cin fully consumed
      // pass 2: radix 8 over s2 -> rows x1 = i + KA*m
      for (int tau = tid; tau < KA * KYP; tau += NTH) {
        const int q = tau % KYP, i = tau / KYP;
        float2 v[8];
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) v[s2] = Gb[(s2 * KA + i) * KYP + q];
        dft8<1>(v);
#pragma unroll
        for (int m = 0; m < 8; ++m) Gb[(i + KA * m) * KYP + q] = v[m];
      }
      named_bar(kGComputeBar, NTH);
#pragma unroll 1
      for (int j = 0; j < IPC; ++j) {
        const int x1 = j * TEAMS + team;
        float2* tbt = tb + buf * G::TB + team * V * TS;
        if (G::NTB == 1 && j > 0) gteam_sync<M>(team);  // previous row's stage B is done with tbt
        // ---- stage A: (r, a) -- bins r + V*k (k < T), twiddle w_M^{+k a}, V-point iDFT over k
        if (r_ < RN) {
          float2 u[V];
#pragma unroll
          for (int c = 0; c < V; ++c) u[c] = make_float2(0.f, 0.f);
#pragma unroll
          for (int k = 0; k < T; ++k) {
            float2 g = Gb[x1 * KYP + r_ + V * k];
            if (A > 1 && k > 0) g = cmul_p(g, tw3[k]);
            u[k % V] = (k < V) ? g : cadd(u[k % V], g);
          }
          dft_in<V, 1, (T < V ? T : V)>(u);
#pragma unroll
          for (int c = 0; c < V; ++c) tbt[r_ * TS + a_ + A * c] = u[c];
        }
        gteam_sync<M>(team);
        // ---- stage B: thread tt -- twiddle w_DY^{+r tt}, V-point iDFT over r, streaming stores
        {
          float2 v[V];
#pragma unroll
          for (int r = 0; r < V; ++r) v[r] = r < RN ? tbt[r * TS + tt] : make_float2(0.f, 0.f);
#pragma unroll
          for (int r = 1; r < RN; ++r) v[r] = cmul_p(v[r], tw1[r]);
          dft_in<V, 1, RN>(v);
          float2* orow = yp + (int64_t)(x0 + R * x1) * DY;
#pragma unroll
          for (int y2 = 0; y2 < V; ++y2) __stcs(orow + tt + M * y2, v[y2]);
        }
        if (G::NTB == 2) buf ^= 1;
      }
    }
  }
}

// ============================================================== inverse + channel mix
// One kernel for the second half of the rank-2 layer (N1: the contraction is
// no longer a pass of its own).  Work unit = task (b, n0 .. n0+GN-1):
//   mix warps (the last 4 warps): C[b, n0+g, m] = alpha * sum_h A[b, h, m] W[h, n0+g]
//     in FP32 SIMT (packed FFMA2, h ascending like cgemm.gemm_kloop,
//     cgemm.py:83-95).  A[b, h0:h0+HC, m0:m0+MC] chunks stream into a shared
//     ring with TMA bulk copies (afull / aempty mbarriers); the W columns of
//     the task sit in shared memory as (wr, wi, -wi, wr).  The task's C planes
//     go to a per-CTA two-slot ring in global memory (L2-resident, it is read
//     back within one task) -- one task ahead of the inverse warps.
//   inverse warps (the first NTH threads): plane_inv_g's padded 2D inverse of
//     each plane of the task, its mode tile TMA-loaded from the ring slot once
//     the mix warps have published it (cready) and the slot handed back
//     (cfree) when the last plane's tile has landed.
// The mode tensor A therefore makes one HBM round trip (written by the
// forward, read here) and C never leaves L2 in steady state; the reference
// keeps C on chip the same way (pipeline.py:185-206, 245-250).
constexpr int kMixThreads = 128;  // 4 mix warps
constexpr int kMixBar = 14;       // named barrier of the mix warps

// a twiddle and its companion from a (w, -w.y, w.x) shared-memory entry
__device__ __forceinline__ twp twp_ld(float4 t) {
#ifdef TFNO_TWP_REBUILD_INV  // A/B: companion rebuilt from w (ptxas rematerialises it per use)
  return make_twp(make_float2(t.x, t.y));
#else
  return twp{make_float2(t.x, t.y), make_float2(t.z, t.w)};
#endif
}

template <int MQ>
struct MixGeo {
  static constexpr int MC = MQ < 512 ? MQ : 512;  // modes per chunk (128 * MI)
  static constexpr int MI = MC / 128;              // modes per mix thread
  static constexpr int HC = 2048 / MC;             // hidden channels per chunk (16 KiB chunks)
  static constexpr int SA_MAX = 8;                 // ring depth: as many chunks as shared memory allows
  static_assert(MC % 128 == 0 && MQ % MC == 0, "mode chunking");
};

// PREC 0: FP32 SIMT mix (above).  PREC 1 / 3: the mix on the tensor cores --
// tcgen05.mma kind::tf32 (TF32, or 3xTF32 = hi*hi + hi*lo + lo*hi with
// lo = x - tf32(x)), M = 128 modes (TMEM lanes) x N = 2*GN real columns
// (re / im of the GN output channels) x K = 8 (4 hidden channels, real-
// embedded: K' = 2h + c, W'[2h+c][2n+c'] = [[Wr, Wi], [-Wi, Wr]][c][c']).
// The task's whole C (MQ/128 mode tiles x 2*GN columns, <= 512 columns) sits in
// TMEM; the mix warps stage A (global -> registers -> K-major canonical
// shared tiles, split hi/lo), one elected thread issues the MMAs and commits
// to an mbarrier per stage, and at the end of the task the four mix warps
// read their TMEM lane quarters (tcgen05.ld) into the C ring.
template <int MQ>
__host__ __device__ constexpr int invmix_tmem_cols() {
  return (MQ / 128) * 16 <= 32 ? 32 : (MQ / 128) * 16 <= 64 ? 64 : (MQ / 128) * 16 <= 128 ? 128 : (MQ / 128) * 16 <= 256 ? 256 : 512;
}

template <class G, int GN, int PREC = 0>
__global__ void __launch_bounds__(G::NTH + kMixThreads, 1)
    plane_invmix_g(const float2* __restrict__ Ain, const float2* __restrict__ W, float2* __restrict__ Cs,
                   float2* __restrict__ y, int B, int H, int N, int dx, const float2* __restrict__ twg,
                   float alpha, int SA) {
  constexpr int DY = G::DY, V = G::V, M = G::M, A = G::A, T = G::T, RN = G::RN, TEAMS = G::TEAMS;
  constexpr int KXP = G::KXP, KYP = G::KYP, KA = G::KA, IPC = G::IPC, TS = G::TS, NTH = G::NTH;
  constexpr int MQ = KXP * KYP;
  using X = MixGeo<MQ>;
  constexpr int MC = X::MC, MI = X::MI, HC = X::HC;
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int NPASS = PREC == 3 ? 2 : 1;
  static_assert(PREC == 0 || GN == 8, "tensor-core mix: N = 16 real columns");
  float2* ring = reinterpret_cast<float2*>(smem);          // SA x HC x MC (TMA targets / TC: A stages)
  float4* Wt = reinterpret_cast<float4*>(ring + SA * HC * MC);  // H x GN packed W columns (TC: W' tiles)
  const int Hp = (H + 3) & ~3;
  float2* cin = reinterpret_cast<float2*>(Wt + (size_t)(PREC ? NPASS * Hp : H) * GN);  // MQ (TMA target)
  float2* Gb = cin + MQ;                                   // MQ
  float2* tb = Gb + MQ;                                    // NTB x TB
  // conj w_DY^k with its FFMA2 companion, loaded (not rebuilt per use) like the forward's
  float4* twy = reinterpret_cast<float4*>(tb + G::NTB * G::TB);
  float2* twk = reinterpret_cast<float2*>(twy + DY);
  float2* twx = twk + KXP;
  uint64_t* bar = reinterpret_cast<uint64_t*>(twx + dx);   // cin landed
  uint64_t* cready = bar + 1;                              // [2] C slot written (128 arrivals)
  uint64_t* cfree = cready + 2;                            // [2] C slot read back (1 arrival)
  uint64_t* afull = cfree + 2;                             // [SA_MAX]
  uint64_t* aempty = afull + X::SA_MAX;                    // [SA_MAX] (4 warp arrivals)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(aempty + X::SA_MAX);  // TC: TMEM base address

  const int tid = threadIdx.x;
  const int R = dx / KXP;
  const int NG = (N + GN - 1) / GN;
  const int64_t tasks = (int64_t)B * NG;
  const int64_t nmine = tasks > blockIdx.x ? (tasks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  float2* myC = Cs + (int64_t)blockIdx.x * 2 * GN * MQ;  // this CTA's two task slots

  for (int k = tid; k < DY; k += blockDim.x) {
    const float2 w = conjf2(__ldg(&twg[(size_t)k * (TFNO_TW_MAX / DY)]));
    twy[k] = make_float4(w.x, w.y, -w.y, w.x);
  }
  for (int k = tid; k < KXP; k += blockDim.x) twk[k] = conjf2(__ldg(&twg[(size_t)k * (TFNO_TW_MAX / KXP)]));
  for (int k = tid; k < dx; k += blockDim.x) twx[k] = conjf2(__ldg(&twg[(size_t)k * (TFNO_TW_MAX / dx)]));
  if (tid == 0) {
    mbar_init(bar, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&cready[s], kMixThreads);
      mbar_init(&cfree[s], 1);
    }
    for (int s = 0; s < SA; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], kMixThreads / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();

  if (PREC != 0 && tid >= NTH) {
    if constexpr (PREC != 0) {
    // ================= mix warps, tcgen05 contraction
    constexpr int NT = MC / 128;                // M tiles per chunk
    constexpr int NMB = MQ / MC;
    constexpr int A_LBO = 2048, B_LBO = 256;    // K-group strides (16 M / 2 N' groups of 128 B)
    constexpr int ATILE = 128 * 8 * 4;          // one M tile x one K step (K' = 8), bytes
    constexpr int STAGE = NPASS * NT * ATILE;
    constexpr int NCOLS = invmix_tmem_cols<MQ>();
    constexpr uint32_t IDESC = tc::make_idesc(128, 2 * GN, true);
    constexpr int AI = NT;                      // (mode pair, channel pair) items per thread
    const int ct = tid - NTH, mw = ct >> 5, lane = tid & 31;
    uint8_t* stg = reinterpret_cast<uint8_t*>(ring);
    uint8_t* wp = reinterpret_cast<uint8_t*>(Wt);
    const int wpass = Hp * 128;                 // bytes of one W' pass (K' = 2 Hp rows of 16 columns)
    uint64_t* mmadone = afull;                  // [2] a stage's MMAs completed
    uint64_t* tdone = afull + 2;                // the task's MMAs completed
    if (mw == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::saddr(tslot)),
                   "n"(NCOLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc::fence_before();
    named_bar(kMixBar, kMixThreads);
    tc::fence_after();
    const uint32_t tmem = *tslot;
    const int NHC = Hp / 4;
    const int64_t per_task = (int64_t)NMB * NHC;
    const int64_t nch = nmine * per_task;
    float4 ra[AI][2];
    auto load_chunk = [&](int64_t c) {
      const int64_t k = c / per_task;
      const int r = (int)(c - k * per_task), mb = r / NHC, hc = r % NHC;
      const int64_t b = (blockIdx.x + k * gridDim.x) / NG;
#pragma unroll
      for (int i = 0; i < AI; ++i) {
        const int idx = ct + i * kMixThreads, mp = idx % (MC / 2), hp = idx / (MC / 2);
        const int m = mb * MC + 2 * mp, h = hc * 4 + 2 * hp;
#pragma unroll
        for (int rr = 0; rr < 2; ++rr)
          ra[i][rr] = (h + rr < H) ? __ldg(reinterpret_cast<const float4*>(Ain + ((b * H + h + rr) * (int64_t)MQ + m)))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto store_chunk = [&](int st) {
      uint8_t* sA = stg + st * STAGE;
#pragma unroll
      for (int i = 0; i < AI; ++i) {
        const int idx = ct + i * kMixThreads, mp = idx % (MC / 2), hp = idx / (MC / 2);
        const int m = 2 * mp, t = m / 128, ml = m % 128;
        const float4 v0 = ra[i][0], v1 = ra[i][1];  // (re, im) of modes m, m+1 at h; at h+1
        const float4 r0 = make_float4(v0.x, v0.y, v1.x, v1.y), r1 = make_float4(v0.z, v0.w, v1.z, v1.w);
        const uint32_t o0 = t * ATILE + cm_off(ml, 4 * hp, A_LBO), o1 = t * ATILE + cm_off(ml + 1, 4 * hp, A_LBO);
        if constexpr (NPASS == 1) {
          *reinterpret_cast<float4*>(sA + o0) = r0;
          *reinterpret_cast<float4*>(sA + o1) = r1;
        } else {
          const float4 h0 = hi4(r0), h1 = hi4(r1);
          *reinterpret_cast<float4*>(sA + o0) = h0;
          *reinterpret_cast<float4*>(sA + o1) = h1;
          *reinterpret_cast<float4*>(sA + NT * ATILE + o0) = sub4(r0, h0);
          *reinterpret_cast<float4*>(sA + NT * ATILE + o1) = sub4(r1, h1);
        }
      }
    };
    int64_t gch = 0;
    if (nch > 0) load_chunk(0);
    for (int64_t k = 0; k < nmine; ++k) {
      const int64_t t = blockIdx.x + k * gridDim.x;
      const int n0 = (int)(t % NG) * GN;
      const int gn = min(GN, N - n0);
      named_bar(kMixBar, kMixThreads);  // the previous task's MMAs have completed (tdone): W' is free
      // W' of the task, K-major canonical: row n' = 2n + c' holds K' = 2h + c
      for (int i = ct; i < GN * (Hp / 2); i += kMixThreads) {
        const int nl = i % GN, hp = i / GN, h = 2 * hp;
        const bool okn = nl < gn;
        const float2 w0 = (okn && h < H) ? __ldg(&W[(int64_t)h * N + n0 + nl]) : make_float2(0.f, 0.f);
        const float2 w1 = (okn && h + 1 < H) ? __ldg(&W[(int64_t)(h + 1) * N + n0 + nl]) : make_float2(0.f, 0.f);
        const float4 re_row = make_float4(w0.x, -w0.y, w1.x, -w1.y), im_row = make_float4(w0.y, w0.x, w1.y, w1.x);
        const uint32_t o0 = cm_off(2 * nl, 4 * hp, B_LBO), o1 = cm_off(2 * nl + 1, 4 * hp, B_LBO);
        if constexpr (NPASS == 1) {
          *reinterpret_cast<float4*>(wp + o0) = re_row;
          *reinterpret_cast<float4*>(wp + o1) = im_row;
        } else {
          const float4 h0 = hi4(re_row), h1 = hi4(im_row);
          *reinterpret_cast<float4*>(wp + o0) = h0;
          *reinterpret_cast<float4*>(wp + o1) = h1;
          *reinterpret_cast<float4*>(wp + wpass + o0) = sub4(re_row, h0);
          *reinterpret_cast<float4*>(wp + wpass + o1) = sub4(im_row, h1);
        }
      }
      const int s = (int)(k & 1);
      if (k >= 2) mbar_wait(&cfree[s], (uint32_t)(((k >> 1) - 1) & 1));  // the inverse has read slot s back
      float2* cdst = myC + (int64_t)s * GN * MQ;
#pragma unroll 1
      for (int mb = 0; mb < NMB; ++mb) {
#pragma unroll 1
        for (int hc = 0; hc < NHC; ++hc, ++gch) {
          const int st = (int)(gch & 1);
          if (gch >= 2) mbar_wait(&mmadone[st], (uint32_t)(((gch - 2) >> 1) & 1));  // stage st drained
          store_chunk(st);
          if (gch + 1 < nch) load_chunk(gch + 1);
          fence_proxy_async();  // generic smem stores -> the tensor core's reads
          named_bar(kMixBar, kMixThreads);
          if (ct == 0) {
            tc::fence_after();
            const uint32_t a0 = tc::saddr(stg + st * STAGE), b0 = tc::saddr(wp) + 2 * hc * B_LBO;
#pragma unroll
            for (int tt = 0; tt < NT; ++tt) {
              const uint32_t d = tmem + (uint32_t)((mb * NT + tt) * 2 * GN);
              const uint64_t ad = tc::make_desc(a0 + tt * ATILE, A_LBO, 128), bd = tc::make_desc(b0, B_LBO, 128);
              tc::mma_tf32(d, ad, bd, IDESC, hc > 0 ? 1u : 0u);
              if constexpr (NPASS == 2) {
                tc::mma_tf32(d, ad, tc::make_desc(b0 + wpass, B_LBO, 128), IDESC, 1u);
                tc::mma_tf32(d, tc::make_desc(a0 + NT * ATILE + tt * ATILE, A_LBO, 128), bd, IDESC, 1u);
              }
            }
            tc::commit(&mmadone[st]);
          }
        }
      }
      if (ct == 0) tc::commit(tdone);
      mbar_wait(tdone, (uint32_t)(k & 1));
      tc::fence_after();
      // drain: this warp's 32 TMEM lanes = modes tg*128 + 32*mw + lane of every mode tile tg
#pragma unroll 1
      for (int tp = 0; tp < MQ / 256; ++tp) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(mw * 32) << 16) + (uint32_t)(tp * 32), v);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int m = (2 * tp + hf) * 128 + mw * 32 + lane;
#pragma unroll
          for (int g = 0; g < GN; ++g)
            if (g < gn)
              cdst[(int64_t)g * MQ + m] = make_float2(alpha * v[hf * 16 + 2 * g], alpha * v[hf * 16 + 2 * g + 1]);
        }
      }
      tc::fence_before();   // TMEM reads complete before the next task's MMAs (after the next barrier)
      fence_proxy_async_global();  // the C tile is read back with cp.async.bulk
      mbar_arrive(&cready[s]);
    }
    tc::fence_before();
    named_bar(kMixBar, kMixThreads);
    if (mw == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(NCOLS) : "memory");
    }
    return;
  }
  if (tid >= NTH) {
    // ================= mix warps
    const int ct = tid - NTH;
    constexpr int NMB = MQ / MC;
    const int NHC = (H + HC - 1) / HC;
    const int64_t per_task = (int64_t)NMB * NHC;
    const int64_t nch = nmine * per_task;
    const uint64_t pol_a = policy_evict_last();  // A[b] is read by the NG tasks of batch b
    auto issue_chunk = [&](int64_t c, int slot) {
      const int64_t k = c / per_task;
      const int r = (int)(c - k * per_task), mb = r / NHC, hc = r % NHC;
      const int64_t b = (blockIdx.x + k * gridDim.x) / NG;
      const int h0 = hc * HC, hn = min(HC, H - h0);
      mbar_expect_tx(&afull[slot], (uint32_t)(hn * MC * 8));
      const float2* src = Ain + ((b * H + h0) * (int64_t)MQ + (int64_t)mb * MC);
      for (int kk = 0; kk < hn; ++kk)
        tma_load_1d(ring + (slot * HC + kk) * MC, src + (int64_t)kk * MQ, MC * 8, &afull[slot], pol_a);
    };
    if (ct == 0)
      for (int64_t c = 0; c < SA && c < nch; ++c) issue_chunk(c, (int)c);
    int64_t c = 0;
    int aslot = 0;
    uint32_t aphase = 0;
    for (int64_t k = 0; k < nmine; ++k) {
      const int64_t t = blockIdx.x + k * gridDim.x;
      const int n0 = (int)(t % NG) * GN;
      const int gn = min(GN, N - n0);
      named_bar(kMixBar, kMixThreads);  // all mix warps are done with the previous task's Wt
      for (int i = ct; i < H * GN; i += kMixThreads) {
        const int h = i / GN, g = i % GN;
        const float2 w = (g < gn) ? __ldg(&W[(int64_t)h * N + n0 + g]) : make_float2(0.f, 0.f);
        Wt[i] = make_float4(w.x, w.y, -w.y, w.x);
      }
      named_bar(kMixBar, kMixThreads);
      const int s = (int)(k & 1);
      if (k >= 2) mbar_wait(&cfree[s], (uint32_t)(((k >> 1) - 1) & 1));  // the inverse has read slot s back
      float2* cdst = myC + (int64_t)s * GN * MQ;
#pragma unroll 1
      for (int mb = 0; mb < NMB; ++mb) {
        float2 acc[MI][GN];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int g = 0; g < GN; ++g) acc[i][g] = make_float2(0.f, 0.f);
#pragma unroll 1
        for (int hc = 0; hc < NHC; ++hc, ++c) {
          const int slot = aslot;
          mbar_wait(&afull[slot], aphase);
          const float2* As = ring + slot * HC * MC + ct;
          const float4* wt = Wt + hc * HC * GN;
          const int hn = min(HC, H - hc * HC);
#pragma unroll 2
          for (int kk = 0; kk < hn; ++kk) {
            float2 a[MI];
#pragma unroll
            for (int i = 0; i < MI; ++i) a[i] = As[kk * MC + 128 * i];
#pragma unroll
            for (int g = 0; g < GN; ++g) {
              const float4 w = wt[kk * GN + g];
#pragma unroll
              for (int i = 0; i < MI; ++i) {
                acc[i][g] = fma2(make_float2(a[i].x, a[i].x), make_float2(w.x, w.y), acc[i][g]);
                acc[i][g] = fma2(make_float2(a[i].y, a[i].y), make_float2(w.z, w.w), acc[i][g]);
              }
            }
          }
          __syncwarp();
          if ((ct & 31) == 0) mbar_arrive(&aempty[slot]);
          if (ct == 0 && c + SA < nch) {  // refill the slot once all four mix warps are done with it
            mbar_wait(&aempty[slot], aphase);
            issue_chunk(c + SA, slot);
          }
          if (++aslot == SA) {
            aslot = 0;
            aphase ^= 1u;
          }
        }
#pragma unroll
        for (int g = 0; g < GN; ++g)
          if (g < gn)
#pragma unroll
            for (int i = 0; i < MI; ++i) cdst[(int64_t)g * MQ + mb * MC + ct + 128 * i] = cscale(acc[i][g], alpha);
      }
      fence_proxy_async_global();  // the C tile is read back with cp.async.bulk
      mbar_arrive(&cready[s]);
    }
    return;
  }

  // ================= inverse warps (plane_inv_g per plane of each task)
  const int team = tid / M, tt = tid % M;
  const int r_ = tt / A, a_ = tt % A;
  const uint64_t pol = policy_evict_first();
  auto task_gn = [&](int64_t k) {
    const int64_t t = blockIdx.x + k * gridDim.x;
    return min(GN, N - (int)(t % NG) * GN);
  };
  // tid 0: mode tile of plane g of task k -> cin (waits for the slot to be published)
  auto issue = [&](int64_t k, int g) {
    const int s = (int)(k & 1);
    if (g == 0) mbar_wait(&cready[s], (uint32_t)((k >> 1) & 1));
    mbar_expect_tx(bar, MQ * 8);
    tma_load_1d(cin, myC + ((int64_t)s * GN + g) * MQ, MQ * 8, bar, pol);
  };
  if (tid == 0 && nmine > 0) issue(0, 0);

  twp tw1[V], tw3[T];
#pragma unroll
  for (int r = 0; r < V; ++r) tw1[r] = twp_ld(twy[r * tt]);
#pragma unroll
  for (int k = 0; k < T; ++k) tw3[k] = twp_ld(twy[(V * k * a_) % DY]);
  int buf = 0;
  uint32_t pc = 0;  // planes done (cin phase)
  for (int64_t k = 0; k < nmine; ++k) {
    const int64_t t = blockIdx.x + k * gridDim.x;
    const int64_t b = t / NG;
    const int n0 = (int)(t % NG) * GN;
    const int gn = min(GN, N - n0);
    for (int g = 0; g < gn; ++g, ++pc) {
      mbar_wait(bar, pc & 1u);
      if (tid == 0 && g == gn - 1) mbar_arrive(&cfree[k & 1]);  // slot fully read back
      float2* yp = y + (b * N + n0 + g) * (int64_t)dx * DY;
      for (int x0 = 0; x0 < R; ++x0) {
        named_bar(kGComputeBar, NTH);  // previous class's rows are done with Gb
        for (int tau = tid; tau < 8 * KYP; tau += NTH) {
          const int q = tau % KYP, s2 = tau / KYP;
          float2 w[KA];
#pragma unroll
          for (int u = 0; u < KA; ++u) {
            const int p = s2 + 8 * u;
            w[u] = cmul(cin[p * KYP + q], twx[p * x0]);
          }
          dft<KA, 1>(w);
#pragma unroll
          for (int i = 1; i < KA; ++i) w[i] = cmul(w[i], twk[s2 * i]);
#pragma unroll
          for (int i = 0; i < KA; ++i) Gb[(s2 * KA + i) * KYP + q] = w[i];
        }
        named_bar(kGComputeBar, NTH);
        if (x0 == R - 1 && tid == 0) {  // cin fully consumed: next plane's tile
          if (g + 1 < gn)
            issue(k, g + 1);
          else if (k + 1 < nmine)
            issue(k + 1, 0);
        }
        for (int tau = tid; tau < KA * KYP; tau += NTH) {
          const int q = tau % KYP, i = tau / KYP;
          float2 v[8];
#pragma unroll
          for (int s2 = 0; s2 < 8; ++s2) v[s2] = Gb[(s2 * KA + i) * KYP + q];
          dft8<1>(v);
#pragma unroll
          for (int m = 0; m < 8; ++m) Gb[(i + KA * m) * KYP + q] = v[m];
        }
        named_bar(kGComputeBar, NTH);
#pragma unroll 1
        for (int j = 0; j < IPC; ++j) {
          const int x1 = j * TEAMS + team;
          float2* tbt = tb + buf * G::TB + team * V * TS;
          if (G::NTB == 1 && j > 0) gteam_sync<M>(team);
          if (r_ < RN) {
            float2 u[V];
#pragma unroll
            for (int c = 0; c < V; ++c) u[c] = make_float2(0.f, 0.f);
#pragma unroll
            for (int kb = 0; kb < T; ++kb) {
              float2 gv = Gb[x1 * KYP + r_ + V * kb];
              if (A > 1 && kb > 0) gv = cmul_p(gv, tw3[kb]);
              u[kb % V] = (kb < V) ? gv : cadd(u[kb % V], gv);
            }
            dft_in<V, 1, (T < V ? T : V)>(u);
#pragma unroll
            for (int c = 0; c < V; ++c) tbt[r_ * TS + a_ + A * c] = u[c];
          }
          gteam_sync<M>(team);
          {
            float2 v[V];
#pragma unroll
            for (int r = 0; r < V; ++r) v[r] = r < RN ? tbt[r * TS + tt] : make_float2(0.f, 0.f);
#pragma unroll
            for (int r = 1; r < RN; ++r) v[r] = cmul_p(v[r], tw1[r]);
            dft_in<V, 1, RN>(v);
            float2* orow = yp + (int64_t)(x0 + R * x1) * DY;
#pragma unroll
            for (int y2 = 0; y2 < V; ++y2) __stcs(orow + tt + M * y2, v[y2]);
          }
          if (G::NTB == 2) buf ^= 1;
        }
      }
    }
  }
}

}  // namespace tfno
