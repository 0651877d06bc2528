// Fused 1D Fourier layer (K6, reference pipeline.py:185-206 + 236-275 for
// rank 1): FFT -> truncate -> channel CGEMM -> zero-pad -> iFFT in ONE
// persistent sm_100a kernel; only x, y (and the L2-resident W) touch HBM.
//
// Warp-specialised, one CTA per SM, 20 warps (registers split with setmaxnreg):
//   8 FFT warps     TEAMS = 256/L row teams (L = 16: N = 256 per half warp;
//                   L = 32: N = 1024 per warp).  Per work item g (a batch
//                   element for rank 1) they walk the hidden dimension in
//                   chunks of KC = TEAMS channel rows, in step with the GEMM
//                   k-loop: load the row from its TMA slot into registers,
//                   release the slot, truncated register FFT (wf_dft.cuh:
//                   DFT_L, twiddle, swizzled smem transpose, first-KP DFT_L),
//                   kept bins -> A chunk ring As[s][h][q].  After the forward
//                   of item i they run the zero-padded inverse of item i-1's
//                   output rows from the C tile (scaled 1/N, streaming stores).
//   8 GEMM warps    acc[q][n] += As[h][q] * W[h][n], FP32 FFMA, TI x TJ complex
//                   register tile per thread, k ascending like cgemm.gemm_kloop;
//                   at the end of an item the tile goes to Cs for the FFT warps.
//   producer WG     one thread: cp.async.bulk of each team's next input row into its slot
//                   (L2 evict-first) and of the chunk's W rows W[h0:h0+KC][:]
//                   into a 2-slot ring (evict-last).
// Every hand-off is an mbarrier (full/empty pairs for rows, W chunks, A chunks
// and the C tile), so the GEMM of item i overlaps the forward FFTs of item i
// and the inverse FFTs of item i-1; there is no CTA-wide barrier in the loop.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"
#include "wf_dft.cuh"

namespace tfno {

template <int L, int V, int KP, int TI, int TJ, int NOUT>
struct F1Geo;

// A element e of the chunk ring: a (AW = 1) or (a.x, a.y, -a.y, a.x) (AW = 2)
template <int AW>
__device__ __forceinline__ void put_a(float2* As, int e, float2 a) {
  if constexpr (AW == 2)
    reinterpret_cast<float4*>(As)[e] = make_float4(a.x, a.y, -a.y, a.x);
  else
    As[e] = a;
}

// acc += a * b with a staged as (a.x, a.y, -a.y, a.x): acc += b.x * a + b.y * (-a.y, a.x)
__device__ __forceinline__ void cmac_comp(float2& acc, float4 a, float2 b) {
#ifdef TFNO_SCALAR_COMPLEX
  acc.x = fmaf(b.y, a.z, fmaf(b.x, a.x, acc.x));
  acc.y = fmaf(b.y, a.w, fmaf(b.x, a.y, acc.y));
#else
  acc = fma2(make_float2(b.x, b.x), make_float2(a.x, a.y), acc);
  acc = fma2(make_float2(b.y, b.y), make_float2(a.z, a.w), acc);
#endif
}

template <int L, int V, int KP, int TI, int TJ, int NOUT>
struct F1Geo {
  // N = L * V: L lanes per row team, V values per lane (V = L: square rows N = 256 / 1024;
  // V = 8 with L = 16: N = 128)
  static constexpr int N = L * V, NFT = 256, NGT = 256, TEAMS = NFT / L, KC = TEAMS, KT = KP * L;
  static constexpr int NTH = NFT + NGT + 128;  // + one producer warpgroup (3 warps idle)
  static constexpr int NA = 2;                 // A chunk ring depth
  static constexpr int MT = KT / TI, NTG = NOUT / TJ;
  static_assert(MT * NTG == NGT, "GEMM thread grid must cover the GEMM warps");
  static_assert(NOUT % TEAMS == 0, "inverse rows per team");
  static constexpr int BAR_BYTES = 2048;  // >= 8 * (2 * TEAMS * NSLOT + 2 + 2 + 2 * NA + 2)
  // float2 units after the barrier block; NSLOT input-row slots per team; AW float2 per A element
  static constexpr size_t total_aw(int ns, int aw) {
    return (size_t)TEAMS * N * ns + 2 * KC * NOUT + NA * KC * KT * aw + KT * NOUT + TEAMS * N + N + L;
  }
  // A elements staged with their companion (a.x, a.y, -a.y, a.x) when it fits: the GEMM
  // warps then issue only FFMA2 (b.x broadcast * a, b.y broadcast * companion) -- without it
  // ptxas builds (-b.y, b.x) pairs with MOV / FADD, ~0.6 extra issue slots per FFMA2
#ifdef TFNO_F1_NO_ACOMP
  static constexpr int AW = 1;
#else
  // (only where it does not cost an input-row slot)
  static constexpr int NS1 = (BAR_BYTES + 8 * total_aw(4, 1) <= 220 * 1024) ? 4 : (BAR_BYTES + 8 * total_aw(2, 1) <= 220 * 1024) ? 2 : 1;
  static constexpr int AW = (BAR_BYTES + 8 * total_aw(NS1, 2) <= 220 * 1024) ? 2 : 1;
#endif
  static constexpr size_t total(int ns) { return total_aw(ns, AW); }
  // input-row slots per team: as deep a prefetch as fits (4 rows in flight per team at N <= 256)
  static constexpr int NSLOT = (BAR_BYTES + 8 * total(4) <= 220 * 1024) ? 4 : (BAR_BYTES + 8 * total(2) <= 220 * 1024) ? 2 : 1;
  static_assert(8 * (2 * TEAMS * NSLOT + 4 + 2 * NA + 2) <= BAR_BYTES, "mbarrier block");
  static constexpr int OFF_SLOT = 0;
  static constexpr int OFF_W = OFF_SLOT + TEAMS * N * NSLOT;
  static constexpr int OFF_A = OFF_W + 2 * KC * NOUT;
  static constexpr int OFF_C = OFF_A + NA * KC * KT * AW;
  static constexpr int OFF_TR = OFF_C + KT * NOUT;
  static constexpr int OFF_TWN = OFF_TR + TEAMS * N;
  static constexpr int OFF_TWL = OFF_TWN + N;
  static constexpr int TOTAL = OFF_TWL + L;
  static constexpr size_t smem_bytes() { return BAR_BYTES + sizeof(float2) * (size_t)TOTAL; }
  // register split (setmaxnreg) inside the CTA's launch allocation of 640 x 96:
  // producer warpgroup 24, FFT warps 96 (unchanged), GEMM warps 128
  // (L = 32 rows hold 32 complex values per lane: FFT warps get 112, GEMM warps 112)
  // (an 88 / 136 split for the large tiles measured no faster: N256 H256 0.541 ms either way)
  static constexpr int REG_LAUNCH = 96, REG_PROD = 24, REG_FFT = L == 32 ? 112 : 96, REG_GEMM = L == 32 ? 112 : 128;
  static_assert(128 * REG_PROD + NFT * REG_FFT + NGT * REG_GEMM <= NTH * REG_LAUNCH, "register pool");
};

// L x L transpose tile without padding: column XOR-swizzled by the row, so
// both the row-wise writes and the column-wise reads of a team are
// bank-conflict free.
template <int L>
__device__ __forceinline__ int tsw(int r, int c) {
  return r * L + (c ^ r);
}
// ---- cluster / DSMEM helpers (hidden-channel split over a thread-block cluster)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ float2 ld_dsmem(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(10000000u)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 8 x 16 tile of the N = 128 rows ([k1][t]): the column is XOR-ed with 2*k1 so
// the row writes (16 consecutive t) and the (k1 = lane/2, t = lane%2 + 2t')
// reads of a half warp are both conflict free.
__device__ __forceinline__ int tsw8(int r, int c) { return r * 16 + (c ^ (2 * r)); }

// PART: 0 = the full layer; 1 = K4 (fused_fft_gemm: FFT + GEMM, the C tile goes to
// a.C and the padded y-iFFT runs as its own pass); 2 = K5 (fused_gemm_ifft: the
// kept bins are read from a.A -- written by the y-FFT pass -- instead of being
// transformed, then GEMM + padded iFFT as usual)
template <int L, int V, int KP, int TI, int TJ, int NOUT, int CS, int PART = 0>
__global__ void __launch_bounds__(640, 1) fused1d_kernel(FusedArgs a) {
  // CS > 1: a cluster of CS CTAs shares each item: CTA r transforms and mixes
  // the hidden channels [r*H/CS, (r+1)*H/CS), the CS partial C tiles are summed
  // in a fixed order over distributed shared memory, and CTA r runs the
  // inverse of output rows [r*NOUT/CS, (r+1)*NOUT/CS).
  using G = F1Geo<L, V, KP, TI, TJ, NOUT>;
  constexpr int N = G::N, TEAMS = G::TEAMS, KC = G::KC, KT = G::KT, MT = G::MT, NTG = G::NTG, NA = G::NA;
  constexpr int NGW = G::NGT / 32, NS = G::NSLOT;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [TEAMS][NS] row slot filled
  uint64_t* empty = full + TEAMS * NS;                  // [TEAMS][NS] row slot free
  uint64_t* wfull = empty + TEAMS * NS;                 // [2]
  uint64_t* wempty = wfull + 2;                         // [2]
  uint64_t* afull = wempty + 2;                         // [NA]
  uint64_t* aempty = afull + NA;                        // [NA]
  uint64_t* cfull = aempty + NA;                        // C tile written
  uint64_t* cempty = cfull + 1;                         // C tile consumed
  float2* base = reinterpret_cast<float2*>(smem + G::BAR_BYTES);
  float2* slots = base + G::OFF_SLOT;
  float2* Wr = base + G::OFF_W;
  float2* As = base + G::OFF_A;
  float2* Cs = base + G::OFF_C;
  float2* tr = base + G::OFF_TR;
  float2* twN = base + G::OFF_TWN;
  float2* twL = base + G::OFF_TWL;

  const int tid = threadIdx.x;
  const int keep = a.keep;
  const int cr = CS > 1 ? (int)cluster_rank() : 0;
  const int Hc = a.H / CS, h_off = cr * Hc;  // this CTA's hidden channels
  const int nchunks = Hc / KC;
  const int S = (CS == 1 && a.nsplit > 1) ? a.nsplit : 1;  // items = row groups x output-channel splits
  const int64_t items = a.G * S;
  const int64_t first = CS > 1 ? (int64_t)(blockIdx.x / CS) : (int64_t)blockIdx.x;  // item stride: units
  const int64_t units = CS > 1 ? (int64_t)(gridDim.x / CS) : (int64_t)gridDim.x;
  for (int k = tid; k < L; k += blockDim.x) twL[k] = __ldg(&a.twg[(size_t)k * (TFNO_TW_MAX / L)]);
  for (int i = tid; i < N; i += blockDim.x) {  // [k1][t] = w_N^{t k1}, k1 < V, t < L
    const int k1 = i / L, t = i % L;
    twN[i] = __ldg(&a.twg[(size_t)((t * k1) % N) * (TFNO_TW_MAX / N)]);
  }
  if (tid == 0) {
    for (int t = 0; t < TEAMS * NS; ++t) {
      mbar_init(&full[t], 1);
      mbar_init(&empty[t], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], NGW);
    }
    for (int s = 0; s < NA; ++s) {
      mbar_init(&afull[s], TEAMS);
      mbar_init(&aempty[s], NGW);
    }
    mbar_init(cfull, CS * NGW);    // every CTA of the cluster publishes its partial C
    mbar_init(cempty, CS * TEAMS); // every CTA of the cluster has read this CTA's partial
    fence_mbar_init();
  }
  __syncthreads();
  if constexpr (CS > 1) cluster_sync_all();  // peers' barriers initialised before any remote arrive
  // PDL: the prologue above (barriers, twiddle tables) overlapped the previous layer's tail;
  // x / W / y are touched only after it has completed
  pdl_wait();
  pdl_launch_dependents();

  if (tid >= G::NFT + G::NGT) {
    // ================= producer warpgroup (one elected thread issues)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(G::REG_PROD));
    if (tid == G::NFT + G::NGT) {
      const int64_t nmine = (items - first + units - 1) / units;
      const uint64_t pol_x = policy_evict_first();
      const uint64_t pol_w = policy_evict_last();
      const uint32_t wbytes = (uint32_t)(KC * NOUT * sizeof(float2));
      int64_t kk = 0;  // chunks issued so far (the same count for every team)
      for (int64_t it = 0; it < nmine; ++it) {
        const int64_t item = first + it * units;
        const int64_t g = item / S, n0 = (item % S) * NOUT;
        const int64_t bb = g / a.gx, pp = g % a.gx;
        // PART 2 streams the y-FFT's kept bins (keep complex per row) instead of the input rows
        const float2* xg = PART == 2 ? a.A + bb * a.a_sb + pp * a.a_sp : a.x + bb * a.x_sb + pp * a.x_sp;
        const int64_t rstride = PART == 2 ? a.a_sh : a.x_sh;
        const uint32_t rbytes = (uint32_t)((PART == 2 ? keep : N) * sizeof(float2));
        for (int c = 0; c < nchunks; ++c, ++kk) {
          const int rs = (int)(kk % NS);
          const int64_t use = kk / NS;
#pragma unroll 1
          for (int t = 0; t < TEAMS; ++t) {
            const int b = t * NS + rs;
            if (use >= 1) mbar_wait(&empty[b], (uint32_t)((use - 1) & 1));
            mbar_expect_tx(&full[b], rbytes);
            tma_load_1d(slots + b * N, xg + (int64_t)(h_off + c * KC + t) * rstride, rbytes, &full[b], pol_x);
          }
          const int ws = (int)(kk & 1);
          if (kk >= 2) mbar_wait(&wempty[ws], (uint32_t)(((kk >> 1) - 1) & 1));
          mbar_expect_tx(&wfull[ws], wbytes);
          if (S == 1) {
            tma_load_1d(Wr + ws * KC * NOUT, a.W + (int64_t)(h_off + c * KC) * NOUT, wbytes, &wfull[ws], pol_w);
          } else {  // this split's columns W[h][n0:n0+NOUT], one bulk copy per row
#pragma unroll 1
            for (int r = 0; r < KC; ++r)
              tma_load_1d(Wr + (ws * KC + r) * NOUT, a.W + (int64_t)(c * KC + r) * a.N + n0, NOUT * sizeof(float2),
                          &wfull[ws], pol_w);
          }
        }
      }
    }
    return;
  }

  if (tid >= G::NFT) {
    // ================= GEMM warps
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(G::REG_GEMM));
    const int64_t nmine = (items - first + units - 1) / units;
    const int gt = tid - G::NFT;
    const int tm = gt % MT, tn = gt / MT;
    int64_t kk = 0;
    for (int64_t it = 0; it < nmine; ++it) {
      float2 acc[TI][TJ];
#pragma unroll
      for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < TJ; ++j) acc[i][j] = make_float2(0.f, 0.f);
      for (int c = 0; c < nchunks; ++c, ++kk) {
        const int s = (int)(kk % NA), ws = (int)(kk & 1);
        mbar_wait(&afull[s], (uint32_t)((kk / NA) & 1));
        mbar_wait(&wfull[ws], (uint32_t)((kk >> 1) & 1));
        const float2* Wc = Wr + ws * KC * NOUT;
        if constexpr (G::AW == 2) {
          const float4* Ab = reinterpret_cast<const float4*>(As) + s * KC * KT;
#pragma unroll 4
          for (int hl = 0; hl < KC; ++hl) {
            float4 av[TI];
            float2 bv[TJ];
#pragma unroll
            for (int i = 0; i < TI; ++i) av[i] = Ab[hl * KT + tm + MT * i];
#pragma unroll
            for (int j = 0; j < TJ; ++j) bv[j] = Wc[hl * NOUT + tn + NTG * j];
#pragma unroll
            for (int i = 0; i < TI; ++i)
#pragma unroll
              for (int j = 0; j < TJ; ++j) cmac_comp(acc[i][j], av[i], bv[j]);
          }
        } else {
          const float2* Ab = As + s * KC * KT;
#pragma unroll 4
          for (int hl = 0; hl < KC; ++hl) {
            float2 av[TI], bv[TJ];
#pragma unroll
            for (int i = 0; i < TI; ++i) av[i] = Ab[hl * KT + tm + MT * i];
#pragma unroll
            for (int j = 0; j < TJ; ++j) bv[j] = Wc[hl * NOUT + tn + NTG * j];
#pragma unroll
            for (int i = 0; i < TI; ++i)
#pragma unroll
              for (int j = 0; j < TJ; ++j) cmac(acc[i][j], av[i], bv[j]);
          }
        }
        __syncwarp();
        if ((gt & 31) == 0) {
          mbar_arrive(&aempty[s]);
          mbar_arrive(&wempty[ws]);
        }
      }
      // hand the C tile to the FFT warps (once they are done with the previous one)
      if (it >= 1) {
        if constexpr (CS > 1)
          mbar_wait_cluster(cempty, (uint32_t)((it - 1) & 1));
        else
          mbar_wait(cempty, (uint32_t)((it - 1) & 1));
      }
#pragma unroll
      for (int j = 0; j < TJ; ++j)
#pragma unroll
        for (int i = 0; i < TI; ++i) Cs[(tn + NTG * j) * KT + tm + MT * i] = acc[i][j];
      if constexpr (CS > 1) {
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        __syncwarp();
        if ((gt & 31) == 0)
          for (int r = 0; r < CS; ++r) mbar_arrive_cluster(mapa_rank(cfull, (uint32_t)r));
      } else {
        __syncwarp();
        if ((gt & 31) == 0) mbar_arrive(cfull);
      }
    }
    return;
  }

  // ================= FFT warps
  if constexpr (G::REG_FFT > G::REG_LAUNCH) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(G::REG_FFT));
  if constexpr (G::REG_FFT < G::REG_LAUNCH) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(G::REG_FFT));
  const int64_t nmine = (items - first + units - 1) / units;  // grid <= items
  const int lane = tid % L, team = tid / L;
  const unsigned tmask = L == 32 ? 0xffffffffu : (0xffffu << (16 * (team & 1)));
  float2* trr = tr + team * N;
  int64_t kk = 0;
  for (int64_t it = 0; it <= nmine; ++it) {
    if (it < nmine) {
      // ---- forward of item it: channel rows h = c*KC + team -> A chunk ring
      for (int c = 0; c < nchunks; ++c, ++kk) {
        const int b = team * NS + (int)(kk % NS);
        mbar_wait(&full[b], (uint32_t)((kk / NS) & 1));
        const float2* slot = slots + b * N;
        const int s = (int)(kk % NA);  // A chunk slot
        if constexpr (PART == 2) {
          // the kept bins of this row, as the y-FFT pass wrote them (slot[q], q < keep)
          constexpr int QB = V == L ? KP : 2 * KP;  // bins per lane
          float2 o[QB];
#pragma unroll
          for (int k2 = 0; k2 < QB; ++k2) {
            const int q = V == L ? lane + L * k2 : (lane >> 1) + 8 * k2;
            o[k2] = (q < keep && (V == L || (k2 & 1) == (lane & 1))) ? slot[q] : make_float2(0.f, 0.f);
          }
          __syncwarp(tmask);
          if (lane == 0) mbar_arrive(&empty[b]);
          if (kk >= NA) mbar_wait(&aempty[s], (uint32_t)(((kk / NA) - 1) & 1));
#pragma unroll
          for (int k2 = 0; k2 < QB; ++k2) {
            if (V != L && (k2 & 1) != (lane & 1)) continue;
            const int q = V == L ? lane + L * k2 : (lane >> 1) + 8 * k2;
            put_a<G::AW>(As, s * KC * KT + team * KT + q, q < keep ? o[k2] : make_float2(0.f, 0.f));
          }
        } else if constexpr (V == L) {
        float2 v[L];
#pragma unroll
        for (int j = 0; j < L; ++j) v[j] = slot[lane + L * j];
        __syncwarp(tmask);
        if (lane == 0) mbar_arrive(&empty[b]);  // the producer refills the slot now
        wf::dftL<L, -1>(v, twL);
#pragma unroll
        for (int k1 = 1; k1 < L; ++k1) v[k1] = cmul(v[k1], twN[k1 * L + lane]);
#pragma unroll
        for (int k1 = 0; k1 < L; ++k1) trr[tsw<L>(k1, lane)] = v[k1];
        __syncwarp(tmask);
#pragma unroll
        for (int t = 0; t < L; ++t) v[t] = trr[tsw<L>(lane, t)];
        __syncwarp(tmask);
        float2 o[KP];
        wf::dftL_first<L, KP>(v, o, twL);
        if (kk >= NA) mbar_wait(&aempty[s], (uint32_t)(((kk / NA) - 1) & 1));
#pragma unroll
        for (int k2 = 0; k2 < KP; ++k2) {
          const int q = lane + L * k2;
          put_a<G::AW>(As, s * KC * KT + team * KT + q, q < keep ? o[k2] : make_float2(0.f, 0.f));
        }
        } else {
        // N = 128 = 16 lanes x 8: Y_t[k1] = DFT8_j x[t + 16 j] * w_128^{t k1};
        // X[k1 + 8 k2] = sum over t = hf + 2 t' of w_16^{hf k2} DFT8_t'(Y)[k2],
        // lane = (k1, hf): the two halves are summed with one shuffle.
        static_assert(V == 8 && L == 16, "row shape");
        constexpr int K2 = 2 * KP;  // bins k1 + 8 k2 < KT
        float2 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = slot[lane + 16 * j];
        __syncwarp(tmask);
        if (lane == 0) mbar_arrive(&empty[b]);
        dft8<-1>(v);
#pragma unroll
        for (int k1 = 1; k1 < 8; ++k1) v[k1] = cmul(v[k1], twN[k1 * 16 + lane]);
#pragma unroll
        for (int k1 = 0; k1 < 8; ++k1) trr[tsw8(k1, lane)] = v[k1];
        __syncwarp(tmask);
        const int k1 = lane >> 1, hf = lane & 1;
#pragma unroll
        for (int t2 = 0; t2 < 8; ++t2) v[t2] = trr[tsw8(k1, hf + 2 * t2)];
        __syncwarp(tmask);
        dft8<-1>(v);
#pragma unroll
        for (int k2 = 1; k2 < K2; ++k2)
          if (hf) v[k2] = cmul(v[k2], twL[k2]);
#pragma unroll
        for (int k2 = 0; k2 < K2; ++k2) {
          const float2 p = make_float2(__shfl_xor_sync(tmask, v[k2].x, 1), __shfl_xor_sync(tmask, v[k2].y, 1));
          v[k2] = cadd(v[k2], p);
        }
        if (kk >= NA) mbar_wait(&aempty[s], (uint32_t)(((kk / NA) - 1) & 1));
#pragma unroll
        for (int k2 = 0; k2 < K2; ++k2) {
          if ((k2 & 1) != hf) continue;
          const int q = k1 + 8 * k2;
          put_a<G::AW>(As, s * KC * KT + team * KT + q, q < keep ? v[k2] : make_float2(0.f, 0.f));
        }
        }
        __syncwarp(tmask);
        if (lane == 0) mbar_arrive(&afull[s]);
      }
    }
    if (it >= 1) {
      // ---- zero-padded inverse of item it-1's output rows from the C tile
      const int64_t item = first + (it - 1) * units;
      const int64_t g = item / S, n0 = (item % S) * NOUT;
      const int64_t bb = g / a.gx, pp = g % a.gx;
      float2* yg = a.y + bb * a.y_sb + pp * a.y_sp + n0 * a.y_sn;
      constexpr int NC = NOUT / CS;  // output rows of this CTA: [cr*NC, (cr+1)*NC)
      if constexpr (CS > 1)
        mbar_wait_cluster(cfull, (uint32_t)((it - 1) & 1));
      else
        mbar_wait(cfull, (uint32_t)((it - 1) & 1));
      // C[n][q]: own tile, or the fixed-order sum of the cluster's partial tiles (DSMEM)
      auto cval = [&](int n, int q) -> float2 {
        if constexpr (CS == 1) {
          return Cs[n * KT + q];
        } else {
          float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int r = 0; r < CS; ++r) s2 = cadd(s2, ld_dsmem(mapa_rank(Cs + n * KT + q, (uint32_t)r)));
          return s2;
        }
      };
      for (int n = cr * NC + team; n < (cr + 1) * NC; n += TEAMS) {
        float2* dst = yg + (int64_t)n * a.y_sn;
        if constexpr (PART == 1) {
          // K4: the unscaled C row (first keep bins) for the separate padded y-iFFT pass
          float2* cdst = a.C + bb * a.c_sb + pp * a.c_sp + (n0 + n) * a.c_sn;
          for (int q = lane; q < keep; q += L) __stcs(cdst + q, cval(n, q));
        } else if constexpr (V == L) {
        float2 xk[KP];
#pragma unroll
        for (int k2 = 0; k2 < KP; ++k2) {
          const int q = lane + L * k2;
          xk[k2] = q < keep ? cval(n, q) : make_float2(0.f, 0.f);
        }
        float2 z[L];
        wf::idftL_padded<L, KP>(xk, z, twL);
#pragma unroll
        for (int t = 1; t < L; ++t) z[t] = cmul(z[t], conjf2(twN[t * L + lane]));
#pragma unroll
        for (int t = 0; t < L; ++t) trr[tsw<L>(t, lane)] = z[t];
        __syncwarp(tmask);
#pragma unroll
        for (int k1 = 0; k1 < L; ++k1) z[k1] = trr[tsw<L>(lane, k1)];
        __syncwarp(tmask);
        wf::dftL<L, 1>(z, twL);
#pragma unroll
        for (int j = 0; j < L; ++j) __stcs(dst + lane + L * j, cscale(z[j], a.inv_scale));
        } else {
        // N = 128: lane (k1, hf) forms Y_t[k1] for t = hf + 2 t' from its
        // nonzero bins X[k1 + 8 k2], twiddles by w_128^{+k1 t}, transposes;
        // lane t then runs the inverse DFT8 over k1 -> y[t + 16 j]
        constexpr int K2 = 2 * KP;
        const int k1 = lane >> 1, hf = lane & 1;
        float2 z[8];
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) {
          const int q = k1 + 8 * k2;
          z[k2] = (k2 < K2 && q < keep) ? cval(n, q) : make_float2(0.f, 0.f);
          if (k2 < K2 && k2 && hf) z[k2] = cmul(z[k2], conjf2(twL[k2]));
        }
        dft8<1>(z);
#pragma unroll
        for (int t2 = 0; t2 < 8; ++t2) {
          const int t = hf + 2 * t2;
          trr[tsw8(k1, t)] = k1 ? cmul(z[t2], conjf2(twN[k1 * 16 + t])) : z[t2];
        }
        __syncwarp(tmask);
#pragma unroll
        for (int r = 0; r < 8; ++r) z[r] = trr[tsw8(r, lane)];
        __syncwarp(tmask);
        dft8<1>(z);
#pragma unroll
        for (int j = 0; j < 8; ++j) __stcs(dst + lane + 16 * j, cscale(z[j], a.inv_scale));
        }
      }
      __syncwarp(tmask);
      if (lane == 0) {
        if constexpr (CS > 1) {
          for (int r = 0; r < CS; ++r) mbar_arrive_cluster(mapa_rank(cempty, (uint32_t)r));
        } else {
          mbar_arrive(cempty);
        }
      }
    }
  }
  // peers read this CTA's last partial tile over DSMEM: stay resident until they are done
  if constexpr (CS > 1)
    if (nmine > 0) mbar_wait_cluster(cempty, (uint32_t)((nmine - 1) & 1));
}

// ---------------------------------------------------------------- dispatch
struct F1Shape {
  int L, V, KP, TI, TJ, NOUT;
};
// instantiated shapes: keep <= KP*L (masked), H % (256/L) == 0, N_out == NOUT
static const F1Shape kF1Shapes[] = {
    {16, 16, 1, 1, 4, 64}, {16, 16, 1, 1, 8, 128}, {16, 16, 1, 2, 8, 256},  // keep <= 16 (N = 256)
    {16, 16, 2, 1, 4, 32},                                                  // keep <= 32, N_out (per split) 32
    {16, 16, 2, 2, 4, 64}, {16, 16, 2, 2, 8, 128}, {16, 16, 2, 4, 8, 256},  // keep <= 32
    {16, 16, 4, 4, 4, 64}, {16, 16, 4, 4, 8, 128},                          // keep <= 64
    {32, 32, 2, 4, 4, 64},                                                  // keep <= 64 (N = 1024)
    {32, 32, 4, 8, 4, 64},                                                  // keep <= 128
    {16, 8, 2, 1, 2, 16}, {16, 8, 2, 1, 4, 32}, {16, 8, 2, 2, 4, 64},      // N = 128, keep <= 32 (C1)
};

static const F1Shape* f1_pick(int n, int keep, int H, int NO) {
  const int L = (n == 256 || n == 128) ? 16 : (n == 1024 ? 32 : 0);
  const int V = n == 128 ? 8 : L;
  if (!L || keep < 1 || H < 1 || H % (256 / L) != 0) return nullptr;
  const int kp = (keep + L - 1) / L;
  for (const F1Shape& s : kF1Shapes)
    if (s.L == L && s.V == V && s.NOUT == NO && (s.KP == kp || (kp == 3 && s.KP == 4))) return &s;
  return nullptr;
}

bool fused1d_supported(int n, int keep, int H, int NO) { return f1_pick(n, keep, H, NO) != nullptr; }

template <int L, int V, int KP, int TI, int TJ, int NOUT, int CS, int PART = 0>
static cudaError_t launch_f1(const FusedArgs& a, cudaStream_t s) {
  using G = F1Geo<L, V, KP, TI, TJ, NOUT>;
  static_assert(G::smem_bytes() <= 227 * 1024, "shared memory");
  const size_t smem = G::smem_bytes();
  if ((uintptr_t)a.x % 16 || (uintptr_t)a.W % 16 || (a.x_sh % 2) || (a.x_sb % 2) || (a.x_sp % 2))
    return cudaErrorNotSupported;  // TMA bulk copies need 16-byte aligned rows
  auto kern = fused1d_kernel<L, V, KP, TI, TJ, NOUT, CS, PART>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (CS == 1) {
    const int64_t items = a.G * (a.nsplit > 1 ? a.nsplit : 1);
    const int grid = (int)(items < sms ? items : sms);
    if (grid < 1) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(G::NTH);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, kern, a);
    if (e != cudaSuccess) return e;
  } else {
    const int64_t units = a.G < sms / CS ? a.G : sms / CS;
    if (units < 1) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(units * CS));
    cfg.blockDim = dim3(G::NTH);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    e = cudaLaunchKernelEx(&cfg, kern, a);
    if (e != cudaSuccess) return e;
  }
  ++g_launches;
  return cudaGetLastError();
}

int fused1d_split(int n, int keep, int H, int NO, int64_t G) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int S = 1;
  if (!f1_pick(n, keep, H, NO)) {
    // the full C tile does not fit one CTA (e.g. N = 1024, N_out = 128): split the
    // output channels (forward recomputed per split) when the batch is small
    // (measured: S = 2 wins, N1024 H128 B64 0.110 -> 0.077 ms; S = 4 loses, N1024 H256 B64 0.185 -> 0.235)
    if (NO % 2 || !f1_pick(n, keep, H, NO / 2) || G * 2 > sms) return 0;
    S = 2;
  }
  // split further while the doubled item count still fits one wave of SMs
  while (S < 4 && NO % (2 * S) == 0 && G * 2 * S <= sms && f1_pick(n, keep, H, NO / (2 * S))) S *= 2;
  return S;
}

// K5 (GEMM + padded iFFT from the y-FFT's A): splitting the output channels recomputes nothing
// (each split item streams the same A rows), so any batch may split until the C tile fits
int fused1d_split_gemm_ifft(int n, int keep, int H, int NO) {
  if (f1_pick(n, keep, H, NO)) return 1;
  for (int S = 2; S <= 8; S *= 2)
    if (NO % S == 0 && f1_pick(n, keep, H, NO / S)) return S;
  return 0;
}

int fused1d_cluster(int n, int keep, int H, int NO, int64_t G) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("TFNO_FUSED1D_CLUSTER");
    env = e ? atoi(e) : -1;
  }
  if (env == 0 || !f1_pick(n, keep, H, NO)) return 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int L = (n == 256 || n == 128) ? 16 : 32, KC = 256 / L;
  int CS = 1;  // split the hidden channels while the clusters still fit one wave of SMs
  while (CS < 4 && G * 2 * CS <= sms && H % (2 * CS * KC) == 0 && NO % (2 * CS) == 0) CS *= 2;
  return CS;
}

cudaError_t launch_fused1d(const FusedArgs& a, cudaStream_t s) {
  const int CS = a.cluster > 1 ? a.cluster : 1;
  const int S = (CS == 1 && a.nsplit > 1) ? a.nsplit : 1;
  if (a.N % S) return cudaErrorNotSupported;
  const F1Shape* p = f1_pick(a.n, a.keep, a.H, a.N / S);
  if (!p) return cudaErrorNotSupported;
#define F1_CASE(LL, VV, KK, TI_, TJ_, NO_)                                                          \
  if (p->L == LL && p->V == VV && p->KP == KK && p->NOUT == NO_) {                                  \
    if (a.part == 1) return CS == 1 ? launch_f1<LL, VV, KK, TI_, TJ_, NO_, 1, 1>(a, s) : cudaErrorNotSupported; \
    if (a.part == 2) return CS == 1 ? launch_f1<LL, VV, KK, TI_, TJ_, NO_, 1, 2>(a, s) : cudaErrorNotSupported; \
    if (CS == 4) return launch_f1<LL, VV, KK, TI_, TJ_, NO_, 4>(a, s);                             \
    if (CS == 2) return launch_f1<LL, VV, KK, TI_, TJ_, NO_, 2>(a, s);                             \
    return launch_f1<LL, VV, KK, TI_, TJ_, NO_, 1>(a, s);                                          \
  }
  F1_CASE(16, 16, 1, 1, 4, 64) F1_CASE(16, 16, 1, 1, 8, 128) F1_CASE(16, 16, 1, 2, 8, 256)
  F1_CASE(16, 16, 2, 1, 4, 32)
  F1_CASE(16, 16, 2, 2, 4, 64) F1_CASE(16, 16, 2, 2, 8, 128) F1_CASE(16, 16, 2, 4, 8, 256)
  F1_CASE(16, 16, 4, 4, 4, 64) F1_CASE(16, 16, 4, 4, 8, 128)
  F1_CASE(32, 32, 2, 4, 4, 64)
  F1_CASE(32, 32, 4, 8, 4, 64)
  F1_CASE(16, 8, 2, 1, 2, 16) F1_CASE(16, 8, 2, 1, 4, 32) F1_CASE(16, 8, 2, 2, 4, 64)
#undef F1_CASE
  return cudaErrorNotSupported;
}

}  // namespace tfno
