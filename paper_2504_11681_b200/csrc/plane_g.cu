// Launchers for the generic per-plane 2D kernels (plane_g.cuh): one
// instantiation per (dy, KP) with dy in {64 ... 1024}, KP in {8 ... 128}.
// The build compiles this file once per row length (-DPLANE_G_DY=64 ... 1024)
// so the units compile in parallel; plane2d.cu routes a config to its unit.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"
#include "plane2d.cuh"
#include "plane_g.cuh"

#ifndef PLANE_G_DY
#error "compile with -DPLANE_G_DY=<dy>"
#endif

namespace tfno {

namespace {

template <int DY, int KP>
struct PGCfg {
  static constexpr int V = DY >= 256 ? 16 : 8;
  static constexpr int M = DY / V;
  static constexpr int CAPF = KP >= 128 ? 128 : 256;
  static constexpr int NTHF = M * (KP < CAPF / M ? KP : CAPF / M);
  static constexpr int NTHI = M * (KP < 256 / M ? KP : 256 / M);
  // 512^2 / keep 64 (C4): a 4-slot ring with the class accumulators in registers beats
  // 3 slots with shared-memory accumulators (same box, alternating: 14.10 / 14.21 ->
  // 13.98 / 14.06 ms per C4 layer, profiles/r02/s4_ab.txt); -DTFNO_PG_S3 restores it
#ifndef TFNO_PG_S3
  static constexpr bool S4 = DY == 512 && KP == 64;
#else
  static constexpr bool S4 = false;
#endif
  static constexpr int S = S4 ? 4 : KP >= 128 ? 2 : 3;
  static constexpr bool BIG = KP >= 128;  // accumulate classes in global, mode tile read from L2
  using GF = PG<DY, KP, KP, NTHF>;
  using GI = PG<DY, KP, KP, NTHI>;
  // forward accumulators in shared memory when they fit next to everything else (frees registers
  // for the hoisted twiddle companions; 1024 keeps registers)
  static constexpr size_t FWD_BASE = sizeof(float2) * ((size_t)S * GF::TEAMS * DY + (size_t)GF::NTB * GF::TB +
                                                       (size_t)KP * KP + 2 * DY + KP + 1024) + 16 * S + 16;
  static constexpr size_t ACC_BYTES = sizeof(float2) * (size_t)GF::TASKS2 * GF::KA * GF::NTH;
  static constexpr bool ACCS = !S4 && !BIG && FWD_BASE + ACC_BYTES <= 227 * 1024;
};

template <class G>
size_t g_fwd_smem(int S, bool accs, int dx) {
  return sizeof(float2) * ((size_t)S * G::TEAMS * G::DY + (size_t)G::NTB * G::TB + (size_t)G::KXP * G::KYP +
                           (accs ? (size_t)G::TASKS2 * G::KA * G::NTH : 0) + 2 * G::DY + G::KXP + dx) +
         16 * S + 16;
}
template <class G>
size_t g_inv_smem(bool cing, int dx) {
  return sizeof(float2) * ((cing ? 0 : (size_t)G::KXP * G::KYP) + (size_t)G::KXP * G::KYP +
                           (size_t)G::NTB * G::TB + G::DY + G::KXP + dx) +
         16;
}

template <class K>
cudaError_t persistent_grid(K kernel, int threads, size_t smem, int64_t planes, int* grid) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem)) != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const int64_t cap = (int64_t)device_sms() * occ;
  *grid = (int)(planes < cap ? planes : cap);
  return cudaSuccess;
}

template <int DY, int KP>
cudaError_t g_fwd(const float2* x, float2* A, int64_t planes, int dx, int kx, int ky, const float2* tw,
                  cudaStream_t st) {
  using C = PGCfg<DY, KP>;
  using G = typename C::GF;
  if (planes <= 0) return cudaSuccess;
  auto kern = plane_fwd_g<G, C::S, C::BIG, C::ACCS>;
  const size_t smem = g_fwd_smem<G>(C::S, C::ACCS, dx);
  int grid = 0;
  cudaError_t e = persistent_grid(kern, G::NTH + 32, smem, planes, &grid);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kern, dim3(grid), dim3(G::NTH + 32), smem, st, x, A, planes, dx, kx, ky, tw);
  if (e != cudaSuccess) return e;
  ++g_launches;
  return cudaGetLastError();
}

template <int DY, int KP>
cudaError_t g_inv(const float2* Cm, float2* y, int64_t planes, int dx, const float2* tw, float scale,
                  cudaStream_t st) {
  using C = PGCfg<DY, KP>;
  using G = typename C::GI;
  if (planes <= 0) return cudaSuccess;
  auto kern = plane_inv_g<G, C::BIG>;
  const size_t smem = g_inv_smem<G>(C::BIG, dx);
  int grid = 0;
  cudaError_t e = persistent_grid(kern, G::NTH, smem, planes, &grid);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kern, dim3(grid), dim3(G::NTH), smem, st, Cm, y, planes, dx, tw, scale);
  if (e != cudaSuccess) return e;
  ++g_launches;
  return cudaGetLastError();
}

// fused inverse + channel mix (plane_invmix_g): tasks of kMixGN output channels
constexpr int kMixGN = 8;
// A-ring depth: as many 16 KiB chunks (<= SA_MAX) as fit next to the inverse's buffers; >= 3.
// prec 1 / 3 (tensor-core mix): the ring holds the two staged A chunks (hi [, lo] canonical
// tiles) and the W' tiles replace the packed W columns (depth >= 3 keeps three mbarriers).
template <class G>
int g_invmix_depth(int H, int dx, int prec, size_t* bytes) {
  using X = MixGeo<G::KXP * G::KYP>;
  const int npass = prec == 3 ? 2 : 1, Hp = (H + 3) & ~3;
  const size_t wt = prec ? (size_t)npass * Hp * 128 : sizeof(float4) * (size_t)H * kMixGN;
  const size_t rest = wt + sizeof(float2) * (2 * (size_t)G::KXP * G::KYP + (size_t)G::NTB * G::TB + 2 * G::DY + G::KXP + dx) +
                      8 * (5 + 2 * X::SA_MAX) + 8;
  const size_t chunk = sizeof(float2) * (size_t)X::HC * X::MC, cap = 227 * 1024;
  const int need = prec ? (2 * npass * X::MC * 32 + (int)chunk - 1) / (int)chunk : 3;
  const int lo = need > 3 ? need : 3;
  if (rest + lo * chunk > cap) return 0;
  int sa = prec ? lo : (int)((cap - rest) / chunk);
  if (sa > X::SA_MAX) sa = X::SA_MAX;
  if (sa < lo) return 0;
  *bytes = rest + sa * chunk;
  return sa;
}

template <int DY, int KP>
size_t g_invmix_bytes(int H, int dx, int prec, int* sa = nullptr) {
  if constexpr (KP < 16 || KP > 64 || KP > DY) {
    return 0;
  } else {
    size_t b = 0;
    const int d = g_invmix_depth<typename PGCfg<DY, KP>::GI>(H, dx, prec, &b);
    if (sa) *sa = d;
    return d ? b : 0;
  }
}

template <int DY, int KP, int PREC>
cudaError_t g_invmix_p(const float2* A, const float2* W, float2* Cs, float2* y, int B, int H, int N, int dx,
                       const float2* tw, float alpha, cudaStream_t st) {
  using G = typename PGCfg<DY, KP>::GI;
  int sa = 0;
  const size_t smem = g_invmix_bytes<DY, KP>(H, dx, PREC, &sa);
  if (!smem) return cudaErrorNotSupported;
  const int64_t tasks = (int64_t)B * ((N + kMixGN - 1) / kMixGN);
  if (tasks <= 0) return cudaSuccess;
  auto kern = plane_invmix_g<G, kMixGN, PREC>;
  int grid = 0;
  cudaError_t e = persistent_grid(kern, G::NTH + kMixThreads, smem, tasks, &grid);
  if (e != cudaSuccess) return e;
  if (grid > device_sms()) grid = device_sms();  // the C ring is sized for one CTA per SM
  e = launch_pdl(kern, dim3(grid), dim3(G::NTH + kMixThreads), smem, st, A, W, Cs, y, B, H, N, dx, tw, alpha, sa);
  if (e != cudaSuccess) return e;
  ++g_launches;
  return cudaGetLastError();
}

template <int DY, int KP>
cudaError_t g_invmix(const float2* A, const float2* W, float2* Cs, float2* y, int B, int H, int N, int dx,
                     const float2* tw, float alpha, int prec, cudaStream_t st) {
  if constexpr (KP < 16 || KP > 64 || KP > DY) {
    return cudaErrorNotSupported;
  } else {
    if (prec == 0) return g_invmix_p<DY, KP, 0>(A, W, Cs, y, B, H, N, dx, tw, alpha, st);
    if (prec == 1) return g_invmix_p<DY, KP, 1>(A, W, Cs, y, B, H, N, dx, tw, alpha, st);
    if (prec == 3) return g_invmix_p<DY, KP, 3>(A, W, Cs, y, B, H, N, dx, tw, alpha, st);
    return cudaErrorNotSupported;
  }
}

template <int DY>
cudaError_t g_dispatch(int KP, int dir, const float2* in, float2* out, int64_t planes, int dx, int kx, int ky,
                       const float2* tw, float scale, cudaStream_t st) {
#define TFNO_G_CASE(K)                                                                       \
  case K:                                                                                    \
    if constexpr (K <= DY)                                                                   \
      return dir < 0 ? g_fwd<DY, K>(in, out, planes, dx, kx, ky, tw, st)                     \
                     : g_inv<DY, K>(in, out, planes, dx, tw, scale, st);                     \
    break;
  switch (KP) {
    TFNO_G_CASE(8)
    TFNO_G_CASE(16)
    TFNO_G_CASE(32)
    TFNO_G_CASE(64)
    TFNO_G_CASE(128)
    default: break;
  }
#undef TFNO_G_CASE
  return cudaErrorNotSupported;
}

template <int DY>
size_t g_invmix_query(int KP, int H, int dx, int prec) {
  switch (KP) {
    case 16: return g_invmix_bytes<DY, 16>(H, dx, prec);
    case 32: return g_invmix_bytes<DY, 32>(H, dx, prec);
    case 64: return g_invmix_bytes<DY, 64>(H, dx, prec);
    default: return 0;
  }
}
template <int DY>
cudaError_t g_invmix_dispatch(int KP, const float2* A, const float2* W, float2* Cs, float2* y, int B, int H, int N,
                              int dx, const float2* tw, float alpha, int prec, cudaStream_t st) {
  switch (KP) {
    case 16: return g_invmix<DY, 16>(A, W, Cs, y, B, H, N, dx, tw, alpha, prec, st);
    case 32: return g_invmix<DY, 32>(A, W, Cs, y, B, H, N, dx, tw, alpha, prec, st);
    case 64: return g_invmix<DY, 64>(A, W, Cs, y, B, H, N, dx, tw, alpha, prec, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace

#define TFNO_CAT2(a, b) a##b
#define TFNO_CAT(a, b) TFNO_CAT2(a, b)
// entry point of this translation unit: plane_g_run_<dy>
cudaError_t TFNO_CAT(plane_g_run_, PLANE_G_DY)(int KP, int dir, const float2* in, float2* out, int64_t planes,
                                               int dx, int kx, int ky, const float2* tw, float scale,
                                               cudaStream_t st) {
  return g_dispatch<PLANE_G_DY>(KP, dir, in, out, planes, dx, kx, ky, tw, scale, st);
}
// fused inverse + channel mix (prec 0 FP32 SIMT, 1 TF32, 3 3xTF32 tcgen05): shared-memory
// bytes (0 = unsupported) and launch
size_t TFNO_CAT(plane_g_invmix_smem_, PLANE_G_DY)(int KP, int H, int dx, int prec) {
  return g_invmix_query<PLANE_G_DY>(KP, H, dx, prec);
}
cudaError_t TFNO_CAT(plane_g_invmix_run_, PLANE_G_DY)(int KP, const float2* A, const float2* W, float2* Cs,
                                                      float2* y, int B, int H, int N, int dx, const float2* tw,
                                                      float alpha, int prec, cudaStream_t st) {
  return g_invmix_dispatch<PLANE_G_DY>(KP, A, W, Cs, y, B, H, N, dx, tw, alpha, prec, st);
}

}  // namespace tfno
