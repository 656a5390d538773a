// tmop_launch.cuh -- compile-time dispatch of the element kernels over
// (n_q, kind) for one (dim, p+1); included by one small .cu per (dim, p+1)
// so the instantiations compile in parallel.
#pragma once

#include <algorithm>

#include <cstdlib>
#include <cstring>

#include "tmop_lim.cuh"
#include "tmop_xl.cuh"
#include "tmop_xld.cuh"
#include "tmop_diag.cuh"
#include "tmop_elem.cuh"
#include "tmop_internal.h"

namespace tmop {

#ifndef TMOP_XL_GRAD_P3
#define TMOP_XL_GRAD_P3 1
#endif

// TMOP_XL=0 forces the work-item kernels (elem_kernel) everywhere (A/B and
// parity of the two implementations).
inline bool xl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = std::getenv("TMOP_XL");
    v = (e && std::strcmp(e, "0") == 0) ? 0 : 1;
  }
  return v == 1;
}

// Which kinds run in x-line form, per order (measured, profiles/round1_*):
// p <= 3 all of them; p = 4 only the forward-only energy / min det -- its
// backward kinds and setup keep ~90+ doubles live per line and spill, and
// the work-item kernel is faster there.
template <int N, int KIND>
constexpr bool xl_kind() {
  if constexpr (KIND == K_SETUP_DIAG) return N <= 4;
  if constexpr (N >= 5) return KIND == K_ENERGY || KIND == K_MINDET;
  // p = 3 gradient: x-line with W in shared memory (tmop_xl.cuh WSM), C3
  // 8.3 -> 7.4-7.7 ms; with W in registers it spilled ~320 B per thread at
  // 255 registers and the work-item kernel was faster (8.5 vs 9.1 ms)
  if constexpr (N == 4 && KIND == K_GRAD) return TMOP_XL_GRAD_P3 != 0;
  return KIND == K_APPLY || KIND == K_APPLY_NT || KIND == K_GRAD || KIND == K_SETUP || KIND == K_ENERGY ||
         KIND == K_MINDET;
}

// 3D x-line kernels (tmop_xl.cuh) where selected (xl_kind) and the CTA fits.  The grid is
// one persistent wave: SMs x the occupancy the kernel achieves, capped at
// GRID_CAP (the per-CTA reduction partials).
template <int N, int Q, int KIND>
int launch_xl(ElemArgs &a, const Tab &t, cudaStream_t s) {
  using XC = XlCfg<N, Q>;
  constexpr int smem = XC::template smem<KIND>();
  a.ngroups = (a.ne + XC::EPB - 1) / XC::EPB;
  static_assert(XC::EPB == 16 || XC::EPB == 8 || XC::EPB == 4 || XC::EPB == 1,
                "e_es assumes 1-, 4-, 8- or 16-element groups");
  if constexpr (xl_backward<KIND>() || KIND == K_SETUP_DIAG)
    a.e_es = XC::EPB == 16 ? 4 : XC::EPB == 8 ? 3 : XC::EPB == 4 ? 2 : 0;
  auto kfn = xl_kernel<N, Q, KIND>;
  static int per_sm = 0;
  if (per_sm == 0) {
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -2;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kfn, XC::NT, smem) != cudaSuccess || nb < 1) nb = 1;
    per_sm = nb;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(std::min<int64_t>(a.ngroups, (int64_t)sms * per_sm), GRID_CAP);
  if (grid == 0) return 0;
  kfn<<<grid, XC::NT, smem, s>>>(a, t);
  return grid;
}

// TMOP_XLD=0 keeps the work-item diagonal (diag2_kernel) everywhere.
inline bool xld_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = std::getenv("TMOP_XLD");
    v = (e && std::strcmp(e, "0") == 0) ? 0 : 1;
  }
  return v == 1;
}

// 3D p <= 3 diagonal in x-line form (tmop_xld.cuh): one persistent wave.
template <int N, int Q, bool NTM>
int launch_xld(ElemArgs &a, const Tab &t, cudaStream_t s) {
  using XC = XldCfg<N, Q>;
  a.ngroups = (a.ne + XC::EPB - 1) / XC::EPB;
  a.e_es = XC::EPB == 16 ? 4 : XC::EPB == 8 ? 3 : 2;
  auto kfn = xld_kernel<N, Q, NTM>;
  static int per_sm = 0;
  if (per_sm == 0) {
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, XC::SMEM) != cudaSuccess) return -2;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kfn, XC::NT, XC::SMEM) != cudaSuccess || nb < 1) nb = 1;
    per_sm = nb;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(std::min<int64_t>(a.ngroups, (int64_t)sms * per_sm), GRID_CAP);
  if (grid == 0) return 0;
  kfn<<<grid, XC::NT, XC::SMEM, s>>>(a, t);
  return grid;
}

template <int DIM, int N, int Q, bool NTM>
int launch_diag(ElemArgs &a, const Tab &t, cudaStream_t s) {
  if constexpr (DIM == 3 && xld_supported<N, Q>()) {
    if (xld_enabled()) return launch_xld<N, Q, NTM>(a, t, s);
  }
  using DC = DiagCfg<DIM, N, Q>;
  a.ngroups = (a.ne + DC::EPB - 1) / DC::EPB;
  const int grid = (int)std::min<int64_t>(a.ngroups, GRID_CAP);
  if (grid == 0) return 0;
  auto kfn = diag2_kernel<DIM, N, Q, NTM>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, DC::SMEM) != cudaSuccess) return -2;
    configured = true;
  }
  kfn<<<grid, ELEM_NT, DC::SMEM, s>>>(a, t);
  return grid;
}

template <int DIM, int N, int Q, int KIND>
int launch_lim(ElemArgs &a, const Tab &t, cudaStream_t s) {
  using LC = LimCfg<DIM, N, Q>;
  a.ngroups = (a.ne + LC::EPB - 1) / LC::EPB;
  a.e_es = 0;
  const int grid = (int)std::min<int64_t>(a.ngroups, GRID_CAP);
  if (grid == 0) return 0;
  auto kfn = lim_kernel<DIM, N, Q, KIND>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, LC::SMEM) != cudaSuccess) return -2;
    configured = true;
  }
  kfn<<<grid, LC::NT, LC::SMEM, s>>>(a, t);
  return grid;
}

template <int DIM, int N, int Q, int KIND>
int launch_one(ElemArgs &a, const Tab &t, cudaStream_t s) {
  using CF = Cfg<DIM, N, Q>;
  if constexpr (KIND == K_LIM_VALUE || KIND == K_LIM_FIELD || KIND == K_LIM_DIAG || KIND == K_TSCALE) {
    return launch_lim<DIM, N, Q, KIND>(a, t, s);
  } else if constexpr (KIND == K_DIAG || KIND == K_DIAG_NT) {
    return launch_diag<DIM, N, Q, KIND == K_DIAG_NT>(a, t, s);
  } else {
    if constexpr (KIND == K_SETUP_DIAG) {
      // fused setup + diagonal: 3D x-line only (callers fall back to the two
      // separate passes on -1)
      // (the fused kind lays the diagonal out with the action's group size
      // and the records-overlay layout: tuning variants that change either
      // keep the two passes)
      if constexpr (DIM == 3 && xl_kind<N, KIND>() && XlCfg<N, Q>::template smem<KIND>() <= 227 * 1024 &&
                    XldCfg<N, Q>::EPB == XlCfg<N, Q>::EPB) {
        if (xl_enabled() && xld_enabled()) return launch_xl<N, Q, KIND>(a, t, s);
      }
      return -1;
    } else {
    if constexpr (DIM == 3 && xl_kind<N, KIND>() && xl_supported<N, Q>() &&
                  (!xl_ldg<N, Q>() || KIND == K_APPLY)) {
      if (xl_enabled()) return launch_xl<N, Q, KIND>(a, t, s);
    }
    a.ngroups = (a.ne + CF::EPB - 1) / CF::EPB;
    const int grid = (int)std::min<int64_t>(a.ngroups, GRID_CAP);
    if (grid == 0) return 0;
    auto kfn = elem_kernel<DIM, N, Q, KIND>;
    constexpr int smem = (KIND == K_APPLY || KIND == K_APPLY_NT) ? CF::SMEM_TMA : CF::SMEM;
    static bool configured = false;
    if (!configured) {
      if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -2;
      configured = true;
    }
    kfn<<<grid, CF::NT, smem, s>>>(a, t);
    return grid;
    }
  }
}

template <int DIM, int N, int Q>
int launch_kind(int kind, ElemArgs &a, const Tab &t, cudaStream_t s) {
  switch (kind) {
    case K_SETUP: return launch_one<DIM, N, Q, K_SETUP>(a, t, s);
    case K_APPLY: return launch_one<DIM, N, Q, K_APPLY>(a, t, s);
    case K_GRAD: return launch_one<DIM, N, Q, K_GRAD>(a, t, s);
    case K_ENERGY: return launch_one<DIM, N, Q, K_ENERGY>(a, t, s);
    case K_MINDET: return launch_one<DIM, N, Q, K_MINDET>(a, t, s);
    case K_ELEMDET: return launch_one<DIM, N, Q, K_ELEMDET>(a, t, s);
    case K_VOLUME: return launch_one<DIM, N, Q, K_VOLUME>(a, t, s);
    case K_DIAG: return launch_one<DIM, N, Q, K_DIAG>(a, t, s);
    case K_APPLY_NT: return launch_one<DIM, N, Q, K_APPLY_NT>(a, t, s);
    case K_DIAG_NT: return launch_one<DIM, N, Q, K_DIAG_NT>(a, t, s);
    case K_LIM_VALUE: return launch_one<DIM, N, Q, K_LIM_VALUE>(a, t, s);
    case K_LIM_FIELD: return launch_one<DIM, N, Q, K_LIM_FIELD>(a, t, s);
    case K_LIM_DIAG: return launch_one<DIM, N, Q, K_LIM_DIAG>(a, t, s);
    case K_TSCALE: return launch_one<DIM, N, Q, K_TSCALE>(a, t, s);
    case K_SETUP_DIAG: return launch_one<DIM, N, Q, K_SETUP_DIAG>(a, t, s);
    default: return -1;
  }
}

// Supported n_q: 2..9 for every p.
template <int DIM, int N>
int launch_q(int nq, int kind, ElemArgs &a, const Tab &t, cudaStream_t s) {
  switch (nq) {
    case 2: return launch_kind<DIM, N, 2>(kind, a, t, s);
    case 3: return launch_kind<DIM, N, 3>(kind, a, t, s);
    case 4: return launch_kind<DIM, N, 4>(kind, a, t, s);
    case 5: return launch_kind<DIM, N, 5>(kind, a, t, s);
    case 6: return launch_kind<DIM, N, 6>(kind, a, t, s);
    case 7: return launch_kind<DIM, N, 7>(kind, a, t, s);
    case 8: return launch_kind<DIM, N, 8>(kind, a, t, s);
    case 9: return launch_kind<DIM, N, 9>(kind, a, t, s);
    default: return -1;
  }
}

}  // namespace tmop
