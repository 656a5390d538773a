// tmop_launch.cuh -- compile-time dispatch of the element kernels over
// (n_q, kind) for one (dim, p+1); included by one small .cu per (dim, p+1)
// so the instantiations compile in parallel.
#pragma once

#include <algorithm>

#include <cstdlib>
#include <cstring>

#include "tmop_apply_col.cuh"
#include "tmop_diag.cuh"
#include "tmop_elem.cuh"
#include "tmop_internal.h"

namespace tmop {

// The work-item kernel (elem_kernel<K_APPLY>) is the default Hessian action;
// TMOP_APPLY_KERNEL=col selects the column kernel (apply_col_kernel), which
// measured slower for p >= 2 in round 1 (profiles/round1_apply_ab.md).
inline bool use_generic_apply() {
  static int v = -1;
  if (v < 0) {
    const char *e = std::getenv("TMOP_APPLY_KERNEL");
    v = (e && std::strcmp(e, "col") == 0) ? 0 : 1;
  }
  return v == 1;
}

template <int N, int Q, bool NTM>
int launch_col(ElemArgs &a, const Tab &t, cudaStream_t s) {
  using CC = ColCfg<N, Q>;
  a.ngroups = (a.ne + CC::E - 1) / CC::E;
  const int grid = (int)std::min<int64_t>(a.ngroups, GRID_CAP);
  if (grid == 0) return 0;
  auto kfn = apply_col_kernel<N, Q, NTM>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM) != cudaSuccess) return -2;
    configured = true;
  }
  kfn<<<grid, CC::NT, CC::SMEM, s>>>(a, t);
  return grid;
}

template <int DIM, int N, int Q, bool NTM>
int launch_diag(ElemArgs &a, const Tab &t, cudaStream_t s) {
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
int launch_one(ElemArgs &a, const Tab &t, cudaStream_t s) {
  using CF = Cfg<DIM, N, Q>;
  if constexpr (KIND == K_DIAG || KIND == K_DIAG_NT) {
    return launch_diag<DIM, N, Q, KIND == K_DIAG_NT>(a, t, s);
  } else {
    if constexpr (DIM == 3 && (KIND == K_APPLY || KIND == K_APPLY_NT) && col_supported<N, Q>()) {
      if (!use_generic_apply()) return launch_col<N, Q, KIND == K_APPLY_NT>(a, t, s);
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
