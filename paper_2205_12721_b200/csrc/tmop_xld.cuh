// tmop_xld.cuh -- the exact diagonal of the partially assembled Hessian
// (AssembleGradDiagonalPA; reference hessian_diagonal, operator.py:420-459)
// in x-line form, for 3D p <= 3:
//
//   diag[(c,i)] = sum_q sum_{n<=p} h_{c,np}(q) prod_axis P_{sel(axis,np)}[q_a, i_a]
//
// with h the H-pair values (off-diagonal pairs doubled, operator.py:437-448)
// and P_sel in {B.B, B.G, G.G} the per-axis product tables (Tab::P).
//
// One CTA owns EPB = xl_epb(p+1) elements per group, thread e + EPB * line
// (line = qy + Q qz), like the Hessian action (tmop_xl.cuh):
//   Q-data  the group's lean records arrive by one TMA bulk copy issued a
//           group ahead into QB (the record's qx-slowest slot order gives
//           unit-stride reads per line)
//   X       per line: for each qx the 18 H-pair values (3 components x 6
//           pairs) from the record, accumulated straight into the x^T sweep
//           acc[c][f][kx] (registers); written to A[c][f][qz][qy][kx]
//   Y       item (qz, kx): y^T sweep of the 6 pairs, pairs with the same z
//           table summed (6 -> 3 groups per component): Bv[c][g][qz][ky][kx]
//   Z       item (ky, kx): z^T sweep of the 3 groups -> element-interleaved
//           E-vector (the apply's layout), summed to nodes by e2l_kernel
//           (mode 2: constrained dofs -> 1, operator.py:458)
// Replaces diag2_kernel's work-item stages (27 % bank-conflicted shared
// wavefronts, 3.9 barrier stalls per issue at p = 2, profiles/round1_*).
// The stages live in tmop_xld_parts.cuh (shared with xl_kernel<K_SETUP_DIAG>).
#pragma once

#include "tmop_xl.cuh"
#include "tmop_xld_parts.cuh"

namespace tmop {

template <int N, int Q>
__host__ __device__ constexpr bool xld_supported() {
  return N <= 4 && XldCfg<N, Q>::SMEM <= 227 * 1024;
}

template <int N, int Q, bool NTM>
__global__ void __launch_bounds__(XldCfg<N, Q>::NT, XldCfg<N, Q>::MINB)
    xld_kernel(const ElemArgs a, const __grid_constant__ Tab t) {
  using XC = XldCfg<N, Q>;
  constexpr int EPB = XC::EPB, QS = XC::QS;
  extern __shared__ __align__(16) double smem[];
  double *QB = smem;                           // staged records ...
  double *A = smem + XC::AOFF;                 // ... overlaid by the x^T output (OVL) or beside them
  double *Bv = XC::BVA ? A : smem + XC::R1P;    // (BVA: inside A's consumed slots)
  __shared__ __align__(8) uint64_t qbar;

  const int tid = threadIdx.x;
  const int e = tid % EPB, item = tid / EPB;

  auto issue = [&](int64_t grp) {
    const int64_t e0 = grp * EPB;
    const int64_t cnt = (a.ne - e0) < EPB ? (a.ne - e0) : EPB;
    const uint32_t bytes = (uint32_t)(cnt * QS * 8);
    mbar_expect_tx(&qbar, bytes);
    tma_load_1d(QB, a.qdata + e0 * QS, bytes, &qbar);
  };
  if (tid == 0) {
    mbar_init(&qbar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0 && (int64_t)blockIdx.x < a.ngroups) issue(blockIdx.x);
  uint32_t phase = 0;

  for (int64_t grp = blockIdx.x; grp < a.ngroups; grp += gridDim.x) {
    mbar_wait(&qbar, phase);
    phase ^= 1u;
    double acc[3][6][N];
    xld_line<N, Q, NTM>(a.metric, QB + e * QS + item, t, acc);
    __syncthreads();                           // every record read: A may overwrite QB
    if constexpr (!XC::OVL) {                  // records consumed: stream in the next group's
      if (tid == 0 && grp + gridDim.x < a.ngroups) issue(grp + gridDim.x);
    }
    xld_store_a<N, Q>(A, item, e, acc);
    __syncthreads();
    if (item < Q * N) xld_y<N, Q, XC::BVA>(A, Bv, item, e, t);
    __syncthreads();                           // A (= QB) consumed: stream in the next group's records
    if constexpr (XC::OVL) {
      if (tid == 0 && grp + gridDim.x < a.ngroups) issue(grp + gridDim.x);
    }
    if (item < N * N) xld_z<N, Q, XC::BVA>(Bv, a.E, grp, item, e, t);
    // (the next group's X stage writes only registers; its A writes come
    // after the barrier that follows its record reads, and Bv is rewritten
    // only after the next Y barrier -- Z of this group is ordered before
    // both by the X-stage barrier)
  }
}

}  // namespace tmop

