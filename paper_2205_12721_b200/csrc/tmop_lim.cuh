// tmop_lim.cuh -- the displacement-limiting term (operator.py:463-533):
//
//   c_q = 2 weight det_w w_q / delta_q^2           (_limiting_point_scale)
//   value     = 1/2 sum_q c_q |d_q|^2,  d = B (x - x0)            (K_LIM_VALUE)
//   gradient  = B^T (c_q d_q)           apply = B^T (c_q B v)       (K_LIM_FIELD)
//   diagonal  = (B.B)^T c_q  (added to every component)             (K_LIM_DIAG)
//
// delta is a scalar or a nodal field interpolated with B (fe.py:227-239).
// All contractions use the value table B only (a mass-like operator), so
// this is a small work-item kernel: per group of LEPB elements the D input
// components (+ nodal delta) are gathered into shared memory, interpolated to
// the points by three (2D: two) B sweeps, scaled at the points, and pulled
// back by the transposed sweeps (x axis first, fe.py:242-253) into an
// element-blocked E-vector E[e][c][l] that e2l_kernel sums to nodes; the
// result is added to the main operator's node sums (operator.py:325, 343-344,
// 415-416, 452-457).  The value reduces per CTA in a fixed order.
#pragma once

#include "tmop_elem.cuh"

namespace tmop {

template <int DIM, int N, int Q>
struct LimCfg {
  static constexpr int NP = ipow(N, DIM), QP = ipow(Q, DIM);
  static constexpr int F = DIM + 1;                  // components (+ nodal delta)
  static constexpr int R = F * cmax(cmax(NP, QP), cmax(Q * ipow(N, DIM - 1), ipow(Q, DIM - 1) * N));
  static constexpr int NT = 128;
  static constexpr int EPB = cclamp(6144 / (2 * R), 1, 16);
  static constexpr int SMEM = (EPB * 2 * R + 2 * Q * N) * 8;
};

// out[f][o][t][i] = sum_j T[t][j] in[f][o][j][i]  for every element of the
// group: a (F x O x J x I) -> (F x O x TO x I) contraction along axis J.
template <int DIM, int N, int Q, int O, int J, int I, int TO>
__device__ __forceinline__ void lim_contract(const double *T, const double *in, double *out, int nf) {
  using LC = LimCfg<DIM, N, Q>;
  const int items = LC::EPB * nf * O * I;
  for (int w = threadIdx.x; w < items; w += LC::NT) {
    const int e = w / (nf * O * I), r = w % (nf * O * I);
    const int f = r / (O * I), oi = r % (O * I), o = oi / I, i = oi % I;
    const double *src = in + e * LC::R + f * O * J * I + o * J * I + i;
    double x[J];
#pragma unroll
    for (int j = 0; j < J; ++j) x[j] = src[j * I];
    double *dst = out + e * LC::R + f * O * TO * I + o * TO * I + i;
#pragma unroll
    for (int t = 0; t < TO; ++t) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) s += T[t * J + j] * x[j];
      dst[t * I] = s;
    }
  }
}

template <int DIM, int N, int Q, int KIND>
__global__ void __launch_bounds__(LimCfg<DIM, N, Q>::NT) lim_kernel(const ElemArgs a, const __grid_constant__ Tab t) {
  using LC = LimCfg<DIM, N, Q>;
  constexpr int NP = LC::NP, QP = LC::QP, EPB = LC::EPB, NT = LC::NT, R = LC::R;
  extern __shared__ __align__(16) double smem[];
  double *P0 = smem, *P1 = smem + EPB * R;
  double *TB = smem + 2 * EPB * R;          // B  (Q x N), forward
  double *TT = TB + Q * N;                  // B^T or (B.B)^T (N x Q), backward
  __shared__ double red[NT / 32];
  for (int i = threadIdx.x; i < Q * N; i += NT) {
    TB[i] = t.B[i];
    const int k = i / Q, q = i % Q;         // TT[k][q]
    const double b = t.B[q * N + k];
    TT[i] = KIND == K_LIM_DIAG ? b * b : b;
  }
  const bool nodal = a.lim_dn != nullptr;
  // K_TSCALE (size-field targets): the nodal target volume rides in lim_dn
  const int nf = (KIND == K_LIM_DIAG || KIND == K_TSCALE) ? (nodal ? 1 : 0) : DIM + (nodal ? 1 : 0);
  const int fd = (KIND == K_LIM_DIAG || KIND == K_TSCALE) ? 0 : DIM;   // field index of the nodal scalar
  double acc = 0.0;
  __syncthreads();

  for (int64_t grp = blockIdx.x; grp < a.ngroups; grp += gridDim.x) {
    const int64_t e0 = grp * EPB;
    // ---- gather: components of (in - x0) or in (masked), nodal delta
    for (int w = threadIdx.x; w < EPB * nf * NP; w += NT) {
      const int e = w / (nf * NP), r = w % (nf * NP), f = r / NP, l = r % NP;
      const int64_t eg = e0 + e;
      double val = 0.0;
      if (eg < a.ne) {
        const int node = __ldg(a.restr + eg * NP + l);
        if (f == fd && nodal) {
          val = __ldg(a.lim_dn + node);
        } else {
          val = __ldg(a.in + f * a.nn + node);
          if (a.lim_x0) val -= __ldg(a.lim_x0 + f * a.nn + node);
          if (a.lim_mask && ((__ldg(a.fixed + node) >> f) & 1)) val = 0.0;
        }
      }
      P0[e * R + f * NP + l] = val;
    }
    __syncthreads();
    // ---- forward B sweeps, z axis first (contract_dofs_to_quad, fe.py:227-239)
    double *V = P0;
    if (nf > 0) {
      if constexpr (DIM == 3) {
        lim_contract<3, N, Q, 1, N, N * N, Q>(TB, P0, P1, nf);
        __syncthreads();
        lim_contract<3, N, Q, Q, N, N, Q>(TB, P1, P0, nf);
        __syncthreads();
        lim_contract<3, N, Q, Q * Q, N, 1, Q>(TB, P0, P1, nf);
      } else {
        lim_contract<2, N, Q, 1, N, N, Q>(TB, P0, P1, nf);
        __syncthreads();
        lim_contract<2, N, Q, Q, N, 1, Q>(TB, P1, P0, nf);
      }
      __syncthreads();
      V = DIM == 3 ? P1 : P0;
    }
    // ---- point stage: c_q, then value / scaled field (in place in V)
    double *Z = V;
    for (int w = threadIdx.x; w < EPB * QP; w += NT) {
      const int e = w / QP, q = w % QP;
      const int64_t eg = e0 + e;
      double *vq = V + e * R + q;
      if constexpr (KIND == K_TSCALE) {
        // W_q = v_q^(1/d) I from the interpolated target volume v_q: store 1 / s_q
        // (NaN marks v_q <= 0, checked by the caller)
        const double vv = vq[0];
        if (eg < a.ne) a.qout[eg * QP + q] = vv > 0.0 ? (DIM == 3 ? 1.0 / cbrt(vv) : 1.0 / sqrt(vv)) : NAN;
        continue;
      }
      const double dq = nodal ? vq[fd * QP] : a.lim_delta;
      const double cq = (a.lim_base * wq<DIM, Q>(t, q)) / (dq * dq);
      if constexpr (KIND == K_LIM_VALUE) {
        if (eg < a.ne) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < DIM; ++c) s += cq * vq[c * QP] * vq[c * QP];
          acc += s;
        }
      } else if constexpr (KIND == K_LIM_FIELD) {
#pragma unroll
        for (int c = 0; c < DIM; ++c) vq[c * QP] *= cq;
      } else {
        vq[0] = cq;   // one field; replicated to every component at the E write
      }
    }
    __syncthreads();
    if constexpr (KIND != K_LIM_VALUE && KIND != K_TSCALE) {
      // ---- transposed sweeps, x axis first (contract_quad_to_dofs, fe.py:242-253)
      const int nz = KIND == K_LIM_DIAG ? 1 : DIM;
      double *W = (Z == P0) ? P1 : P0;
      double *outp;
      if constexpr (DIM == 3) {
        lim_contract<3, N, Q, Q * Q, Q, 1, N>(TT, Z, W, nz);
        __syncthreads();
        lim_contract<3, N, Q, Q, Q, N, N>(TT, W, Z, nz);
        __syncthreads();
        lim_contract<3, N, Q, 1, Q, N * N, N>(TT, Z, W, nz);
        outp = W;
      } else {
        lim_contract<2, N, Q, Q, Q, 1, N>(TT, Z, W, nz);
        __syncthreads();
        lim_contract<2, N, Q, 1, Q, N, N>(TT, W, Z, nz);
        outp = Z;
      }
      __syncthreads();
      for (int w = threadIdx.x; w < EPB * DIM * NP; w += NT) {
        const int e = w / (DIM * NP), r = w % (DIM * NP), c = r / NP, l = r % NP;
        const int64_t eg = e0 + e;
        if (eg < a.ne) a.E[(eg * DIM + c) * NP + l] = outp[e * R + (KIND == K_LIM_DIAG ? 0 : c) * NP + l];
      }
    }
    __syncthreads();
  }
  if constexpr (KIND == K_LIM_VALUE) {
    const double s = block_sum<NT>(acc, red);
    if (threadIdx.x == 0) a.part_sum[blockIdx.x] = s;
  }
}

}  // namespace tmop
