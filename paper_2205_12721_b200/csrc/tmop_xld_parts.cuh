// tmop_xld_parts.cuh -- the stages of the x-line diagonal (tmop_xld.cuh),
// shared by the stand-alone diagonal kernel (xld_kernel) and the fused
// setup + diagonal kind of the x-line kernel (xl_kernel<K_SETUP_DIAG>).
#pragma once

#include "tmop_diag.cuh"

namespace tmop {

// register target of the p = 2 diagonal (tools/build_variant.sh A/B)
#ifndef TMOP_XLD_REG3
#define TMOP_XLD_REG3 200
#endif

// group size of the p = 2 diagonal (0: the Hessian action's 8) and whether
// the x^T output overlays the staged records (1) or has its own region (0:
// the next group's record copy is then issued right after the X stage)
#ifndef TMOP_XLD_EPB3
#define TMOP_XLD_EPB3 0
#endif
#ifndef TMOP_XLD_OVL
#define TMOP_XLD_OVL 1
#endif
// p <= 2: the records keep their own region, the x^T output A follows them
// and the y^T output Bv is written into A's own consumed slots (item (qz,kx)
// reads only A[.][.][qz][.][kx]), so the next group's record copy is issued
// right after the X stage and lands during the A store / Y / Z stages, in
// 100 KB per CTA at p = 2 (2 CTAs / SM, like the overlay layout)
#ifndef TMOP_XLD_BVA
#define TMOP_XLD_BVA 1
#endif

template <int N, int Q>
struct XldCfg {
  static constexpr int EPB = (N == 3 && TMOP_XLD_EPB3) ? TMOP_XLD_EPB3 : xl_epb(N);
  static constexpr bool BVA = TMOP_XLD_BVA != 0 && N <= 3;
  static constexpr bool OVL = !BVA && TMOP_XLD_OVL != 0;
  static constexpr int NP = N * N * N, QP = Q * Q * Q;
  static constexpr int LINES = Q * Q;
  static constexpr int NT = EPB * LINES;
  static constexpr int NF = 18;                         // (component, pair) fields
  static constexpr int NA = N | 1;                      // A x-line stride (odd: distinct bank pairs)
  static constexpr int A_SZ = NF * LINES * NA;          // slots (one slot = EPB doubles)
  static constexpr int NB = N * N;                      // Bv (ky, kx) plane
  static constexpr int BV_SZ = 9 * Q * NB;              // [c][g][qz][ky][kx]
  static constexpr int QS = lean_stride(11 * QP, xl_epb(N));   // record element stride (doubles)
  // A overlays the staged records (read-only during X; a barrier separates
  // the last record read from the first A write) or follows them (!OVL);
  // Bv has its own region
  static constexpr int AOFF = OVL ? 0 : ((EPB * QS + 1) & ~1);
  static constexpr int R1 = OVL ? cmax(A_SZ * EPB, EPB * QS) : AOFF + A_SZ * EPB;
  static constexpr int R1P = (R1 + 1) & ~1;             // 16-byte aligned Bv
  static constexpr int SMEM = (R1P + (BVA ? 0 : BV_SZ * EPB)) * 8;
  // the fused setup + diagonal kind (xl_kernel<K_SETUP_DIAG>) always lays A
  // over its records and Bv after them
  static constexpr int R1OP = (cmax(A_SZ * EPB, EPB * QS) + 1) & ~1;
  static constexpr int WARPS = (NT + 31) / 32;
  // occupancy hint: the register target per order, but no more CTAs than
  // fit in shared memory (BVA p = 1: 2 CTAs, so no 128-register cap / spill)
  static constexpr int MINB = cmax(1, cmin(65536 / (WARPS * 32 * (N <= 2 ? 128 : N == 3 ? TMOP_XLD_REG3 : 240)),
                                           (228 * 1024) / (SMEM + 1024 + 1024)));
};

// X: the 18 H-pair values of every point of this thread's line (template or
// non-template metric) from the lean records at qb (field 0 of point qx = 0
// of the line, slots line + Q^2 qx), accumulated into the x^T sweep.
template <int N, int Q, bool NTM>
__device__ __forceinline__ void xld_line(int metric, const double *qb, const Tab &t, double (&acc)[3][6][N]) {
  using PR = Pairs<3>;
  constexpr int QP = Q * Q * Q;
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int f = 0; f < 6; ++f)
#pragma unroll
      for (int k = 0; k < N; ++k) acc[c][f][k] = 0.0;
#pragma unroll
  for (int qx = 0; qx < Q; ++qx) {
    double T[3][3], C[3][3], S[3][3];
    const double *qp = qb + Q * Q * qx;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) T[i][j] = qp[(i * 3 + j) * QP];
    const double k0 = qp[9 * QP], itau = qp[10 * QP];
    mcof<3>(T, C);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) S[i][j] = C[i][j] * itau;
    double hv[3][6];
    if constexpr (!NTM) {
      // c1 (S_n T_p + T_n S_p) + (c2 + c3) S_n S_p = S_n u_p + S_p u_n with
      // u_k = c1 T_k + (c2 + c3)/2 S_k (operator.py:437-441 regrouped): the
      // doubled off-diagonal pairs are S_n u'_p + S_p u'_n, u' = 2u, and the
      // diagonal pairs S_n u'_n + c0 -- 21 instead of 36 FP64 ops per row
      double c[4];
      lean_coeffs(metric, k0, itau, mfro2<3>(T), c);
      const double c1x2 = 2.0 * c[1], c23 = c[2] + c[3];
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) {
        double u[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) u[k] = c1x2 * T[cc][k] + c23 * S[cc][k];
#pragma unroll
        for (int f = 0; f < 6; ++f) {
          const int n = PR::n(f), p = PR::p(f);
          hv[cc][f] = (n == p) ? S[cc][n] * u[n] + c[0] : S[cc][n] * u[p] + S[cc][p] * u[n];
        }
      }
    } else {
      const NtDiag<3> nd(S, T);               // column (c,p): z[n] = H[(c,n),(c,p)] (unit-direction nt_hess)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          double z[3];
          nd.col(metric, k0, S, T, cc, p, z);
#pragma unroll
          for (int f = 0; f < 6; ++f) {
            const int n = PR::n(f), pp = PR::p(f);
            if (pp == p) hv[cc][f] = (n == p) ? z[n] : 2.0 * z[n];
          }
        }
    }
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
#pragma unroll
      for (int f = 0; f < 6; ++f)
#pragma unroll
        for (int k = 0; k < N; ++k) acc[cc][f][k] += t.P[PR::sel(0, f)][qx * N + k] * hv[cc][f];
  }
}

// A[c][f][qz][qy][kx] (element-interleaved slots) <- this line's x^T output
template <int N, int Q>
__device__ __forceinline__ void xld_store_a(double *A, int line, int e, const double (&acc)[3][6][N]) {
  using XC = XldCfg<N, Q>;
  constexpr int EPB = XC::EPB, NA = XC::NA, AV = XC::LINES * NA * EPB;
#pragma unroll
  for (int cc = 0; cc < 3; ++cc)
#pragma unroll
    for (int f = 0; f < 6; ++f)
#pragma unroll
      for (int k = 0; k < N; ++k) A[(cc * 6 + f) * AV + (line * NA + k) * EPB + e] = acc[cc][f][k];
}

// Y: item (qz, kx) -- y^T sweep of every pair, pairs with equal z table
// summed (Pairs::zgroup): Bv[c][g][qz][ky][kx]
template <int N, int Q, bool BVA = false>
__device__ __forceinline__ void xld_y(double *A, double *Bv, int item, int e, const Tab &t) {
  using XC = XldCfg<N, Q>;
  using PR = Pairs<3>;
  constexpr int EPB = XC::EPB, NA = XC::NA, NB = XC::NB, AV = XC::LINES * NA * EPB;
  constexpr int BQ = NB * EPB, BG = Q * BQ;
  const int y_qz = item / N, y_kx = item % N;
#pragma unroll
  for (int cc = 0; cc < 3; ++cc) {
    double s[3][N];
#pragma unroll
    for (int g = 0; g < 3; ++g)
#pragma unroll
      for (int k = 0; k < N; ++k) s[g][k] = 0.0;
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      const double *ap = A + (cc * 6 + f) * AV + ((y_qz * Q) * NA + y_kx) * EPB + e;
      double av[Q];
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) av[qy] = ap[qy * NA * EPB];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double u = 0.0;
#pragma unroll
        for (int qy = 0; qy < Q; ++qy) u += t.P[PR::sel(1, f)][qy * N + k] * av[qy];
        s[PR::zgroup(f)][k] += u;
      }
    }
#pragma unroll
    for (int g = 0; g < 3; ++g)
#pragma unroll
      for (int k = 0; k < N; ++k) {
        if constexpr (BVA) {
          // into this item's consumed A slots of component cc: field g, qy = ky
          A[(cc * 6 + g) * AV + ((y_qz * Q + k) * NA + y_kx) * EPB + e] = s[g][k];
        } else {
          Bv[(cc * 3 + g) * BG + y_qz * BQ + (k * N + y_kx) * EPB + e] = s[g][k];
        }
      }
  }
}

// Z: item (ky, kx) -- z^T sweep of the 3 groups into the element-interleaved
// E-vector of group grp (the Hessian action's layout)
template <int N, int Q, bool BVA = false>
__device__ __forceinline__ void xld_z(const double *Bv, double *E, int64_t grp, int item, int e, const Tab &t) {
  using XC = XldCfg<N, Q>;
  constexpr int EPB = XC::EPB, NP = XC::NP, NB = XC::NB;
  constexpr int BQ = NB * EPB, BG = Q * BQ;
  constexpr int NA = XC::NA, AV = XC::LINES * NA * EPB;
  const int z_ky = item / N, z_kx = item % N;
  double *out = E + (grp * 3 * NP + item) * EPB + e;
#pragma unroll
  for (int cc = 0; cc < 3; ++cc) {
    double o[N];
#pragma unroll
    for (int k = 0; k < N; ++k) o[k] = 0.0;
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      // BVA: Bv lives in A (field g, qy = ky) of component cc (xld_y)
      const double *bp = BVA ? Bv + (cc * 6 + g) * AV + (z_ky * NA + z_kx) * EPB + e
                             : Bv + (cc * 3 + g) * BG + item * EPB + e;
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) {
        const double b = bp[qz * (BVA ? Q * NA * EPB : BQ)];
#pragma unroll
        for (int k = 0; k < N; ++k) o[k] += t.P[g][qz * N + k] * b;
      }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) out[(cc * NP + k * N * N) * EPB] = o[k];
  }
}

}  // namespace tmop
