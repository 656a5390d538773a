// tmop_device.cuh -- device building blocks of the B200 TMOP kernels.
//
// * Tab: 1D basis tables B[q][i], G[q][i] and 1D weights, passed BY VALUE
//   as a __grid_constant__ kernel parameter so every table read is a
//   constant-bank operand (no shared-memory or register pressure).
//   (fe.py:143-160, fe.py:126-140)
// * Point algebra: det / cofactor / metric values, first derivatives and the
//   4-coefficient Hessian template (metrics.py:7-13, 173-262;
//   _kernels.py:20-258), plus the non-template mu_302 / mu_321 Hessian
//   actions (extensions, derived in DESIGN.md section 3).
// * Sum-factorised stages over shared memory (fe.py:218-253 restated as
//   per-line register-blocked contractions, one work item = one 1D line).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tmop {

constexpr int MAXN = 5;   // p <= 4
constexpr int MAXQ = 9;   // n_q <= 9 (paper table uses 9)

struct Tab {
  double B[MAXQ * MAXN];
  double G[MAXQ * MAXN];
  double w1[MAXQ];
  // elementwise products B.B, B.G, G.G (the diagonal's per-axis tables,
  // operator.py:443-448), indexed like B
  double P[3][MAXQ * MAXN];
};

template <int Q, int N>
__device__ __forceinline__ double tB(const Tab &t, int q, int i) { return t.B[q * N + i]; }
template <int Q, int N>
__device__ __forceinline__ double tG(const Tab &t, int q, int i) { return t.G[q * N + i]; }

// tensor weight of flat point q (x fastest): w[qz] * (w[qy] * w[qx]),
// the association order of np.multiply.outer in fe.py:134-140.
template <int DIM, int Q>
__device__ __forceinline__ double wq(const Tab &t, int q) {
  if constexpr (DIM == 2) {
    return t.w1[q / Q] * t.w1[q % Q];
  } else {
    return t.w1[q / (Q * Q)] * (t.w1[(q / Q) % Q] * t.w1[q % Q]);
  }
}

// ---------------------------------------------------------------- metrics
enum : int { MU2 = 2, MU7 = 7, MU55 = 55, MU302 = 302, MU303 = 303, MU321 = 321 };

__host__ __device__ inline bool metric_is_template(int m) {
  return m == MU2 || m == MU7 || m == MU55 || m == MU303;
}

template <int D>
__device__ __forceinline__ double mdet(const double (&A)[D][D]) {
  if constexpr (D == 2) {
    return A[0][0] * A[1][1] - A[0][1] * A[1][0];
  } else {
    return A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) -
           A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
           A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
  }
}

// cof(A) with A^{-T} = cof(A)/det(A) (metrics.py:79-97, _kernels.py:115-131)
template <int D>
__device__ __forceinline__ void mcof(const double (&A)[D][D], double (&C)[D][D]) {
  if constexpr (D == 2) {
    C[0][0] = A[1][1];  C[0][1] = -A[1][0];
    C[1][0] = -A[0][1]; C[1][1] = A[0][0];
  } else {
    C[0][0] = A[1][1] * A[2][2] - A[1][2] * A[2][1];
    C[0][1] = A[1][2] * A[2][0] - A[1][0] * A[2][2];
    C[0][2] = A[1][0] * A[2][1] - A[1][1] * A[2][0];
    C[1][0] = A[0][2] * A[2][1] - A[0][1] * A[2][2];
    C[1][1] = A[0][0] * A[2][2] - A[0][2] * A[2][0];
    C[1][2] = A[0][1] * A[2][0] - A[0][0] * A[2][1];
    C[2][0] = A[0][1] * A[1][2] - A[0][2] * A[1][1];
    C[2][1] = A[0][2] * A[1][0] - A[0][0] * A[1][2];
    C[2][2] = A[0][0] * A[1][1] - A[0][1] * A[1][0];
  }
}

template <int D>
__device__ __forceinline__ double mfro2(const double (&A)[D][D]) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) s += A[i][j] * A[i][j];
  return s;
}

template <int D>
__device__ __forceinline__ double mdot(const double (&A)[D][D], const double (&B)[D][D]) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) s += A[i][j] * B[i][j];
  return s;
}

// C = A * B^T * C0 style helpers
template <int D>
__device__ __forceinline__ void mmul(const double (&A)[D][D], const double (&B)[D][D], double (&C)[D][D]) {
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += A[i][k] * B[k][j];
      C[i][j] = s;
    }
}
template <int D>
__device__ __forceinline__ void mmulT(const double (&A)[D][D], const double (&B)[D][D], double (&C)[D][D]) {
  // C = A * B^T
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += A[i][k] * B[j][k];
      C[i][j] = s;
    }
}

// mu(T) given tau = det T, I1 = |T|^2 and (for non-template metrics) S.
template <int D>
__device__ __forceinline__ double metric_mu(int metric, double tau, double I1, const double (&S)[D][D]) {
  switch (metric) {
    case MU2: return I1 / (2.0 * tau) - 1.0;
    case MU55: { double t = tau - 1.0; return t * t; }
    case MU303: return I1 * rcbrt(tau * tau) * (1.0 / 3.0) - 1.0;
    case MU7: return I1 + mfro2<D>(S) - 2.0 * D;
    case MU302: return I1 * mfro2<D>(S) * (1.0 / 9.0) - 1.0;
    default: /* MU321 */ return I1 + mfro2<D>(S) - 2.0 * D;
  }
}

// (a_t, a_s): dmu/dT = a_t T + a_s S  (metrics.py:188-196, _kernels.py:89-98)
__device__ __forceinline__ void metric_first_coeffs(int metric, double tau, double I1, double &at, double &as) {
  switch (metric) {
    case MU2: at = 1.0 / tau; as = -I1 / (2.0 * tau); break;
    case MU55: at = 0.0; as = 2.0 * tau * (tau - 1.0); break;
    case MU7: { double it2 = 1.0 / (tau * tau); at = 2.0 * (1.0 + it2); as = -2.0 * I1 * it2; } break;
    default: /* MU303 */ {
      double r = rcbrt(tau * tau);
      at = (2.0 / 3.0) * r; as = -(2.0 / 9.0) * I1 * r;
    }
  }
}

// mu (when `want_mu`) and (a_t, a_s) of a template metric from one rcbrt:
// bitwise the values metric_mu / metric_first_coeffs return (the gradient
// kernel's fused line-search energy, solvers.py:210-216).
template <int D>
__device__ __forceinline__ void metric_mu_first(int metric, double tau, double I1, const double (&S)[D][D],
                                                bool want_mu, double &mu, double &at, double &as) {
  if (metric == MU303) {
    const double r = rcbrt(tau * tau);
    if (want_mu) mu = I1 * r * (1.0 / 3.0) - 1.0;
    at = (2.0 / 3.0) * r; as = -(2.0 / 9.0) * I1 * r;
  } else {
    if (want_mu) mu = metric_mu<D>(metric, tau, I1, S);
    metric_first_coeffs(metric, tau, I1, at, as);
  }
}

// (c_id, c_ts, c_ss, c_x) of the Hessian template (metrics.py:199-210,
// _kernels.py:155-171); mu_7 derived in DESIGN.md.
__device__ __forceinline__ void metric_second_coeffs(int metric, double tau, double I1, double (&c)[4]) {
  switch (metric) {
    case MU2: { double h = I1 / (2.0 * tau); c[0] = 1.0 / tau; c[1] = -1.0 / tau; c[2] = h; c[3] = h; } break;
    case MU55: c[0] = 0.0; c[1] = 0.0; c[2] = 2.0 * tau * (2.0 * tau - 1.0); c[3] = -2.0 * tau * (tau - 1.0); break;
    case MU7: { double it2 = 1.0 / (tau * tau);
      c[0] = 2.0 * (1.0 + it2); c[1] = -4.0 * it2; c[2] = 4.0 * I1 * it2; c[3] = 2.0 * I1 * it2; } break;
    default: /* MU303 */ {
      double r = rcbrt(tau * tau);
      c[0] = (2.0 / 3.0) * r; c[1] = -(4.0 / 9.0) * r;
      c[2] = (4.0 / 27.0) * I1 * r; c[3] = (2.0 / 9.0) * I1 * r;
    }
  }
}

// ---- lean Q-data (the B200 format) -------------------
// Per point: T (d*d), k0, itau = 1/det T.  S = cof(T) * itau and I1 = |T|^2
// are recomputed in the apply, and the four template coefficients follow
// from (k0, itau, I1) -- 11 doubles per 3D point instead of the reference's
// 4 + 2 d^2 = 22 (operator.py:91-113), with identical information.
//   mu_303: k0 = sw r, r = tau^{-2/3}:  c = k0 (2/3, -4/9, 4/27 I1, 2/9 I1)
//   mu_2:   k0 = sw / tau:              c = k0 (1, -1, I1/2, I1/2)
//   mu_7:   k0 = sw:                    c = k0 (2(1+it2), -4 it2, 4 I1 it2, 2 I1 it2)
//   mu_55:  k0 = sw:                    c = k0 (0, 0, 2 tau(2 tau-1), -2 tau(tau-1))
//   mu_302 / mu_321: k0 = sw (non-template action, nt_hess)
__device__ __forceinline__ double lean_k0(int metric, double sw, double tau) {
  switch (metric) {
    case MU303: return sw * rcbrt(tau * tau);
    case MU2: return sw / tau;
    default: return sw;
  }
}
__device__ __forceinline__ void lean_coeffs(int metric, double k0, double itau, double I1, double (&c)[4]) {
  switch (metric) {
    case MU303: {
      const double h = k0 * I1;
      c[0] = (2.0 / 3.0) * k0; c[1] = -(4.0 / 9.0) * k0; c[2] = (4.0 / 27.0) * h; c[3] = (2.0 / 9.0) * h;
    } break;
    case MU2: { const double h = 0.5 * k0 * I1; c[0] = k0; c[1] = -k0; c[2] = h; c[3] = h; } break;
    case MU7: {
      const double it2 = itau * itau, h = k0 * it2;
      c[0] = 2.0 * k0 * (1.0 + it2); c[1] = -4.0 * h; c[2] = 4.0 * h * I1; c[3] = 2.0 * h * I1;
    } break;
    default: /* MU55 */ {
      const double tau = 1.0 / itau;
      c[0] = 0.0; c[1] = 0.0; c[2] = 2.0 * k0 * tau * (2.0 * tau - 1.0); c[3] = -2.0 * k0 * tau * (tau - 1.0);
    }
  }
}

// z = H g for the template block  c0 I + c1 (S(x)T + T(x)S) + c2 S(x)S + c3 S_mp S_on
// (_kernels.py:235-258).
template <int D>
__device__ __forceinline__ void hess_template(const double (&c)[4], const double (&S)[D][D], const double (&T)[D][D],
                                              const double (&g)[D][D], double (&z)[D][D]) {
  const double dt = mdot<D>(T, g);
  const double ds = mdot<D>(S, g);
  const double w1 = c[1] * dt + c[2] * ds;
  const double w2 = c[1] * ds;
  // gs[p][n] = sum_o g[o][p] S[o][n] ; cross[a][n] = sum_p S[a][p] gs[p][n]
  double gs[D][D];
#pragma unroll
  for (int p = 0; p < D; ++p)
#pragma unroll
    for (int n = 0; n < D; ++n) {
      double s = 0.0;
#pragma unroll
      for (int o = 0; o < D; ++o) s += g[o][p] * S[o][n];
      gs[p][n] = s;
    }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int n = 0; n < D; ++n) {
      double cross = 0.0;
#pragma unroll
      for (int p = 0; p < D; ++p) cross += S[a][p] * gs[p][n];
      z[a][n] = c[0] * g[a][n] + w1 * S[a][n] + w2 * T[a][n] + c[3] * cross;
    }
}

// 3D template block from C = cof(T) (S = itau C) without forming S g^T S:
// with tau = det T, C g^T C = (C:g) C - tau dcof(T)[g] (differentiate
// cof(T) = tau T^-T), so
//   z = c0 g + (w1 + k3 ds) C + w2 T - k3 dcof(T)[g],  k3 = c3 itau,
// w1 = (c1 T:g + c2 ds) itau, w2 = c1 ds, ds = itau C:g -- 72 FP64 ops for
// the g-dependent part instead of 90 (two 3x3 products).  dcof(T)[g]_ij is
// the cyclic 2x2 minor rule of mcof differentiated: 4 products per entry.
#ifndef TMOP_DCOF
#define TMOP_DCOF 1
#endif
__device__ __forceinline__ void hess_tpl_cof3(const double (&c)[4], const double (&C)[3][3], const double (&T)[3][3],
                                              double itau, const double (&g)[3][3], double (&z)[3][3]) {
  double dt = 0.0, cgd = 0.0;
  {
    double r[3], q[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      r[i] = T[i][0] * g[i][0] + T[i][1] * g[i][1] + T[i][2] * g[i][2];
      q[i] = C[i][0] * g[i][0] + C[i][1] * g[i][1] + C[i][2] * g[i][2];
    }
    dt = (r[0] + r[1]) + r[2];
    cgd = (q[0] + q[1]) + q[2];
  }
  const double ds = itau * cgd;
  const double w1 = (c[1] * dt + c[2] * ds) * itau;
  const double w2 = c[1] * ds;
  const double k3 = c[3] * itau;
  const double wc = w1 + k3 * ds;
  if constexpr (TMOP_DCOF == 2) {
    // rows: wc C_i - k3 dcof_i = (wc T_i1 + h_i1) x T_i2 + T_i1 x h_i2 with
    // h = -k3 g (C_i = T_i1 x T_i2, i1 = i+1, i2 = i+2 cyclic): 6 FP64 ops
    // per entry + 18 (72) instead of 9 per entry (81)
    double h[3][3], u[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        h[i][j] = -k3 * g[i][j];
        u[i][j] = wc * T[i][j] + h[i][j];
      }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int i1 = (i + 1) % 3, i2 = (i + 2) % 3;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int j1 = (j + 1) % 3, j2 = (j + 2) % 3;
        // one FMA chain: 1 DMUL + 5 DFMA
        double r = c[0] * g[i][j];
        r = fma(w2, T[i][j], r);
        r = fma(u[i1][j1], T[i2][j2], r);
        r = fma(-u[i1][j2], T[i2][j1], r);
        r = fma(T[i1][j1], h[i2][j2], r);
        z[i][j] = fma(-T[i1][j2], h[i2][j1], r);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int i1 = (i + 1) % 3, i2 = (i + 2) % 3;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int j1 = (j + 1) % 3, j2 = (j + 2) % 3;
        const double dc = (g[i1][j1] * T[i2][j2] + T[i1][j1] * g[i2][j2]) -
                          (g[i1][j2] * T[i2][j1] + T[i1][j2] * g[i2][j1]);
        z[i][j] = c[0] * g[i][j] + wc * C[i][j] + w2 * T[i][j] - k3 * dc;
      }
    }
  }
}

// Non-template metrics (mu_302, mu_321): first derivative and Hessian action
// from T and S = T^{-T}.  With I1 = |T|^2, J = |S|^2, M = S S^T S:
//   dJ/dT = -2 M,  dS[g] = -S g^T S,  dM[g] = dS S^T S + S dS^T S + S S^T dS.
//   mu_321 = I1 + J - 6:      P = 2T - 2M;              H g = 2g - 2 dM[g]
//   mu_302 = I1 J / 9 - 1:    P = (2 J T - 2 I1 M)/9;
//       H g = (2 dJ T + 2 J g - 2 dI1 M - 2 I1 dM[g]) / 9, dJ = -2 M:g, dI1 = 2 T:g
// Symmetric products S S^T and S^T S (6 / 3 unique entries).
template <int D>
__device__ __forceinline__ void nt_sym(const double (&S)[D][D], double (&SSt)[D][D], double (&StS)[D][D]) {
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = i; j < D; ++j) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        a += S[i][k] * S[j][k];
        b += S[k][i] * S[k][j];
      }
      SSt[i][j] = SSt[j][i] = a;
      StS[i][j] = StS[j][i] = b;
    }
}

template <int D>
__device__ __forceinline__ void nt_first(int metric, const double (&T)[D][D], const double (&S)[D][D], double (&P)[D][D]) {
  double SSt[D][D], StS[D][D], M[D][D];
  nt_sym<D>(S, SSt, StS);
  mmul<D>(SSt, S, M);
  if (metric == MU302) {
    const double I1 = mfro2<D>(T), J = mfro2<D>(S);
    const double ct = (2.0 / 9.0) * J, cm = -(2.0 / 9.0) * I1;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) P[i][j] = ct * T[i][j] + cm * M[i][j];
  } else {
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) P[i][j] = 2.0 * T[i][j] - 2.0 * M[i][j];
  }
}

// With dS = -S g^T S:  dM = dS S^T S + S dS^T S + S S^T dS
//                         = -[(S g^T) M + (S S^T g)(S^T S) + (M g^T) S]
// (S (S^T S) = (S S^T) S = M), three 3x3 products instead of seven.
template <int D>
__device__ __forceinline__ void nt_hess(int metric, double w, const double (&S)[D][D], const double (&T)[D][D],
                                        const double (&g)[D][D], double (&z)[D][D]) {
  // -dM[g] = S g^T M + S S^T g S^T S + M g^T S with M = S S^T S regrouped as
  //   B = S (g^T S):  -dM[g] = B (S^T S) + (S S^T)(g S^T S + B)
  // -- five 3x3 products instead of six plus M (M itself only for mu_302)
  double SSt[D][D], StS[D][D];
  nt_sym<D>(S, SSt, StS);
  double A[D][D], B[D][D], Cm[D][D];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s0 = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s0 += g[k][i] * S[k][j];
      A[i][j] = s0;                       // g^T S
    }
  mmul<D>(S, A, B);
  mmul<D>(g, StS, Cm);
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) Cm[i][j] += B[i][j];
  double nM[D][D];               // -dM[g]
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s0 = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s0 += B[i][k] * StS[k][j] + SSt[i][k] * Cm[k][j];
      nM[i][j] = s0;
    }
  if (metric == MU302) {
    double M[D][D];
    mmul<D>(SSt, S, M);
    const double I1 = mfro2<D>(T), J = mfro2<D>(S);
    const double dJ = -2.0 * mdot<D>(M, g), dI1 = 2.0 * mdot<D>(T, g);
    const double c = (2.0 / 9.0) * w;
    const double ct = c * dJ, cg = c * J, cm = -c * dI1, cn = c * I1;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) z[i][j] = ct * T[i][j] + cg * g[i][j] + cm * M[i][j] + cn * nM[i][j];
  } else {
    const double c = 2.0 * w;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) z[i][j] = c * (g[i][j] + nM[i][j]);
  }
}

// Row c of nt_hess for the unit direction g = e_c e_p^T (column (c, p) of
// the Hessian block, the diagonal's need): with g a unit matrix the three
// products of nt_hess collapse to rank-one terms,
//   -dM[g]_cj = S_cp M_cj + (S S^T)_cc (S^T S)_pj + M_cp S_cj,
// so a column costs ~15 FP64 operations instead of a full Hessian action.
template <int D>
struct NtDiag {
  double SSt[D][D], StS[D][D], M[D][D], I1, J;
  __device__ __forceinline__ NtDiag(const double (&S)[D][D], const double (&T)[D][D]) {
    nt_sym<D>(S, SSt, StS);
    mmul<D>(SSt, S, M);
    I1 = mfro2<D>(T);
    J = mfro2<D>(S);
  }
  // z[n] = H[(c,n),(c,p)] for n = 0..D-1 (metric MU302 / MU321, scale w)
  __device__ __forceinline__ void col(int metric, double w, const double (&S)[D][D], const double (&T)[D][D], int c,
                                      int p, double (&z)[D]) const {
    double nM[D];
#pragma unroll
    for (int j = 0; j < D; ++j) nM[j] = S[c][p] * M[c][j] + SSt[c][c] * StS[p][j] + M[c][p] * S[c][j];
    if (metric == MU302) {
      const double cc = (2.0 / 9.0) * w;
      const double dJ = -2.0 * M[c][p], dI1 = 2.0 * T[c][p];
#pragma unroll
      for (int j = 0; j < D; ++j) z[j] = cc * (dJ * T[c][j] + (j == p ? J : 0.0) - dI1 * M[c][j] + I1 * nM[j]);
    } else {
      const double cc = 2.0 * w;
#pragma unroll
      for (int j = 0; j < D; ++j) z[j] = cc * ((j == p ? 1.0 : 0.0) + nM[j]);
    }
  }
};

// ------------------------------------------- TMA bulk copy + mbarrier
// One elected thread streams a contiguous global range into shared memory
// with cp.async.bulk (the TMA engine, no register staging); consumers wait
// on an mbarrier phase.  Sizes and addresses must be multiples of 16 B.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// cp.async (LDGSTS): global -> shared without register staging.
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// Bulk L2 prefetch (no shared-memory destination): bytes % 16 == 0, src 16-byte aligned.
__device__ __forceinline__ void l2_prefetch_bulk(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// ------------------------------------------------ deterministic reductions
struct MinLoc {
  double v;
  int64_t i;
};
__device__ __forceinline__ MinLoc minloc(MinLoc a, MinLoc b) {
  if (b.v < a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

// Fixed-order block reduction (warp shuffles in a fixed butterfly, then a
// fixed pass over warp results).  Result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) r += scratch[w];
  }
  return r;
}

template <int NT>
__device__ __forceinline__ MinLoc block_minloc(MinLoc m, double *sv, int64_t *si) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    MinLoc other;
    other.v = __shfl_down_sync(0xffffffffu, m.v, o);
    other.i = __shfl_down_sync(0xffffffffu, m.i, o);
    m = minloc(m, other);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) { sv[wid] = m.v; si[wid] = m.i; }
  __syncthreads();
  MinLoc r{sv[0], si[0]};
  if (threadIdx.x == 0) {
    for (int w = 1; w < NT / 32; ++w) r = minloc(r, MinLoc{sv[w], si[w]});
  }
  return r;
}

}  // namespace tmop
