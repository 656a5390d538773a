/*
 * tmop_cpu.c -- C/OpenMP restatement of the reference Hessian action
 * (TEST INFRASTRUCTURE / CPU BASELINE ONLY -- see oracle/__init__.py).
 *
 * Restates TmopProblem.hessian_apply (operator.py:401-418) for 3D hexes:
 *   vin = where(fixed, 0, v)                                  (op:409)
 *   per element: gather (fe:180-187), for each reference direction p the
 *   3-axis contraction with G on axis p and B elsewhere, z axis first
 *   (fe:227-239, fe:256-260); the factored block multiply per point
 *   (_kernels.py:235-258) on the reference's PLANAR Q-data (op:105-113);
 *   per direction n the transposed contraction, x axis first
 *   (fe:242-253), summed over n (op:286-290);
 *   E -> L sum in ascending element order (np.add.at, fe:189-204; op:277)
 *   through a node -> (element, local) map;
 *   out[fixed] = v[fixed]                                     (op:417)
 * Parallelism: OpenMP over elements (element-local work is independent,
 * _kernels.py:3-6) and over nodes for the E -> L sum, so the result is
 * independent of the thread count.
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXN 5
#define MAXQ 9

/* out[c][b][a] = sum_k M[c][k] * in[k][b][a]  (z axis contraction, extents) */
static void contract_z(int n_in, int n_out, int nb, int na, const double *M, const double *in, double *out) {
  for (int c = 0; c < n_out; ++c)
    for (int ba = 0; ba < nb * na; ++ba) {
      double s = 0.0;
      for (int k = 0; k < n_in; ++k) s += M[c * n_in + k] * in[k * nb * na + ba];
      out[c * nb * na + ba] = s;
    }
}
/* y axis: in[z][k][a] -> out[z][c][a] */
static void contract_y(int nz, int n_in, int n_out, int na, const double *M, const double *in, double *out) {
  for (int z = 0; z < nz; ++z)
    for (int c = 0; c < n_out; ++c)
      for (int a = 0; a < na; ++a) {
        double s = 0.0;
        for (int k = 0; k < n_in; ++k) s += M[c * n_in + k] * in[(z * n_in + k) * na + a];
        out[(z * n_out + c) * na + a] = s;
      }
}
/* x axis: in[zy][k] -> out[zy][c] */
static void contract_x(int nzy, int n_in, int n_out, const double *M, const double *in, double *out) {
  for (int r = 0; r < nzy; ++r)
    for (int c = 0; c < n_out; ++c) {
      double s = 0.0;
      for (int k = 0; k < n_in; ++k) s += M[c * n_in + k] * in[r * n_in + k];
      out[r * n_out + c] = s;
    }
}

static void transpose(int r, int c, const double *M, double *MT) {
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) MT[j * r + i] = M[i * c + j];
}

int oracle_hessian_apply3d(int n1, int nq, int64_t ne, int64_t nn, const int32_t *restr, const uint8_t *fixed,
                           const double *B, const double *G, const double *coeffs, const double *smat,
                           const double *tmat, const double *v, double *y, const int64_t *l2e_off,
                           const uint32_t *l2e_idx, double *E, int nthreads) {
  const int NP = n1 * n1 * n1, QP = nq * nq * nq;
  const int64_t NQ = ne * QP;
  if (n1 > MAXN || nq > MAXQ) return 1;
  double BT[MAXQ * MAXN], GT[MAXQ * MAXN];
  transpose(nq, n1, B, BT);
  transpose(nq, n1, G, GT);
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
  {
    double X[3 * MAXN * MAXN * MAXN];
    double t1[MAXQ * MAXN * MAXN], t2[MAXQ * MAXQ * MAXN];
    double g[3][3][MAXQ * MAXQ * MAXQ], z[3][3][MAXQ * MAXQ * MAXQ];
    double u1[MAXQ * MAXQ * MAXN], u2[MAXQ * MAXN * MAXN], part[MAXN * MAXN * MAXN];
#pragma omp for schedule(static)
    for (int64_t e = 0; e < ne; ++e) {
      for (int c = 0; c < 3; ++c)
        for (int l = 0; l < NP; ++l) {
          const int32_t node = restr[e * NP + l];
          X[c * NP + l] = ((fixed[node] >> c) & 1) ? 0.0 : v[c * nn + node];
        }
      for (int c = 0; c < 3; ++c)
        for (int p = 0; p < 3; ++p) {
          const double *Mx = (p == 0) ? G : B, *My = (p == 1) ? G : B, *Mz = (p == 2) ? G : B;
          contract_z(n1, nq, n1, n1, Mz, X + c * NP, t1);
          contract_y(nq, n1, nq, n1, My, t1, t2);
          contract_x(nq * nq, n1, nq, Mx, t2, g[c][p]);
        }
      for (int q = 0; q < QP; ++q) {
        const int64_t k = e * QP + q;
        double S[3][3], T[3][3], gg[3][3];
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) {
            S[a][b] = smat[(a * 3 + b) * NQ + k];
            T[a][b] = tmat[(a * 3 + b) * NQ + k];
            gg[a][b] = g[a][b][q];
          }
        double dt = 0.0, ds = 0.0;
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) {
            dt += T[a][b] * gg[a][b];
            ds += S[a][b] * gg[a][b];
          }
        const double c0 = coeffs[0 * NQ + k], c1 = coeffs[1 * NQ + k], c2 = coeffs[2 * NQ + k],
                     c3 = coeffs[3 * NQ + k];
        const double w1 = c1 * dt + c2 * ds, w2 = c1 * ds;
        for (int a = 0; a < 3; ++a)
          for (int n = 0; n < 3; ++n) {
            double cross = 0.0;
            for (int p = 0; p < 3; ++p) {
              double gs = 0.0;
              for (int o = 0; o < 3; ++o) gs += gg[o][p] * S[o][n];
              cross += S[a][p] * gs;
            }
            z[a][n][q] = c0 * gg[a][n] + w1 * S[a][n] + w2 * T[a][n] + c3 * cross;
          }
      }
      for (int c = 0; c < 3; ++c) {
        double *out = E + (e * 3 + c) * NP;
        for (int n = 0; n < 3; ++n) {
          const double *Mx = (n == 0) ? GT : BT, *My = (n == 1) ? GT : BT, *Mz = (n == 2) ? GT : BT;
          contract_x(nq * nq, nq, n1, Mx, z[c][n], u1);
          contract_y(nq, nq, n1, n1, My, u1, u2);
          contract_z(nq, n1, n1, n1, Mz, u2, part);
          if (n == 0)
            memcpy(out, part, sizeof(double) * NP);
          else
            for (int l = 0; l < NP; ++l) out[l] += part[l];
        }
      }
    }
#pragma omp for schedule(static)
    for (int64_t node = 0; node < nn; ++node) {
      double acc[3] = {0.0, 0.0, 0.0};
      for (int64_t k = l2e_off[node]; k < l2e_off[node + 1]; ++k) {
        const uint32_t u = l2e_idx[k];
        const int64_t e = u / NP, l = u % NP;
        for (int c = 0; c < 3; ++c) acc[c] += E[(e * 3 + c) * NP + l];
      }
      for (int c = 0; c < 3; ++c) y[c * nn + node] = ((fixed[node] >> c) & 1) ? v[c * nn + node] : acc[c];
    }
  }
  return 0;
}

int oracle_max_threads(void) { return omp_get_max_threads(); }
