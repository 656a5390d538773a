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
#pragma once

#include "tmop_diag.cuh"
#include "tmop_xl.cuh"

namespace tmop {

// register target of the p = 2 diagonal (tools/build_variant.sh A/B)
#ifndef TMOP_XLD_REG3
#define TMOP_XLD_REG3 200
#endif

template <int N, int Q>
struct XldCfg {
  static constexpr int EPB = xl_epb(N);
  static constexpr int NP = N * N * N, QP = Q * Q * Q;
  static constexpr int LINES = Q * Q;
  static constexpr int NT = EPB * LINES;
  static constexpr int NF = 18;                         // (component, pair) fields
  static constexpr int NA = N | 1;                      // A x-line stride (odd: distinct bank pairs)
  static constexpr int A_SZ = NF * LINES * NA;          // slots (one slot = EPB doubles)
  static constexpr int NB = N * N;                      // Bv (ky, kx) plane
  static constexpr int BV_SZ = 9 * Q * NB;              // [c][g][qz][ky][kx]
  static constexpr int QS = lean_stride(11 * QP, EPB);  // record element stride (doubles)
  // A overlays the staged records (read-only during X; a barrier separates
  // the last record read from the first A write), Bv has its own region
  static constexpr int R1 = cmax(A_SZ * EPB, EPB * QS);
  static constexpr int R1P = (R1 + 1) & ~1;             // 16-byte aligned Bv
  static constexpr int SMEM = (R1P + BV_SZ * EPB) * 8;
  static constexpr int WARPS = (NT + 31) / 32;
  static constexpr int MINB = cmax(1, 65536 / (WARPS * 32 * (N <= 2 ? 128 : N == 3 ? TMOP_XLD_REG3 : 240)));
};

template <int N, int Q>
__host__ __device__ constexpr bool xld_supported() {
  return N <= 4 && XldCfg<N, Q>::SMEM <= 227 * 1024;
}

template <int N, int Q, bool NTM>
__global__ void __launch_bounds__(XldCfg<N, Q>::NT, XldCfg<N, Q>::MINB)
    xld_kernel(const ElemArgs a, const __grid_constant__ Tab t) {
  using XC = XldCfg<N, Q>;
  using PR = Pairs<3>;
  constexpr int EPB = XC::EPB, NP = XC::NP, QP = XC::QP, QS = XC::QS, NA = XC::NA, NB = XC::NB;
  constexpr int AV = XC::LINES * NA * EPB;     // A stride of one (c, f) field
  constexpr int BQ = NB * EPB;                 // Bv stride of qz
  constexpr int BG = Q * BQ;                   // Bv stride of (c, g)
  extern __shared__ __align__(16) double smem[];
  double *QB = smem;                           // staged records ...
  double *A = smem;                            // ... overlaid by the x^T output
  double *Bv = smem + XC::R1P;
  __shared__ __align__(8) uint64_t qbar;

  const int tid = threadIdx.x;
  const int e = tid % EPB, item = tid / EPB;
  const int line = item;                       // X: line = qy + Q qz
  const bool ry = item < Q * N;                // Y: (qz, kx)
  const int y_qz = item / N, y_kx = item % N;
  const bool rz = item < N * N;                // Z: (ky, kx)

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
    // ---- X: H-pair values per point, x^T sweep in registers
    double acc[3][6][N];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int f = 0; f < 6; ++f)
#pragma unroll
        for (int k = 0; k < N; ++k) acc[c][f][k] = 0.0;
    const double *qb = QB + e * QS + line;     // field 0, point (qx = 0) of this line
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
        double c[4];
        lean_coeffs(a.metric, k0, itau, mfro2<3>(T), c);
        const double c23 = c[2] + c[3];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
#pragma unroll
          for (int f = 0; f < 6; ++f) {
            const int n = PR::n(f), p = PR::p(f);
            const double sn = S[cc][n], sp = S[cc][p], tn = T[cc][n], tp = T[cc][p];
            double v = c[1] * (sn * tp + tn * sp) + c23 * sn * sp;
            if (n == p)
              v += c[0];
            else
              v *= 2.0;
            hv[cc][f] = v;
          }
      } else {
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
#pragma unroll
          for (int p = 0; p < 3; ++p) {
            double g[3][3] = {}, z[3][3];
            g[cc][p] = 1.0;
            nt_hess<3>(a.metric, k0, S, T, g, z);   // column (c,p) of the block: z[c][n] = H[(c,n),(c,p)]
#pragma unroll
            for (int f = 0; f < 6; ++f) {
              const int n = PR::n(f), pp = PR::p(f);
              if (pp == p) hv[cc][f] = (n == p) ? z[cc][n] : 2.0 * z[cc][n];
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
    __syncthreads();                           // every record read: A may overwrite QB
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
#pragma unroll
      for (int f = 0; f < 6; ++f)
#pragma unroll
        for (int k = 0; k < N; ++k) A[(cc * 6 + f) * AV + (line * NA + k) * EPB + e] = acc[cc][f][k];
    __syncthreads();
    // ---- Y: y^T sweep per pair, pairs with equal z table summed
    if (ry) {
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
          for (int k = 0; k < N; ++k) Bv[(cc * 3 + g) * BG + y_qz * BQ + (k * N + y_kx) * EPB + e] = s[g][k];
      }
    }
    __syncthreads();                           // A (= QB) consumed: stream in the next group's records
    if (tid == 0 && grp + gridDim.x < a.ngroups) issue(grp + gridDim.x);
    // ---- Z: z^T sweep of the 3 groups -> element-interleaved E-vector
    if (rz) {
      double *out = a.E + (grp * 3 * NP + item) * EPB + e;
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) {
        double o[N];
#pragma unroll
        for (int k = 0; k < N; ++k) o[k] = 0.0;
#pragma unroll
        for (int g = 0; g < 3; ++g) {
          const double *bp = Bv + (cc * 3 + g) * BG + item * EPB + e;
#pragma unroll
          for (int qz = 0; qz < Q; ++qz) {
            const double b = bp[qz * BQ];
#pragma unroll
            for (int k = 0; k < N; ++k) o[k] += t.P[g][qz * N + k] * b;
          }
        }
#pragma unroll
        for (int k = 0; k < N; ++k) out[(cc * NP + k * N * N) * EPB] = o[k];
      }
    }
    // (the next group's X stage writes only registers; its A writes come
    // after the barrier that follows its record reads, and Bv is rewritten
    // only after the next Y barrier -- Z of this group is ordered before
    // both by the X-stage barrier)
  }
}

}  // namespace tmop
