// tmop_diag.cuh -- exact diagonal of the partially assembled Hessian
// (AssembleGradDiagonalPA; reference hessian_diagonal, operator.py:420-459).
//
//   diag[(c,i)] = sum_q sum_{n,p} D_n(q,i) H[(c,n),(c,p)](q) D_p(q,i)
//
// with D_n(q,i) D_p(q,i) = prod_axis (M_n,axis .* M_p,axis)[q_a, i_a] and
// M = G on the differentiated axis, B elsewhere (operator.py:443-448).  The
// summand is symmetric in (n, p), so only the d(d+1)/2 unique pairs are
// formed (off-diagonal pairs doubled).  Per element: one point stage builds
// H-pair values for every component from the lean record, then ONE batched
// transposed contraction over all (component, pair) fields with the
// per-axis product tables (BB, BG, GG) held in shared memory.
#pragma once

#include "tmop_elem.cuh"

namespace tmop {

template <int DIM, int N, int Q>
struct DiagCfg {
  static constexpr int NPAIR = DIM * (DIM + 1) / 2;
  static constexpr int NF = DIM * NPAIR;                      // (component, pair) fields
  static constexpr int QP = ipow(Q, DIM), NP = ipow(N, DIM);
  static constexpr int RA = DIM == 3 ? cmax(NF * QP, NF * Q * N * N) : NF * QP;   // points / y-sweep out
  static constexpr int RB = DIM == 3 ? NF * Q * Q * N : NF * Q * N;               // x-sweep out
  static constexpr int PER = RA + RB;
  static constexpr int EPB = cclamp(8192 / PER, 1, 32);
  static constexpr int PT = 3 * Q * N;                        // product tables BB, BG, GG
  static constexpr int SMEM = (EPB * PER + PT) * 8;
};

// pair index -> (n, p), n <= p: diagonal pairs first
template <int DIM>
__device__ __forceinline__ void pair_np(int f, int &n, int &p) {
  if constexpr (DIM == 2) {
    n = f == 2 ? 0 : f;
    p = f == 2 ? 1 : f;
  } else {
    const int nn[6] = {0, 1, 2, 0, 0, 1}, pp[6] = {0, 1, 2, 1, 2, 2};
    n = nn[f];
    p = pp[f];
  }
}

template <int DIM, int N, int Q, bool NTM>
__global__ void __launch_bounds__(ELEM_NT) diag2_kernel(const ElemArgs a, const __grid_constant__ Tab t) {
  using DC = DiagCfg<DIM, N, Q>;
  constexpr int QP = DC::QP, NP = DC::NP, EPB = DC::EPB, NF = DC::NF, NPAIR = DC::NPAIR;
  constexpr int QS = Cfg<DIM, N, Q>::QS;
  extern __shared__ __align__(16) double smem[];
  double *PT = smem;                       // [sel][q][k], sel: 0 = BB, 1 = BG, 2 = GG
  double *RA = smem + DC::PT;
  double *RB = RA + EPB * DC::RA;
  for (int i = threadIdx.x; i < Q * N; i += ELEM_NT) {
    const double b = t.B[i], g = t.G[i];
    PT[i] = b * b;
    PT[Q * N + i] = b * g;
    PT[2 * Q * N + i] = g * g;
  }
  __syncthreads();

  for (int64_t grp = blockIdx.x; grp < a.ngroups; grp += gridDim.x) {
    const int64_t e0 = grp * EPB;
    // ---- point stage: Hpair[c*NPAIR + f][q]
    for (int w = threadIdx.x; w < EPB * QP; w += ELEM_NT) {
      const int e = w / QP, q = w % QP;
      const int64_t eg = e0 + e;
      double *hp = RA + e * DC::RA + q;
      if (eg >= a.ne) {
#pragma unroll
        for (int f = 0; f < NF; ++f) hp[f * QP] = 0.0;
        continue;
      }
      double T[DIM][DIM], S[DIM][DIM], k0, itau;
      lean_load<DIM>(a.qdata + eg * QS + lean_slot<DIM, Q>(q), QP, T, S, k0, itau);
      if constexpr (!NTM) {
        double c[4];
        lean_coeffs(a.metric, k0, itau, mfro2<DIM>(T), c);
        const double c23 = c[2] + c[3];
#pragma unroll
        for (int cc = 0; cc < DIM; ++cc)
#pragma unroll
          for (int f = 0; f < NPAIR; ++f) {
            int n, p;
            pair_np<DIM>(f, n, p);
            const double sn = S[cc][n], sp = S[cc][p], tn = T[cc][n], tp = T[cc][p];
            double v = c[1] * (sn * tp + tn * sp) + c23 * sn * sp;
            if (n == p)
              v += c[0];
            else
              v *= 2.0;
            hp[(cc * NPAIR + f) * QP] = v;
          }
      } else {
#pragma unroll
        for (int cc = 0; cc < DIM; ++cc)
#pragma unroll
          for (int p = 0; p < DIM; ++p) {
            double g[DIM][DIM] = {}, z[DIM][DIM];
            g[cc][p] = 1.0;
            nt_hess<DIM>(a.metric, k0, S, T, g, z);   // column (c,p) of the block: z[c][n] = H[(c,n),(c,p)]
#pragma unroll
            for (int f = 0; f < NPAIR; ++f) {
              int n, pp;
              pair_np<DIM>(f, n, pp);
              if (pp == p) hp[(cc * NPAIR + f) * QP] = (n == p) ? z[cc][n] : 2.0 * z[cc][n];
            }
          }
      }
    }
    __syncthreads();
    // ---- x-sweep: RA [f][.., qy][qx] -> RB [f][.., qy][kx]
    constexpr int XL = DIM == 3 ? Q * Q : Q;   // x-lines per field
    for (int w = threadIdx.x; w < EPB * NF * XL; w += ELEM_NT) {
      const int e = w / (NF * XL), r = w % (NF * XL), fc = r / XL, line = r % XL;
      int n, p;
      pair_np<DIM>(fc % NPAIR, n, p);
      const double *tab = PT + ((n == 0) + (p == 0)) * Q * N;
      const double *z = RA + e * DC::RA + fc * QP + line * Q;
      double zv[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) zv[q] = z[q];
      double *o = RB + e * DC::RB + (fc * XL + line) * N;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) s += tab[q * N + k] * zv[q];
        o[k] = s;
      }
    }
    __syncthreads();
    if constexpr (DIM == 3) {
      // ---- y-sweep: RB [f][qz][qy][kx] -> RA [f][qz][ky][kx]
      for (int w = threadIdx.x; w < EPB * NF * Q * N; w += ELEM_NT) {
        const int e = w / (NF * Q * N), r = w % (NF * Q * N), fc = r / (Q * N), r2 = r % (Q * N), qz = r2 / N,
                  kx = r2 % N;
        int n, p;
        pair_np<DIM>(fc % NPAIR, n, p);
        const double *tab = PT + ((n == 1) + (p == 1)) * Q * N;
        const double *z = RB + e * DC::RB + (fc * Q + qz) * Q * N + kx;
        double zv[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) zv[q] = z[q * N];
        double *o = RA + e * DC::RA + (fc * Q + qz) * N * N + kx;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < Q; ++q) s += tab[q * N + k] * zv[q];
          o[k * N] = s;
        }
      }
      __syncthreads();
      // ---- z-sweep + pair sum: RA [c*NPAIR+f][qz][ky][kx] -> E[e][c][kz][ky][kx]
      for (int w = threadIdx.x; w < EPB * 3 * N * N; w += ELEM_NT) {
        const int e = w / (3 * N * N), r = w % (3 * N * N), c = r / (N * N), kk = r % (N * N);
        if (e0 + e >= a.ne) continue;
        double acc[N];
#pragma unroll
        for (int k = 0; k < N; ++k) acc[k] = 0.0;
#pragma unroll
        for (int f = 0; f < NPAIR; ++f) {
          int n, p;
          pair_np<DIM>(f, n, p);
          const double *tab = PT + ((n == 2) + (p == 2)) * Q * N;
          const double *z = RA + e * DC::RA + (c * NPAIR + f) * Q * N * N + kk;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const double zq = z[q * N * N];
#pragma unroll
            for (int k = 0; k < N; ++k) acc[k] += tab[q * N + k] * zq;
          }
        }
        double *o = a.E + ((e0 + e) * 3 + c) * NP + kk;
#pragma unroll
        for (int k = 0; k < N; ++k) o[k * N * N] = acc[k];
      }
    } else {
      // ---- y-sweep + pair sum: RB [c*NPAIR+f][qy][kx] -> E[e][c][ky][kx]
      for (int w = threadIdx.x; w < EPB * 2 * N; w += ELEM_NT) {
        const int e = w / (2 * N), r = w % (2 * N), c = r / N, kx = r % N;
        if (e0 + e >= a.ne) continue;
        double acc[N];
#pragma unroll
        for (int k = 0; k < N; ++k) acc[k] = 0.0;
#pragma unroll
        for (int f = 0; f < NPAIR; ++f) {
          int n, p;
          pair_np<DIM>(f, n, p);
          const double *tab = PT + ((n == 1) + (p == 1)) * Q * N;
          const double *z = RB + e * DC::RB + (c * NPAIR + f) * Q * N + kx;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const double zq = z[q * N];
#pragma unroll
            for (int k = 0; k < N; ++k) acc[k] += tab[q * N + k] * zq;
          }
        }
        double *o = a.E + ((e0 + e) * 2 + c) * NP + kx;
#pragma unroll
        for (int k = 0; k < N; ++k) o[k * N] = acc[k];
      }
    }
    __syncthreads();
  }
}

}  // namespace tmop
