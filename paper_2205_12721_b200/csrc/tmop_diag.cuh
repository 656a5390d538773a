// tmop_diag.cuh -- exact diagonal of the partially assembled Hessian
// (AssembleGradDiagonalPA; reference hessian_diagonal, operator.py:420-459).
//
//   diag[(c,i)] = sum_q sum_{n,p} D_n(q,i) H[(c,n),(c,p)](q) D_p(q,i)
//
// with D_n(q,i) D_p(q,i) = prod_axis (M_n,axis .* M_p,axis)[q_a, i_a] and
// M = G on the differentiated axis, B elsewhere (operator.py:443-448).  The
// summand is symmetric in (n, p), so only the d(d+1)/2 unique pairs are
// formed (off-diagonal pairs doubled).  Per element group:
//   point    H-pair values of every (component, pair) from the lean record,
//            stored in the record's slot order (coalesced global reads,
//            conflict-free shared writes)
//   x^T      one work item per (element, component, x-line), all pairs
//            unrolled: the per-pair axis table (BB / BG / GG) is a
//            compile-time choice, read from the constant bank (Tab::P)
//   y^T      per (element, component, qz, kx), all pairs; pairs sharing the
//            same z table are summed here (6 -> 3 fields per component in
//            3D; 2D sums all pairs and writes the E-vector)
//   z^T      per (element, component, ky, kx) -> element-blocked E-vector
// The E-vector is summed to nodes by e2l_kernel (mode 2: constrained -> 1).
#pragma once

#include "tmop_elem.cuh"

namespace tmop {

template <int DIM>
struct Pairs {
  static constexpr int NPAIR = DIM * (DIM + 1) / 2;
  // pair index -> (n, p), n <= p: diagonal pairs first
  __host__ __device__ static constexpr int n(int f) {
    return DIM == 2 ? (f == 2 ? 0 : f) : (f < 3 ? f : (f == 5 ? 1 : 0));
  }
  __host__ __device__ static constexpr int p(int f) {
    return DIM == 2 ? (f == 2 ? 1 : f) : (f < 3 ? f : (f == 3 ? 1 : 2));
  }
  // product table of pair f along axis a: 0 = B.B, 1 = B.G, 2 = G.G
  __host__ __device__ static constexpr int sel(int a, int f) { return (n(f) == a) + (p(f) == a); }
  // 3D: z-table groups (pairs with equal z table are summed after the y sweep)
  __host__ __device__ static constexpr int zgroup(int f) { return sel(2, f); }
};

// Shared doubles per CTA; 0 = per-order default, measured in round 1
// (p=1,2: 8 K; p=3: 12 K; p=4: 16 K -- tools/build_variant.sh A/B).
#ifndef TMOP_DIAG_BUDGET
#define TMOP_DIAG_BUDGET 0
#endif

template <int DIM, int N, int Q>
struct DiagCfg {
  static constexpr int NPAIR = Pairs<DIM>::NPAIR;
  static constexpr int NF = DIM * NPAIR;                      // (component, pair) fields
  static constexpr int QP = ipow(Q, DIM), NP = ipow(N, DIM);
  static constexpr int XL = DIM == 3 ? Q * Q : Q;             // x-lines per field
  static constexpr int XLS = N | 1;                           // x^T output line stride (odd)
  static constexpr int RA = DIM == 3 ? cmax(NF * QP, DIM * 3 * Q * N * N) : NF * QP;   // points / y^T out
  static constexpr int RB = NF * XL * XLS;                                           // x^T out
  static constexpr int PER = RA + RB;
  static constexpr int BUDGET = TMOP_DIAG_BUDGET ? TMOP_DIAG_BUDGET : (N <= 3 ? 8192 : N == 4 ? 12288 : 16384);
  static constexpr int EPB = cclamp(BUDGET / PER, 1, 32);
  static constexpr int SMEM = EPB * PER * 8;
};

template <int Q, int N>
__device__ __forceinline__ double tP(const Tab &t, int sel, int q, int k) { return t.P[sel][q * N + k]; }

template <int DIM, int N, int Q, bool NTM>
__global__ void __launch_bounds__(ELEM_NT) diag2_kernel(const ElemArgs a, const __grid_constant__ Tab t) {
  using DC = DiagCfg<DIM, N, Q>;
  using PR = Pairs<DIM>;
  constexpr int QP = DC::QP, NP = DC::NP, EPB = DC::EPB, NF = DC::NF, NPAIR = DC::NPAIR, XL = DC::XL,
                XLS = DC::XLS;
  constexpr int QS = Cfg<DIM, N, Q>::QS;
  extern __shared__ __align__(16) double smem[];
  double *RA = smem;
  double *RB = RA + EPB * DC::RA;

  // Lean point records of the NEXT group are loaded into registers while the
  // current group runs its sweeps (one or two points per thread), so the
  // point stage never waits on DRAM latency.
  constexpr int PTS = (EPB * QP + ELEM_NT - 1) / ELEM_NT, LW = DIM * DIM + 2;
  double qn[PTS][LW];
  auto fetch = [&](int64_t g) {
#pragma unroll
    for (int j = 0; j < PTS; ++j) {
      const int w = threadIdx.x + j * ELEM_NT;
      const int64_t eg = g * EPB + w / QP;
      if (w < EPB * QP && g < a.ngroups && eg < a.ne) {
        const double *q = a.qdata + eg * QS + w % QP;
#pragma unroll
        for (int k = 0; k < LW; ++k) qn[j][k] = __ldg(q + k * QP);
      }
    }
  };
  fetch(blockIdx.x);
  for (int64_t grp = blockIdx.x; grp < a.ngroups; grp += gridDim.x) {
    const int64_t e0 = grp * EPB;
    // ---- point stage: Hpair[c*NPAIR + f][slot]
#pragma unroll
    for (int j = 0; j < PTS; ++j) {
      const int w = threadIdx.x + j * ELEM_NT;
      if (w >= EPB * QP) break;
      const int e = w / QP, slot = w % QP;
      const int64_t eg = e0 + e;
      double *hp = RA + e * DC::RA + slot;
      if (eg >= a.ne) {
#pragma unroll
        for (int f = 0; f < NF; ++f) hp[f * QP] = 0.0;
        continue;
      }
      double T[DIM][DIM], S[DIM][DIM], C[DIM][DIM], k0 = qn[j][DIM * DIM], itau = qn[j][DIM * DIM + 1];
#pragma unroll
      for (int r = 0; r < DIM; ++r)
#pragma unroll
        for (int cc = 0; cc < DIM; ++cc) T[r][cc] = qn[j][r * DIM + cc];
      mcof<DIM>(T, C);
#pragma unroll
      for (int r = 0; r < DIM; ++r)
#pragma unroll
        for (int cc = 0; cc < DIM; ++cc) S[r][cc] = C[r][cc] * itau;
      if constexpr (!NTM) {
        // regrouped as in xld_line (tmop_xld_parts.cuh): S_n u'_p + S_p u'_n,
        // u'_k = 2 c1 T_k + (c2 + c3) S_k
        double c[4];
        lean_coeffs(a.metric, k0, itau, mfro2<DIM>(T), c);
        const double c1x2 = 2.0 * c[1], c23 = c[2] + c[3];
#pragma unroll
        for (int cc = 0; cc < DIM; ++cc) {
          double u[DIM];
#pragma unroll
          for (int k = 0; k < DIM; ++k) u[k] = c1x2 * T[cc][k] + c23 * S[cc][k];
#pragma unroll
          for (int f = 0; f < NPAIR; ++f) {
            const int n = PR::n(f), p = PR::p(f);
            hp[(cc * NPAIR + f) * QP] = (n == p) ? S[cc][n] * u[n] + c[0] : S[cc][n] * u[p] + S[cc][p] * u[n];
          }
        }
      } else {
        const NtDiag<DIM> nd(S, T);             // column (c,p): z[n] = H[(c,n),(c,p)] (unit-direction nt_hess)
#pragma unroll
        for (int cc = 0; cc < DIM; ++cc)
#pragma unroll
          for (int p = 0; p < DIM; ++p) {
            double z[DIM];
            nd.col(a.metric, k0, S, T, cc, p, z);
#pragma unroll
            for (int f = 0; f < NPAIR; ++f) {
              const int n = PR::n(f), pp = PR::p(f);
              if (pp == p) hp[(cc * NPAIR + f) * QP] = (n == p) ? z[n] : 2.0 * z[n];
            }
          }
      }
    }
    __syncthreads();
    fetch(grp + gridDim.x);
    // ---- x^T: RA [c*NPAIR+f][slot] -> RB [c*NPAIR+f][line][kx]
    for (int w = threadIdx.x; w < EPB * DIM * XL; w += ELEM_NT) {
      const int e = w / (DIM * XL), r = w % (DIM * XL), c = r / XL, line = r % XL;
#pragma unroll
      for (int f = 0; f < NPAIR; ++f) {
        const int fc = c * NPAIR + f;
        // 3D slots: line + XL qx (qx slowest); 2D slots are the point index qx + Q qy
        const double *z = RA + e * DC::RA + fc * QP + (DIM == 3 ? line : line * Q);
        double zv[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) zv[q] = z[q * (DIM == 3 ? XL : 1)];
        double *o = RB + e * DC::RB + (fc * XL + line) * XLS;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < Q; ++q) s += tP<Q, N>(t, PR::sel(0, f), q, k) * zv[q];
          o[k] = s;
        }
      }
    }
    __syncthreads();
    if constexpr (DIM == 3) {
      // ---- y^T + z-group sum: RB [c*6+f][qz*Q+qy][kx] -> RA [c][g][qz][ky][kx]
      for (int w = threadIdx.x; w < EPB * 3 * Q * N; w += ELEM_NT) {
        const int e = w / (3 * Q * N), r = w % (3 * Q * N), c = r / (Q * N), r2 = r % (Q * N), qz = r2 / N,
                  kx = r2 % N;
        double acc[3][N];
#pragma unroll
        for (int g = 0; g < 3; ++g)
#pragma unroll
          for (int k = 0; k < N; ++k) acc[g][k] = 0.0;
#pragma unroll
        for (int f = 0; f < NPAIR; ++f) {
          const double *z = RB + e * DC::RB + ((c * NPAIR + f) * XL + qz * Q) * XLS + kx;
          double zv[Q];
#pragma unroll
          for (int q = 0; q < Q; ++q) zv[q] = z[q * XLS];
#pragma unroll
          for (int k = 0; k < N; ++k) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < Q; ++q) s += tP<Q, N>(t, PR::sel(1, f), q, k) * zv[q];
            acc[PR::zgroup(f)][k] += s;
          }
        }
#pragma unroll
        for (int g = 0; g < 3; ++g) {
          double *o = RA + e * DC::RA + ((c * 3 + g) * Q + qz) * N * N + kx;
#pragma unroll
          for (int k = 0; k < N; ++k) o[k * N] = acc[g][k];
        }
      }
      __syncthreads();
      // ---- z^T: RA [c][g][qz][ky][kx] -> E[e][c][kz][ky][kx]
      for (int w = threadIdx.x; w < EPB * 3 * N * N; w += ELEM_NT) {
        const int e = w / (3 * N * N), r = w % (3 * N * N), c = r / (N * N), kk = r % (N * N);
        if (e0 + e >= a.ne) continue;
        double acc[N];
#pragma unroll
        for (int k = 0; k < N; ++k) acc[k] = 0.0;
#pragma unroll
        for (int g = 0; g < 3; ++g) {
          const double *z = RA + e * DC::RA + (c * 3 + g) * Q * N * N + kk;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const double zq = z[q * N * N];
#pragma unroll
            for (int k = 0; k < N; ++k) acc[k] += tP<Q, N>(t, g, q, k) * zq;
          }
        }
        double *o = a.E + ((e0 + e) * 3 + c) * NP + kk;
#pragma unroll
        for (int k = 0; k < N; ++k) o[k * N * N] = acc[k];
      }
    } else {
      // ---- y^T + pair sum: RB [c*3+f][qy][kx] -> E[e][c][ky][kx]
      for (int w = threadIdx.x; w < EPB * 2 * N; w += ELEM_NT) {
        const int e = w / (2 * N), r = w % (2 * N), c = r / N, kx = r % N;
        if (e0 + e >= a.ne) continue;
        double acc[N];
#pragma unroll
        for (int k = 0; k < N; ++k) acc[k] = 0.0;
#pragma unroll
        for (int f = 0; f < NPAIR; ++f) {
          const double *z = RB + e * DC::RB + (c * NPAIR + f) * XL * XLS + kx;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const double zq = z[q * XLS];
#pragma unroll
            for (int k = 0; k < N; ++k) acc[k] += tP<Q, N>(t, PR::sel(1, f), q, k) * zq;
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
