// tmop_apply_col.cuh -- the 3D Hessian-action kernel (AddMultGradPA,
// operator.py:401-418) in "column" form.
//
// Every element gets a Q x Q tile of threads; thread (tx, ty) owns the
// quadrature column (qx = tx, qy = ty, qz = 0..Q-1) and keeps the nine
// gradient fields g[c][d][qz] in registers from the x-sweep through the
// point stage into the transposed x-sweep.  The z- and y-sweeps go through
// shared memory one component at a time, so the per-element work buffers
// stay small and most of the shared memory holds the element group's lean
// Q-data, streamed in by a TMA bulk copy one group ahead.  All shared
// offsets are compile-time constants plus a per-thread base computed once;
// thread-dependent basis rows/columns come from the constant bank (Tab).
//
//   forward (per component c):  gather (z-columns, prefetched one group
//     ahead into registers)  -z->  U(B,G) [smem]  -y->  W(BB,BG,GB) [smem]
//     -x->  g[c][*][qz] [registers]
//   point:  z = H(T, k0, itau) g per point, Q-data from the TMA stage
//   backward (per component c):  g -> Z [smem]  -x^T->  A [smem]  -y^T->
//     Bv [smem]  -z^T->  element-blocked E-vector (global)
#pragma once

#include "tmop_elem.cuh"

namespace tmop {

template <int N, int Q>
struct ColCfg {
  static constexpr int TPE = Q * Q;                    // threads per element
  static constexpr int NL = N | 1, QL = Q | 1;         // odd line strides (bank-conflict free)
  static constexpr int NP = N * N * N, QP = Q * Q * Q;
  static constexpr int F = 11;                         // lean fields: T (9), k0, itau
  static constexpr int QS = (F * QP + 1) & ~1;         // element stride of the Q-data
  static constexpr int P1 = 3 * Q * Q * NL;            // W_c / A_c (one component)
  static constexpr int P2 = cmax(2 * Q * N * N, 3 * Q * Q * QL);  // U_c / Z_c / Bv_c
  static constexpr int PERE = QS + ((P1 + P2 + 1) & ~1);
  // elements per CTA: ~128 threads, at most ~72 KB of shared memory
  static constexpr int E0 = cmax(1, 128 / TPE);
  static constexpr int E = cmax(1, (E0 * PERE * 8 > 73728) ? 73728 / (PERE * 8) : E0);
  static constexpr int NT = E * TPE;
  static constexpr int SMEM = E * PERE * 8;
};

template <int N, int Q>
__host__ __device__ constexpr bool col_supported() {
  return Q <= 6;   // nine Q-long register columns: Q <= 6 keeps it under ~168 registers
}

template <int N, int Q, bool NTM>
__global__ void __launch_bounds__(ColCfg<N, Q>::NT, cmax(1, 384 / ColCfg<N, Q>::NT)) apply_col_kernel(const ElemArgs a,
                                                                      const __grid_constant__ Tab t) {
  using CC = ColCfg<N, Q>;
  constexpr int E = CC::E, TPE = CC::TPE, NL = CC::NL, QL = CC::QL, QS = CC::QS, QP = CC::QP;
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t qbar;

  const int tid = threadIdx.x;
  const int el = tid / TPE;          // element slot in the group
  const int tx = tid % Q;
  const int ty = (tid / Q) % Q;
  double *QB = smem;                                       // [E][QS] staged lean Q-data
  double *P1 = smem + E * QS + el * (CC::PERE - QS);       // this element's W / A
  double *P2 = P1 + CC::P1;                                // this element's U / Z / Bv
  const double *qb = QB + el * QS + ty * Q + tx;           // field 0 of point (tx, ty, qz = 0)

  auto issue = [&](int64_t grp) {
    const int64_t e0 = grp * E;
    const int64_t cnt = (a.ne - e0) < E ? (a.ne - e0) : E;
    const uint32_t bytes = (uint32_t)(cnt * QS * 8);
    mbar_expect_tx(&qbar, bytes);
    tma_load_1d(QB, a.qdata + e0 * QS, bytes, &qbar);
  };

  // z-column of the gathered direction v for (kx, ky) = (tx, ty), all three
  // components, loaded one group ahead
  const bool colthr = (tx < N) && (ty < N);
  double xv[3][N];
  auto gather_col = [&](int64_t grp) {
    const int64_t eg = grp * E + el;
    if (colthr && eg < a.ne) {
      const int32_t *rr = a.restr + eg * CC::NP + ty * N + tx;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const int node = __ldg(rr + k * N * N);
        const uint8_t f = __ldg(a.fixed + node);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double val = __ldg(a.in + c * a.nn + node);
          xv[c][k] = ((f >> c) & 1) ? 0.0 : val;
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < N; ++k) xv[c][k] = 0.0;
    }
  };

  if (tid == 0) {
    mbar_init(&qbar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0 && (int64_t)blockIdx.x < a.ngroups) issue(blockIdx.x);
  uint32_t phase = 0;
  if ((int64_t)blockIdx.x < a.ngroups) gather_col(blockIdx.x);

  for (int64_t grp = blockIdx.x; grp < a.ngroups; grp += gridDim.x) {
    const int64_t eg = grp * E + el;
    double g[3][3][Q];

    // ------------------------------------------------------------ forward
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      // z-sweep: U_B / U_G [qz][ky][kx]
      if (colthr) {
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) {
          double sb = 0.0, sg = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            sb += tB<Q, N>(t, qz, k) * xv[c][k];
            sg += tG<Q, N>(t, qz, k) * xv[c][k];
          }
          P2[(qz * N + ty) * N + tx] = sb;
          P2[Q * N * N + (qz * N + ty) * N + tx] = sg;
        }
      }
      __syncthreads();
      // y-sweep: (kx = tx < N, qy = ty) -> W_BB / W_BG / W_GB [qz][qy][kx]
      if (tx < N) {
        double by[N], gy[N];
#pragma unroll
        for (int k = 0; k < N; ++k) { by[k] = t.B[ty * N + k]; gy[k] = t.G[ty * N + k]; }
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            const double ub = P2[(qz * N + k) * N + tx], ug = P2[Q * N * N + (qz * N + k) * N + tx];
            s0 += by[k] * ub;
            s1 += gy[k] * ub;
            s2 += by[k] * ug;
          }
          P1[(qz * Q + ty) * NL + tx] = s0;
          P1[Q * Q * NL + (qz * Q + ty) * NL + tx] = s1;
          P1[2 * Q * Q * NL + (qz * Q + ty) * NL + tx] = s2;
        }
      }
      __syncthreads();
      // x-sweep: (qx = tx, qy = ty) -> g[c][d][qz] in registers
      {
        double bx[N], gx[N];
#pragma unroll
        for (int k = 0; k < N; ++k) { bx[k] = t.B[tx * N + k]; gx[k] = t.G[tx * N + k]; }
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            const int o = (qz * Q + ty) * NL + k;
            s0 += gx[k] * P1[o];
            s1 += bx[k] * P1[Q * Q * NL + o];
            s2 += bx[k] * P1[2 * Q * Q * NL + o];
          }
          g[c][0][qz] = s0;
          g[c][1][qz] = s1;
          g[c][2][qz] = s2;
        }
      }
    }

    // ---------------------------------------------------------- point stage
    mbar_wait(&qbar, phase);
    phase ^= 1u;
    if (eg < a.ne) {
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) {
        double A[3][3], z[3][3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = 0; d < 3; ++d) A[c][d] = g[c][d][qz];
        lean_hess<3, NTM>(a.metric, qb + qz * Q * Q, QP, A, z);
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = 0; d < 3; ++d) g[c][d][qz] = z[c][d];
      }
    }
    // prefetch the next group's direction columns while the sweeps run
    const int64_t nxt = grp + gridDim.x;
    if (nxt < a.ngroups) gather_col(nxt);
    __syncthreads();   // staged Q-data consumed (and P1/P2 free)
    if (tid == 0 && nxt < a.ngroups) issue(nxt);

    // ----------------------------------------------------------- backward
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      // Z_c[d][qz][qy][qx] <- g[c][d][qz]
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) P2[(d * Q * Q + qz * Q + ty) * QL + tx] = g[c][d][qz];
      __syncthreads();
      // x^T: (kx = tx < N, qy = ty): A0 = Gx^T z0, A1 = Bx^T z1, A2 = Bx^T z2
      if (tx < N) {
        double bc[Q], gc[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) { bc[q] = t.B[q * N + tx]; gc[q] = t.G[q * N + tx]; }
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const int o = (qz * Q + ty) * QL + q;
            s0 += gc[q] * P2[o];
            s1 += bc[q] * P2[Q * Q * QL + o];
            s2 += bc[q] * P2[2 * Q * Q * QL + o];
          }
          P1[(qz * Q + ty) * NL + tx] = s0;
          P1[Q * Q * NL + (qz * Q + ty) * NL + tx] = s1;
          P1[2 * Q * Q * NL + (qz * Q + ty) * NL + tx] = s2;
        }
      }
      __syncthreads();
      // y^T: (kx = tx < N, ky = ty < N): b0 = By^T A0 + Gy^T A1, b1 = By^T A2
      if (colthr) {
        double bc[Q], gc[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) { bc[q] = t.B[q * N + ty]; gc[q] = t.G[q * N + ty]; }
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) {
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const int o = (qz * Q + q) * NL + tx;
            s0 += bc[q] * P1[o] + gc[q] * P1[Q * Q * NL + o];
            s1 += bc[q] * P1[2 * Q * Q * NL + o];
          }
          P2[(qz * N + ty) * N + tx] = s0;
          P2[Q * N * N + (qz * N + ty) * N + tx] = s1;
        }
      }
      __syncthreads();
      // z^T: E[eg][c][kz][ky][kx] = Bz^T b0 + Gz^T b1
      if (colthr && eg < a.ne) {
        double b0[Q], b1[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          b0[q] = P2[(q * N + ty) * N + tx];
          b1[q] = P2[Q * N * N + (q * N + ty) * N + tx];
        }
        double *out = a.E + (eg * 3 + c) * CC::NP + ty * N + tx;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < Q; ++q) s += tB<Q, N>(t, q, k) * b0[q] + tG<Q, N>(t, q, k) * b1[q];
          out[k * N * N] = s;
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace tmop
