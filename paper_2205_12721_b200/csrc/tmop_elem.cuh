// tmop_elem.cuh -- element kernels of the TMOP operator (one template for
// every per-element entry point, specialised by KIND at compile time).
//
// A CTA owns EPB elements at a time and walks element groups with a
// grid-stride loop (grid = min(#groups, GRID_CAP): a fixed function of the
// mesh size, so every reduction below is bitwise reproducible run to run).
// Per group:
//   gather   restriction -> shared memory (coalesced index reads; nodal
//            values come through L2, neighbours share nodes)
//   forward  3 (2D: 2) sum-factorised 1D sweeps, B/G from the constant bank,
//            z axis first like contract_dofs_to_quad (fe.py:227-239):
//            X --z--> U(B,G) --y--> W(BB,BG,GB) --x--> grad[c][dir] at points
//   point    KIND-specific quadrature-point work (setup / Hessian block /
//            first derivative / energy / det)
//   backward the transposed sweeps (fe.py:242-253), x axis first, with the
//            three direction terms summed inside the sweeps, written as an
//            element-blocked E-vector E[e][c][local]
// The E-vector is summed to nodes by e2l_kernel in ascending element
// order (np.add.at order, fe.py:189-204) -- no atomics anywhere.
#pragma once

#include <cfloat>
#include <climits>

#include "tmop_device.cuh"
#include "tmop_elem_pad.h"

namespace tmop {

enum Kind : int {
  K_SETUP = 0,    // hessian_setup        (operator.py:350-371)
  K_APPLY = 1,    // hessian_apply        (operator.py:401-418)
  K_GRAD = 2,     // gradient             (operator.py:328-346)
  K_ENERGY = 3,   // objective            (operator.py:311-326)
  K_MINDET = 4,   // min_det_jacobian     (operator.py:296-304)
  K_ELEMDET = 5,  // per-element min det  (operator.py:267-272 diagnostics)
  K_VOLUME = 6,   // mesh_volume          (metrics.py:319-330)
  K_DIAG = 7,     // hessian_diagonal     (operator.py:420-459)
  K_APPLY_NT = 8, // hessian_apply, non-template metrics (mu_302 / mu_321)
  K_DIAG_NT = 9,  // hessian_diagonal, non-template metrics
  K_LIM_VALUE = 10,  // limiting_value        (operator.py:488-495)
  K_LIM_FIELD = 11,  // limiting gradient / Hessian action (operator.py:497-533)
  K_LIM_DIAG = 12,   // limiting part of hessian_diagonal (operator.py:452-457)
  K_TSCALE = 13,     // size-field targets: per-point 1/scale from a nodal target volume (extension)
  K_SETUP_DIAG = 14, // hessian_setup + hessian_diagonal from one element pass (3D p <= 3, template metrics)
  K_COUNT = 15
};

// Tuning knobs (compile-time overrides for tools/build_variant.sh; 0 = the
// per-order defaults in Cfg): threads per CTA, shared-memory budget per CTA
// in doubles, and the occupancy hint.
#ifndef TMOP_ELEM_NT
#define TMOP_ELEM_NT 0
#endif
#ifndef TMOP_SMEM_BUDGET
#define TMOP_SMEM_BUDGET 0
#endif
#ifndef TMOP_WIDE_LDG
#define TMOP_WIDE_LDG 1
#endif
#ifndef TMOP_WIDE_MINB
#define TMOP_WIDE_MINB 2
#endif
#ifndef TMOP_MIN_BLOCKS
#define TMOP_MIN_BLOCKS 0
#endif
constexpr int GRID_CAP = 148 * 8;
constexpr int ELEM_NT = 256;   // diagonal kernel

__host__ __device__ constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int cclamp(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Element-group size of the 3D x-line kernels (tmop_xl.cuh): 16 elements per
// CTA for p = 1 (9 lines per element: 144 threads), 8 for p = 2, 4 for
// p >= 3 (shared-memory budget).
__host__ __device__ constexpr int xl_epb(int n1) { return n1 <= 2 ? 16 : (n1 == 3 ? 8 : 4); }

// Element stride of the lean Q-data record (doubles): the smallest value
// >= fields * points with stride == 16 / epb (mod 16) (2 for epb = 16).
// Even, so every element block is 16-byte aligned (TMA bulk copies), and
// with that residue the epb element-interleaved threads of a half-warp
// reading the same field / slot of consecutive staged elements hit distinct
// bank pairs (2-way for epb = 16, where an odd stride would break the TMA
// alignment).
__host__ __device__ constexpr int lean_stride(int n, int epb) {
  return n + ((16 + (epb >= 16 ? 2 : 16 / epb) - n % 16) % 16);
}

template <int DIM, int N, int Q>
struct Cfg {
  static constexpr int NP = ipow(N, DIM);
  static constexpr int QP = ipow(Q, DIM);
  // x-lines of the W/A (length N) and grad/z (length Q) buffers are padded to
  // an odd number of doubles: a half-warp walking consecutive lines then hits
  // 16 distinct bank pairs (even strides caused 2- to 8-way conflicts).
  static constexpr int NL = N | 1;
  // grad / z x-lines: odd Q unpadded (odd strides are conflict-free); Q a
  // power of two unpadded but XOR-swizzled (slot x of line l holds point
  // x ^ ((l / (16/Q)) mod Q)), which keeps both the x-sweep writes (one line per
  // thread) and the point-stage reads (one point per thread) conflict-free;
  // other even Q (6) padded to Q + 1.
  static constexpr bool SWZ = (Q & (Q - 1)) == 0 && Q <= 16;
  static constexpr int QL = (Q & 1) || SWZ ? Q : Q + 1;
  __device__ __forceinline__ static int gs(int l, int x) {
    if constexpr (SWZ) {
      return l * Q + (x ^ ((l / (16 / Q)) & (Q - 1)));
    } else {
      return l * QL + x;
    }
  }
  static constexpr int WF = Q * Q * NL;                       // one (c, variant) block of W / A (2D layout)
  // 3D sweep buffers (strides from tools/elem_banks.py, tmop_elem_pad.h)
  using PAD = ElemPad<N, Q>;
  static constexpr int UZ = PAD::UZ, UV = PAD::UV, UC = PAD::UC;
  static constexpr int WY = PAD::WY, WZ = PAD::WZ, WV = PAD::WV, WC = PAD::WC;
  static constexpr int GF = DIM == 3 ? Q * Q * QL : Q * QL;   // one field of grad / z
  // 3D: R1 holds X / W / A (and det scratch); R2 holds U / grad+z / Bv.
  // 2D: R1 holds X / grad+z (and diag x-sweep); R2 holds U / A (and diag points).
  static constexpr int R1 =
      DIM == 3 ? cmax(cmax(3 * NP, 2 * WC + 3 * WV), cmax(QP, GF)) : cmax(cmax(2 * NP, 4 * GF), 2 * Q * N);
  static constexpr int R2 = DIM == 3 ? cmax(2 * UC + 2 * UV, 9 * GF) : cmax(4 * Q * NL, 2 * QP);
  static constexpr int PER = R1 + R2;
  // lean Q-data: T (d*d), k0, itau per point; element stride rounded to an
  // even number of doubles so every element block is 16-byte aligned (TMA).
  static constexpr int F = DIM * DIM + 2;
  static constexpr int QS = lean_stride(F * QP, xl_epb(N));
  // Launch shape, from the A/B sweep of round 1 (profiles/round1_apply_ab.md):
  // 128-thread CTAs with ~56 KB (4 CTAs / SM) for p = 1, 2, 4; 256-thread
  // CTAs with ~72 KB (3 CTAs / SM) for p = 3.
  // 256-thread CTAs for n_q >= 7 (one element's Q-data + work arrays fill the
  // CTA's shared memory; measured 1.4-1.8x faster at n_q = 9, round 1)
  static constexpr bool WIDE = Q >= 7;
  static constexpr int NT = TMOP_ELEM_NT ? TMOP_ELEM_NT : (WIDE ? 256 : 128);
  // n_q >= 7 Hessian action: the point stage reads its Q-data straight from
  // HBM (unit stride in slot order) instead of staging a 64 KB element block,
  // which halves the CTA's shared memory and doubles the resident CTAs
  static constexpr bool QLDG = WIDE && TMOP_WIDE_LDG;
  static constexpr int MINB = TMOP_MIN_BLOCKS ? TMOP_MIN_BLOCKS : (WIDE ? (QLDG ? TMOP_WIDE_MINB : 1) : 4);
  // n_q >= 7: the work arrays (~70-82 KB) allow 2-3 CTAs / SM; the register
  // target follows (the forward-only kinds need ~80 registers)
  template <int KIND>
  static constexpr int minb() {
    return (!WIDE || TMOP_MIN_BLOCKS) ? MINB
           : KIND == K_APPLY ? MINB
           : KIND == K_APPLY_NT ? 1
           : (KIND == K_SETUP || KIND == K_GRAD || KIND == K_DIAG || KIND == K_DIAG_NT) ? 2
           : cmin(3, (227 * 1024) / (EPB * PER * 8 + 1024));
  }
  static constexpr int BUDGET = TMOP_SMEM_BUDGET ? TMOP_SMEM_BUDGET : (WIDE ? 9216 : 7168);
  // elements per CTA: work arrays + staged Q-data within BUDGET doubles
  static constexpr int EPB = cclamp(BUDGET / (PER + (QLDG ? 0 : QS)), 1, 32);
  static constexpr int QOFF = (EPB * PER + 1) & ~1;          // Q-data staging offset (doubles)
  static constexpr int SMEM = EPB * PER * 8;                 // kernels without staging
  static constexpr int SMEM_TMA = QLDG ? SMEM : (QOFF + EPB * QS) * 8;   // Hessian-action kernels
};

struct ElemArgs {
  int64_t ne, nn, ngroups;
  int e_es;                           // out: log2 of the E-vector element interleave (e2l_kernel)
  const int32_t *__restrict__ restr;
  const uint8_t *__restrict__ fixed;
  const double *__restrict__ in;      // x (positions) or v (direction), T-vector
  const double *__restrict__ qdata;   // K_APPLY / K_DIAG input (lean, element stride QS)
  double *__restrict__ qout;          // K_SETUP output (lean)
  double *__restrict__ E;             // K_APPLY / K_GRAD / K_DIAG E-vector output
  double *__restrict__ part_sum;      // per-CTA partial sums (energy / volume)
  double *__restrict__ part_min;      // per-CTA partial min det
  int64_t *__restrict__ part_arg;
  double *__restrict__ elem_min;      // K_ELEMDET
  int32_t *__restrict__ elem_arg;
  int metric;
  double inv_s;       // 1 / target scale
  double inv_s_dm1;   // inv_s^(d-1)
  double inv_s_d;     // inv_s^d
  double coef_e;      // omega * det_w               (operator.py:314)
  double coef_g;      // omega * det_w * inv_s       (operator.py:330)
  double coef_h;      // omega * det_w * inv_s^2     (operator.py:358-359)
  // limiting term (tmop_lim.cuh)
  const double *__restrict__ lim_x0;   // reference positions subtracted from `in` (NULL: none)
  const double *__restrict__ lim_dn;   // nodal delta (NULL: scalar lim_delta)
  double lim_delta;
  double lim_base;    // 2 * weight * det_w  (operator.py:477)
  int lim_mask;       // zero constrained input components (hessian_apply)
  int energy;         // K_GRAD: also accumulate the energy into part_sum
  const int32_t *stop;   // if non-NULL and *stop != 0 the launch is a no-op (converged MINRES)
  // size-field targets (extension; metrics.py:282-345 has constant W only):
  // W_q = s_q I with tscale[e * QP + q] = 1 / s_q (reference point order);
  // NULL = the constant target above.  When set, the context passes
  // inv_s = det_w = 1 and the per-point factors come from PtScale.
  const double *__restrict__ tscale;
  double omega;       // spatial weight
};

// Target factors of one quadrature point (k = e * QP + q): the constant
// target's uniform values, or the size field's s_q^-1 with det W_q = s_q^d.
struct PtScale {
  double is, is_dm1, is_d, cg, ch, ew;
};
template <int DIM>
__device__ __forceinline__ PtScale pt_scale(const ElemArgs &a, int64_t k) {
  PtScale s;
  if (a.tscale == nullptr) {
    s.is = a.inv_s;
    s.is_dm1 = a.inv_s_dm1;
    s.is_d = a.inv_s_d;
    s.cg = a.coef_g;
    s.ch = a.coef_h;
    s.ew = 1.0;
    return s;
  }
  const double is = __ldg(a.tscale + k);
  s.is = is;
  s.is_dm1 = DIM == 3 ? is * is : is;
  s.is_d = s.is_dm1 * is;
  s.ew = 1.0 / s.is_d;              // det W_q (energy weight; coef_e = omega)
  s.cg = a.omega * s.ew * is;       // omega det_w inv_s   (operator.py:330)
  s.ch = s.cg * is;                 // omega det_w inv_s^2 (operator.py:358-359)
  return s;
}

// Point slot of quadrature point q (x fastest, fe.py:134-140) inside a lean
// Q-data field: 3D records store qx as the SLOWEST index (slot = line +
// Q^2 qx, line = qy + Q qz), so the x-line kernel's threads (one per line)
// read each field of one point with unit stride.  2D: identity.
template <int DIM, int Q>
__host__ __device__ __forceinline__ int lean_slot(int q) {
  if constexpr (DIM == 3) {
    return q / Q + Q * Q * (q % Q);
  } else {
    return q;
  }
}

// ------------------------------------------------------------- gather
template <int DIM, int N, int Q, int C, bool MASK>
__device__ __forceinline__ void gather(const ElemArgs &a, int64_t e0, double *R1) {
  using CF = Cfg<DIM, N, Q>;
  constexpr int NP = CF::NP, ITEMS = C * NP;
  for (int w = threadIdx.x; w < CF::EPB * ITEMS; w += CF::NT) {
    const int e = w / ITEMS, r = w % ITEMS, c = r / NP, l = r % NP;
    const int64_t eg = e0 + e;
    double val = 0.0;
    if (eg < a.ne) {
      const int node = __ldg(a.restr + eg * NP + l);
      val = __ldg(a.in + c * a.nn + node);
      if (MASK && ((__ldg(a.fixed + node) >> c) & 1)) val = 0.0;
    }
    R1[e * CF::R1 + c * NP + l] = val;
  }
}

// Register-prefetching gather (Hessian action).  Two stages so no load is
// consumed right after it is issued: the restriction indices of group g+2
// and the nodal values of group g+1 are loaded while group g's transposed
// sweeps run; values are masked and stored to shared memory at the top of
// the next iteration.
template <int DIM, int N, int Q>
struct GatherPrefetch {
  using CF = Cfg<DIM, N, Q>;
  static constexpr int ITEMS = DIM * CF::NP, TOTAL = CF::EPB * ITEMS;
  static constexpr int PER_THREAD = (TOTAL + CF::NT - 1) / CF::NT;
  int node[PER_THREAD];       // restriction of the group after next (-1: none)
  double val[PER_THREAD];     // raw v of the next group
  uint8_t fl[PER_THREAD];     // fixed flags of the next group
  __device__ __forceinline__ void load_index(const ElemArgs &a, int64_t e0) {
#pragma unroll
    for (int j = 0; j < PER_THREAD; ++j) {
      const int w = threadIdx.x + j * CF::NT;
      int nd = -1;
      if (w < TOTAL) {
        const int e = w / ITEMS, r = w % ITEMS, l = r % CF::NP;
        const int64_t eg = e0 + e;
        if (eg < a.ne) nd = __ldg(a.restr + eg * CF::NP + l);
      }
      node[j] = nd;
    }
  }
  __device__ __forceinline__ void load_values(const ElemArgs &a) {
#pragma unroll
    for (int j = 0; j < PER_THREAD; ++j) {
      const int w = threadIdx.x + j * CF::NT;
      const int c = (w % ITEMS) / CF::NP;
      if (node[j] >= 0) {
        val[j] = __ldg(a.in + c * a.nn + node[j]);
        fl[j] = __ldg(a.fixed + node[j]);
      } else {
        val[j] = 0.0;
        fl[j] = 0;
      }
    }
  }
  __device__ __forceinline__ void store(double *R1) const {
#pragma unroll
    for (int j = 0; j < PER_THREAD; ++j) {
      const int w = threadIdx.x + j * CF::NT;
      if (w < TOTAL) {
        const int e = w / ITEMS, r = w % ITEMS, c = r / CF::NP;
        R1[e * CF::R1 + r] = ((fl[j] >> c) & 1) ? 0.0 : val[j];
      }
    }
  }
};

// --------------------------------------------------------- 3D forward
// X[c][kz][ky][kx] (R1) -> U[c][v][qz][ky][kx] (R2), v in {B, G}
template <int N, int Q, int C>
__device__ __forceinline__ void f1_3d(const Tab &t, const double *R1, double *R2) {
  using CF = Cfg<3, N, Q>;
  constexpr int ITEMS = C * N * N;
  for (int w = threadIdx.x; w < CF::EPB * ITEMS; w += CF::NT) {
    const int e = w / ITEMS, r = w % ITEMS, c = r / (N * N), kk = r % (N * N);
    const double *x = R1 + e * CF::R1 + c * N * N * N + kk;
    double xv[N];
#pragma unroll
    for (int k = 0; k < N; ++k) xv[k] = x[k * N * N];
    double *u = R2 + e * CF::R2 + c * CF::UC + kk;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      double sb = 0.0, sg = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        sb += tB<Q, N>(t, q, k) * xv[k];
        sg += tG<Q, N>(t, q, k) * xv[k];
      }
      u[q * CF::UZ] = sb;
      u[CF::UV + q * CF::UZ] = sg;
    }
  }
}

// U (R2) -> W[c][v3][qz][qy][kx] (R1), v3 in {BB, BG, GB} (z-table, y-table)
template <int N, int Q, int C>
__device__ __forceinline__ void f2_3d(const Tab &t, const double *R2, double *R1) {
  using CF = Cfg<3, N, Q>;
  constexpr int ITEMS = C * Q * N;
  for (int w = threadIdx.x; w < CF::EPB * ITEMS; w += CF::NT) {
    const int e = w / ITEMS, r = w % ITEMS, c = r / (Q * N), r2 = r % (Q * N), qz = r2 / N, kx = r2 % N;
    const double *ub = R2 + e * CF::R2 + c * CF::UC + qz * CF::UZ + kx;
    const double *ug = ub + CF::UV;
    double vb[N], vg[N];
#pragma unroll
    for (int k = 0; k < N; ++k) { vb[k] = ub[k * N]; vg[k] = ug[k * N]; }
    constexpr int NL = CF::WY, WF = CF::WV;
    double *wb = R1 + e * CF::R1 + c * CF::WC + qz * CF::WZ + kx;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        s0 += tB<Q, N>(t, q, k) * vb[k];
        s1 += tG<Q, N>(t, q, k) * vb[k];
        s2 += tB<Q, N>(t, q, k) * vg[k];
      }
      wb[q * NL] = s0;
      wb[WF + q * NL] = s1;
      wb[2 * WF + q * NL] = s2;
    }
  }
}

// W (R1) -> grad[c*3+dir][qz][qy][qx] (R2); dir 0 = d/dx (G on x), 1 = d/dy, 2 = d/dz
template <int N, int Q, int C>
__device__ __forceinline__ void f3_3d(const Tab &t, const double *R1, double *R2) {
  using CF = Cfg<3, N, Q>;
  constexpr int ITEMS = C * Q * Q;
  for (int w = threadIdx.x; w < CF::EPB * ITEMS; w += CF::NT) {
    const int e = w / ITEMS, r = w % ITEMS, c = r / (Q * Q), qq = r % (Q * Q);
    constexpr int WF = CF::WV, GF = CF::GF;
    const double *wb = R1 + e * CF::R1 + c * CF::WC + (qq / Q) * CF::WZ + (qq % Q) * CF::WY;
    double bb[N], bg[N], gb[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      bb[k] = wb[k];
      bg[k] = wb[WF + k];
      gb[k] = wb[2 * WF + k];
    }
    double *g = R2 + e * CF::R2 + (c * 3) * GF;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        s0 += tG<Q, N>(t, q, k) * bb[k];
        s1 += tB<Q, N>(t, q, k) * bg[k];
        s2 += tB<Q, N>(t, q, k) * gb[k];
      }
      const int o = CF::gs(qq, q);
      g[o] = s0;
      g[GF + o] = s1;
      g[2 * GF + o] = s2;
    }
  }
}

// -------------------------------------------------------- 3D backward
// z[c*3+dir][q] (R2) -> A[c][v3][qz][qy][kx] (R1): A0 = Gx^T z0, A1 = Bx^T z1, A2 = Bx^T z2
template <int N, int Q>
__device__ __forceinline__ void b3_3d(const Tab &t, const double *R2, double *R1) {
  using CF = Cfg<3, N, Q>;
  constexpr int ITEMS = 3 * Q * Q;
  for (int w = threadIdx.x; w < CF::EPB * ITEMS; w += CF::NT) {
    const int e = w / ITEMS, r = w % ITEMS, c = r / (Q * Q), qq = r % (Q * Q);
    constexpr int WF = CF::WV, GF = CF::GF;
    const double *z = R2 + e * CF::R2 + (c * 3) * GF;
    double z0[Q], z1[Q], z2[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int o = CF::gs(qq, q);
      z0[q] = z[o];
      z1[q] = z[GF + o];
      z2[q] = z[2 * GF + o];
    }
    double *A = R1 + e * CF::R1 + c * CF::WC + (qq / Q) * CF::WZ + (qq % Q) * CF::WY;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        s0 += tG<Q, N>(t, q, k) * z0[q];
        s1 += tB<Q, N>(t, q, k) * z1[q];
        s2 += tB<Q, N>(t, q, k) * z2[q];
      }
      A[k] = s0;
      A[WF + k] = s1;
      A[2 * WF + k] = s2;
    }
  }
}

// A (R1) -> Bv[c][2][qz][ky][kx] (R2): b0 = By^T A0 + Gy^T A1, b1 = By^T A2
template <int N, int Q>
__device__ __forceinline__ void b2_3d(const Tab &t, const double *R1, double *R2) {
  using CF = Cfg<3, N, Q>;
  constexpr int ITEMS = 3 * Q * N;
  for (int w = threadIdx.x; w < CF::EPB * ITEMS; w += CF::NT) {
    const int e = w / ITEMS, r = w % ITEMS, c = r / (Q * N), r2 = r % (Q * N), qz = r2 / N, kx = r2 % N;
    constexpr int NL = CF::WY, WF = CF::WV;
    const double *A = R1 + e * CF::R1 + c * CF::WC + qz * CF::WZ + kx;
    double a0[Q], a1[Q], a2[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      a0[q] = A[q * NL];
      a1[q] = A[WF + q * NL];
      a2[q] = A[2 * WF + q * NL];
    }
    double *b = R2 + e * CF::R2 + c * CF::UC + qz * CF::UZ + kx;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        s0 += tB<Q, N>(t, q, k) * a0[q] + tG<Q, N>(t, q, k) * a1[q];
        s1 += tB<Q, N>(t, q, k) * a2[q];
      }
      b[k * N] = s0;
      b[CF::UV + k * N] = s1;
    }
  }
}

// Bv (R2) -> E[e][c][kz][ky][kx] (global) = Bz^T b0 + Gz^T b1
template <int N, int Q>
__device__ __forceinline__ void b1_3d(const Tab &t, const double *R2, double *__restrict__ E, int64_t e0,
                                      int64_t ne) {
  using CF = Cfg<3, N, Q>;
  constexpr int ITEMS = 3 * N * N, NP = N * N * N;
  for (int w = threadIdx.x; w < CF::EPB * ITEMS; w += CF::NT) {
    const int e = w / ITEMS, r = w % ITEMS, c = r / (N * N), kk = r % (N * N);
    if (e0 + e >= ne) continue;
    const double *b = R2 + e * CF::R2 + c * CF::UC + kk;
    double b0[Q], b1[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) { b0[q] = b[q * CF::UZ]; b1[q] = b[CF::UV + q * CF::UZ]; }
    double *out = E + ((e0 + e) * 3 + c) * NP + kk;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) s += tB<Q, N>(t, q, k) * b0[q] + tG<Q, N>(t, q, k) * b1[q];
      out[k * N * N] = s;
    }
  }
}

// --------------------------------------------------------- 2D sweeps
// X[c][ky][kx] (R1) -> U[c][v][qy][kx] (R2)
template <int N, int Q, int C>
__device__ __forceinline__ void f1_2d(const Tab &t, const double *R1, double *R2) {
  using CF = Cfg<2, N, Q>;
  constexpr int ITEMS = C * N;
  for (int w = threadIdx.x; w < CF::EPB * ITEMS; w += CF::NT) {
    const int e = w / ITEMS, r = w % ITEMS, c = r / N, kx = r % N;
    const double *x = R1 + e * CF::R1 + c * N * N + kx;
    double xv[N];
#pragma unroll
    for (int k = 0; k < N; ++k) xv[k] = x[k * N];
    constexpr int NL = CF::NL;
    double *u = R2 + e * CF::R2 + c * 2 * Q * NL + kx;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      double sb = 0.0, sg = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        sb += tB<Q, N>(t, q, k) * xv[k];
        sg += tG<Q, N>(t, q, k) * xv[k];
      }
      u[q * NL] = sb;
      u[Q * NL + q * NL] = sg;
    }
  }
}

// U (R2) -> grad[c*2+dir][qy][qx] (R1)
template <int N, int Q, int C>
__device__ __forceinline__ void f2_2d(const Tab &t, const double *R2, double *G) {
  using CF = Cfg<2, N, Q>;
  constexpr int ITEMS = C * Q;
  for (int w = threadIdx.x; w < CF::EPB * ITEMS; w += CF::NT) {
    const int e = w / ITEMS, r = w % ITEMS, c = r / Q, qy = r % Q;
    constexpr int NL = CF::NL, GF = CF::GF;
    const double *ub = R2 + e * CF::R2 + (c * 2) * Q * NL + qy * NL;
    const double *ug = ub + Q * NL;
    double vb[N], vg[N];
#pragma unroll
    for (int k = 0; k < N; ++k) { vb[k] = ub[k]; vg[k] = ug[k]; }
    double *g = G + e * CF::R1 + (c * 2) * GF;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        s0 += tG<Q, N>(t, q, k) * vb[k];
        s1 += tB<Q, N>(t, q, k) * vg[k];
      }
      const int o = CF::gs(qy, q);
      g[o] = s0;
      g[GF + o] = s1;
    }
  }
}

// z[c*2+dir][q] (R1) -> A[c][v][qy][kx] (R2): A0 = Gx^T z0, A1 = Bx^T z1
template <int N, int Q>
__device__ __forceinline__ void b2_2d(const Tab &t, const double *Z, double *R2) {
  using CF = Cfg<2, N, Q>;
  constexpr int ITEMS = 2 * Q;
  for (int w = threadIdx.x; w < CF::EPB * ITEMS; w += CF::NT) {
    const int e = w / ITEMS, r = w % ITEMS, c = r / Q, qy = r % Q;
    constexpr int NL = CF::NL, GF = CF::GF;
    const double *z = Z + e * CF::R1 + (c * 2) * GF;
    double z0[Q], z1[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int o = CF::gs(qy, q);
      z0[q] = z[o];
      z1[q] = z[GF + o];
    }
    double *A = R2 + e * CF::R2 + (c * 2) * Q * NL + qy * NL;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        s0 += tG<Q, N>(t, q, k) * z0[q];
        s1 += tB<Q, N>(t, q, k) * z1[q];
      }
      A[k] = s0;
      A[Q * NL + k] = s1;
    }
  }
}

// A (R2) -> E[e][c][ky][kx] = By^T A0 + Gy^T A1
template <int N, int Q>
__device__ __forceinline__ void b1_2d(const Tab &t, const double *R2, double *__restrict__ E, int64_t e0,
                                      int64_t ne) {
  using CF = Cfg<2, N, Q>;
  constexpr int ITEMS = 2 * N, NP = N * N;
  for (int w = threadIdx.x; w < CF::EPB * ITEMS; w += CF::NT) {
    const int e = w / ITEMS, r = w % ITEMS, c = r / N, kx = r % N;
    if (e0 + e >= ne) continue;
    constexpr int NL = CF::NL;
    const double *A = R2 + e * CF::R2 + (c * 2) * Q * NL + kx;
    double a0[Q], a1[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) { a0[q] = A[q * NL]; a1[q] = A[Q * NL + q * NL]; }
    double *out = E + ((e0 + e) * 2 + c) * NP + kx;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) s += tB<Q, N>(t, q, k) * a0[q] + tG<Q, N>(t, q, k) * a1[q];
      out[k * N] = s;
    }
  }
}

// ------------------------------------------------ point-level helpers
template <int D>
__device__ __forceinline__ void load_point(const double *g, int stride, double (&A)[D][D]) {
#pragma unroll
  for (int c = 0; c < D; ++c)
#pragma unroll
    for (int d = 0; d < D; ++d) A[c][d] = g[(c * D + d) * stride];
}
template <int D>
__device__ __forceinline__ void store_point(double *g, int stride, const double (&A)[D][D]) {
#pragma unroll
  for (int c = 0; c < D; ++c)
#pragma unroll
    for (int d = 0; d < D; ++d) g[(c * D + d) * stride] = A[c][d];
}

// Lean point record -> (T, S, coefficient scalars).  qd points at field 0 of
// the point (field stride QP).
template <int D>
__device__ __forceinline__ void lean_load(const double *qd, int QP, double (&T)[D][D], double (&S)[D][D],
                                          double &k0, double &itau) {
  load_point<D>(qd, QP, T);
  k0 = qd[D * D * QP];
  itau = qd[(D * D + 1) * QP];
  double C[D][D];
  mcof<D>(T, C);
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) S[i][j] = C[i][j] * itau;
}

// z = (d2 mu / dT2 scaled) : g from a lean point record.
template <int D, bool NTM>
__device__ __forceinline__ void lean_hess(int metric, const double *qd, int QP, const double (&g)[D][D],
                                          double (&z)[D][D]) {
  if constexpr (D == 3 && !NTM && TMOP_DCOF) {
    double T[3][3], C[3][3], c[4];
    load_point<3>(qd, QP, T);
    const double k0 = qd[9 * QP], itau = qd[10 * QP];
    mcof<3>(T, C);
    lean_coeffs(metric, k0, itau, mfro2<3>(T), c);
    hess_tpl_cof3(c, C, T, itau, g, z);
    return;
  }
  double T[D][D], S[D][D], k0, itau;
  lean_load<D>(qd, QP, T, S, k0, itau);
  if constexpr (!NTM) {
    double c[4];
    lean_coeffs(metric, k0, itau, mfro2<D>(T), c);
    hess_template<D>(c, S, T, g, z);
  } else {
    nt_hess<D>(metric, k0, S, T, g, z);
  }
}

// ------------------------------------------------------ the kernel
template <int DIM, int N, int Q, int KIND>
__global__ void __launch_bounds__(Cfg<DIM, N, Q>::NT, Cfg<DIM, N, Q>::template minb<KIND>()) elem_kernel(const ElemArgs a, const __grid_constant__ Tab t) {
  using CF = Cfg<DIM, N, Q>;
  constexpr int QP = CF::QP, EPB = CF::EPB, QS = CF::QS;
  constexpr bool APPLY = (KIND == K_APPLY || KIND == K_APPLY_NT);
  constexpr bool STAGE = APPLY && !CF::QLDG;   // Q-data staged in shared memory by TMA
  extern __shared__ __align__(16) double smem[];
  double *R1 = smem;
  double *R2 = smem + EPB * CF::R1;
  double *QB = smem + CF::QOFF;   // staged Q-data of the current group (apply only)
  __shared__ double red_v[CF::NT / 32];
  __shared__ int64_t red_i[CF::NT / 32];
  __shared__ __align__(8) uint64_t qbar;

  if (a.stop && *a.stop) return;
  double acc = 0.0;
  MinLoc mn{DBL_MAX, LLONG_MAX};

  // The Hessian action streams each group's Q-data (one contiguous block of
  // EPB * QS doubles) into shared memory with one TMA bulk copy, issued a
  // whole group ahead: the copy for group g + grid overlaps the transposed
  // sweeps of group g and the gather / forward sweeps of the next group.
  auto issue = [&](int64_t grp) {
    const int64_t e0 = grp * EPB;
    const int64_t cnt = (a.ne - e0) < EPB ? (a.ne - e0) : EPB;
    const uint32_t bytes = (uint32_t)(cnt * QS * 8);
    mbar_expect_tx(&qbar, bytes);
    tma_load_1d(QB, a.qdata + e0 * QS, bytes, &qbar);
  };
  uint32_t phase = 0;
  if constexpr (STAGE) {
    if (threadIdx.x == 0) {
      mbar_init(&qbar, 1);
      mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && (int64_t)blockIdx.x < a.ngroups) issue(blockIdx.x);
  }

  GatherPrefetch<DIM, N, Q> pre;
  if constexpr (APPLY) {
    pre.load_index(a, (int64_t)blockIdx.x * EPB);      // (empty when blockIdx.x >= ngroups)
    pre.load_values(a);
    pre.load_index(a, ((int64_t)blockIdx.x + gridDim.x) * EPB);
  }

  for (int64_t grp = blockIdx.x; grp < a.ngroups; grp += gridDim.x) {
    const int64_t e0 = grp * EPB;
    if constexpr (APPLY && CF::QLDG) {
      // the next group's Q-data block -> L2 while this group runs, so the
      // point stage's direct loads of it hit L2
      const int64_t nxt = grp + gridDim.x;
      if (threadIdx.x == 0 && nxt < a.ngroups) {
        const int64_t cnt = (a.ne - nxt * EPB) < EPB ? (a.ne - nxt * EPB) : EPB;
        l2_prefetch_bulk(a.qdata + nxt * EPB * QS, (uint32_t)(cnt * QS * 8));
      }
    }
    if constexpr (APPLY) {
      pre.store(R1);
    } else {
      gather<DIM, N, Q, DIM, false>(a, e0, R1);
    }
    __syncthreads();
    // ---- forward: gradients of the gathered field at the points
    double *Gp;
    int gstride;
    if constexpr (DIM == 3) {
      f1_3d<N, Q, 3>(t, R1, R2);
      __syncthreads();
      f2_3d<N, Q, 3>(t, R2, R1);
      __syncthreads();
      f3_3d<N, Q, 3>(t, R1, R2);
      Gp = R2;
      gstride = CF::R2;
    } else {
      f1_2d<N, Q, 2>(t, R1, R2);
      __syncthreads();
      f2_2d<N, Q, 2>(t, R2, R1);
      Gp = R1;
      gstride = CF::R1;
    }
    if constexpr (STAGE) mbar_wait(&qbar, phase);
    __syncthreads();

    // ---- point stage
    for (int w = threadIdx.x; w < EPB * QP; w += CF::NT) {
      // 3D, unswizzled lines: threads walk the lean record's slot order
      // (qx slowest) -- unit-stride Q-data reads / setup writes and odd-stride
      // (conflict-free) gradient-buffer accesses; otherwise point order
      constexpr bool SLOTW = DIM == 3 && !CF::SWZ;
      const int e = w / QP, r = w % QP;
      const int q = SLOTW ? (r / (Q * Q)) + Q * (r % (Q * Q)) : r;
      const int64_t eg = e0 + e;
      if (eg >= a.ne) continue;
      const int gi = CF::gs(q / Q, q % Q);   // (padded / swizzled) slot of the point
      double *gp = Gp + e * gstride + gi;
      double A[DIM][DIM];
      load_point<DIM>(gp, CF::GF, A);

      if constexpr (APPLY) {
        double z[DIM][DIM];
        const double *qp = (CF::QLDG ? a.qdata + eg * QS : QB + e * QS) + lean_slot<DIM, Q>(q);
        lean_hess<DIM, KIND == K_APPLY_NT>(a.metric, qp, QP, A, z);
        store_point<DIM>(gp, CF::GF, z);
      } else {
        // A is the Jacobian dx/dxi at the point
        const double dj = mdet<DIM>(A);
        if constexpr (KIND == K_VOLUME) {
          acc += dj * wq<DIM, Q>(t, q);
        } else if constexpr (KIND == K_ELEMDET) {
          R1[e * CF::R1 + gi] = dj;  // own field-0 slot (2D: in place over this point's grad)
        } else {
          mn = minloc(mn, MinLoc{dj, eg * QP + q});
        }
        if constexpr (KIND == K_SETUP || KIND == K_GRAD || KIND == K_ENERGY) {
          const PtScale ps = pt_scale<DIM>(a, eg * QP + q);
          const double tau = dj * ps.is_d;
          const double I1 = mfro2<DIM>(A) * (ps.is * ps.is);
          const double itau = 1.0 / tau;   // the one division of the point
          const double cs = ps.is_dm1 * itau;
          const double wpt = wq<DIM, Q>(t, q);
          // S = cof(T) / det T and T only where the metric / kind reads them
          // (the template metrics' energy and gradient need neither)
          const bool uses_s = a.metric == MU7 || !metric_is_template(a.metric);
          auto mk_s = [&](const double (&Cof)[DIM][DIM], double (&S)[DIM][DIM]) {
#pragma unroll
            for (int i = 0; i < DIM; ++i)
#pragma unroll
              for (int j = 0; j < DIM; ++j) S[i][j] = cs * Cof[i][j];
          };
          auto mk_t = [&](double (&T)[DIM][DIM]) {
#pragma unroll
            for (int i = 0; i < DIM; ++i)
#pragma unroll
              for (int j = 0; j < DIM; ++j) T[i][j] = ps.is * A[i][j];
          };
          if constexpr (KIND == K_ENERGY) {
            double mu;
            if (uses_s) {
              double Cof[DIM][DIM], S[DIM][DIM];
              mcof<DIM>(A, Cof);
              mk_s(Cof, S);
              mu = metric_mu<DIM>(a.metric, tau, I1, S);
            } else {
              const double Z[DIM][DIM] = {};
              mu = metric_mu<DIM>(a.metric, tau, I1, Z);
            }
            acc += (wpt * ps.ew) * mu;
          } else if constexpr (KIND == K_SETUP) {
            // lean record (operator.py:350-371 restated; see lean_k0)
            double T[DIM][DIM];
            mk_t(T);
            double *qo = a.qout + eg * QS + lean_slot<DIM, Q>(q);
            store_point<DIM>(qo, QP, T);
            qo[DIM * DIM * QP] = lean_k0(a.metric, ps.ch * wpt, tau);
            qo[(DIM * DIM + 1) * QP] = itau;
          } else {  // K_GRAD (+ the energy, for the fused line-search evaluation)
            double Cof[DIM][DIM];
            mcof<DIM>(A, Cof);
            const double cw = ps.cg * wpt;
            double P[DIM][DIM];
            if (metric_is_template(a.metric)) {
              double at, as, mu = 0.0;
              if (uses_s && a.energy) {
                double S[DIM][DIM];
                mk_s(Cof, S);
                metric_mu_first<DIM>(a.metric, tau, I1, S, a.energy, mu, at, as);
              } else {
                const double Z[DIM][DIM] = {};
                metric_mu_first<DIM>(a.metric, tau, I1, Z, a.energy, mu, at, as);
              }
              if (a.energy) acc += (wpt * ps.ew) * mu;
              const double ct = cw * at * ps.is;
              const double cc = cw * as * ps.is_dm1 * itau;
#pragma unroll
              for (int i = 0; i < DIM; ++i)
#pragma unroll
                for (int j = 0; j < DIM; ++j) P[i][j] = ct * A[i][j] + cc * Cof[i][j];
            } else {
              double S[DIM][DIM], T[DIM][DIM];
              mk_s(Cof, S);
              mk_t(T);
              if (a.energy) acc += (wpt * ps.ew) * metric_mu<DIM>(a.metric, tau, I1, S);
              nt_first<DIM>(a.metric, T, S, P);
#pragma unroll
              for (int i = 0; i < DIM; ++i)
#pragma unroll
                for (int j = 0; j < DIM; ++j) P[i][j] *= cw;
            }
            store_point<DIM>(gp, CF::GF, P);
          }
        }
      }
    }
    __syncthreads();
    if constexpr (APPLY) {
      // the staging buffer is free again: stream in the next group's Q-data
      phase ^= 1u;
      const int64_t nxt = grp + gridDim.x;
      if (STAGE && threadIdx.x == 0 && nxt < a.ngroups) issue(nxt);
      pre.load_values(a);                              // group nxt (indices loaded last iteration)
      pre.load_index(a, (nxt + gridDim.x) * EPB);       // group after nxt
    }

    if constexpr (KIND == K_ELEMDET) {
      for (int e = threadIdx.x; e < EPB; e += CF::NT) {
        const int64_t eg = e0 + e;
        if (eg >= a.ne) continue;
        double m = R1[e * CF::R1];
        int arg = 0;
        for (int q = 1; q < QP; ++q) {
          const double v = R1[e * CF::R1 + CF::gs(q / Q, q % Q)];
          if (v < m) { m = v; arg = q; }
        }
        a.elem_min[eg] = m;
        a.elem_arg[eg] = arg;
      }
      __syncthreads();
    }

    // ---- backward sweeps to the element-blocked E-vector
    if constexpr (APPLY || KIND == K_GRAD) {
      if constexpr (DIM == 3) {
        b3_3d<N, Q>(t, R2, R1);
        __syncthreads();
        b2_3d<N, Q>(t, R1, R2);
        __syncthreads();
        b1_3d<N, Q>(t, R2, a.E, e0, a.ne);
      } else {
        b2_2d<N, Q>(t, R1, R2);
        __syncthreads();
        b1_2d<N, Q>(t, R2, a.E, e0, a.ne);
      }
      __syncthreads();
    }
  }

  // ---- per-CTA deterministic partials
  if constexpr (KIND == K_ENERGY || KIND == K_VOLUME || KIND == K_GRAD) {
    const double s = block_sum<CF::NT>(acc, red_v);
    if (threadIdx.x == 0) a.part_sum[blockIdx.x] = s;
  }
  if constexpr (KIND == K_SETUP || KIND == K_GRAD || KIND == K_ENERGY || KIND == K_MINDET) {
    const MinLoc m = block_minloc<CF::NT>(mn, red_v, red_i);
    if (threadIdx.x == 0) {
      a.part_min[blockIdx.x] = m.v;
      a.part_arg[blockIdx.x] = m.i;
    }
  }
}

// ------------------------------------------ lean -> reference Q-data
// Materialises the reference's planar HessQData arrays (operator.py:105-113)
// from the lean record: template metrics -> coeffs (4), S, T; non-template
// -> w (1), S, T.  out is (fields_ref, ne * QP) planar.
template <int D>
__global__ void qdata_expand_kernel(int metric, int64_t ne, int q1d, int QP, int QS, const double *__restrict__ qd,
                                    double *__restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nq = ne * QP;
  if (k >= nq) return;
  const int64_t e = k / QP;
  const int q = (int)(k - e * QP);
  double T[D][D], S[D][D], k0, itau;
  const int slot = D == 3 ? q / q1d + q1d * q1d * (q % q1d) : q;   // lean_slot
  lean_load<D>(qd + e * QS + slot, QP, T, S, k0, itau);
  int f = 0;
  if (metric_is_template(metric)) {
    double c[4];
    lean_coeffs(metric, k0, itau, mfro2<D>(T), c);
    for (; f < 4; ++f) out[f * nq + k] = c[f];
  } else {
    out[k] = k0;
    f = 1;
  }
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) out[(f + i * D + j) * nq + k] = S[i][j];
  f += D * D;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) out[(f + i * D + j) * nq + k] = T[i][j];
}

}  // namespace tmop
