// tmop_xl.cuh -- the 3D element kernels in "x-line" form: the Hessian action
// (AddMultGradPA, operator.py:401-418), the gradient (AddMultPA,
// operator.py:328-346), the Hessian setup (AssembleGradPA,
// operator.py:350-371), the energy (GetLocalStateEnergyPA,
// operator.py:311-326) and min det(A) (operator.py:296-304).
//
// Why this shape (profiles/round1_*.md): on B200 the FP64 pipe is shared by
// DFMA and DMMA (measured: mixed DFMA+DMMA loops sum to the same ~35 TF/s),
// so the element contractions stay on DFMA, and the previous work-item
// kernel was co-limited by shared-memory bandwidth (~6.5 K doubles of
// shared traffic per p=2 element, 69 % of the LSU wavefront budget) and
// FP64 issue.  Here one thread owns one x-line (qy, qz) of an element for
// all three components and keeps, in registers, the y/x-sweep results W, the
// nine gradient entries of the current point, the point's result (Hessian
// action / first Piola-Kirchhoff term) and the transposed x-sweep
// accumulators A -- the quadrature-point fields never touch shared memory.
// For the Hessian action the group's lean Q-data arrives by one TMA bulk
// copy issued a group ahead (the lean record stores qx as the slowest point
// index, lean_slot(), and the element stride is 2 mod 16 doubles, so the X
// stage reads it conflict-free); the setup writes the record the same way,
// one coalesced 32-byte run per (element, field, qx) and warp.
//
// Layout: a CTA owns EPB = 8 (p <= 2) or 4 (p >= 3) elements per group;
// thread id = e + EPB * item and every shared buffer is element-interleaved
// (slot * EPB + e), so a half-warp touches 16 / EPB items x EPB elements;
// the padded strides (XlPad, searched by tools/xl_banks.py) make every 64-bit
// shared access pattern of the kernel conflict-free.
//
// Stages per group (z axis first like contract_dofs_to_quad, fe.py:227-239):
//   G   all threads:    cp.async gather of the input T-vector (x or v) and the
//                       fixed flags of the NEXT group into shared memory
//   F1  item (ky,kx):   z-sweep -> U[c][v][qz][ky][kx], v in {B, G}
//   X   item (qy,qz):   U -> W (y-sweep of row qy: BB, BG, GB; registers) ->
//                       gradient at the Q points of the line -> point work
//                       (KIND) -> A (x^T sweep) -> A[c][v3][qz][qy][kx]
//   B2  item (qz,kx):   A -> Bv[c][v][qz][ky][kx]   (y^T sweep, fe.py:242-253)
//   B1  item (ky,kx):   Bv -> element-interleaved E-vector (z^T sweep)
// B2 / B1 run for the Hessian action and the gradient only.  The E-vector is
// summed to nodes by e2l_kernel (EPB-element interleave) in ascending element
// order, no atomics; energies and min det reduce per CTA in a fixed order.
#pragma once

#include "tmop_elem.cuh"
#include "tmop_xld_parts.cuh"

namespace tmop {

// Tuning knob (tools/build_variant.sh): occupancy hint (CTAs / SM; 0 = per
// order default).
#ifndef TMOP_XL_MINB
#define TMOP_XL_MINB 0
#endif

template <int KIND>
__host__ __device__ constexpr bool xl_backward() {
  return KIND == K_APPLY || KIND == K_APPLY_NT || KIND == K_GRAD;
}
template <int KIND>
__host__ __device__ constexpr bool xl_qdata() {
  return KIND == K_APPLY || KIND == K_APPLY_NT;
}

// Padded strides (in slots) chosen by tools/xl_banks.py so that every shared
// access pattern of the kernel is bank-conflict free for the group size.
// n_q >= 7 (the paper's Kershaw table uses 9): one element per CTA and the
// Hessian action reads its record straight from global memory (the record,
// 11 n_q^3 doubles, is too large to stage), Q^2 = 49..81 x-line threads.
template <int N, int Q>
__host__ __device__ constexpr bool xl_ldg() { return Q >= 7; }

template <int N, int Q>
struct XlPad {
  static constexpr int EPB = xl_ldg<N, Q>() ? 1 : xl_epb(N);
  // EPB = 16: a half-warp is one item x 16 elements -- conflict-free unpadded;
  // EPB = 1: a half-warp is 16 consecutive lines (odd W_QY: distinct banks)
  static constexpr int U_QZ = (EPB == 16 || EPB == 1) ? N * N
                            : EPB == 8 ? (N * N) | (Q & 1) : (N == 4 ? (Q % 4 == 0 ? 16 : 17) : 25);
  static constexpr int W_QY = EPB == 16 ? N : (EPB == 8 || EPB == 1) ? (N | 1)
                                                 : ((N == 5 && (Q == 3 || Q == 7)) ? 7 : 5);
  static constexpr int W_QZ = EPB == 16 ? Q * N
                            : EPB == 1 ? Q * W_QY
                            : EPB == 8 ? Q * W_QY + ((N & 1) && !(Q & 1) ? 1 : 0)
                                       : (N == 4 ? Q * 5 : (Q == 3 ? 21 : Q == 4 ? 21 : Q == 6 ? 33 : Q * W_QY));
};

// software prefetch of the next point's record fields in the x-line apply
// (registers): -1 = per order (measured at C3: p = 3 6.81 -> 5.78 ms element
// kernel; p = 2 slower, 7.27 -> 7.58 ms; p = 1 slower, 6.6 -> 8.1 ms), 0 = never, 1 = always
#ifndef TMOP_XL_QPF
#define TMOP_XL_QPF -1
#endif

// x-line Hessian action at n_q >= 7 (xl_ldg): 1 = on, 0 = work-item kernel
#ifndef TMOP_XL_LDG
#define TMOP_XL_LDG 1
#endif
// (bulk L2 prefetch of the next element's record: measured slower at
// 24^3 n_q = 9, p = 1 0.242 -> 0.254 ms, with 31 % more DRAM reads)
#ifndef TMOP_XL_LDG_L2PF
#define TMOP_XL_LDG_L2PF 0
#endif
#ifndef TMOP_XL_LDG_MINB
#define TMOP_XL_LDG_MINB 0
#endif
// y-sweep results W of the x-line in the thread's own A slots instead of
// registers (-1 = per configuration, 0 = never, 1 = always)
#ifndef TMOP_XL_WSM
#define TMOP_XL_WSM -1
#endif
#ifndef TMOP_XL_LDG_NMIN
#define TMOP_XL_LDG_NMIN 3
#endif
#ifndef TMOP_XL_LDG_NMAX
#define TMOP_XL_LDG_NMAX 3
#endif
// (p = 3 gradient unrolled by 2: C3 6.67 -> 6.43 ms; fully: 7.7 ms)
#ifndef TMOP_XL_P3_GRAD_UNROLL
#define TMOP_XL_P3_GRAD_UNROLL 2
#endif
// (p = 3 action unrolled by 2: C3 6.23 -> 6.14 ms; fully unrolled it spills)
#ifndef TMOP_XL_P3_APPLY_UNROLL
#define TMOP_XL_P3_APPLY_UNROLL 2
#endif
// unroll factor of the X stage's point loop (0 = per order)
#ifndef TMOP_XL_QX_UNROLL
#define TMOP_XL_QX_UNROLL 0
#endif
#ifndef TMOP_XL_GRAD_MINB
#define TMOP_XL_GRAD_MINB 0
#endif
#ifndef TMOP_XL_P1_MINB
#define TMOP_XL_P1_MINB 3
#endif
#ifndef TMOP_XL_NT_MINB
#define TMOP_XL_NT_MINB 0
#endif

template <int N, int Q>
struct XlCfg {
  static constexpr int EPB = XlPad<N, Q>::EPB;
  static constexpr int NP = N * N * N, QP = Q * Q * Q;
  static constexpr int LINES = Q * Q;
  static constexpr int NT = EPB * LINES;
  // U / Bv: [c][v][qz][ky*N+kx]          (slots; one slot = EPB doubles)
  static constexpr int U_QZ = XlPad<N, Q>::U_QZ;
  static constexpr int U_SZ = 6 * Q * U_QZ;
  // W / A:  [c][v3][qz][qy][kx]
  static constexpr int W_QY = XlPad<N, Q>::W_QY;
  static constexpr int W_QZ = XlPad<N, Q>::W_QZ;
  static constexpr int W_SZ = 9 * Q * W_QZ;
  static constexpr int SLOTS = (U_SZ + W_SZ + 1) & ~1;
  static constexpr int F = 11;                 // lean fields (T, k0, itau)
  static constexpr int QS = lean_stride(F * QP, xl_epb(N));   // the record's element stride (Cfg::QS)
  static constexpr bool LDG = xl_ldg<N, Q>();              // apply: record read from global memory
  static constexpr bool GRAD3 = Q == N + 1;                // gradient: W in shared memory, 3 CTAs / SM
  static constexpr int XOFF = SLOTS * EPB;                 // gathered input: XS[c][l][e]
  static constexpr int FOFF = XOFF + 3 * NP * EPB;         // fixed-flag words: FS[l][e] (uint32)
  static constexpr int BOFF = FOFF + (NP * EPB + 1) / 2;   // flag byte offsets: FB[l][e] (uint8)
  static constexpr int QOFF = (BOFF + (NP * EPB + 7) / 8 + 1) & ~1;   // staged Q-data, 16-byte aligned
  static constexpr int SMEM = (QOFF + EPB * QS) * 8;      // Hessian action
  // kinds without the A buffer / staged Q-data: U + gather buffers only
  static constexpr int XOFF_F = U_SZ * EPB;
  static constexpr int FOFF_F = XOFF_F + 3 * NP * EPB;
  static constexpr int BOFF_F = FOFF_F + (NP * EPB + 1) / 2;
  static constexpr int SMEM_F = (BOFF_F + (NP * EPB + 7) / 8 + 1) * 8;
  // setup: the group's lean records are assembled in shared memory and
  // written back by one TMA bulk store
  static constexpr int QOFF_S = (BOFF_F + (NP * EPB + 7) / 8 + 1) & ~1;
  static constexpr int SMEM_S = (QOFF_S + EPB * QS) * 8;
  // setup + diagonal: the diagonal's x^T output A overlays the group's
  // records once they are stored (XldCfg::R1), its y^T output Bv follows
  static constexpr int SMEM_SD = (QOFF_S + XldCfg<N, Q>::R1OP + XldCfg<N, Q>::BV_SZ * EPB) * 8;
  template <int KIND>
  static constexpr int smem() {
    return xl_qdata<KIND>() ? (LDG ? QOFF * 8 : SMEM)
           : (xl_backward<KIND>() ? QOFF * 8
                                  : (KIND == K_SETUP ? SMEM_S : (KIND == K_SETUP_DIAG ? SMEM_SD : SMEM_F)));
  }
  static constexpr int GJ = (EPB * NP + NT - 1) / NT;      // gather (element, node) pairs per thread
  // CTAs / SM: the backward kinds keep ~110 doubles live in the x-line
  // (p = 2: ~240 registers); forward-only kinds ~half
  static constexpr int WARPS = (NT + 31) / 32;
  template <int KIND>
  static constexpr int minb() {
    return TMOP_XL_MINB ? TMOP_XL_MINB
           : KIND == K_SETUP_DIAG ? XldCfg<N, Q>::MINB
           : (KIND == K_APPLY_NT && TMOP_XL_NT_MINB) ? TMOP_XL_NT_MINB
           // p = 1, n_q = 3 action (144-thread CTAs): 3 CTAs / SM at a 128-register cap (small spill)
           // beat 2 CTAs at 166 registers: overlapped apply 6.46 -> 6.12 ms
           : (KIND == K_APPLY && N <= 2 && Q == 3) ? TMOP_XL_P1_MINB
           : (KIND == K_APPLY && xl_ldg<N, Q>()) ? (TMOP_XL_LDG_MINB ? TMOP_XL_LDG_MINB : (N <= 3 ? 4 : 2))
           : (KIND == K_GRAD && TMOP_XL_GRAD_MINB) ? TMOP_XL_GRAD_MINB
           // gradient at n_q = p + 2 (W in shared memory): 3 CTAs / SM (p = 3 at
           // 2 CTAs: 7.5 ms, at 3: 6.7 ms; with W in registers 3 CTAs were slower
           // at p = 2, 9.6 vs 7.5 ms)
           : (KIND == K_GRAD && GRAD3) ? 3
                        : cmax(1, 65536 / (WARPS * 32 *
                                           (xl_backward<KIND>() ? (N <= 2 ? 168 : N == 3 ? 248 : 255)
                                                                : (N <= 3 ? 128 : 168))));
  }
};

template <int N, int Q>
__host__ __device__ constexpr bool xl_supported() {
  // the CTA's work buffers + staged Q-data within 227 KB; n_q >= 7: the
  // Hessian action only (p <= 2), record from global memory
  if constexpr (xl_ldg<N, Q>()) {
    // (24^3 n_q = 9 action p = 2 0.291 -> 0.284 ms with W in shared memory
    // at 4 CTAs / SM (0.363 ms with W in registers, 243 registers, 2 CTAs);
    // p = 3 slower, 0.325 -> 0.50 ms.  p = 1 is faster, 0.265 -> 0.242 ms,
    // but off by default (TMOP_XL_LDG_NMIN=2 enables it): its different
    // rounding flips the paper-table p = 1 Kershaw solve -- chaotic, see
    // from converged in 69 Newton iterations to the
    // 100-iteration cap)
    return TMOP_XL_LDG != 0 && N >= TMOP_XL_LDG_NMIN && N <= TMOP_XL_LDG_NMAX && XlCfg<N, Q>::NT <= 1024 &&
           XlCfg<N, Q>::QOFF * 8 <= 227 * 1024;
  } else {
    return Q >= 2 && XlCfg<N, Q>::SMEM <= 227 * 1024;
  }
}

// Fixed-order block reductions for any CTA size (partial warps allowed):
// every thread stores its partial, thread 0 combines them in thread order.
template <int NT>
__device__ __forceinline__ double xl_block_sum(double v, double *sv) {
  __syncthreads();
  sv[threadIdx.x] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < NT; ++i) r += sv[i];
  return r;
}
template <int NT>
__device__ __forceinline__ MinLoc xl_block_minloc(MinLoc m, double *sv, int64_t *si) {
  __syncthreads();
  sv[threadIdx.x] = m.v;
  si[threadIdx.x] = m.i;
  __syncthreads();
  MinLoc r{DBL_MAX, LLONG_MAX};
  if (threadIdx.x == 0)
    for (int i = 0; i < NT; ++i) r = minloc(r, MinLoc{sv[i], si[i]});
  return r;
}

// A:B as three row sums added pairwise (dependency depth 4 instead of 9).
__device__ __forceinline__ double tdot(const double (&A)[3][3], const double (&B)[3][3]) {
  double r[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) r[i] = A[i][0] * B[i][0] + A[i][1] * B[i][1] + A[i][2] * B[i][2];
  return (r[0] + r[1]) + r[2];
}

// Point stage of the x-line: z = (scaled d2mu/dT2) : g from the lean record
// (T, k0, itau), accumulated straight into the transposed x-sweep:
// av[c][0][k] += G(qx,k) z[c][0], av[c][v][k] += B(qx,k) z[c][v] (v = 1, 2).
// Template metrics: S = itau cof(T) is folded into the coefficients and the
// block (_kernels.py:235-258) is applied with C = cof(T) directly.
template <int N, bool NTM>
__device__ __forceinline__ void xl_point(int metric, const double (&qd)[11], const double (&g)[3][3],
                                         const double (&tg)[N], const double (&tb)[N], double (&av)[3][3][N]) {
  double T[3][3], C[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) T[i][j] = qd[i * 3 + j];
  mcof<3>(T, C);
  auto acc = [&](int c, int n, double z) {
#pragma unroll
    for (int k = 0; k < N; ++k) av[c][n][k] += (n == 0 ? tg[k] : tb[k]) * z;
  };
  if constexpr (!NTM && TMOP_DCOF) {
    const double k0 = qd[9], itau = qd[10];
    double c[4], z[3][3];
    lean_coeffs(metric, k0, itau, tdot(T, T), c);
    hess_tpl_cof3(c, C, T, itau, g, z);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int n = 0; n < 3; ++n) acc(a, n, z[a][n]);
  } else if constexpr (!NTM) {
    const double k0 = qd[9], itau = qd[10];
    double c[4];
    lean_coeffs(metric, k0, itau, tdot(T, T), c);
    const double dt = tdot(T, g);
    const double ds = itau * tdot(C, g);
    const double w1 = (c[1] * dt + c[2] * ds) * itau;
    const double w2 = c[1] * ds;
    const double c3 = c[3] * (itau * itau);
    double gs[3][3];
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int n = 0; n < 3; ++n) gs[p][n] = g[0][p] * C[0][n] + g[1][p] * C[1][n] + g[2][p] * C[2][n];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        const double cross = C[a][0] * gs[0][n] + C[a][1] * gs[1][n] + C[a][2] * gs[2][n];
        acc(a, n, c[0] * g[a][n] + w1 * C[a][n] + w2 * T[a][n] + c3 * cross);
      }
  } else {
    double S[3][3], z[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) S[i][j] = C[i][j] * qd[10];
    nt_hess<3>(metric, qd[9], S, T, g, z);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int n = 0; n < 3; ++n) acc(a, n, z[a][n]);
  }
}


// TMA bulk store shared -> global (bulk_group completion) and its fences.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_store(void *dst, const void *src, uint32_t bytes) {
  asm volatile(
      "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
      "cp.async.bulk.commit_group;" ::"l"(dst),
      "r"(smem_u32(src)), "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// x-line point work of the forward-only / gradient kinds at one point:
// J = the Jacobian dx/dxi (operator.py:252-292 restated like the work-item
// kernel's point stage, same operation order).
template <int KIND, int N, int Q>
__device__ __forceinline__ void xl_point_x(const ElemArgs &a, const Tab &t, int64_t eg, int line, int qx,
                                           const double (&J)[3][3], const double (&tg)[N], const double (&tb)[N],
                                           double (&av)[3][3][N], double &acc, MinLoc &mn, double *rec) {
  constexpr int QP = Q * Q * Q;
  const int q = qx + Q * line;                       // reference point index (x fastest)
  const double dj = mdet<3>(J);
  if (eg < a.ne) mn = minloc(mn, MinLoc{dj, eg * QP + q});
  if constexpr (KIND == K_SETUP || KIND == K_GRAD || KIND == K_ENERGY) {
    const PtScale ps = pt_scale<3>(a, (eg < a.ne ? eg : 0) * QP + q);
    const double tau = dj * ps.is_d;
    const double I1 = mfro2<3>(J) * (ps.is * ps.is);
    const double wpt = wq<3, Q>(t, q);
    // S = cof(T) / det T and T itself only where the metric / kind reads them
    // (the template metrics' energy and gradient need neither)
    auto mk_s = [&](const double (&Cof)[3][3], double cs, double (&S)[3][3]) {
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) S[i][j] = cs * Cof[i][j];
    };
    auto mk_t = [&](double (&T)[3][3]) {
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) T[i][j] = ps.is * J[i][j];
    };
    const bool uses_s = a.metric == MU7 || !metric_is_template(a.metric);
    if constexpr (KIND == K_ENERGY) {
      double mu;
      if (uses_s) {
        const double itau = 1.0 / tau;
        double Cof[3][3], S[3][3];
        mcof<3>(J, Cof);
        mk_s(Cof, ps.is_dm1 * itau, S);
        mu = metric_mu<3>(a.metric, tau, I1, S);
      } else {
        const double Z[3][3] = {};
        mu = metric_mu<3>(a.metric, tau, I1, Z);
      }
      if (eg < a.ne) acc += (wpt * ps.ew) * mu;
    } else if constexpr (KIND == K_SETUP) {
      const double itau = 1.0 / tau;   // the one division of the point
      double T[3][3];
      mk_t(T);
      // lean record (operator.py:350-371 restated; see lean_k0), staged in
      // shared memory at slot = line + Q^2 qx of this thread's element
      double *qo = rec + line + Q * Q * qx;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) qo[(i * 3 + j) * QP] = T[i][j];
      qo[9 * QP] = lean_k0(a.metric, ps.ch * wpt, tau);
      qo[10 * QP] = itau;
    } else {  // K_GRAD: P = cw (a_t T + a_s S) (operator.py:328-346), + the energy
      const double itau = 1.0 / tau;
      const double cs = ps.is_dm1 * itau;
      double Cof[3][3];
      mcof<3>(J, Cof);
      const double cw = ps.cg * wpt;
      const bool en = a.energy && eg < a.ne;   // (line-search evaluation)
      double P[3][3];
      if (metric_is_template(a.metric)) {
        double at, as, mu = 0.0;
        if (uses_s && en) {
          double S[3][3];
          mk_s(Cof, cs, S);
          metric_mu_first<3>(a.metric, tau, I1, S, en, mu, at, as);
        } else {
          const double Z[3][3] = {};
          metric_mu_first<3>(a.metric, tau, I1, Z, en, mu, at, as);
        }
        if (en) acc += (wpt * ps.ew) * mu;
        const double ct = cw * at * ps.is;
        const double cc = cw * as * ps.is_dm1 * itau;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j) P[i][j] = ct * J[i][j] + cc * Cof[i][j];
      } else {
        double S[3][3], T[3][3];
        mk_s(Cof, cs, S);
        mk_t(T);
        if (en) acc += (wpt * ps.ew) * metric_mu<3>(a.metric, tau, I1, S);
        nt_first<3>(a.metric, T, S, P);
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j) P[i][j] *= cw;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < N; ++k) {
          av[c][0][k] += tg[k] * P[c][0];
          av[c][1][k] += tb[k] * P[c][1];
          av[c][2][k] += tb[k] * P[c][2];
        }
    }
  } else if constexpr (KIND == K_VOLUME) {
    if (eg < a.ne) acc += dj * wq<3, Q>(t, q);
  }
}


template <int N, int Q, int KIND>
__global__ void __launch_bounds__(XlCfg<N, Q>::NT, XlCfg<N, Q>::template minb<KIND>())
    xl_kernel(const ElemArgs a, const __grid_constant__ Tab t) {
  using XC = XlCfg<N, Q>;
  constexpr bool APPLY = xl_qdata<KIND>();
  constexpr bool LDG = APPLY && XC::LDG;   // record fields loaded from global memory (n_q >= 7)
  constexpr bool BACK = xl_backward<KIND>();
  constexpr bool MASK = APPLY;          // the apply zeroes constrained inputs (operator.py:409)
  constexpr bool NTM = KIND == K_APPLY_NT;
  constexpr bool RSUM = KIND == K_ENERGY || KIND == K_VOLUME || KIND == K_GRAD;
  constexpr bool SD = KIND == K_SETUP_DIAG;
  constexpr bool RMIN = KIND == K_SETUP || SD || KIND == K_GRAD || KIND == K_ENERGY || KIND == K_MINDET;
  constexpr int EPB = XC::EPB, NP = XC::NP, QP = XC::QP, QS = XC::QS, NT = XC::NT;
  constexpr int U_QZ = XC::U_QZ, W_QY = XC::W_QY, W_QZ = XC::W_QZ;
  constexpr int XOFF = BACK ? XC::XOFF : XC::XOFF_F;
  constexpr int FOFF = BACK ? XC::FOFF : XC::FOFF_F;
  constexpr int BOFF = BACK ? XC::BOFF : XC::BOFF_F;
  extern __shared__ __align__(16) double smem[];
  double *U = smem;                       // U / Bv
  double *W = smem + XC::U_SZ * EPB;      // A (backward kinds)
  double *QB = smem + ((KIND == K_SETUP || SD) ? XC::QOFF_S : XC::QOFF);   // the group's lean Q-data (TMA-staged)
  __shared__ __align__(8) uint64_t qbar;
  __shared__ double red_v[(RSUM || RMIN) ? NT : 1];
  __shared__ int64_t red_i[RMIN ? NT : 1];

  if (a.stop && *a.stop) return;          // converged MINRES: the step is a no-op
  const int tid = threadIdx.x;
  const int e = tid % EPB;                // element slot of this thread (all stages)
  const int item = tid / EPB;
  double *QS_rec = QB + e * QS;           // setup: this thread's staged element record

  // per-stage roles (loop-invariant)
  const bool r1 = item < N * N;                 // F1 / B1: (ky, kx)
  const bool r2 = item < Q * N;                 // B2: (qz, kx)
  const int i2_kx = item % N, i2_qz = item / N;
  const int lqy = item % Q, lqz = item / Q;     // X stage: line (qy, qz); all threads
  const int line = item;

  // shared offsets (doubles) of each stage's item base
  const int o1 = item * EPB + e;                                     // U[..][qz=0][item]
  const int o2u = (i2_qz * U_QZ + i2_kx) * EPB + e;                 // U[..][qz][ky=0][kx]
  const int o2w = (i2_qz * W_QZ + i2_kx) * EPB + e;                 // A[..][qz][qy=0][kx]
  const int ox = (lqz * W_QZ + lqy * W_QY) * EPB + e;               // A[..][qz][qy][k=0]
  const int ou = lqz * U_QZ * EPB + e;                              // U[..][qz][ky=0][kx=0]
  double ty_b[N], ty_g[N];                                          // B, G rows of qy
#pragma unroll
  for (int k = 0; k < N; ++k) {
    ty_b[k] = t.B[lqy * N + k];
    ty_g[k] = t.G[lqy * N + k];
  }
  constexpr int UV = Q * U_QZ * EPB;      // U stride of v (c stride = 2 UV)
  constexpr int WV = Q * W_QZ * EPB;      // A stride of v3 (c stride = 3 WV)

  // ---- gather: asynchronous.  Every thread owns GJ (element, local node)
  // pairs of a group (element-fastest, matching the interleaved buffers);
  // the restriction indices of group g + 2 are loaded during group g, and
  // once F1 has consumed the gather buffer, cp.async copies in[c][node] (and,
  // for the apply, the 4-byte word holding fixed[node]) of group g + 1
  // straight into shared memory, landing during X / B2 / B1.
  double *XS = smem + XOFF;
  uint32_t *FS = reinterpret_cast<uint32_t *>(smem + FOFF);
  uint8_t *FB = reinterpret_cast<uint8_t *>(smem + BOFF);
  int nd[XC::GJ];
  auto load_index = [&](int64_t grp) {
#pragma unroll
    for (int j = 0; j < XC::GJ; ++j) {
      const int w = tid + j * NT;
      const int64_t eg = grp * EPB + w % EPB;
      nd[j] = (w < EPB * NP && grp < a.ngroups && eg < a.ne) ? __ldg(a.restr + eg * NP + w / EPB) : -1;
    }
  };
  auto issue_gather = [&]() {
#pragma unroll
    for (int j = 0; j < XC::GJ; ++j) {
      const int w = tid + j * NT;
      if (nd[j] >= 0) {
        const int ge = w % EPB, l = w / EPB;
        const int64_t node = nd[j];
#pragma unroll
        for (int c = 0; c < 3; ++c) cp_async8(XS + (c * NP + l) * EPB + ge, a.in + c * a.nn + node);
        if constexpr (MASK) {
          cp_async4(FS + l * EPB + ge, reinterpret_cast<const uint32_t *>(a.fixed + (node & ~(int64_t)3)));
          FB[l * EPB + ge] = (uint8_t)(8 * (node & 3));
        }
      }
    }
    cp_async_commit();
  };
  // ---- lean Q-data (apply): the group's EPB contiguous element records are
  // streamed into QB by one TMA bulk copy, issued one group ahead (after the
  // X stage has consumed the previous group's copy).
  auto issue = [&](int64_t grp) {
    const int64_t e0 = grp * EPB;
    const int64_t cnt = (a.ne - e0) < EPB ? (a.ne - e0) : EPB;
    const uint32_t bytes = (uint32_t)(cnt * QS * 8);
    mbar_expect_tx(&qbar, bytes);
    tma_load_1d(QB, a.qdata + e0 * QS, bytes, &qbar);
  };
  const double *qb = QB + e * QS + lqy + Q * lqz;   // field 0 of point (qx = 0) of this line (LDG: per group)
  auto qload = [&](int qx, double (&qd)[11]) {
#pragma unroll
    for (int f = 0; f < 11; ++f) qd[f] = LDG ? __ldg(qb + f * QP + Q * Q * qx) : qb[f * QP + Q * Q * qx];
  };
  uint32_t phase = 0;
  if constexpr (APPLY && !LDG) {
    if (tid == 0) {
      mbar_init(&qbar, 1);
      mbar_fence_init();
    }
    __syncthreads();
    if (tid == 0 && (int64_t)blockIdx.x < a.ngroups) issue(blockIdx.x);
  }
  double acc = 0.0;
  MinLoc mn{DBL_MAX, LLONG_MAX};

  load_index(blockIdx.x);
  issue_gather();
  load_index((int64_t)blockIdx.x + gridDim.x);
  for (int64_t grp = blockIdx.x; grp < a.ngroups; grp += gridDim.x) {
    const int64_t eg = grp * EPB + e;
    if constexpr (KIND == K_SETUP) {
      if (tid == 0) bulk_wait_read();   // previous group's record store has read QB
    }
    if constexpr (LDG) {
      // this line's record in global memory (and, with TMOP_XL_LDG_L2PF, the
      // next group's record block -> L2)
      qb = a.qdata + (grp * EPB + e) * QS + lqy + Q * lqz;
      const int64_t g2 = grp + gridDim.x;
      if (TMOP_XL_LDG_L2PF && tid == 0 && g2 < a.ngroups) {
        const int64_t e2 = g2 * EPB;
        const int64_t cnt = (a.ne - e2) < EPB ? (a.ne - e2) : EPB;
        l2_prefetch_bulk(a.qdata + e2 * QS, (uint32_t)(cnt * QS * 8));
      }
    }
    cp_async_wait_all();
    __syncthreads();
    // ---- F1: z-sweep of the gathered z-lines
    if (r1) {
      double xv[3][N];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const int l = k * N * N + item;
        if constexpr (MASK) {
          const uint32_t fw = FS[l * EPB + e] >> FB[l * EPB + e];
#pragma unroll
          for (int c = 0; c < 3; ++c) xv[c][k] = ((fw >> c) & 1u) ? 0.0 : XS[(c * NP + l) * EPB + e];
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) xv[c][k] = XS[(c * NP + l) * EPB + e];
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double *u = U + c * 2 * UV + o1;
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) {
          double sb = 0.0, sg = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            sb += tB<Q, N>(t, qz, k) * xv[c][k];
            sg += tG<Q, N>(t, qz, k) * xv[c][k];
          }
          u[qz * U_QZ * EPB] = sb;
          u[UV + qz * U_QZ * EPB] = sg;
        }
      }
    }
    __syncthreads();
    issue_gather();                             // group grp + grid: lands during X / B2 / B1
    load_index(grp + 2 * (int64_t)gridDim.x);   // consumed one group from now
    if constexpr (APPLY && !LDG) mbar_wait(&qbar, phase);   // this group's Q-data
    // ---- X: y-sweep of this line's row qy, x-sweep, point stage,
    // transposed x-sweep -- all in registers
    {
      // (per configuration: the n_q >= 7 action, 4 CTAs / SM; the gradient at
      // n_q = p + 2, 3 CTAs / SM: C3 p = 1 / 2 / 3 5.9 / 8.0 / 8.3 -> 5.4-5.5 /
      // 7.6-7.7 / 6.7 ms -- p = 3 spilled ~320 B with W in registers)
      constexpr bool WSM =
          BACK && (TMOP_XL_WSM == 1 || (TMOP_XL_WSM == -1 && ((LDG && N >= 3) || (KIND == K_GRAD && XC::GRAD3))));
      double wv[3][3][N], av[3][3][N];
      double *wo = W + ox;   // (WSM: this thread's own A slots hold W until the x^T output)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double *ub = U + c * 2 * UV + ou;
#pragma unroll
        for (int kx = 0; kx < N; ++kx) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
          for (int ky = 0; ky < N; ++ky) {
            const double vb = ub[(ky * N + kx) * EPB], vg = ub[UV + (ky * N + kx) * EPB];
            s0 += ty_b[ky] * vb;
            s1 += ty_g[ky] * vb;
            s2 += ty_b[ky] * vg;
          }
          if constexpr (WSM) {
            wo[(c * 3 + 0) * WV + kx * EPB] = s0;
            wo[(c * 3 + 1) * WV + kx * EPB] = s1;
            wo[(c * 3 + 2) * WV + kx * EPB] = s2;
          } else {
            wv[c][0][kx] = s0;
            wv[c][1][kx] = s1;
            wv[c][2][kx] = s2;
          }
          av[c][0][kx] = av[c][1][kx] = av[c][2][kx] = 0.0;
        }
      }
      constexpr bool QPF = APPLY && (TMOP_XL_QPF == 1 || (TMOP_XL_QPF == -1 && (N == 4 || LDG)));
      double qnext[11];
      if constexpr (QPF) qload(0, qnext);
      // (fully unrolled for p <= 2: C3 p = 1 / 2 action 6.57 -> 5.90 / 7.37 -> 7.30 ms,
      // setup, gradient and energy 2-18 % faster; p = 3: fully unrolled the
      // action spills, 6.23 -> 7.44 ms, by 2 6.23 -> 6.14 ms)
      constexpr int QXU = TMOP_XL_QX_UNROLL ? TMOP_XL_QX_UNROLL
                          : XC::LDG ? 1
                          : N >= 4 ? (KIND == K_APPLY ? TMOP_XL_P3_APPLY_UNROLL
                                                      : KIND == K_GRAD ? TMOP_XL_P3_GRAD_UNROLL : 1)
                                   : Q;
#pragma unroll QXU
      for (int qx = 0; qx < Q; ++qx) {
        double tg[N], tb[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          tg[k] = tG<Q, N>(t, qx, k);
          tb[k] = tB<Q, N>(t, qx, k);
        }
        double g[3][3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            if constexpr (WSM) {
              s0 += tg[k] * wo[(c * 3 + 0) * WV + k * EPB];
              s1 += tb[k] * wo[(c * 3 + 1) * WV + k * EPB];
              s2 += tb[k] * wo[(c * 3 + 2) * WV + k * EPB];
            } else {
              s0 += tg[k] * wv[c][0][k];
              s1 += tb[k] * wv[c][1][k];
              s2 += tb[k] * wv[c][2][k];
            }
          }
          g[c][0] = s0;
          g[c][1] = s1;
          g[c][2] = s2;
        }
        if constexpr (APPLY) {
          double qd[11];
          if constexpr (QPF) {
            // this point's record was loaded during the previous point; fetch the next one now
#pragma unroll
            for (int f = 0; f < 11; ++f) qd[f] = qnext[f];
            if (qx + 1 < Q) qload(qx + 1, qnext);
          } else {
            qload(qx, qd);
          }
          xl_point<N, NTM>(a.metric, qd, g, tg, tb, av);
        } else {
          xl_point_x<SD ? K_SETUP : KIND, N, Q>(a, t, eg, line, qx, g, tg, tb, av, acc, mn, QS_rec);
        }
      }
      if constexpr (BACK) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int v = 0; v < 3; ++v)
#pragma unroll
            for (int k = 0; k < N; ++k) W[(c * 3 + v) * WV + ox + k * EPB] = av[c][v][k];
      }
    }
    if constexpr (BACK) {
      __syncthreads();
      if constexpr (APPLY && !LDG) {
        // QB is free again: stream in the next group's Q-data
        phase ^= 1u;
        if (tid == 0 && grp + gridDim.x < a.ngroups) issue(grp + gridDim.x);
      }
      // ---- B2: y^T sweep  A -> Bv (U region)
      if (r2) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double *A = W + c * 3 * WV + o2w;
          double a0[Q], a1[Q], a2[Q];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            a0[q] = A[q * W_QY * EPB];
            a1[q] = A[WV + q * W_QY * EPB];
            a2[q] = A[2 * WV + q * W_QY * EPB];
          }
          double *b = U + c * 2 * UV + o2u;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              s0 += tB<Q, N>(t, q, k) * a0[q] + tG<Q, N>(t, q, k) * a1[q];
              s1 += tB<Q, N>(t, q, k) * a2[q];
            }
            b[k * N * EPB] = s0;
            b[UV + k * N * EPB] = s1;
          }
        }
      }
      __syncthreads();
      // ---- B1: z^T sweep -> element-interleaved E-vector
      if (r1) {
        double *out = a.E + (grp * 3 * NP + item) * EPB + e;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double *b = U + c * 2 * UV + o1;
          double b0[Q], b1[Q];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            b0[q] = b[q * U_QZ * EPB];
            b1[q] = b[UV + q * U_QZ * EPB];
          }
#pragma unroll
          for (int k = 0; k < N; ++k) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < Q; ++q) s += tB<Q, N>(t, q, k) * b0[q] + tG<Q, N>(t, q, k) * b1[q];
            out[(c * NP + k * N * N) * EPB] = s;
          }
        }
      }
    }
    if constexpr (KIND == K_SETUP || SD) {
      // the group's records are complete in QB: one TMA bulk store
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        const int64_t e0 = grp * EPB;
        const int64_t cnt = (a.ne - e0) < EPB ? (a.ne - e0) : EPB;
        bulk_store(a.qout + e0 * QS, QB, (uint32_t)(cnt * QS * 8));
      }
    }
    if constexpr (SD) {
      // the diagonal (operator.py:420-459) from the records still in shared
      // memory (tmop_xld_parts.cuh): no re-read of the record from HBM
      double dacc[3][6][N];
      xld_line<N, Q, false>(a.metric, QB + e * QS + line, t, dacc);
      if (tid == 0) bulk_wait_read();   // the store has read QB ...
      __syncthreads();                  // ... and so has every thread: A may overlay it
      xld_store_a<N, Q>(QB, line, e, dacc);
      __syncthreads();
      if (item < Q * N) xld_y<N, Q>(QB, QB + XldCfg<N, Q>::R1OP, item, e, t);
      __syncthreads();
      if (item < N * N) xld_z<N, Q>(QB + XldCfg<N, Q>::R1OP, a.E, grp, item, e, t);
    }
    // (no end-of-group barrier: the top-of-loop barrier orders this group's
    // reads of U / Bv before the next F1 writes U)
  }
  if constexpr (KIND == K_SETUP || SD) {
    if (tid == 0) bulk_wait_all();
  }

  // ---- per-CTA deterministic partials
  if constexpr (RSUM) {
    const double sum = xl_block_sum<NT>(acc, red_v);
    if (tid == 0) a.part_sum[blockIdx.x] = sum;
  }
  if constexpr (RMIN) {
    const MinLoc m = xl_block_minloc<NT>(mn, red_v, red_i);
    if (tid == 0) {
      a.part_min[blockIdx.x] = m.v;
      a.part_arg[blockIdx.x] = m.i;
    }
  }
}

}  // namespace tmop
