// tmop_core.cu -- mesh-level kernels: deterministic E->L gather-sum, the
// fixed-order finalisation of per-CTA partials, pointwise metric
// evaluation, and the fused vector kernels of the device MINRES.
#include <cfloat>
#include <climits>
#include <cmath>

#include "../../include/tmop_b200.h"
#include "tmop_core.h"
#include "tmop_elem.cuh"

namespace tmop {

// ---------------------------------------------------------------- E -> L
// y[c][node] = sum over the node's element copies, ascending element order
// (np.add.at order, fe.py:189-204).  mode: 0 = apply (constrained entries
// copy v, operator.py:417), 1 = gradient (constrained -> 0, operator.py:345),
// 2 = diagonal (constrained -> 1, operator.py:458).  `add` (may be NULL) is
// an extra T-vector added before the constraint fix-up (limiting term).
// E layout: element groups of 2^es elements interleaved (element fastest):
// E[((e >> es) * D * np + c * np + l) << es | (e & (2^es - 1))]; es = 0 is
// the plain element-blocked layout E[e][c][l].
__device__ __forceinline__ const double *e_src(const double *E, uint32_t u, int np, int D, int es, int64_t &cs) {
  const uint32_t e = u / (uint32_t)np, l = u - e * (uint32_t)np;
  cs = (int64_t)np << es;
  return E + ((((int64_t)(e >> es) * D * np + l) << es) | (int64_t)(e & ((1u << es) - 1u)));
}

template <int D>
__global__ void e2l_kernel(int64_t nn, int np, int es, const int64_t *__restrict__ off, const uint32_t *__restrict__ idx,
                           const double *__restrict__ E, const uint8_t *__restrict__ fixed, int mode,
                           const double *__restrict__ v, const double *__restrict__ add, double *__restrict__ y) {
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int64_t b = off[node], end = off[node + 1];
  double acc[D];
#pragma unroll
  for (int c = 0; c < D; ++c) acc[c] = 0.0;
  for (int64_t k = b; k < end; ++k) {
    int64_t cs;
    const double *src = e_src(E, __ldg(idx + k), np, D, es, cs);
#pragma unroll
    for (int c = 0; c < D; ++c) acc[c] += __ldg(src + c * cs);
  }
  const uint8_t f = __ldg(fixed + node);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const int64_t i = c * nn + node;
    double r = acc[c];
    if (add) r += add[i];
    if ((f >> c) & 1) r = (mode == 0) ? v[i] : (mode == 1 ? 0.0 : 1.0);
    y[i] = r;
  }
}

int launch_e2l(int dim, int64_t nn, int np, int es, const int64_t *off, const uint32_t *idx, const double *E,
               const uint8_t *fixed, int mode, const double *v, const double *add, double *y, cudaStream_t s) {
  const int nt = 256;
  const int64_t grid = (nn + nt - 1) / nt;
  if (grid == 0) return 0;
  if (dim == 2)
    e2l_kernel<2><<<(unsigned)grid, nt, 0, s>>>(nn, np, es, off, idx, E, fixed, mode, v, add, y);
  else
    e2l_kernel<3><<<(unsigned)grid, nt, 0, s>>>(nn, np, es, off, idx, E, fixed, mode, v, add, y);
  return 0;
}

// ------------------------------------------------------- finalisation
// One CTA reduces the per-CTA partials in a fixed order.
__global__ void fin_kernel(int nparts, const double *__restrict__ psum, const double *__restrict__ pmin,
                           const int64_t *__restrict__ parg, double sum_scale, double *__restrict__ sum_out,
                           double sum_add_scale, const double *__restrict__ sum_add,
                           tmop_det_status *__restrict__ det_out) {
  __shared__ double sv[32];
  __shared__ int64_t si[32];
  if (psum) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += psum[i];
    s = block_sum<1024>(s, sv);
    if (threadIdx.x == 0) {
      double r = sum_scale * s;
      if (sum_add) r += sum_add_scale * sum_add[0];
      sum_out[0] = r;
    }
  }
  if (pmin) {
    MinLoc m{DBL_MAX, LLONG_MAX};
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) m = minloc(m, MinLoc{pmin[i], parg[i]});
    m = block_minloc<1024>(m, sv, si);
    if (threadIdx.x == 0) {
      det_out->min_det = m.v;
      det_out->argmin = m.i;
    }
  }
}

void launch_fin(int nparts, const double *psum, const double *pmin, const int64_t *parg, double sum_scale,
                double *sum_out, double add_scale, const double *add, tmop_det_status *det_out, cudaStream_t s) {
  fin_kernel<<<1, 1024, 0, s>>>(nparts, psum, pmin, parg, sum_scale, sum_out, add_scale, add, det_out);
}

// -------------------------------------------------------- metric eval
template <int D>
__global__ void metric_eval_kernel(int metric, int64_t n, const double *__restrict__ Tin, double *mu, double *P,
                                   double *H) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double T[D][D];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) T[i][j] = Tin[k * D * D + i * D + j];
  const double tau = mdet<D>(T);
  const double I1 = mfro2<D>(T);
  double C[D][D], S[D][D];
  mcof<D>(T, C);
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) S[i][j] = C[i][j] / tau;
  if (mu) mu[k] = metric_mu<D>(metric, tau, I1, S);
  const bool tmpl = metric_is_template(metric);
  if (P) {
    double Pm[D][D];
    if (tmpl) {
      double at, as;
      metric_first_coeffs(metric, tau, I1, at, as);
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) Pm[i][j] = at * T[i][j] + as * S[i][j];
    } else {
      nt_first<D>(metric, T, S, Pm);
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) P[k * D * D + i * D + j] = Pm[i][j];
  }
  if (H) {
    double c[4];
    if (tmpl) metric_second_coeffs(metric, tau, I1, c);
    for (int col = 0; col < D * D; ++col) {
      double g[D][D] = {}, z[D][D];
      g[col / D][col % D] = 1.0;
      if (tmpl)
        hess_template<D>(c, S, T, g, z);
      else
        nt_hess<D>(metric, 1.0, S, T, g, z);
      for (int row = 0; row < D * D; ++row) H[(k * D * D + row) * D * D + col] = z[row / D][row % D];
    }
  }
}

int launch_metric_eval(int metric, int dim, int64_t n, const double *T, double *mu, double *P, double *H) {
  if (n <= 0) return 0;
  const int nt = 128;
  const unsigned grid = (unsigned)((n + nt - 1) / nt);
  if (dim == 2)
    metric_eval_kernel<2><<<grid, nt>>>(metric, n, T, mu, P, H);
  else
    metric_eval_kernel<3><<<grid, nt>>>(metric, n, T, mu, P, H);
  return 0;
}

// -------------------------------------------------------- vector ops
// Grid of the vector kernels: a fixed function of n (determinism).
int vec_grid(int64_t n) {
  const int64_t g = (n + VEC_NT * 4 - 1) / (VEC_NT * 4);
  return (int)(g < 1 ? 1 : (g > VEC_GRID_CAP ? VEC_GRID_CAP : g));
}

// Every CTA re-reduces the same partial array in the same fixed order, so
// all CTAs obtain the bitwise-identical scalar without a grid barrier.
__device__ __forceinline__ double reduce_partials(const double *__restrict__ part, int np, double *sv) {
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += VEC_NT) s += part[i];
  s = block_sum<VEC_NT>(s, sv);
  __shared__ double bc;
  if (threadIdx.x == 0) bc = s;
  __syncthreads();
  return bc;
}

__global__ void __launch_bounds__(VEC_NT) dot_kernel(int64_t n, const double *__restrict__ a,
                                                     const double *__restrict__ b, double *__restrict__ part) {
  __shared__ double sv[VEC_NT / 32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT)
    s += a[i] * b[i];
  s = block_sum<VEC_NT>(s, sv);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_partials_kernel(int np, const double *__restrict__ part, double *__restrict__ out) {
  __shared__ double sv[VEC_NT / 32];
  const double s = reduce_partials(part, np, sv);
  if (threadIdx.x == 0) out[0] = s;
}

void launch_dot(int64_t n, const double *a, const double *b, double *part, double *out, cudaStream_t s) {
  const int g = vec_grid(n);
  dot_kernel<<<g, VEC_NT, 0, s>>>(n, a, b, part);
  sum_partials_kernel<<<1, VEC_NT, 0, s>>>(g, part, out);
}

__global__ void axpby_kernel(int64_t n, double a, const double *__restrict__ x, double b, double *__restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT)
    y[i] = a * x[i] + b * y[i];
}
void launch_axpby(int64_t n, double a, const double *x, double b, double *y, cudaStream_t s) {
  axpby_kernel<<<vec_grid(n), VEC_NT, 0, s>>>(n, a, x, b, y);
}

__global__ void trial_kernel(int64_t n, const double *__restrict__ x, const double *__restrict__ dx, double alpha,
                             double *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT)
    out[i] = x[i] - alpha * dx[i];
}
void launch_trial(int64_t n, const double *x, const double *dx, double alpha, double *out, cudaStream_t s) {
  trial_kernel<<<vec_grid(n), VEC_NT, 0, s>>>(n, x, dx, alpha, out);
}

__global__ void jacobi_kernel(int64_t n, const double *__restrict__ d, double fl, double *__restrict__ inv,
                              int32_t *__restrict__ nonfinite) {
  for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT) {
    const double v = d[i];
    if (!isfinite(v)) *nonfinite = 1;
    inv[i] = 1.0 / fmax(fabs(v), fl);
  }
}
void launch_jacobi(int64_t n, const double *d, double fl, double *inv, int32_t *nonfinite, cudaStream_t s) {
  jacobi_kernel<<<vec_grid(n), VEC_NT, 0, s>>>(n, d, fl, inv, nonfinite);
}

// ------------------------------------------------------------- MINRES
// Reference recurrence: solvers.py:117-178.  Scalars live in device
// memory; two state slots alternate by iteration parity so that the CTAs of
// the last fused kernel can all read the old state while CTA 0 writes the
// new one.
__global__ void __launch_bounds__(VEC_NT) minres_init_kernel(int64_t n, const double *__restrict__ b,
                                                             const double *__restrict__ inv, double *x, double *r1,
                                                             double *r2, double *z, double *w, double *w2,
                                                             double *__restrict__ part) {
  __shared__ double sv[VEC_NT / 32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT) {
    const double bi = b[i];
    const double zi = inv ? inv[i] * bi : bi;
    r1[i] = bi;
    r2[i] = bi;
    z[i] = zi;
    x[i] = 0.0;
    w[i] = 0.0;
    w2[i] = 0.0;
    s += bi * zi;
  }
  s = block_sum<VEC_NT>(s, sv);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(VEC_NT) minres_init2_kernel(int64_t n, const double *__restrict__ z,
                                                              double *__restrict__ v,
                                                              const double *__restrict__ part, int np,
                                                              tmop_minres_state *st) {
  __shared__ double sv[VEC_NT / 32];
  const double b2 = reduce_partials(part, np, sv);
  const double beta1 = sqrt(fmax(b2, 0.0));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    tmop_minres_state s;
    s.beta1 = beta1;
    s.beta = beta1;
    s.oldb = 0.0;
    s.alfa = 0.0;
    s.beta2 = b2;
    s.dbar = 0.0;
    s.epsln = 0.0;
    s.sn = 0.0;
    s.cs = -1.0;
    s.phibar = beta1;
    s.relres = 1.0;
    s.gamma = 0.0;
    s.itn = 0;
    s.nonpd = b2 < 0.0;
    s.done = (b2 < 0.0) || (beta1 == 0.0);
    s.breakdown = 0;
    st[0] = s;
  }
  if (beta1 == 0.0 || b2 < 0.0) return;
  for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT)
    v[i] = z[i] / beta1;
}

// K1: Av -= (beta/oldb) r1 (itn >= 2); partial alfa = v . Av
__global__ void __launch_bounds__(VEC_NT) minres_k1(int64_t n, double *__restrict__ Av, const double *__restrict__ r1,
                                                    const double *__restrict__ v, const tmop_minres_state *cur,
                                                    double *__restrict__ part) {
  if (cur->done) return;
  __shared__ double sv[VEC_NT / 32];
  const bool sub = cur->itn >= 1;
  const double f = sub ? cur->beta / cur->oldb : 0.0;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT) {
    double y = Av[i];
    if (sub) {
      y = y - f * r1[i];
      Av[i] = y;
    }
    s += v[i] * y;
  }
  s = block_sum<VEC_NT>(s, sv);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// K2: alfa = sum(part1); Av -= (alfa/beta) r2; z = inv .* Av; partial beta2 = Av . z
__global__ void __launch_bounds__(VEC_NT) minres_k2(int64_t n, double *__restrict__ Av, const double *__restrict__ r2,
                                                    const double *__restrict__ inv, double *__restrict__ z,
                                                    const tmop_minres_state *cur, const double *__restrict__ part1,
                                                    double *__restrict__ part2, int np) {
  if (cur->done) return;
  __shared__ double sv[VEC_NT / 32];
  const double alfa = reduce_partials(part1, np, sv);
  const double f = alfa / cur->beta;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT) {
    const double y = Av[i] - f * r2[i];
    Av[i] = y;
    const double zi = inv ? inv[i] * y : y;
    z[i] = zi;
    s += y * zi;
  }
  s = block_sum<VEC_NT>(s, sv);
  if (threadIdx.x == 0) part2[blockIdx.x] = s;
}

// K3: beta2 = sum(part2); Givens recurrence; w_new (into w1buf); x += phi w_new; v = z / beta
__global__ void __launch_bounds__(VEC_NT) minres_k3(int64_t n, const double *__restrict__ z, double *__restrict__ v,
                                                    const double *__restrict__ w, double *__restrict__ w1buf,
                                                    const double *__restrict__ w2, double *__restrict__ x,
                                                    const tmop_minres_state *cur, tmop_minres_state *nxt,
                                                    const double *__restrict__ part1,
                                                    const double *__restrict__ part2, int np, double rtol,
                                                    double *__restrict__ hist, int hist_cap) {
  const tmop_minres_state c = *cur;
  if (c.done) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *nxt = c;
    return;
  }
  __shared__ double sv[VEC_NT / 32];
  const double alfa = reduce_partials(part1, np, sv);
  const double beta2 = reduce_partials(part2, np, sv);
  tmop_minres_state s = c;
  s.itn = c.itn + 1;
  s.alfa = alfa;
  s.beta2 = beta2;
  s.oldb = c.beta;
  if (beta2 < 0.0) {  // solvers.py:141-142: preconditioner not positive definite
    s.nonpd = 1;
    s.done = 1;
    if (blockIdx.x == 0 && threadIdx.x == 0) *nxt = s;
    return;
  }
  const double beta = sqrt(beta2);
  s.beta = beta;
  const double oldeps = c.epsln;
  const double delta = c.cs * c.dbar + c.sn * alfa;
  const double gbar = c.sn * c.dbar - c.cs * alfa;
  s.epsln = c.sn * beta;
  s.dbar = -c.cs * beta;
  const double gamma = fmax(hypot(gbar, beta), DBL_EPSILON);
  s.gamma = gamma;
  s.cs = gbar / gamma;
  s.sn = beta / gamma;
  const double phi = s.cs * c.phibar;
  s.phibar = s.sn * c.phibar;
  s.relres = s.phibar / c.beta1;
  const double rg = 1.0 / gamma;  // (v - oldeps w1 - delta w2) / gamma, solvers.py:158
  (void)rg;
  for (int64_t i = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VEC_NT) {
    const double vi = v[i];
    const double wn = (vi - oldeps * w2[i] - delta * w[i]) / gamma;
    w1buf[i] = wn;
    x[i] = x[i] + phi * wn;
    v[i] = z[i] / beta;
  }
  if (beta == 0.0) {
    s.breakdown = 1;
    s.done = 1;
  } else if (s.relres <= rtol) {
    s.done = 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *nxt = s;
    if (hist && s.itn < hist_cap) hist[s.itn] = s.relres;   // residual history (solvers.py:168-176)
  }
}

void launch_minres_init(int64_t n, const double *b, const double *inv, double *x, double *r1, double *r2, double *z,
                        double *v, double *w, double *w2, double *part, tmop_minres_state *st, cudaStream_t s) {
  const int g = vec_grid(n);
  minres_init_kernel<<<g, VEC_NT, 0, s>>>(n, b, inv, x, r1, r2, z, w, w2, part);
  minres_init2_kernel<<<g, VEC_NT, 0, s>>>(n, z, v, part, g, st);
}

// Fused E->L gather + MINRES K1 for the TMOP operator (one pass over Av
// instead of a gather write followed by a K1 read-modify-write):
//   Av[i] = (fixed ? v : sum_E) ; Av -= (beta/oldb) r1 (itn >= 2) ; alfa partial v.Av
// Grid = vec_grid(n), grid-stride over nodes, so the partial array has the
// same length the following K2 / K3 expect.
template <int D>
__global__ void __launch_bounds__(VEC_NT) e2l_minres_k1(int64_t nn, int np, int es, const int64_t *__restrict__ off,
                                                        const uint32_t *__restrict__ idx, const double *__restrict__ E,
                                                        const uint8_t *__restrict__ fixed, const double *__restrict__ v,
                                                        const double *__restrict__ r1, double *__restrict__ Av,
                                                        const tmop_minres_state *cur, double *__restrict__ part) {
  if (cur->done) return;
  __shared__ double sv[VEC_NT / 32];
  const bool sub = cur->itn >= 1;
  const double f = sub ? cur->beta / cur->oldb : 0.0;
  double s = 0.0;
  for (int64_t node = (int64_t)blockIdx.x * VEC_NT + threadIdx.x; node < nn; node += (int64_t)gridDim.x * VEC_NT) {
    double acc[D];
#pragma unroll
    for (int c = 0; c < D; ++c) acc[c] = 0.0;
    for (int64_t k = off[node]; k < off[node + 1]; ++k) {
      int64_t cs;
      const double *src = e_src(E, __ldg(idx + k), np, D, es, cs);
#pragma unroll
      for (int c = 0; c < D; ++c) acc[c] += __ldg(src + c * cs);
    }
    const uint8_t fl = __ldg(fixed + node);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const int64_t i = c * nn + node;
      const double vi = v[i];
      double y = ((fl >> c) & 1) ? vi : acc[c];
      if (sub) y = y - f * r1[i];
      Av[i] = y;
      s += vi * y;
    }
  }
  s = block_sum<VEC_NT>(s, sv);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

void launch_minres_step_op(int dim, int64_t nn, int np, int es, const int64_t *off, const uint32_t *idx, const double *E,
                           const uint8_t *fixed, int64_t n, double *Av, const double *r1, const double *r2,
                           const double *inv, double *z, double *v, const double *w, double *w1buf, const double *w2,
                           double *x, double rtol, tmop_minres_state *cur, tmop_minres_state *nxt, double *part1,
                           double *part2, double *hist, int hist_cap, cudaStream_t s) {
  const int g = vec_grid(n);
  if (dim == 2)
    e2l_minres_k1<2><<<g, VEC_NT, 0, s>>>(nn, np, es, off, idx, E, fixed, v, r1, Av, cur, part1);
  else
    e2l_minres_k1<3><<<g, VEC_NT, 0, s>>>(nn, np, es, off, idx, E, fixed, v, r1, Av, cur, part1);
  minres_k2<<<g, VEC_NT, 0, s>>>(n, Av, r2, inv, z, cur, part1, part2, g);
  minres_k3<<<g, VEC_NT, 0, s>>>(n, z, v, w, w1buf, w2, x, cur, nxt, part1, part2, g, rtol, hist, hist_cap);
}

void launch_minres_step(int64_t n, double *Av, const double *r1, const double *r2, const double *inv, double *z,
                        double *v, const double *w, double *w1buf, const double *w2, double *x, double rtol,
                        tmop_minres_state *cur, tmop_minres_state *nxt, double *part1, double *part2,
                        double *hist, int hist_cap, cudaStream_t s) {
  const int g = vec_grid(n);
  minres_k1<<<g, VEC_NT, 0, s>>>(n, Av, r1, v, cur, part1);
  minres_k2<<<g, VEC_NT, 0, s>>>(n, Av, r2, inv, z, cur, part1, part2, g);
  minres_k3<<<g, VEC_NT, 0, s>>>(n, z, v, w, w1buf, w2, x, cur, nxt, part1, part2, g, rtol, hist, hist_cap);
}

}  // namespace tmop
