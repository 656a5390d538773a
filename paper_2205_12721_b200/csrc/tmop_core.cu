// tmop_core.cu -- mesh-level kernels: deterministic E->L gather-sum, the
// fixed-order finalisation of per-CTA partials, pointwise metric
// evaluation, and the fused vector kernels of the device MINRES.
#include <algorithm>
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
// 2 = diagonal (constrained -> 1, operator.py:458), 3 = raw sums (no fix-up;
// the limiting term's node sums).  `add` (may be NULL) is
// an extra T-vector added before the constraint fix-up (limiting term).
// E layout: element groups of 2^es elements interleaved (element fastest):
// E[((e >> es) * D * np + c * np + l) << es | (e & (2^es - 1))]; es = 0 is
// the plain element-blocked layout E[e][c][l].
__device__ __forceinline__ const double *e_src(const double *E, uint32_t u, int np, int D, int es, int64_t &cs) {
  const uint32_t e = u / (uint32_t)np, l = u - e * (uint32_t)np;
  cs = (int64_t)np << es;
  return E + ((((int64_t)(e >> es) * D * np + l) << es) | (int64_t)(e & ((1u << es) - 1u)));
}

// Copies of lattice node index i along one axis of a box with `ncell`
// elements of order p: (element, local) pairs in ascending element order.
struct LatAxis {
  int e[2], l[2], n;
};
__device__ __forceinline__ void lat_axis(int i, int ncell, int p, LatAxis &o) {
  const int q = i / p, r = i - q * p;
  o.e[1] = o.l[1] = 0;
  if (r != 0) {
    o.n = 1; o.e[0] = q; o.l[0] = r;
  } else if (q == 0) {
    o.n = 1; o.e[0] = 0; o.l[0] = 0;
  } else if (q == ncell) {
    o.n = 1; o.e[0] = q - 1; o.l[0] = p;
  } else {
    o.n = 2; o.e[0] = q - 1; o.l[0] = p; o.e[1] = q; o.l[1] = 0;
  }
}

// Sum of the E copies of `node` (all D components) in ascending element
// order -- through the transpose map, or arithmetically on a lattice.
template <int D, bool LAT>
__device__ __forceinline__ void e2l_node(int64_t node, const E2LMap &m, const double *__restrict__ E,
                                         double (&acc)[D]) {
#pragma unroll
  for (int c = 0; c < D; ++c) acc[c] = 0.0;
  if constexpr (LAT) {
    static_assert(D == 3, "lattice E->L is 3D");
    const int p = m.lat_p, n1 = p + 1;
    const uint32_t NX = (uint32_t)m.lat_n[0] * p + 1, NY = (uint32_t)m.lat_n[1] * p + 1;
    const uint32_t nd = (uint32_t)node;
    const uint32_t t = (uint32_t)(((uint64_t)nd * m.mag_x) >> m.sh_x);      // nd / NX
    const uint32_t iz = (uint32_t)(((uint64_t)t * m.mag_y) >> m.sh_y);     // t / NY
    const int ix = (int)(nd - t * NX), iy = (int)(t - iz * NY);
    LatAxis ax, ay, az;
    lat_axis(ix, m.lat_n[0], p, ax);
    lat_axis(iy, m.lat_n[1], p, ay);
    lat_axis((int)iz, m.lat_n[2], p, az);
    const int64_t cs = (int64_t)m.np << m.es;
    const uint32_t msk = (1u << m.es) - 1u;
    // all (up to 8) copies' loads are issued before any is summed; the sum
    // then runs in ascending element order (z, y, x lexicographic)
    double val[8][D];
#pragma unroll
    for (int kz = 0; kz < 2; ++kz)
#pragma unroll
      for (int ky = 0; ky < 2; ++ky)
#pragma unroll
        for (int kx = 0; kx < 2; ++kx) {
          const int k = (kz * 2 + ky) * 2 + kx;
          if (kz < az.n && ky < ay.n && kx < ax.n) {
            const uint32_t e = ax.e[kx] + (uint32_t)m.lat_n[0] * (ay.e[ky] + (uint32_t)m.lat_n[1] * az.e[kz]);
            const int l = ax.l[kx] + n1 * (ay.l[ky] + n1 * az.l[kz]);
            const double *src = E + (((((int64_t)(e >> m.es)) * D * m.np + l) << m.es) | (int64_t)(e & msk));
#pragma unroll
            for (int c = 0; c < D; ++c) val[k][c] = __ldg(src + c * cs);
          }
        }
#pragma unroll
    for (int kz = 0; kz < 2; ++kz)
#pragma unroll
      for (int ky = 0; ky < 2; ++ky)
#pragma unroll
        for (int kx = 0; kx < 2; ++kx) {
          const int k = (kz * 2 + ky) * 2 + kx;
          if (kz < az.n && ky < ay.n && kx < ax.n) {
#pragma unroll
            for (int c = 0; c < D; ++c) acc[c] += val[k][c];
          }
        }
  } else {
    const int64_t b = m.off[node], end = m.off[node + 1];
    for (int64_t k = b; k < end; ++k) {
      int64_t cs;
      const double *src = e_src(E, __ldg(m.idx + k), m.np, D, m.es, cs);
#pragma unroll
      for (int c = 0; c < D; ++c) acc[c] += __ldg(src + c * cs);
    }
  }
}

template <int D, bool LAT>
__global__ void e2l_kernel(int64_t nn, int64_t n0, int64_t n1, const E2LMap m, const double *__restrict__ E,
                           const uint8_t *__restrict__ fixed, int mode, const double *__restrict__ v,
                           const double *__restrict__ add, double *__restrict__ y) {
  const int64_t node = n0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= n1) return;
  double acc[D];
  e2l_node<D, LAT>(node, m, E, acc);
  const uint8_t f = __ldg(fixed + node);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const int64_t i = c * nn + node;
    double r = acc[c];
    if (add) r += add[i];
    if (mode != 3 && ((f >> c) & 1)) r = (mode == 0) ? v[i] : (mode == 1 ? 0.0 : 1.0);
    y[i] = r;
  }
}

int launch_e2l(int dim, int64_t nn, const E2LMap &m, const double *E, const uint8_t *fixed, int mode, const double *v,
               const double *add, double *y, cudaStream_t s, int64_t n0, int64_t n1, int nt) {
  if (n1 < 0) n1 = nn;
  const int64_t grid = (n1 - n0 + nt - 1) / nt;
  if (grid <= 0) return 0;
  if (dim == 2)
    e2l_kernel<2, false><<<(unsigned)grid, nt, 0, s>>>(nn, n0, n1, m, E, fixed, mode, v, add, y);
  else if (m.lat_p > 0)
    e2l_kernel<3, true><<<(unsigned)grid, nt, 0, s>>>(nn, n0, n1, m, E, fixed, mode, v, add, y);
  else
    e2l_kernel<3, false><<<(unsigned)grid, nt, 0, s>>>(nn, n0, n1, m, E, fixed, mode, v, add, y);
  return 0;
}

// Verifies that a restriction is the box lattice of build_box (mesh.py:118-164):
// node(e, l) = sum_a (e_a p + l_a) stride_a.  Any mismatch sets *flag.
__global__ void lattice_check_kernel(int64_t ne, int np, const int32_t *__restrict__ restr, int nx, int ny, int nz,
                                     int p, int *flag) {
  const int n1 = p + 1;
  const int64_t NX = (int64_t)nx * p + 1, NY = (int64_t)ny * p + 1;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < ne * np; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = k / np;
    const int l = (int)(k - e * np);
    const int64_t ex = e % nx, ey = (e / nx) % ny, ez = e / ((int64_t)nx * ny);
    const int lx = l % n1, ly = (l / n1) % n1, lz = l / (n1 * n1);
    const int64_t want = (ex * p + lx) + NX * ((ey * p + ly) + NY * (ez * p + lz));
    if (ez >= nz || (int64_t)__ldg(restr + k) != want) atomicOr(flag, 1);
  }
}

int launch_lattice_check(int64_t ne, int np, const int32_t *restr, int nx, int ny, int nz, int p, int *flag,
                         cudaStream_t s) {
  lattice_check_kernel<<<148 * 8, 256, 0, s>>>(ne, np, restr, nx, ny, nz, p, flag);
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
// Dot products of a slab partition count each shared node plane once: entry
// i of a component-major (D, nn) local vector is OWNED when its node
// (i mod nn) < n_owned.  nn == 0: every entry is owned (single GPU).
struct Own {
  int64_t nn, n_owned;
  __device__ __forceinline__ bool operator()(int64_t i) const {
    if (nn == 0) return true;
    while (i >= nn) i -= nn;
    return i < n_owned;
  }
};

// Reference recurrence: solvers.py:117-178.  Scalars live in device
// memory; two state slots alternate by iteration parity so that the CTAs of
// the last fused kernel can all read the old state while CTA 0 writes the
// new one.
__global__ void __launch_bounds__(VEC_NT) minres_init_kernel(int64_t n, const double *__restrict__ b,
                                                             const double *__restrict__ inv, double *x, double *r1,
                                                             double *r2, double *z, double *w, double *w2,
                                                             double *__restrict__ part, const Own own) {
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
    if (own(i)) s += bi * zi;
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
                                                    double *__restrict__ part, const Own own) {
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
    if (own(i)) s += v[i] * y;
  }
  s = block_sum<VEC_NT>(s, sv);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// K2: alfa = sum(part1); Av -= (alfa/beta) r2; z = inv .* Av; partial beta2 = Av . z
// V2: 16-byte vector accesses over element pairs (all pointers 16-byte
// aligned; an odd tail element is taken by global thread 0).
template <bool V2>
__global__ void __launch_bounds__(VEC_NT) minres_k2(int64_t n, double *__restrict__ Av, const double *__restrict__ r2,
                                                    const double *__restrict__ inv, double *__restrict__ z,
                                                    const tmop_minres_state *cur, const double *__restrict__ part1,
                                                    int np1, double *__restrict__ part2, const Own own) {
  if (cur->done) return;
  __shared__ double sv[VEC_NT / 32];
  const double alfa = reduce_partials(part1, np1, sv);
  const double f = alfa / cur->beta;
  double s = 0.0;
  auto one = [&](int64_t i) {
    const double y = Av[i] - f * r2[i];
    Av[i] = y;
    const double zi = inv ? inv[i] * y : y;
    z[i] = zi;
    if (own(i)) s += y * zi;
  };
  const int64_t gid = (int64_t)blockIdx.x * VEC_NT + threadIdx.x, stride = (int64_t)gridDim.x * VEC_NT;
  if constexpr (V2) {
    for (int64_t j = gid; j < (n >> 1); j += stride) {
      const double2 a = reinterpret_cast<const double2 *>(Av)[j], r = reinterpret_cast<const double2 *>(r2)[j];
      double2 y, zz;
      y.x = a.x - f * r.x;
      y.y = a.y - f * r.y;
      reinterpret_cast<double2 *>(Av)[j] = y;
      if (inv) {
        const double2 iv = reinterpret_cast<const double2 *>(inv)[j];
        zz.x = iv.x * y.x;
        zz.y = iv.y * y.y;
      } else {
        zz = y;
      }
      reinterpret_cast<double2 *>(z)[j] = zz;
      if (own(2 * j)) s += y.x * zz.x;
      if (own(2 * j + 1)) s += y.y * zz.y;
    }
    if (gid == 0 && (n & 1)) one(n - 1);
  } else {
    for (int64_t i = gid; i < n; i += stride) one(i);
  }
  s = block_sum<VEC_NT>(s, sv);
  if (threadIdx.x == 0) part2[blockIdx.x] = s;
}

// K3: beta2 = sum(part2); Givens recurrence; w_new (into w1buf); x += phi w_new; v = z / beta
template <bool V2>
__global__ void __launch_bounds__(VEC_NT) minres_k3(int64_t n, const double *__restrict__ z, double *__restrict__ v,
                                                    const double *__restrict__ w, double *__restrict__ w1buf,
                                                    const double *__restrict__ w2, double *__restrict__ x,
                                                    const tmop_minres_state *cur, tmop_minres_state *nxt,
                                                    const double *__restrict__ part1, int np1,
                                                    const double *__restrict__ part2, int np, double rtol,
                                                    double *__restrict__ hist, int hist_cap) {
  const tmop_minres_state c = *cur;
  if (c.done) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *nxt = c;
    return;
  }
  __shared__ double sv[VEC_NT / 32];
  const double alfa = reduce_partials(part1, np1, sv);
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
  // w_new = (v - oldeps w1 - delta w2) / gamma (solvers.py:158), true divisions as the reference
  auto one = [&](int64_t i) {
    const double vi = v[i];
    const double wn = (vi - oldeps * w2[i] - delta * w[i]) / gamma;
    w1buf[i] = wn;
    x[i] = x[i] + phi * wn;
    v[i] = z[i] / beta;
  };
  const int64_t gid = (int64_t)blockIdx.x * VEC_NT + threadIdx.x, stride = (int64_t)gridDim.x * VEC_NT;
  if constexpr (V2) {
    for (int64_t j = gid; j < (n >> 1); j += stride) {
      const double2 vi = reinterpret_cast<const double2 *>(v)[j], a = reinterpret_cast<const double2 *>(w2)[j];
      const double2 b = reinterpret_cast<const double2 *>(w)[j], xx = reinterpret_cast<const double2 *>(x)[j];
      const double2 zz = reinterpret_cast<const double2 *>(z)[j];
      double2 wn, xo, vo;
      wn.x = (vi.x - oldeps * a.x - delta * b.x) / gamma;
      wn.y = (vi.y - oldeps * a.y - delta * b.y) / gamma;
      reinterpret_cast<double2 *>(w1buf)[j] = wn;
      xo.x = xx.x + phi * wn.x;
      xo.y = xx.y + phi * wn.y;
      reinterpret_cast<double2 *>(x)[j] = xo;
      vo.x = zz.x / beta;
      vo.y = zz.y / beta;
      reinterpret_cast<double2 *>(v)[j] = vo;
    }
    if (gid == 0 && (n & 1)) one(n - 1);
  } else {
    for (int64_t i = gid; i < n; i += stride) one(i);
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
  minres_init_kernel<<<g, VEC_NT, 0, s>>>(n, b, inv, x, r1, r2, z, w, w2, part, Own{0, 0});
  minres_init2_kernel<<<g, VEC_NT, 0, s>>>(n, z, v, part, g, st);
}

static bool al16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

static void launch_k23(int64_t n, double *Av, const double *r2, const double *inv, double *z, double *v,
                       const double *w, double *w1buf, const double *w2, double *x, double rtol,
                       tmop_minres_state *cur, tmop_minres_state *nxt, double *part1, int np1, double *part2,
                       double *hist, int hist_cap, int g, cudaStream_t s) {
  const bool v2 = al16(Av) && al16(r2) && (!inv || al16(inv)) && al16(z) && al16(v) && al16(w) && al16(w1buf) &&
                  al16(w2) && al16(x);
  if (v2) {
    minres_k2<true><<<g, VEC_NT, 0, s>>>(n, Av, r2, inv, z, cur, part1, np1, part2, Own{0, 0});
    minres_k3<true><<<g, VEC_NT, 0, s>>>(n, z, v, w, w1buf, w2, x, cur, nxt, part1, np1, part2, g, rtol, hist,
                                         hist_cap);
  } else {
    minres_k2<false><<<g, VEC_NT, 0, s>>>(n, Av, r2, inv, z, cur, part1, np1, part2, Own{0, 0});
    minres_k3<false><<<g, VEC_NT, 0, s>>>(n, z, v, w, w1buf, w2, x, cur, nxt, part1, np1, part2, g, rtol, hist,
                                          hist_cap);
  }
}

// Fused E->L gather + MINRES K1 for the TMOP operator (one pass over Av
// instead of a gather write followed by a K1 read-modify-write):
//   Av[i] = (fixed ? v : sum_E) ; Av -= (beta/oldb) r1 (itn >= 2) ; alfa partial v.Av
// Grid = vec_grid(n), grid-stride over nodes, so the partial array has the
// same length the following K2 / K3 expect.
template <int D, bool LAT, int NT = VEC_NT>
__global__ void __launch_bounds__(NT) e2l_minres_k1(int64_t nn, int64_t n0, int64_t n1, const E2LMap m,
                                                    const double *__restrict__ E,
                                                        const double *__restrict__ add,
                                                        const uint8_t *__restrict__ fixed, const double *__restrict__ v,
                                                        const double *__restrict__ r1, double *__restrict__ Av,
                                                        const tmop_minres_state *cur, double *__restrict__ part) {
  if (cur->done) return;
  __shared__ double sv[NT / 32];
  const bool sub = cur->itn >= 1;
  const double f = sub ? cur->beta / cur->oldb : 0.0;
  double s = 0.0;
  for (int64_t node = n0 + (int64_t)blockIdx.x * NT + threadIdx.x; node < n1; node += (int64_t)gridDim.x * NT) {
    double acc[D];
    e2l_node<D, LAT>(node, m, E, acc);
    const uint8_t fl = __ldg(fixed + node);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const int64_t i = c * nn + node;
      const double vi = v[i];
      double y = ((fl >> c) & 1) ? vi : (add ? acc[c] + add[i] : acc[c]);
      if (sub) y = y - f * r1[i];
      Av[i] = y;
      s += vi * y;
    }
  }
  s = block_sum<NT>(s, sv);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

void launch_minres_step_op(int dim, int64_t nn, const E2LMap &m, const double *E, const double *add,
                           const uint8_t *fixed, int64_t n, double *Av, const double *r1, const double *r2,
                           const double *inv, double *z, double *v, const double *w, double *w1buf, const double *w2,
                           double *x, double rtol, tmop_minres_state *cur, tmop_minres_state *nxt, double *part1,
                           double *part2, double *hist, int hist_cap, cudaStream_t s) {
  const int g = vec_grid(n);
  if (dim == 2)
    e2l_minres_k1<2, false><<<g, VEC_NT, 0, s>>>(nn, 0, nn, m, E, add, fixed, v, r1, Av, cur, part1);
  else if (m.lat_p > 0)
    e2l_minres_k1<3, true><<<g, VEC_NT, 0, s>>>(nn, 0, nn, m, E, add, fixed, v, r1, Av, cur, part1);
  else
    e2l_minres_k1<3, false><<<g, VEC_NT, 0, s>>>(nn, 0, nn, m, E, add, fixed, v, r1, Av, cur, part1);
  launch_k23(n, Av, r2, inv, z, v, w, w1buf, w2, x, rtol, cur, nxt, part1, g, part2, hist, hist_cap, g, s);
}

// Overlapped pieces: the fused E->L + K1 over nodes [n0, n1) of a 3D lattice
// in 128-thread CTAs (partials into part[0 .. grid)), and K2/K3 reducing np1
// K1 partials.
void launch_e2l_k1_range(int64_t nn, int64_t n0, int64_t n1, const E2LMap &m, const double *E, const double *add,
                         const uint8_t *fixed, const double *v, const double *r1, double *Av,
                         const tmop_minres_state *cur, double *part, int grid, cudaStream_t s) {
  e2l_minres_k1<3, true, 128><<<grid, 128, 0, s>>>(nn, n0, n1, m, E, add, fixed, v, r1, Av, cur, part);
}

void launch_minres_k23(int64_t n, double *Av, const double *r2, const double *inv, double *z, double *v,
                       const double *w, double *w1buf, const double *w2, double *x, double rtol,
                       tmop_minres_state *cur, tmop_minres_state *nxt, double *part1, int np1, double *part2,
                       double *hist, int hist_cap, cudaStream_t s) {
  const int g = vec_grid(n);
  launch_k23(n, Av, r2, inv, z, v, w, w1buf, w2, x, rtol, cur, nxt, part1, np1, part2, hist, hist_cap, g, s);
}

void launch_minres_step(int64_t n, double *Av, const double *r1, const double *r2, const double *inv, double *z,
                        double *v, const double *w, double *w1buf, const double *w2, double *x, double rtol,
                        tmop_minres_state *cur, tmop_minres_state *nxt, double *part1, double *part2,
                        double *hist, int hist_cap, cudaStream_t s) {
  const int g = vec_grid(n);
  minres_k1<<<g, VEC_NT, 0, s>>>(n, Av, r1, v, cur, part1, Own{0, 0});
  launch_k23(n, Av, r2, inv, z, v, w, w1buf, w2, x, rtol, cur, nxt, part1, g, part2, hist, hist_cap, g, s);
}

// ---- slab-partitioned MINRES phases (tmop_minres_dist_*): every phase that
// ends in a dot product reduces its owned-entry partials in a fixed order
// into scal[k]; the caller all-reduces scal[k] across ranks in between, and
// the next phase reads the global value as a one-entry partial array.
void launch_minres_dist_init_a(int64_t n, int64_t nn, int64_t n_owned, const double *b, const double *inv, double *x,
                               double *r1, double *r2, double *z, double *w, double *w2, double *part, double *scal,
                               cudaStream_t s) {
  const int g = vec_grid(n);
  minres_init_kernel<<<g, VEC_NT, 0, s>>>(n, b, inv, x, r1, r2, z, w, w2, part, Own{nn, n_owned});
  sum_partials_kernel<<<1, VEC_NT, 0, s>>>(g, part, scal);
}

void launch_minres_dist_init_b(int64_t n, const double *z, double *v, const double *scal, tmop_minres_state *st,
                               cudaStream_t s) {
  minres_init2_kernel<<<vec_grid(n), VEC_NT, 0, s>>>(n, z, v, scal, 1, st);
}

void launch_minres_dist_k1(int64_t n, int64_t nn, int64_t n_owned, double *Av, const double *r1, const double *v,
                           const tmop_minres_state *cur, double *part, double *scal, cudaStream_t s) {
  const int g = vec_grid(n);
  minres_k1<<<g, VEC_NT, 0, s>>>(n, Av, r1, v, cur, part, Own{nn, n_owned});
  sum_partials_kernel<<<1, VEC_NT, 0, s>>>(g, part, scal);
}

void launch_minres_dist_k2(int64_t n, int64_t nn, int64_t n_owned, double *Av, const double *r2, const double *inv,
                           double *z, const tmop_minres_state *cur, double *part, double *scal, cudaStream_t s) {
  const int g = vec_grid(n);
  const bool v2 = al16(Av) && al16(r2) && (!inv || al16(inv)) && al16(z);
  if (v2)
    minres_k2<true><<<g, VEC_NT, 0, s>>>(n, Av, r2, inv, z, cur, scal, 1, part, Own{nn, n_owned});
  else
    minres_k2<false><<<g, VEC_NT, 0, s>>>(n, Av, r2, inv, z, cur, scal, 1, part, Own{nn, n_owned});
  sum_partials_kernel<<<1, VEC_NT, 0, s>>>(g, part, scal + 1);
}

void launch_minres_dist_k3(int64_t n, const double *z, double *v, const double *w, double *w1buf, const double *w2,
                           double *x, double rtol, tmop_minres_state *cur, tmop_minres_state *nxt,
                           const double *scal, double *hist, int hist_cap, cudaStream_t s) {
  const int g = vec_grid(n);
  const bool v2 = al16(z) && al16(v) && al16(w) && al16(w1buf) && al16(w2) && al16(x);
  if (v2)
    minres_k3<true><<<g, VEC_NT, 0, s>>>(n, z, v, w, w1buf, w2, x, cur, nxt, scal, 1, scal + 1, 1, rtol, hist,
                                         hist_cap);
  else
    minres_k3<false><<<g, VEC_NT, 0, s>>>(n, z, v, w, w1buf, w2, x, cur, nxt, scal, 1, scal + 1, 1, rtol, hist,
                                          hist_cap);
}

// Shared node planes of a z-slab (component-major local vector (3, nn); the
// planes are nodes [0, pl) and [nn - pl, nn)): pack both into one send
// buffer [lo: 3 pl][hi: 3 pl] ...
__global__ void halo_pack_kernel(int64_t nn, int64_t pl, int lo, int hi, const double *__restrict__ y,
                                 double *__restrict__ send) {
  const int64_t tot = 3 * pl;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / pl, j = i - c * pl;
    if (lo) send[i] = y[c * nn + j];
    if (hi) send[tot + i] = y[c * nn + nn - pl + j];
  }
}

// ... and add the neighbours' partial sums back, re-applying the constraint
// convention on those planes (operator.py:417 / :458): fixed entries take
// vfix[i] (the apply's v) or cfix (the diagonal's 1.0) when vfix == NULL;
// mode 0 leaves fixed entries as summed (the gradient's 0 + 0).
__global__ void halo_unpack_kernel(int64_t nn, int64_t pl, int lo, int hi, const double *__restrict__ recv,
                                   const uint8_t *__restrict__ fixed, int mode, const double *__restrict__ vfix,
                                   double cfix, double *__restrict__ y) {
  const int64_t tot = 3 * pl;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / pl, j = i - c * pl;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      if (side == 0 ? !lo : !hi) continue;
      const int64_t node = side == 0 ? j : nn - pl + j;
      const int64_t k = c * nn + node;
      double val = y[k] + recv[side * tot + i];
      if (mode && ((__ldg(fixed + node) >> c) & 1)) val = vfix ? vfix[k] : cfix;
      y[k] = val;
    }
  }
}

void launch_halo_pack(int64_t nn, int64_t pl, int lo, int hi, const double *y, double *send, cudaStream_t s) {
  const int64_t tot = 3 * pl;
  const int g = (int)std::min<int64_t>((tot + 255) / 256, 148 * 8);
  if (g > 0) halo_pack_kernel<<<g, 256, 0, s>>>(nn, pl, lo, hi, y, send);
}

void launch_halo_unpack(int64_t nn, int64_t pl, int lo, int hi, const double *recv, const uint8_t *fixed, int mode,
                        const double *vfix, double cfix, double *y, cudaStream_t s) {
  const int64_t tot = 3 * pl;
  const int g = (int)std::min<int64_t>((tot + 255) / 256, 148 * 8);
  if (g > 0) halo_unpack_kernel<<<g, 256, 0, s>>>(nn, pl, lo, hi, recv, fixed, mode, vfix, cfix, y);
}

// ---- peer-memory halo (tmop_halo_p2p_*): the shared planes go straight into
// the neighbours' mailboxes (CUDA IPC / NVLink P2P stores), no NCCL on the
// data path.  Mailbox: box[slot][side][3 pl] doubles, side 0 = from the
// lower neighbour (its top plane), side 1 = from the upper neighbour (its
// bottom plane); cnt[side] counts arrivals monotonically (one per put CTA).
int halo_p2p_grid(int64_t pl) {
  const int64_t g = (3 * pl + 255) / 256;
  return (int)std::min<int64_t>(std::max<int64_t>(g, 1), 148 * 4);
}

__global__ void halo_p2p_put_kernel(int64_t nn, int64_t pl, const double *__restrict__ y, double *box_lo,
                                    unsigned long long *cnt_lo, double *box_hi, unsigned long long *cnt_hi,
                                    int slot) {
  const int64_t tot = 3 * pl;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / pl, j = i - c * pl;
    // my bottom plane -> the lower neighbour's side 1; my top plane -> the upper's side 0
    if (box_lo) box_lo[(slot * 2 + 1) * tot + i] = y[c * nn + j];
    if (box_hi) box_hi[(slot * 2 + 0) * tot + i] = y[c * nn + nn - pl + j];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (cnt_lo) asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(cnt_lo + 1) : "memory");
    if (cnt_hi) asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(cnt_hi + 0) : "memory");
  }
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void halo_p2p_get_kernel(int64_t nn, int64_t pl, double *__restrict__ y, const double *box,
                                    const unsigned long long *cnt, int lo, int hi, int slot,
                                    unsigned long long target, const uint8_t *__restrict__ fixed, int mode,
                                    const double *__restrict__ vfix, double cfix, int *err) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    // bounded wait (~4 s): a missing neighbour reports an error instead of
    // hanging the GPU, and every later exchange then returns at once
    int good = *(volatile int *)err == 0;
    for (int side = 0; side < 2 && good; ++side) {
      if (side == 0 ? !lo : !hi) continue;
      long long it = 0;
      while (ld_acquire_sys(cnt + side) < target) {
        __nanosleep(256);
        if (++it > (1ll << 24)) {
          good = 0;
          atomicExch(err, 1);
          break;
        }
      }
    }
    ok = good;
  }
  __syncthreads();
  if (!ok) return;
  const int64_t tot = 3 * pl;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / pl, j = i - c * pl;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      if (side == 0 ? !lo : !hi) continue;
      const int64_t node = side == 0 ? j : nn - pl + j;
      const int64_t k = c * nn + node;
      double val = y[k] + __ldcg(box + (slot * 2 + side) * tot + i);
      if (mode && ((__ldg(fixed + node) >> c) & 1)) val = vfix ? vfix[k] : cfix;
      y[k] = val;
    }
  }
}

void launch_halo_p2p_put(int64_t nn, int64_t pl, const double *y, double *box_lo, unsigned long long *cnt_lo,
                         double *box_hi, unsigned long long *cnt_hi, int slot, cudaStream_t s) {
  halo_p2p_put_kernel<<<halo_p2p_grid(pl), 256, 0, s>>>(nn, pl, y, box_lo, cnt_lo, box_hi, cnt_hi, slot);
}

void launch_halo_p2p_get(int64_t nn, int64_t pl, double *y, const double *box, const unsigned long long *cnt, int lo,
                         int hi, int slot, unsigned long long target, const uint8_t *fixed, int mode,
                         const double *vfix, double cfix, int *err, cudaStream_t s) {
  const int g = (int)std::min<int64_t>((3 * pl + 255) / 256, 148 * 4);
  halo_p2p_get_kernel<<<g > 0 ? g : 1, 256, 0, s>>>(nn, pl, y, box, cnt, lo, hi, slot, target, fixed, mode, vfix,
                                                    cfix, err);
}

}  // namespace tmop
