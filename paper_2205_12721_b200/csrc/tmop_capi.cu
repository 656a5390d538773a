// tmop_capi.cu -- the extern "C" boundary (include/tmop_b200.h).
//
// The context replaces TmopProblem.__init__ (operator.py:230-250): it holds
// the discretisation constants (1D tables as a by-value kernel parameter),
// the caller-owned device mesh arrays, and library-owned scratch (the
// element-blocked E-vector and the per-CTA reduction partials).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "../../include/tmop_b200.h"
#include "tmop_core.h"
#include "tmop_elem.cuh"
#include "tmop_internal.h"

using namespace tmop;

static thread_local char g_err[512] = "";

static int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) return fail(TMOP_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

struct tmop_ctx {
  int dim, order, n1, nq, QP, NP;
  int64_t ne, nn;
  const int32_t *restr;
  const uint8_t *fixed;
  const int64_t *l2e_off;
  const uint32_t *l2e_idx;
  Tab tab;
  int metric;
  double omega, det_w, inv_s;
  cudaStream_t stream;
  double *E;
  int e_es;          // E-vector layout written by the last element kernel (e2l_kernel)
  double *part_sum, *part_min;
  int64_t *part_arg;
  double *vpart1, *vpart2;
  int lat_n[3], lat_p;   // verified box lattice (tmop_ctx_set_lattice), lat_p = 0: none
  uint64_t mag_x, mag_y;
  int sh_x, sh_y;
  int *flag;             // device scratch word
  // displacement limiting (tmop_ctx_set_limiting); buffers allocated on first use
  int lim_on;
  const double *lim_x0, *lim_dn;
  double lim_delta, lim_weight;
  double *E2, *lim_y, *lim_val;
  // overlapped apply (tmop_hessian_apply on lattices): E->L of finished slabs
  // runs on a second stream while the element kernel works on the next slab
  cudaStream_t s2;
  cudaEvent_t ev[33];
  int ov_slabs;
  int64_t ov_min;    // fewest elements for the overlapped path
  double *tscale;    // size-field targets: per-point 1 / s_q (NULL: constant target)
  double *tscale_buf;
  double *hist;      // MINRES residual history (device, optional)
  int hist_cap;
};

// Slab-overlapped paths only pay off for long applies (>= ~0.5 ms); below
// this many elements the extra launches cost more than the hidden gather.
static const int64_t OVERLAP_MIN_ELEMENTS = getenv("TMOP_OVERLAP_MIN") ? atoll(getenv("TMOP_OVERLAP_MIN")) : 262144;

namespace tmop {
int launch_elem(int dim, int n1, int nq, int kind, ElemArgs &a, const Tab &t, cudaStream_t s) {
  if (dim == 2) return launch_elem_2d(n1, nq, kind, a, t, s);
  switch (n1) {
    case 2: return launch_elem_3d_n2(nq, kind, a, t, s);
    case 3: return launch_elem_3d_n3(nq, kind, a, t, s);
    case 4: return launch_elem_3d_n4(nq, kind, a, t, s);
    case 5: return launch_elem_3d_n5(nq, kind, a, t, s);
    default: return -1;
  }
}
bool elem_supported(int dim, int n1, int nq) {
  return (dim == 2 || dim == 3) && n1 >= 2 && n1 <= MAXN && nq >= 2 && nq <= MAXQ;
}
}  // namespace tmop

static bool metric_ok(int metric, int dim) {
  switch (metric) {
    case MU2:
    case MU7: return dim == 2;
    case MU55: return true;
    case MU302:
    case MU303:
    case MU321: return dim == 3;
    default: return false;
  }
}

static ElemArgs base_args(const tmop_ctx *c) {
  ElemArgs a;
  memset(&a, 0, sizeof(a));
  a.ne = c->ne;
  a.nn = c->nn;
  a.restr = c->restr;
  a.fixed = c->fixed;
  a.metric = c->metric;
  const double is = c->inv_s;
  a.inv_s = is;
  a.inv_s_dm1 = c->dim == 3 ? is * is : is;
  a.inv_s_d = c->dim == 3 ? is * is * is : is * is;
  a.coef_e = c->omega * c->det_w;
  a.coef_g = c->omega * c->det_w * is;
  a.coef_h = c->omega * c->det_w * (is * is);
  a.E = c->E;
  a.e_es = 0;
  a.part_sum = c->part_sum;
  a.part_min = c->part_min;
  a.part_arg = c->part_arg;
  a.tscale = c->tscale;
  a.omega = c->omega;
  return a;
}

static E2LMap e2l_map(const tmop_ctx *c) {
  E2LMap m;
  m.off = c->l2e_off;
  m.idx = c->l2e_idx;
  m.np = c->NP;
  m.es = c->e_es;
  for (int i = 0; i < 3; ++i) m.lat_n[i] = c->lat_n[i];
  m.lat_p = c->lat_p;
  m.mag_x = c->mag_x;
  m.mag_y = c->mag_y;
  m.sh_x = c->sh_x;
  m.sh_y = c->sh_y;
  return m;
}

static int run(tmop_ctx *c, int kind, ElemArgs &a, int *grid_out) {
  const int g = launch_elem(c->dim, c->n1, c->nq, kind, a, c->tab, c->stream);
  if (g < 0) return fail(TMOP_ERR_ARG, "no kernel instance for dim=%d p=%d n_q=%d (kind %d)", c->dim, c->order, c->nq, kind);
  CUDA_TRY(cudaGetLastError());
  c->e_es = a.e_es;
  if (grid_out) *grid_out = g;
  return TMOP_OK;
}

// Limiting term node sums into c->lim_y (raw, no constraint fix-up): kind
// K_LIM_FIELD on `in` (minus x0 when given, constrained components zeroed
// when mask) or K_LIM_DIAG; E2 -> e2l mode 3.
static int lim_nodes(tmop_ctx *c, int kind, const double *in, const double *x0, int mask) {
  ElemArgs a = base_args(c);
  a.in = in;
  a.E = c->E2;
  a.lim_x0 = x0;
  a.lim_dn = c->lim_dn;
  a.lim_delta = c->lim_delta;
  a.lim_base = 2.0 * c->lim_weight * c->det_w;
  a.lim_mask = mask;
  const int g = launch_elem(c->dim, c->n1, c->nq, kind, a, c->tab, c->stream);
  if (g < 0) return fail(TMOP_ERR_ARG, "no limiting kernel for dim=%d p=%d n_q=%d", c->dim, c->order, c->nq);
  CUDA_TRY(cudaGetLastError());
  E2LMap m = e2l_map(c);
  m.es = 0;
  launch_e2l(c->dim, c->nn, m, c->E2, c->fixed, 3, nullptr, nullptr, c->lim_y, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

// Limiting value 1/2 sum c_q |B (x - x0)|^2 into c->lim_val (device).
static int lim_value(tmop_ctx *c, const double *x) {
  ElemArgs a = base_args(c);
  a.in = x;
  a.lim_x0 = c->lim_x0;
  a.lim_dn = c->lim_dn;
  a.lim_delta = c->lim_delta;
  a.lim_base = 2.0 * c->lim_weight * c->det_w;
  const int g = launch_elem(c->dim, c->n1, c->nq, K_LIM_VALUE, a, c->tab, c->stream);
  if (g < 0) return fail(TMOP_ERR_ARG, "no limiting kernel for dim=%d p=%d n_q=%d", c->dim, c->order, c->nq);
  CUDA_TRY(cudaGetLastError());
  launch_fin(g, c->part_sum, nullptr, nullptr, 0.5, c->lim_val, 0.0, nullptr, nullptr, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

extern "C" {

const char *tmop_last_error(void) { return g_err; }

int tmop_ctx_create(tmop_ctx **out, int dim, int order, int n_quad, int64_t n_elements, int64_t n_nodes,
                    const int32_t *restriction, const uint8_t *fixed, const int64_t *l2e_offsets,
                    const uint32_t *l2e_index, const double *B, const double *G, const double *w1, int metric,
                    double inv_scale, double det_w, double spatial_weight, void *stream) {
  if (!out) return fail(TMOP_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (!elem_supported(dim, order + 1, n_quad))
    return fail(TMOP_ERR_ARG, "unsupported (dim=%d, p=%d, n_q=%d): need dim in {2,3}, 1<=p<=%d, 2<=n_q<=%d", dim,
                order, n_quad, MAXN - 1, MAXQ);
  if (!metric_ok(metric, dim)) return fail(TMOP_ERR_METRIC, "metric %d is not valid in %dD", metric, dim);
  if (n_elements < 0 || n_nodes < 0) return fail(TMOP_ERR_ARG, "negative sizes");
  const int np = (int)std::lround(std::pow(order + 1, dim));
  if ((double)n_elements * np >= 4294967295.0) return fail(TMOP_ERR_ARG, "mesh too large for uint32 E-indices");
  tmop_ctx *c = new (std::nothrow) tmop_ctx;
  if (!c) return fail(TMOP_ERR_ARG, "out of host memory");
  memset(c, 0, sizeof(*c));
  c->dim = dim;
  c->order = order;
  c->n1 = order + 1;
  c->nq = n_quad;
  c->NP = np;
  c->QP = (int)std::lround(std::pow(n_quad, dim));
  c->ne = n_elements;
  c->nn = n_nodes;
  c->restr = restriction;
  c->fixed = fixed;
  c->l2e_off = l2e_offsets;
  c->l2e_idx = l2e_index;
  for (int q = 0; q < n_quad; ++q) {
    for (int i = 0; i < c->n1; ++i) {
      const double b = B[q * c->n1 + i], g = G[q * c->n1 + i];
      c->tab.B[q * c->n1 + i] = b;
      c->tab.G[q * c->n1 + i] = g;
      c->tab.P[0][q * c->n1 + i] = b * b;
      c->tab.P[1][q * c->n1 + i] = b * g;
      c->tab.P[2][q * c->n1 + i] = g * g;
    }
    c->tab.w1[q] = w1[q];
  }
  c->metric = metric;
  c->omega = spatial_weight;
  c->det_w = det_w;
  c->inv_s = inv_scale;
  c->stream = (cudaStream_t)stream;
  {
    const char *ev = getenv("TMOP_APPLY_SLABS");
    c->ov_slabs = ev ? atoi(ev) : 8;
    if (c->ov_slabs > 30) c->ov_slabs = 30;
    c->ov_min = OVERLAP_MIN_ELEMENTS;
  }
  cudaError_t e = cudaSuccess;
  // E-vector: element count padded to whole 16-element groups (interleaved layout)
  const size_t esz = (size_t)((n_elements + 15) / 16 * 16) * dim * np;
  e = cudaMalloc(&c->E, (esz ? esz : 1) * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&c->part_sum, GRID_CAP * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&c->part_min, GRID_CAP * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&c->part_arg, GRID_CAP * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMalloc(&c->vpart1, VPART_CAP * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&c->vpart2, VPART_CAP * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&c->flag, sizeof(int));
  if (e != cudaSuccess) {
    tmop_ctx_destroy(c);
    return fail(TMOP_ERR_CUDA, "workspace allocation failed: %s", cudaGetErrorString(e));
  }
  *out = c;
  return TMOP_OK;
}

int tmop_ctx_destroy(tmop_ctx *c) {
  if (!c) return TMOP_OK;
  cudaFree(c->E);
  cudaFree(c->part_sum);
  cudaFree(c->part_min);
  cudaFree(c->part_arg);
  cudaFree(c->vpart1);
  cudaFree(c->vpart2);
  cudaFree(c->flag);
  if (c->s2) {
    for (int i = 0; i < 33; ++i) cudaEventDestroy(c->ev[i]);
    cudaStreamDestroy(c->s2);
  }
  cudaFree(c->tscale_buf);
  cudaFree(c->E2);
  cudaFree(c->lim_y);
  cudaFree(c->lim_val);
  delete c;
  return TMOP_OK;
}

int tmop_ctx_set_stream(tmop_ctx *c, void *stream) {
  if (!c) return fail(TMOP_ERR_ARG, "ctx is NULL");
  c->stream = (cudaStream_t)stream;
  return TMOP_OK;
}

int tmop_ctx_set_apply_overlap(tmop_ctx *c, int slabs, int64_t min_elements) {
  if (!c) return fail(TMOP_ERR_ARG, "NULL context");
  if (slabs < 1 || slabs > 30 || min_elements < 0) return fail(TMOP_ERR_ARG, "slabs must be in [1, 30], min >= 0");
  c->ov_slabs = slabs;
  c->ov_min = min_elements;
  return TMOP_OK;
}

int tmop_ctx_set_lattice(tmop_ctx *c, int nx, int ny, int nz, int *accepted) {
  if (!c || !accepted) return fail(TMOP_ERR_ARG, "NULL argument");
  *accepted = 0;
  c->lat_p = 0;
  const int p = c->order;
  if (c->dim != 3 || nx < 1 || ny < 1 || nz < 1) return TMOP_OK;
  if ((int64_t)nx * ny * nz != c->ne) return TMOP_OK;
  if (((int64_t)nx * p + 1) * ((int64_t)ny * p + 1) * ((int64_t)nz * p + 1) != c->nn) return TMOP_OK;
  if (c->nn >= (int64_t)1 << 31 || c->ne >= (int64_t)1 << 31) return TMOP_OK;   // 32-bit lattice arithmetic
  CUDA_TRY(cudaMemsetAsync(c->flag, 0, sizeof(int), c->stream));
  launch_lattice_check(c->ne, c->NP, c->restr, nx, ny, nz, p, c->flag, c->stream);
  CUDA_TRY(cudaGetLastError());
  int bad = 1;
  CUDA_TRY(cudaMemcpyAsync(&bad, c->flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (bad) return TMOP_OK;
  c->lat_n[0] = nx;
  c->lat_n[1] = ny;
  c->lat_n[2] = nz;
  c->lat_p = p;
  // magic numbers for exact n / d with n < 2^31: l = ceil(log2 d), mag = ceil(2^(32+l) / d)
  auto magic = [](uint64_t d, uint64_t &mag, int &sh) {
    int l = 0;
    while (((uint64_t)1 << l) < d) ++l;
    sh = 32 + l;
    mag = (((uint64_t)1 << sh) + d - 1) / d;
  };
  magic((uint64_t)nx * p + 1, c->mag_x, c->sh_x);
  magic((uint64_t)ny * p + 1, c->mag_y, c->sh_y);
  *accepted = 1;
  return TMOP_OK;
}

int tmop_ctx_set_target(tmop_ctx *c, double inv_scale, double det_w) {
  if (!c) return fail(TMOP_ERR_ARG, "ctx is NULL");
  if (!(inv_scale > 0.0) || !(det_w > 0.0)) return fail(TMOP_ERR_ARG, "target scale must be positive");
  c->inv_s = inv_scale;
  c->det_w = det_w;
  c->tscale = nullptr;   // a constant target replaces a size field
  return TMOP_OK;
}

int tmop_ctx_set_size_field(tmop_ctx *c, const double *volume_nodal) {
  if (!c) return fail(TMOP_ERR_ARG, "ctx is NULL");
  if (!volume_nodal) {
    c->tscale = nullptr;
    c->inv_s = c->det_w = 1.0;
    return TMOP_OK;
  }
  if (c->lim_on) return fail(TMOP_ERR_ARG, "size-field targets are not combined with the limiting term");
  const int64_t qp = c->dim == 3 ? (int64_t)c->nq * c->nq * c->nq : (int64_t)c->nq * c->nq;
  if (!c->tscale_buf) CUDA_TRY(cudaMalloc(&c->tscale_buf, (size_t)(c->ne * qp > 0 ? c->ne * qp : 1) * sizeof(double)));
  c->tscale = nullptr;
  c->inv_s = c->det_w = 1.0;
  ElemArgs a = base_args(c);
  a.lim_dn = volume_nodal;
  a.qout = c->tscale_buf;
  const int g = launch_elem(c->dim, c->n1, c->nq, K_TSCALE, a, c->tab, c->stream);
  if (g < 0) return fail(TMOP_ERR_ARG, "no size-field kernel for dim=%d p=%d n_q=%d", c->dim, c->order, c->nq);
  CUDA_TRY(cudaGetLastError());
  c->tscale = c->tscale_buf;
  return TMOP_OK;
}

const double *tmop_ctx_point_scale(const tmop_ctx *c) { return c ? c->tscale : nullptr; }

int tmop_qdata_fields(const tmop_ctx *c) {
  if (!c) return -1;
  return c->dim * c->dim + 2;
}

int64_t tmop_qdata_stride(const tmop_ctx *c) {
  if (!c) return -1;
  return lean_stride(tmop_qdata_fields(c) * c->QP, xl_epb(c->n1));
}

int64_t tmop_qdata_size(const tmop_ctx *c) {
  if (!c) return -1;
  return tmop_qdata_stride(c) * c->ne;
}

int tmop_qdata_reference_fields(const tmop_ctx *c) {
  if (!c) return -1;
  return (metric_is_template(c->metric) ? 4 : 1) + 2 * c->dim * c->dim;
}

int tmop_qdata_to_reference(tmop_ctx *c, const double *qdata, double *out) {
  if (!c || !qdata || !out) return fail(TMOP_ERR_ARG, "NULL argument");
  const int64_t nq = c->ne * c->QP;
  if (nq == 0) return TMOP_OK;
  const int nt = 128;
  const unsigned grid = (unsigned)((nq + nt - 1) / nt);
  const int qs = (int)tmop_qdata_stride(c);
  if (c->dim == 2)
    qdata_expand_kernel<2><<<grid, nt, 0, c->stream>>>(c->metric, c->ne, c->nq, c->QP, qs, qdata, out);
  else
    qdata_expand_kernel<3><<<grid, nt, 0, c->stream>>>(c->metric, c->ne, c->nq, c->QP, qs, qdata, out);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_ctx_set_limiting(tmop_ctx *c, const double *x0, const double *delta_nodal, double delta, double weight) {
  if (!c) return fail(TMOP_ERR_ARG, "ctx is NULL");
  if (!x0) {
    c->lim_on = 0;
    return TMOP_OK;
  }
  if (!(weight > 0.0)) return fail(TMOP_ERR_ARG, "limiting weight must be positive");
  if (c->tscale) return fail(TMOP_ERR_ARG, "the limiting term is not combined with size-field targets");
  if (!delta_nodal && !(delta > 0.0)) return fail(TMOP_ERR_ARG, "limiting delta must be positive");
  if (!c->E2) {
    const size_t esz = (size_t)(c->ne > 0 ? c->ne : 1) * c->dim * c->NP;
    CUDA_TRY(cudaMalloc(&c->E2, esz * sizeof(double)));
    CUDA_TRY(cudaMalloc(&c->lim_y, (size_t)(c->nn > 0 ? c->nn : 1) * c->dim * sizeof(double)));
    CUDA_TRY(cudaMalloc(&c->lim_val, sizeof(double)));
  }
  c->lim_on = 1;
  c->lim_x0 = x0;
  c->lim_dn = delta_nodal;
  c->lim_delta = delta;
  c->lim_weight = weight;
  return TMOP_OK;
}

int tmop_limiting_value(tmop_ctx *c, const double *x, double *out) {
  if (!c || !x || !out) return fail(TMOP_ERR_ARG, "NULL argument");
  if (!c->lim_on) return fail(TMOP_ERR_ARG, "limiting term not configured (tmop_ctx_set_limiting)");
  int rc = lim_value(c, x);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(out, c->lim_val, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  return TMOP_OK;
}

int tmop_limiting_gradient(tmop_ctx *c, const double *x, double *y) {
  if (!c || !x || !y) return fail(TMOP_ERR_ARG, "NULL argument");
  if (!c->lim_on) return fail(TMOP_ERR_ARG, "limiting term not configured (tmop_ctx_set_limiting)");
  int rc = lim_nodes(c, K_LIM_FIELD, x, c->lim_x0, 0);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(y, c->lim_y, (size_t)c->nn * c->dim * sizeof(double), cudaMemcpyDeviceToDevice,
                           c->stream));
  return TMOP_OK;
}

int tmop_limiting_apply(tmop_ctx *c, const double *v, double *y) {
  if (!c || !v || !y) return fail(TMOP_ERR_ARG, "NULL argument");
  if (!c->lim_on) return fail(TMOP_ERR_ARG, "limiting term not configured (tmop_ctx_set_limiting)");
  int rc = lim_nodes(c, K_LIM_FIELD, v, nullptr, 0);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(y, c->lim_y, (size_t)c->nn * c->dim * sizeof(double), cudaMemcpyDeviceToDevice,
                           c->stream));
  return TMOP_OK;
}

int tmop_hessian_setup_diagonal(tmop_ctx *c, const double *x, double *qdata, double *diag,
                                tmop_det_status *det_out) {
  if (!c || !x || !qdata || !diag || !det_out) return fail(TMOP_ERR_ARG, "NULL argument");
  // The one-pass kernel (xl_kernel<K_SETUP_DIAG>) is opt-in: measured slower
  // than the two passes (setup 4.3 ms + x-line diagonal 7.6 ms at C3 p = 2:
  // 11.9 vs 12.5 ms fused; p = 1: 8.8 vs 11.4; p = 3: 10.1 vs 18.0) -- the
  // fused CTA carries the setup's and the diagonal's shared-memory buffers
  // and registers at once (255 registers, 2 CTAs / SM at p = 2, 1 at p = 3)
  // and waits for each group's record store before reusing the buffer.
  static const bool fused_on = getenv("TMOP_SETUP_DIAG_FUSED") && atoi(getenv("TMOP_SETUP_DIAG_FUSED")) != 0;
  if (fused_on && metric_is_template(c->metric) && !c->lim_on) {
    ElemArgs a = base_args(c);
    a.in = x;
    a.qout = qdata;
    const int g = launch_elem(c->dim, c->n1, c->nq, K_SETUP_DIAG, a, c->tab, c->stream);
    if (g >= 0) {   // fused kernel available (3D p <= 3)
      CUDA_TRY(cudaGetLastError());
      c->e_es = a.e_es;
      launch_fin(g, nullptr, c->part_min, c->part_arg, 0.0, nullptr, 0.0, nullptr, det_out, c->stream);
      CUDA_TRY(cudaGetLastError());
      launch_e2l(c->dim, c->nn, e2l_map(c), c->E, c->fixed, 2, nullptr, nullptr, diag, c->stream);
      CUDA_TRY(cudaGetLastError());
      return TMOP_OK;
    }
  }
  int rc = tmop_hessian_setup(c, x, qdata, det_out);   // the two separate passes
  if (rc) return rc;
  return tmop_hessian_diagonal(c, qdata, diag);
}

int tmop_hessian_setup(tmop_ctx *c, const double *x, double *qdata, tmop_det_status *det_out) {
  if (!c || !x || !qdata || !det_out) return fail(TMOP_ERR_ARG, "NULL argument");
  ElemArgs a = base_args(c);
  a.in = x;
  a.qout = qdata;
  int g = 0;
  int rc = run(c, K_SETUP, a, &g);
  if (rc) return rc;
  launch_fin(g, nullptr, c->part_min, c->part_arg, 0.0, nullptr, 0.0, nullptr, det_out, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}


// Overlapped action on a verified lattice: z-slab element launches on the
// context stream; after each, the E->L sum of the node planes that slab
// completes (ascending element order per node, as the one-shot gather) runs
// on a second stream in small CTAs that fit beside the persistent element
// kernel (register headroom), so the memory-bound gather hides under the
// FP64-bound element work.  Results are bitwise identical to the one-shot path.
static int ensure_s2(tmop_ctx *c) {
  if (!c->s2) {
    CUDA_TRY(cudaStreamCreateWithFlags(&c->s2, cudaStreamNonBlocking));
    for (int i = 0; i < 33; ++i) CUDA_TRY(cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming));
  }
  return TMOP_OK;
}

static int apply_overlapped(tmop_ctx *c, const double *qdata, const double *v, double *y) {
  int rc0 = ensure_s2(c);
  if (rc0) return rc0;
  const int64_t layer = (int64_t)c->lat_n[0] * c->lat_n[1];
  const int64_t plane = ((int64_t)c->lat_n[0] * c->lat_p + 1) * ((int64_t)c->lat_n[1] * c->lat_p + 1);
  const int nz = c->lat_n[2];
  const int ns = c->ov_slabs < nz ? c->ov_slabs : nz;
  const E2LMap m0 = e2l_map(c);
  CUDA_TRY(cudaEventRecord(c->ev[31], c->stream));        // fork: s2 follows everything before this call
  CUDA_TRY(cudaStreamWaitEvent(c->s2, c->ev[31], 0));
  int64_t done = 0;
  for (int k = 0; k < ns; ++k) {
    const int64_t e0 = ((int64_t)k * nz / ns) * layer / 16 * 16;
    const int64_t e1 = k + 1 == ns ? c->ne : ((int64_t)(k + 1) * nz / ns) * layer / 16 * 16;
    if (e1 > e0) {
      ElemArgs a = base_args(c);
      a.in = v;
      a.qdata = qdata + e0 * tmop_qdata_stride(c);
      a.restr = c->restr + e0 * c->NP;
      a.E = c->E + e0 * c->dim * c->NP;
      a.ne = e1 - e0;
      int rc = run(c, metric_is_template(c->metric) ? K_APPLY : K_APPLY_NT, a, nullptr);
      if (rc) return rc;
    }
    const int64_t fin = e1 == c->ne ? c->nn : (e1 / layer) * c->lat_p * plane;
    if (fin > done) {
      CUDA_TRY(cudaEventRecord(c->ev[k], c->stream));
      CUDA_TRY(cudaStreamWaitEvent(c->s2, c->ev[k], 0));
      E2LMap m = m0;
      m.es = c->e_es;
      launch_e2l(c->dim, c->nn, m, c->E, c->fixed, 0, v, nullptr, y, c->s2, done, fin, 128);
      CUDA_TRY(cudaGetLastError());
      done = fin;
    }
  }
  CUDA_TRY(cudaEventRecord(c->ev[32], c->s2));            // join
  CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev[32], 0));
  return TMOP_OK;
}

int tmop_hessian_apply(tmop_ctx *c, const double *qdata, const double *v, double *y) {
  if (!c || !qdata || !v || !y) return fail(TMOP_ERR_ARG, "NULL argument");
  // (p <= 3: the x-line element kernel leaves register room for the gather's
  // CTAs; measured 4-5 % faster there, slower at p = 4)
  if (c->lat_p > 0 && c->n1 <= 4 && !c->lim_on && c->ov_slabs > 1 && c->ne >= c->ov_min)
    return apply_overlapped(c, qdata, v, y);
  int rc = tmop_hessian_apply_elements(c, qdata, v);
  if (rc) return rc;
  return tmop_hessian_apply_gather(c, v, y);
}

int tmop_hessian_apply_elements(tmop_ctx *c, const double *qdata, const double *v) {
  if (!c || !qdata || !v) return fail(TMOP_ERR_ARG, "NULL argument");
  ElemArgs a = base_args(c);
  a.in = v;
  a.qdata = qdata;
  int rc = run(c, metric_is_template(c->metric) ? K_APPLY : K_APPLY_NT, a, nullptr);
  if (rc) return rc;
  // limiting part of the action on the masked input (operator.py:415-416)
  return c->lim_on ? lim_nodes(c, K_LIM_FIELD, v, nullptr, 1) : TMOP_OK;
}

int tmop_hessian_apply_elements_range(tmop_ctx *c, const double *qdata, const double *v, int64_t e_begin,
                                      int64_t e_end) {
  if (!c || !qdata || !v) return fail(TMOP_ERR_ARG, "NULL argument");
  if (c->lim_on) return fail(TMOP_ERR_ARG, "range apply does not support the limiting term");
  // both ends on a 16-element group boundary (or end == n_elements): the
  // element kernels write whole groups of the E-vector, so a range ending
  // inside a group would overwrite E entries belonging to the next range
  if (e_begin < 0 || e_end > c->ne || e_begin > e_end || (e_begin & 15) || ((e_end & 15) && e_end != c->ne))
    return fail(TMOP_ERR_ARG,
                "element range [%lld, %lld) invalid (begin and end must be multiples of 16, or end == %lld)",
                (long long)e_begin, (long long)e_end, (long long)c->ne);
  if (e_begin == e_end) return TMOP_OK;
  ElemArgs a = base_args(c);
  a.in = v;
  a.qdata = qdata + e_begin * tmop_qdata_stride(c);
  a.restr = c->restr + e_begin * c->NP;
  a.E = c->E + e_begin * c->dim * c->NP;   // (element groups stay aligned: e_begin % 16 == 0)
  a.ne = e_end - e_begin;
  return run(c, metric_is_template(c->metric) ? K_APPLY : K_APPLY_NT, a, nullptr);
}

int tmop_hessian_apply_gather_range(tmop_ctx *c, const double *v, double *y, int64_t n_begin, int64_t n_end) {
  if (!c || !v || !y) return fail(TMOP_ERR_ARG, "NULL argument");
  if (n_begin < 0 || n_end > c->nn || n_begin > n_end) return fail(TMOP_ERR_ARG, "node range invalid");
  launch_e2l(c->dim, c->nn, e2l_map(c), c->E, c->fixed, 0, v, nullptr, y, c->stream, n_begin, n_end);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_hessian_apply_gather(tmop_ctx *c, const double *v, double *y) {
  if (!c || !v || !y) return fail(TMOP_ERR_ARG, "NULL argument");
  launch_e2l(c->dim, c->nn, e2l_map(c), c->E, c->fixed, 0, v, c->lim_on ? c->lim_y : nullptr, y, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_hessian_diagonal(tmop_ctx *c, const double *qdata, double *diag) {
  if (!c || !qdata || !diag) return fail(TMOP_ERR_ARG, "NULL argument");
  ElemArgs a = base_args(c);
  a.qdata = qdata;
  int rc = run(c, metric_is_template(c->metric) ? K_DIAG : K_DIAG_NT, a, nullptr);
  if (rc) return rc;
  if (c->lim_on) {   // (B.B)^T c_q added to every component (operator.py:452-457)
    rc = lim_nodes(c, K_LIM_DIAG, nullptr, nullptr, 0);
    if (rc) return rc;
  }
  launch_e2l(c->dim, c->nn, e2l_map(c), c->E, c->fixed, 2, nullptr, c->lim_on ? c->lim_y : nullptr, diag, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_gradient(tmop_ctx *c, const double *x, double *grad, tmop_det_status *det_out) {
  return tmop_gradient_energy(c, x, grad, nullptr, det_out);
}

int tmop_gradient_energy(tmop_ctx *c, const double *x, double *grad, double *energy_out, tmop_det_status *det_out) {
  if (!c || !x || !grad || !det_out) return fail(TMOP_ERR_ARG, "NULL argument");
  if (energy_out && c->lim_on) {   // operator.py:324-325: the limiting value joins the energy
    int rc0 = lim_value(c, x);
    if (rc0) return rc0;
  }
  ElemArgs a = base_args(c);
  a.in = x;
  a.energy = energy_out != nullptr;
  int g = 0;
  int rc = run(c, K_GRAD, a, &g);
  if (rc) return rc;
  if (c->lim_on) {   // operator.py:343-344
    rc = lim_nodes(c, K_LIM_FIELD, x, c->lim_x0, 0);
    if (rc) return rc;
  }
  launch_e2l(c->dim, c->nn, e2l_map(c), c->E, c->fixed, 1, nullptr, c->lim_on ? c->lim_y : nullptr, grad, c->stream);
  launch_fin(g, energy_out ? c->part_sum : nullptr, c->part_min, c->part_arg, base_args(c).coef_e, energy_out, 1.0,
             (energy_out && c->lim_on) ? c->lim_val : nullptr, det_out, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_objective(tmop_ctx *c, const double *x, double *energy_out, tmop_det_status *det_out) {
  if (!c || !x || !energy_out || !det_out) return fail(TMOP_ERR_ARG, "NULL argument");
  ElemArgs a = base_args(c);
  a.in = x;
  int g = 0;
  if (c->lim_on) {   // operator.py:324-325 (added after the metric sum)
    int rc0 = lim_value(c, x);
    if (rc0) return rc0;
  }
  int rc = run(c, K_ENERGY, a, &g);
  if (rc) return rc;
  launch_fin(g, c->part_sum, c->part_min, c->part_arg, a.coef_e, energy_out, 1.0, c->lim_on ? c->lim_val : nullptr,
             det_out, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_min_det(tmop_ctx *c, const double *x, tmop_det_status *det_out) {
  if (!c || !x || !det_out) return fail(TMOP_ERR_ARG, "NULL argument");
  ElemArgs a = base_args(c);
  a.in = x;
  int g = 0;
  int rc = run(c, K_MINDET, a, &g);
  if (rc) return rc;
  launch_fin(g, nullptr, c->part_min, c->part_arg, 0.0, nullptr, 0.0, nullptr, det_out, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_element_min_det(tmop_ctx *c, const double *x, double *elem_min, int32_t *elem_arg) {
  if (!c || !x || !elem_min || !elem_arg) return fail(TMOP_ERR_ARG, "NULL argument");
  ElemArgs a = base_args(c);
  a.in = x;
  a.elem_min = elem_min;
  a.elem_arg = elem_arg;
  return run(c, K_ELEMDET, a, nullptr);
}

int tmop_volume(tmop_ctx *c, const double *x, double *vol_out) {
  if (!c || !x || !vol_out) return fail(TMOP_ERR_ARG, "NULL argument");
  ElemArgs a = base_args(c);
  a.in = x;
  int g = 0;
  int rc = run(c, K_VOLUME, a, &g);
  if (rc) return rc;
  launch_fin(g, c->part_sum, nullptr, nullptr, 1.0, vol_out, 0.0, nullptr, nullptr, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_metric_eval(int metric, int dim, int64_t n, const double *T, double *mu, double *P, double *H) {
  if (dim != 2 && dim != 3) return fail(TMOP_ERR_ARG, "dim must be 2 or 3");
  if (!metric_ok(metric, dim)) return fail(TMOP_ERR_METRIC, "metric %d is not valid in %dD", metric, dim);
  launch_metric_eval(metric, dim, n, T, mu, P, H);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  return TMOP_OK;
}

int tmop_dot(tmop_ctx *c, int64_t n, const double *a, const double *b, double *out) {
  if (!c) return fail(TMOP_ERR_ARG, "ctx is NULL");
  launch_dot(n, a, b, c->vpart1, out, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_axpby(tmop_ctx *c, int64_t n, double a, const double *x, double b, double *y) {
  if (!c) return fail(TMOP_ERR_ARG, "ctx is NULL");
  launch_axpby(n, a, x, b, y, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_trial_point(tmop_ctx *c, int64_t n, const double *x, const double *dx, double alpha, double *out) {
  if (!c) return fail(TMOP_ERR_ARG, "ctx is NULL");
  launch_trial(n, x, dx, alpha, out, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_jacobi_inverse(tmop_ctx *c, int64_t n, const double *diag, double floor_value, double *inv,
                        int32_t *nonfinite) {
  if (!c) return fail(TMOP_ERR_ARG, "ctx is NULL");
  launch_jacobi(n, diag, floor_value, inv, nonfinite, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_minres_init(tmop_ctx *c, int64_t n, const double *b, const double *inv, double *x, double *r1, double *r2,
                     double *z, double *v, double *w, double *w2, tmop_minres_state *st2) {
  if (!c || !st2) return fail(TMOP_ERR_ARG, "NULL argument");
  launch_minres_init(n, b, inv, x, r1, r2, z, v, w, w2, c->vpart1, st2, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_minres_step(tmop_ctx *c, int64_t n, double *Av, const double *r1, const double *r2, const double *inv,
                     double *z, double *v, const double *w, double *w1buf, const double *w2, double *x, double rtol,
                     tmop_minres_state *st2, int k) {
  if (!c || !st2) return fail(TMOP_ERR_ARG, "NULL argument");
  launch_minres_step(n, Av, r1, r2, inv, z, v, w, w1buf, w2, x, rtol, st2 + (k & 1), st2 + ((k + 1) & 1), c->vpart1,
                     c->vpart2, c->hist, c->hist_cap, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

// ---- slab-partitioned MINRES (see tmop_b200.h) ----
static int dist_args_ok(tmop_ctx *c, int64_t n, int64_t nn, int64_t n_owned, const void *scal) {
  if (!c || !scal) return fail(TMOP_ERR_ARG, "NULL argument");
  if (nn < 0 || n_owned < 0 || n_owned > nn || (nn && n % nn))
    return fail(TMOP_ERR_ARG, "owned range invalid (n %lld, nn %lld, n_owned %lld)", (long long)n, (long long)nn,
                (long long)n_owned);
  return TMOP_OK;
}

int tmop_minres_dist_init_a(tmop_ctx *c, int64_t n, int64_t nn, int64_t n_owned, const double *b, const double *inv,
                            double *x, double *r1, double *r2, double *z, double *w, double *w2, double *scal) {
  int rc = dist_args_ok(c, n, nn, n_owned, scal);
  if (rc) return rc;
  launch_minres_dist_init_a(n, nn, n_owned, b, inv, x, r1, r2, z, w, w2, c->vpart1, scal, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_minres_dist_init_b(tmop_ctx *c, int64_t n, const double *z, double *v, const double *scal,
                            tmop_minres_state *st2) {
  if (!c || !scal || !st2) return fail(TMOP_ERR_ARG, "NULL argument");
  launch_minres_dist_init_b(n, z, v, scal, st2, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_minres_dist_k1(tmop_ctx *c, int64_t n, int64_t nn, int64_t n_owned, double *Av, const double *r1,
                        const double *v, tmop_minres_state *st2, int k, double *scal) {
  int rc = dist_args_ok(c, n, nn, n_owned, scal);
  if (rc) return rc;
  if (!st2) return fail(TMOP_ERR_ARG, "NULL state");
  launch_minres_dist_k1(n, nn, n_owned, Av, r1, v, st2 + (k & 1), c->vpart1, scal, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_minres_dist_k2(tmop_ctx *c, int64_t n, int64_t nn, int64_t n_owned, double *Av, const double *r2,
                        const double *inv, double *z, tmop_minres_state *st2, int k, double *scal) {
  int rc = dist_args_ok(c, n, nn, n_owned, scal);
  if (rc) return rc;
  if (!st2) return fail(TMOP_ERR_ARG, "NULL state");
  launch_minres_dist_k2(n, nn, n_owned, Av, r2, inv, z, st2 + (k & 1), c->vpart2, scal, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_minres_dist_k3(tmop_ctx *c, int64_t n, const double *z, double *v, const double *w, double *w1buf,
                        const double *w2, double *x, double rtol, tmop_minres_state *st2, int k, const double *scal) {
  if (!c || !scal || !st2) return fail(TMOP_ERR_ARG, "NULL argument");
  launch_minres_dist_k3(n, z, v, w, w1buf, w2, x, rtol, st2 + (k & 1), st2 + ((k + 1) & 1), scal, c->hist,
                        c->hist_cap, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_copy_components(tmop_ctx *c, double *dst, const double *src, int64_t stride, int64_t begin, int64_t count,
                         int ncomp) {
  if (!c || !dst || !src) return fail(TMOP_ERR_ARG, "NULL argument");
  if (ncomp < 1 || begin < 0 || count < 0 || begin + count > stride)
    return fail(TMOP_ERR_ARG, "range [%lld, %lld) outside the component stride %lld", (long long)begin,
                (long long)(begin + count), (long long)stride);
  if (count == 0) return TMOP_OK;
  CUDA_TRY(cudaMemcpy2DAsync(dst + begin, (size_t)stride * 8, src + begin, (size_t)stride * 8, (size_t)count * 8,
                             (size_t)ncomp, cudaMemcpyDefault, c->stream));
  return TMOP_OK;
}

int tmop_halo_pack(tmop_ctx *c, int64_t nn, int64_t plane, int lo, int hi, const double *y, double *send) {
  if (!c || !y || !send) return fail(TMOP_ERR_ARG, "NULL argument");
  if (plane < 0 || 2 * plane > nn + plane) return fail(TMOP_ERR_ARG, "plane size invalid");
  launch_halo_pack(nn, plane, lo, hi, y, send, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_halo_unpack(tmop_ctx *c, int64_t nn, int64_t plane, int lo, int hi, const double *recv, int mode,
                     const double *vfix, double cfix, double *y) {
  if (!c || !y || !recv) return fail(TMOP_ERR_ARG, "NULL argument");
  if (nn != c->nn) return fail(TMOP_ERR_ARG, "node count %lld does not match the context (%lld)", (long long)nn,
                               (long long)c->nn);
  launch_halo_unpack(nn, plane, lo, hi, recv, c->fixed, mode, vfix, cfix, y, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_halo_p2p_put(tmop_ctx *c, int64_t nn, int64_t plane, const double *y, double *peer_lo_box,
                      uint64_t *peer_lo_cnt, double *peer_hi_box, uint64_t *peer_hi_cnt, int slot) {
  if (!c || !y) return fail(TMOP_ERR_ARG, "NULL argument");
  if ((peer_lo_box == nullptr) != (peer_lo_cnt == nullptr) || (peer_hi_box == nullptr) != (peer_hi_cnt == nullptr))
    return fail(TMOP_ERR_ARG, "mailbox and counter must be given together");
  if (slot < 0 || slot > 1 || plane <= 0 || plane > nn) return fail(TMOP_ERR_ARG, "slot / plane invalid");
  launch_halo_p2p_put(nn, plane, y, peer_lo_box, reinterpret_cast<unsigned long long *>(peer_lo_cnt), peer_hi_box,
                      reinterpret_cast<unsigned long long *>(peer_hi_cnt), slot, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int tmop_halo_p2p_get(tmop_ctx *c, int64_t nn, int64_t plane, double *y, const double *own_box,
                      const uint64_t *own_cnt, int lo, int hi, int slot, uint64_t target, int mode,
                      const double *vfix, double cfix, int32_t *err) {
  if (!c || !y || !own_box || !own_cnt || !err) return fail(TMOP_ERR_ARG, "NULL argument");
  if (nn != c->nn) return fail(TMOP_ERR_ARG, "node count does not match the context");
  if (slot < 0 || slot > 1 || plane <= 0 || plane > nn) return fail(TMOP_ERR_ARG, "slot / plane invalid");
  launch_halo_p2p_get(nn, plane, y, own_box, reinterpret_cast<const unsigned long long *>(own_cnt), lo, hi, slot,
                      (unsigned long long)target, c->fixed, mode, vfix, cfix, err, c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

int64_t tmop_halo_p2p_arrivals(int64_t plane) { return halo_p2p_grid(plane); }

int tmop_minres_set_history(tmop_ctx *c, double *hist, int capacity) {
  if (!c) return fail(TMOP_ERR_ARG, "ctx is NULL");
  c->hist = hist;
  c->hist_cap = hist ? capacity : 0;
  return TMOP_OK;
}

int tmop_minres_step_op(tmop_ctx *c, const double *qdata, int64_t n, double *Av, const double *r1, const double *r2,
                        const double *inv, double *z, double *v, const double *w, double *w1buf, const double *w2,
                        double *x, double rtol, tmop_minres_state *st2, int k) {
  if (!c || !qdata || !st2) return fail(TMOP_ERR_ARG, "NULL argument");
  if (n != c->nn * c->dim) return fail(TMOP_ERR_ARG, "vector length %lld != dim * n_nodes", (long long)n);
  tmop_minres_state *cur = st2 + (k & 1), *nxt = st2 + ((k + 1) & 1);
  if (c->lat_p > 0 && c->n1 <= 4 && !c->lim_on && c->ov_slabs > 1 && c->ne >= c->ov_min) {
    // overlapped: element kernel by z-slab on the context stream, the fused
    // E->L + K1 of each finished node range on the second stream (its K1
    // partials in a per-slab block of vpart1), then K2 / K3 reduce them all
    int rc = ensure_s2(c);
    if (rc) return rc;
    const int64_t layer = (int64_t)c->lat_n[0] * c->lat_n[1];
    const int64_t plane = ((int64_t)c->lat_n[0] * c->lat_p + 1) * ((int64_t)c->lat_n[1] * c->lat_p + 1);
    const int nz = c->lat_n[2];
    const int ns = c->ov_slabs < nz ? c->ov_slabs : nz;
    const int gs = VPART_CAP / ns;
    CUDA_TRY(cudaEventRecord(c->ev[31], c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->s2, c->ev[31], 0));
    int64_t done = 0;
    int np1 = 0;
    for (int s_ = 0; s_ < ns; ++s_) {
      const int64_t e0 = ((int64_t)s_ * nz / ns) * layer / 16 * 16;
      const int64_t e1 = s_ + 1 == ns ? c->ne : ((int64_t)(s_ + 1) * nz / ns) * layer / 16 * 16;
      if (e1 > e0) {
        ElemArgs a = base_args(c);
        a.in = v;
        a.qdata = qdata + e0 * tmop_qdata_stride(c);
        a.restr = c->restr + e0 * c->NP;
        a.E = c->E + e0 * c->dim * c->NP;
        a.ne = e1 - e0;
        a.stop = &cur->done;
        rc = run(c, metric_is_template(c->metric) ? K_APPLY : K_APPLY_NT, a, nullptr);
        if (rc) return rc;
      }
      const int64_t fin = e1 == c->ne ? c->nn : (e1 / layer) * c->lat_p * plane;
      if (fin > done) {
        CUDA_TRY(cudaEventRecord(c->ev[s_], c->stream));
        CUDA_TRY(cudaStreamWaitEvent(c->s2, c->ev[s_], 0));
        int64_t want = (fin - done + 4 * 128 - 1) / (4 * 128);
        const int grid = (int)(want < 1 ? 1 : (want > gs ? gs : want));
        launch_e2l_k1_range(c->nn, done, fin, e2l_map(c), c->E, nullptr, c->fixed, v, r1, Av, cur,
                            c->vpart1 + np1, grid, c->s2);
        CUDA_TRY(cudaGetLastError());
        np1 += grid;
        done = fin;
      }
    }
    CUDA_TRY(cudaEventRecord(c->ev[32], c->s2));
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev[32], 0));
    launch_minres_k23(n, Av, r2, inv, z, v, w, w1buf, w2, x, rtol, cur, nxt, c->vpart1, np1, c->vpart2, c->hist,
                      c->hist_cap, c->stream);
    CUDA_TRY(cudaGetLastError());
    return TMOP_OK;
  }
  ElemArgs a = base_args(c);
  a.in = v;
  a.qdata = qdata;
  a.stop = &cur->done;
  int rc = run(c, metric_is_template(c->metric) ? K_APPLY : K_APPLY_NT, a, nullptr);
  if (rc) return rc;
  if (c->lim_on) {
    rc = lim_nodes(c, K_LIM_FIELD, v, nullptr, 1);
    if (rc) return rc;
  }
  launch_minres_step_op(c->dim, c->nn, e2l_map(c), c->E, c->lim_on ? c->lim_y : nullptr, c->fixed, n, Av, r1, r2,
                        inv, z, v, w, w1buf, w2, x, rtol, cur, nxt, c->vpart1, c->vpart2, c->hist, c->hist_cap,
                        c->stream);
  CUDA_TRY(cudaGetLastError());
  return TMOP_OK;
}

}  // extern "C"
