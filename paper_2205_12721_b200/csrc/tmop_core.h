// tmop_core.h -- launchers implemented in tmop_core.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/tmop_b200.h"

namespace tmop {

constexpr int VEC_NT = 256;
constexpr int VEC_GRID_CAP = 148 * 4;
constexpr int VPART_CAP = 4096;   // vector partials capacity (overlapped K1 slabs need more than one grid)

int vec_grid(int64_t n);

// Node-major view of the E-vector: the transposed restriction (CSR by node,
// element-ascending) and the E layout; lat_p > 0 marks a verified
// structured box lattice (lat_n element counts, order lat_p) whose copies
// are enumerated arithmetically instead of through off / idx.
struct E2LMap {
  const int64_t *off;
  const uint32_t *idx;
  int np, es;
  int lat_n[3], lat_p;
  // exact division by the lattice node counts NX, NY for node ids < 2^31:
  // q = (n * mag) >> sh  (host-computed, tmop_ctx_set_lattice)
  uint64_t mag_x, mag_y;
  int sh_x, sh_y;
};
// Node range [n0, n1) (n1 < 0: all nodes).
int launch_e2l(int dim, int64_t nn, const E2LMap &m, const double *E, const uint8_t *fixed, int mode, const double *v, const double *add, double *y, cudaStream_t s,
               int64_t n0 = 0, int64_t n1 = -1, int nt = 256);
void launch_fin(int nparts, const double *psum, const double *pmin, const int64_t *parg, double sum_scale,
                double *sum_out, double add_scale, const double *add, tmop_det_status *det_out, cudaStream_t s);
int launch_metric_eval(int metric, int dim, int64_t n, const double *T, double *mu, double *P, double *H);
void launch_dot(int64_t n, const double *a, const double *b, double *part, double *out, cudaStream_t s);
void launch_axpby(int64_t n, double a, const double *x, double b, double *y, cudaStream_t s);
void launch_trial(int64_t n, const double *x, const double *dx, double alpha, double *out, cudaStream_t s);
void launch_jacobi(int64_t n, const double *d, double fl, double *inv, int32_t *nonfinite, cudaStream_t s);
void launch_minres_init(int64_t n, const double *b, const double *inv, double *x, double *r1, double *r2, double *z,
                        double *v, double *w, double *w2, double *part, tmop_minres_state *st, cudaStream_t s);
void launch_minres_step(int64_t n, double *Av, const double *r1, const double *r2, const double *inv, double *z,
                        double *v, const double *w, double *w1buf, const double *w2, double *x, double rtol,
                        tmop_minres_state *cur, tmop_minres_state *nxt, double *part1, double *part2,
                        double *hist, int hist_cap, cudaStream_t s);

void launch_minres_step_op(int dim, int64_t nn, const E2LMap &m, const double *E, const double *add,
                           const uint8_t *fixed, int64_t n, double *Av, const double *r1, const double *r2,
                           const double *inv, double *z, double *v, const double *w, double *w1buf, const double *w2,
                           double *x, double rtol, tmop_minres_state *cur, tmop_minres_state *nxt, double *part1,
                           double *part2, double *hist, int hist_cap, cudaStream_t s);

void launch_e2l_k1_range(int64_t nn, int64_t n0, int64_t n1, const E2LMap &m, const double *E, const double *add,
                         const uint8_t *fixed, const double *v, const double *r1, double *Av,
                         const tmop_minres_state *cur, double *part, int grid, cudaStream_t s);
void launch_minres_k23(int64_t n, double *Av, const double *r2, const double *inv, double *z, double *v,
                       const double *w, double *w1buf, const double *w2, double *x, double rtol,
                       tmop_minres_state *cur, tmop_minres_state *nxt, double *part1, int np1, double *part2,
                       double *hist, int hist_cap, cudaStream_t s);
void launch_minres_dist_init_a(int64_t n, int64_t nn, int64_t n_owned, const double *b, const double *inv, double *x,
                               double *r1, double *r2, double *z, double *w, double *w2, double *part, double *scal,
                               cudaStream_t s);
void launch_minres_dist_init_b(int64_t n, const double *z, double *v, const double *scal, tmop_minres_state *st,
                               cudaStream_t s);
void launch_minres_dist_k1(int64_t n, int64_t nn, int64_t n_owned, double *Av, const double *r1, const double *v,
                           const tmop_minres_state *cur, double *part, double *scal, cudaStream_t s);
void launch_minres_dist_k2(int64_t n, int64_t nn, int64_t n_owned, double *Av, const double *r2, const double *inv,
                           double *z, const tmop_minres_state *cur, double *part, double *scal, cudaStream_t s);
void launch_minres_dist_k3(int64_t n, const double *z, double *v, const double *w, double *w1buf, const double *w2,
                           double *x, double rtol, tmop_minres_state *cur, tmop_minres_state *nxt,
                           const double *scal, double *hist, int hist_cap, cudaStream_t s);
void launch_halo_pack(int64_t nn, int64_t pl, int lo, int hi, const double *y, double *send, cudaStream_t s);
void launch_halo_unpack(int64_t nn, int64_t pl, int lo, int hi, const double *recv, const uint8_t *fixed, int mode,
                        const double *vfix, double cfix, double *y, cudaStream_t s);
int halo_p2p_grid(int64_t pl);
void launch_halo_p2p_put(int64_t nn, int64_t pl, const double *y, double *box_lo, unsigned long long *cnt_lo,
                         double *box_hi, unsigned long long *cnt_hi, int slot, cudaStream_t s);
void launch_halo_p2p_get(int64_t nn, int64_t pl, double *y, const double *box, const unsigned long long *cnt, int lo,
                         int hi, int slot, unsigned long long target, const uint8_t *fixed, int mode,
                         const double *vfix, double cfix, int *err, cudaStream_t s);
int launch_lattice_check(int64_t ne, int np, const int32_t *restr, int nx, int ny, int nz, int p, int *flag,
                         cudaStream_t s);

}  // namespace tmop
