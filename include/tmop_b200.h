/*
 * tmop_b200.h -- C ABI of the B200-native TMOP hot path (libtmop_b200.so).
 *
 * This is the drop-in boundary for the reference package's `ProblemLike`
 * operator protocol (/root/reference/pkg/src/tmopbench/solvers.py:183-189)
 * and its concrete implementer `TmopProblem`
 * (/root/reference/pkg/src/tmopbench/operator.py:220-459).  Every entry point
 * takes plain device pointers and sizes, is asynchronous on the context's
 * CUDA stream and returns an int status (TMOP_OK == 0).  No torch types.
 *
 * Vector conventions follow the reference (operator.py:10-13, fe.py:1-14):
 * T-vectors are (dim * n_nodes) float64, component-major; node ids and
 * element ids are lexicographic with x fastest; restriction is int32
 * (n_elements, (order+1)^dim) with the local x index fastest.
 *
 * Q-data (the partially assembled Hessian, reference HessQData
 * operator.py:91-138) is stored ELEMENT-BLOCKED and LEAN:
 * qdata[e * stride + field * Q + slot(q)], stride = tmop_qdata_stride(ctx)
 * (== 2 mod 16 doubles: every element block is 16-byte aligned for TMA bulk
 * copies and 8 staged elements map to distinct shared-memory banks); in 3D
 * slot(q) stores qx as the slowest point index, slot = qy + nq*qz +
 * nq^2*qx for q = qx + nq*qy + nq^2*qz (2D: slot = q); fields =
 * T (d*d), k0, itau = 1/det T -- d^2 + 2 doubles per point instead of the
 * reference's 4 + 2 d^2.  S = T^{-T} and the four Hessian-template
 * coefficients are recomputed from them;
 * tmop_qdata_to_reference() materialises the reference's planar
 * coeffs / s_mat / t_mat arrays for inspection and parity tests.
 */
#ifndef TMOP_B200_H
#define TMOP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TMOP_OK = 0,
  TMOP_ERR_ARG = 1,          /* invalid argument / unsupported (dim, p, n_q) */
  TMOP_ERR_CUDA = 2,         /* a CUDA runtime call failed */
  TMOP_ERR_METRIC = 3,       /* metric id not valid for this dimension */
};

/* Metric ids: 2, 55, 303 follow metrics.py:41-44; 7, 302, 321 are the
 * MFEM-numbered extensions named by BASELINE.json (no reference code). */
enum { TMOP_MU_2 = 2, TMOP_MU_7 = 7, TMOP_MU_55 = 55, TMOP_MU_302 = 302,
       TMOP_MU_303 = 303, TMOP_MU_321 = 321 };

typedef struct tmop_ctx tmop_ctx;

/* Determinant status written by kernels that evaluate det(A) (device
 * memory).  min_det = min over all quadrature points of det(A); argmin is
 * the flat point index e * Q + q of the first minimum (ties -> smallest). */
typedef struct {
  double min_det;
  int64_t argmin;
} tmop_det_status;

/* ---- context (replaces TmopProblem.__init__, operator.py:230-250) ------ */

/* Create a context.  restriction/fixed/l2e_* are DEVICE pointers owned by
 * the caller and must outlive the context.  B, G are HOST (n_quad x
 * (order+1)) row-major tables B[q][i] = l_i(chi_q), G[q][i] = l_i'(chi_q)
 * (fe.py:143-160); w1 is the HOST 1D quadrature weight vector (n_quad)
 * (fe.py:126-140).  fixed is uint8 per node, bit a set <=> component a
 * constrained (mesh.py:159-160); the allocation must be readable up to
 * round_up(n_nodes, 4) bytes (the element kernels fetch the aligned 32-bit
 * word holding a node's flags).  l2e_offsets (n_nodes + 1, int64) and
 * l2e_index (n_elements * (order+1)^dim, uint32 = e * Np + local) give, for
 * every node, its element-local copies in ascending element order -- the
 * summation order of np.add.at in fe.py:189-204.  stream is a
 * cudaStream_t (NULL = legacy default stream). */
int tmop_ctx_create(tmop_ctx **out, int dim, int order, int n_quad,
                    int64_t n_elements, int64_t n_nodes,
                    const int32_t *restriction, const uint8_t *fixed,
                    const int64_t *l2e_offsets, const uint32_t *l2e_index,
                    const double *B, const double *G, const double *w1,
                    int metric, double inv_scale, double det_w,
                    double spatial_weight, void *stream);
int tmop_ctx_destroy(tmop_ctx *ctx);
int tmop_ctx_set_stream(tmop_ctx *ctx, void *stream);
/* Slab-overlapped Hessian action on lattices (tmop_hessian_apply, MINRES
 * steps): the element kernel runs in `slabs` z-slabs (1..30; 1 = one-shot)
 * with the E->L of finished node planes on a second stream, for meshes of
 * at least min_elements elements.  Defaults: 8 slabs (TMOP_APPLY_SLABS),
 * 262144 elements (TMOP_OVERLAP_MIN).  Results are bitwise identical. */
int tmop_ctx_set_apply_overlap(tmop_ctx *ctx, int slabs, int64_t min_elements);
/* Change target scale (build_targets, metrics.py:333-345) after creation. */
int tmop_ctx_set_target(tmop_ctx *ctx, double inv_scale, double det_w);
/* Size-field targets (EXTENSION: the reference has constant isotropic W
 * only, metrics.py:282-345; SPEC.md:9 lists space-dependent W as a
 * non-goal).  volume_nodal (DEVICE, n_nodes) is a target element volume per
 * node, interpolated to the quadrature points with B (fe.py:227-239):
 * v_q = sum_i eta_i phi_i(chi_q), W_q = v_q^(1/d) I, so T = A / v_q^(1/d) and
 * det W_q = v_q enter the energy / gradient / Hessian setup point by point
 * (the Hessian action and diagonal read them from the Q-data record).  The
 * field is material (fixed per quadrature point while x moves).  The
 * per-point 1/s_q array is computed here, on the context stream; a v_q <= 0
 * yields NaN (tmop_ctx_point_scale exposes the array for checks).  NULL
 * clears it (constant W = I); tmop_ctx_set_target also clears it. */
int tmop_ctx_set_size_field(tmop_ctx *ctx, const double *volume_nodal);
const double *tmop_ctx_point_scale(const tmop_ctx *ctx);

/* Declare that the mesh is the (nx, ny, nz) box lattice of build_box
 * (mesh.py:118-164).  The restriction is verified on the device; when it
 * matches, *accepted = 1 and the E->L gathers enumerate each node's element
 * copies arithmetically (same ascending element order, bitwise identical
 * sums) instead of reading the transpose map.  3D only; otherwise
 * *accepted = 0 and nothing changes.  Synchronises the context stream. */
int tmop_ctx_set_lattice(tmop_ctx *ctx, int nx, int ny, int nz, int *accepted);
int tmop_qdata_fields(const tmop_ctx *ctx);            /* doubles per point   */
int64_t tmop_qdata_stride(const tmop_ctx *ctx);        /* doubles per element */
int64_t tmop_qdata_size(const tmop_ctx *ctx);          /* doubles total       */
/* Reference-layout view of the Q-data: (fields_ref, n_elements * Q) planar,
 * fields_ref = 4 + 2 d^2 (c_id, c_ts, c_ss, c_x, S, T) for template metrics
 * and 1 + 2 d^2 (w, S, T) for mu_302 / mu_321 (operator.py:105-113). */
int tmop_qdata_reference_fields(const tmop_ctx *ctx);
int tmop_qdata_to_reference(tmop_ctx *ctx, const double *qdata, double *out);
/* Configure the displacement-limiting term (operator.py:57-76, 463-533):
 * x0 (reference positions, T-vector) and delta_nodal (n_nodes, or NULL for
 * the scalar delta) are DEVICE pointers kept by reference; x0 == NULL
 * disables the term.  When enabled, objective / gradient / hessian_apply /
 * hessian_diagonal / minres_step_op include it exactly where the reference
 * adds it (operator.py:324-325, 343-344, 415-416, 452-457). */
int tmop_ctx_set_limiting(tmop_ctx *ctx, const double *x0,
                          const double *delta_nodal, double delta,
                          double weight);
/* The limiting term alone (operator.py:488-533): value into *out (device
 * scalar), raw gradient B^T(c (B(x - x0))) and raw action B^T(c B v) (no
 * constraint handling), as limiting_value / limiting_gradient /
 * limiting_hessian_apply. */
int tmop_limiting_value(tmop_ctx *ctx, const double *x, double *out);
int tmop_limiting_gradient(tmop_ctx *ctx, const double *x, double *y);
int tmop_limiting_apply(tmop_ctx *ctx, const double *v, double *y);
const char *tmop_last_error(void);

/* ---- operator entry points (all async on the context stream) ---------- */

/* AssembleGradPA: hessian_setup (operator.py:350-371). */
int tmop_hessian_setup(tmop_ctx *ctx, const double *x, double *qdata,
                       tmop_det_status *det_out);
/* AddMultGradPA: hessian_apply (operator.py:401-418).  y = H vin on free
 * dofs, y = v on constrained dofs. */
int tmop_hessian_apply(tmop_ctx *ctx, const double *qdata, const double *v,
                       double *y);
/* The two phases of tmop_hessian_apply, exposed for per-kernel timing and
 * for fusing the E->L sum with solver updates: the element kernel (writes
 * the context's element-blocked E-vector) and the deterministic E->L sum
 * with the constrained-dof fix-up. */
int tmop_hessian_apply_elements(tmop_ctx *ctx, const double *qdata,
                                const double *v);
int tmop_hessian_apply_gather(tmop_ctx *ctx, const double *v, double *y);

/* Streaming pieces of the same action for host-resident pipelines
 * (H2D of v / element kernel / E->L / D2H of y overlapped slab by slab):
 * the element kernel over elements [e_begin, e_end) (e_begin % 16 == 0 and
 * e_end % 16 == 0 or e_end == n_elements, else TMOP_ERR_ARG: the kernels
 * write whole 16-element groups of the E-vector; reads v at those elements'
 * nodes only), and the E->L sum + constraint
 * fix-up for nodes [n_begin, n_end) (every element holding those nodes must
 * have been processed).  Results are bitwise identical to
 * tmop_hessian_apply. */
int tmop_hessian_apply_elements_range(tmop_ctx *ctx, const double *qdata, const double *v, int64_t e_begin,
                                      int64_t e_end);
int tmop_hessian_apply_gather_range(tmop_ctx *ctx, const double *v, double *y, int64_t n_begin, int64_t n_end);
/* AssembleGradDiagonalPA: hessian_diagonal (operator.py:420-459). */
int tmop_hessian_diagonal(tmop_ctx *ctx, const double *qdata, double *diag);
/* hessian_setup followed by hessian_diagonal (operator.py:350-371,
 * 420-459) -- what newton_solve does once per iteration when the Jacobi
 * preconditioner is on (solvers.py:292-295).  By default the two passes;
 * with TMOP_SETUP_DIAG_FUSED=1 (3D p <= 3, template metrics, no limiting
 * term) ONE element pass that forms the diagonal's H-pair values from each
 * group's records while they are still in shared memory (records written
 * once, never re-read) -- bitwise the same outputs, measured slower (see
 * DESIGN.md section 3).  diag is garbage when det_out reports an inverted
 * element, like the setup's Q-data. */
int tmop_hessian_setup_diagonal(tmop_ctx *ctx, const double *x, double *qdata, double *diag,
                                tmop_det_status *det_out);
/* AddMultPA: gradient (operator.py:328-346). */
int tmop_gradient(tmop_ctx *ctx, const double *x, double *grad,
                  tmop_det_status *det_out);
/* Gradient, energy and min det(A) from ONE element pass (the line search's
 * trial evaluation, solvers.py:210-216): energy_out (device scalar, may be
 * NULL) = objective(x) up to summation order. */
int tmop_gradient_energy(tmop_ctx *ctx, const double *x, double *grad, double *energy_out,
                         tmop_det_status *det_out);
/* GetLocalStateEnergyPA: objective (operator.py:311-326).  Writes F (incl.
 * the limiting term when configured) to *energy_out (device). */
int tmop_objective(tmop_ctx *ctx, const double *x, double *energy_out,
                   tmop_det_status *det_out);
/* min_det_jacobian (operator.py:296-304). */
int tmop_min_det(tmop_ctx *ctx, const double *x, tmop_det_status *det_out);
/* Per-element min det(A) and its point (diagnostics / exact batch
 * emulation of operator.py:267-272).  elem_min: n_elements doubles,
 * elem_arg: n_elements int32 (device). */
int tmop_element_min_det(tmop_ctx *ctx, const double *x, double *elem_min,
                         int32_t *elem_arg);
/* Volume of the mesh image by quadrature of det(A) (metrics.py:319-330). */
int tmop_volume(tmop_ctx *ctx, const double *x, double *vol_out);

/* Pointwise metric evaluation for n matrices T (n, d, d) row-major:
 * mu (n), P = dmu/dT (n, d, d), H = d2mu/dT2 (n, d*d, d*d); any output may
 * be NULL.  Device pointers, default stream, synchronous. */
int tmop_metric_eval(int metric, int dim, int64_t n, const double *T,
                     double *mu, double *P, double *H);

/* ---- vector kernels for the device MINRES / Newton (solvers.py) ------- */

/* Deterministic dot product (fixed-order two-pass reduction) -> *out (dev). */
int tmop_dot(tmop_ctx *ctx, int64_t n, const double *a, const double *b,
             double *out);
/* y = a * x + b * y (AXPBY). */
int tmop_axpby(tmop_ctx *ctx, int64_t n, double a, const double *x, double b,
               double *y);
/* out = x - alpha * dx (line search trial point, solvers.py:210). */
int tmop_trial_point(tmop_ctx *ctx, int64_t n, const double *x,
                     const double *dx, double alpha, double *out);
/* inv = 1 / max(|diag|, floor) (solvers.py:83-90); *nonfinite (dev int)
 * is set to 1 if any diag entry is not finite. */
int tmop_jacobi_inverse(tmop_ctx *ctx, int64_t n, const double *diag,
                        double floor_value, double *inv, int32_t *nonfinite);

/* Device-resident MINRES state (solvers.py:93-180).  All scalars live in
 * device memory so an iteration needs no host round trip; `done` makes every
 * later step a no-op, so the host may launch several steps per check. */
typedef struct {
  double beta1, beta, oldb, alfa, beta2, dbar, epsln, sn, cs, phibar,
         relres, gamma;
  int32_t itn, done, breakdown, nonpd;
} tmop_minres_state;

/* Initialise (slot 0 of st2): r1 = r2 = b; z = inv .* b (z = b if inv == NULL);
 * beta1 = sqrt(b.z); v = z / beta1; x = w = w2 = 0; st set up as in
 * solvers.py:103-125 (done = 1 when beta1 == 0). */
int tmop_minres_init(tmop_ctx *ctx, int64_t n, const double *b,
                     const double *inv, double *x, double *r1, double *r2,
                     double *z, double *v, double *w, double *w2,
                     tmop_minres_state *st2);
/* One MINRES iteration after the caller computed Av = A v (solvers.py:
 * 131-178).  Fused kernels: Av -= (beta/oldb) r1; alfa = v.Av;
 * Av -= (alfa/beta) r2; z = inv .* Av; beta2 = Av.z; Givens recurrence;
 * w1buf <- (v - oldeps w2 - delta w) / gamma; x += phi w1buf;
 * v <- z / beta.  The caller then rotates buffers:
 *   (r1, r2, free) <- (r2, Av, r1) and (w1, w2, w) <- (w2, w, w1buf).
 * st2 points to TWO state slots (device); init writes slot 0 and step k
 * (0-based) reads slot k&1 and writes slot (k+1)&1, so after K steps the
 * current state is slot K&1. */
int tmop_minres_step(tmop_ctx *ctx, int64_t n, double *Av, const double *r1,
                     const double *r2, const double *inv, double *z,
                     double *v, const double *w, double *w1buf,
                     const double *w2, double *x, double rtol,
                     tmop_minres_state *st2, int k);

/* Optional device array that receives relres after every MINRES iteration
 * (hist[itn] for itn < capacity) -- the reference's residual_history
 * (solvers.py:168-176) without host round trips.  NULL disables. */
int tmop_minres_set_history(tmop_ctx *ctx, double *hist, int capacity);

/* One full MINRES iteration for THIS context's Hessian (AddMultGradPA):
 * Av = H v with the E->L gather fused into the K1 update, then the K2 / K3
 * kernels of tmop_minres_step -- 4 launches, no host round trip.  Same
 * buffer rotation contract as tmop_minres_step. */
int tmop_minres_step_op(tmop_ctx *ctx, const double *qdata, int64_t n,
                        double *Av, const double *r1, const double *r2,
                        const double *inv, double *z, double *v,
                        const double *w, double *w1buf, const double *w2,
                        double *x, double rtol, tmop_minres_state *st2,
                        int k);

/* ---- slab-partitioned (multi-GPU) MINRES and halo planes -------------
 * The paper's MPI assembly P^T -- absent from the
 * reference -- for a z-slab partition of a box lattice: local
 * vectors are component-major (3, nn) with the shared node planes (nodes
 * [0, plane) and [nn - plane, nn)) duplicated on both neighbours.
 *
 * MINRES phases (solvers.py:93-180) with every inner product taken over
 * OWNED entries (node < n_owned in each component; nn = 0: all owned) and
 * reduced in a fixed order into the device scalar scal[k]; between phases
 * the caller all-reduces scal[k] (SUM) across ranks on the context stream
 * (NCCL), so no phase needs a host round trip:
 *   init_a: r1 = r2 = b; z = inv .* b; x = w = w2 = 0; scal[0] = b.z
 *   init_b: beta1 = sqrt(scal[0]); v = z / beta1; state slot 0
 *   k1:     Av -= (beta/oldb) r1 (itn >= 1); scal[0] = v.Av
 *   k2:     alfa = scal[0]; Av -= (alfa/beta) r2; z = inv .* Av; scal[1] = Av.z
 *   k3:     beta2 = scal[1]; Givens recurrence; w1buf, x, v updates
 * Same buffer rotation and state-slot contract as tmop_minres_step; Av must
 * hold the halo-summed, constraint-fixed action on entry to k1. */
int tmop_minres_dist_init_a(tmop_ctx *ctx, int64_t n, int64_t nn, int64_t n_owned, const double *b, const double *inv,
                            double *x, double *r1, double *r2, double *z, double *w, double *w2, double *scal);
int tmop_minres_dist_init_b(tmop_ctx *ctx, int64_t n, const double *z, double *v, const double *scal,
                            tmop_minres_state *st2);
int tmop_minres_dist_k1(tmop_ctx *ctx, int64_t n, int64_t nn, int64_t n_owned, double *Av, const double *r1,
                        const double *v, tmop_minres_state *st2, int k, double *scal);
int tmop_minres_dist_k2(tmop_ctx *ctx, int64_t n, int64_t nn, int64_t n_owned, double *Av, const double *r2,
                        const double *inv, double *z, tmop_minres_state *st2, int k, double *scal);
int tmop_minres_dist_k3(tmop_ctx *ctx, int64_t n, const double *z, double *v, const double *w, double *w1buf,
                        const double *w2, double *x, double rtol, tmop_minres_state *st2, int k, const double *scal);
/* Component ranges of a T-vector between host and device (the pipelined
 * host-resident Hessian action, operator.py:401-418 called with numpy
 * arrays): entries [begin, begin + count) of each of ncomp components
 * (component stride `stride` doubles in both dst and src) as ONE strided copy
 * on the context's stream (cudaMemcpyDefault: host buffers must be pinned
 * for the copy to be asynchronous).  Measured on the B200 box: 16-slab
 * concurrent H2D + D2H of a 99.2 M-double vector 18.3 ms as 2 x 16 strided
 * copies vs 19.0 ms as 2 x 48 plain copies. */
int tmop_copy_components(tmop_ctx *ctx, double *dst, const double *src, int64_t stride, int64_t begin, int64_t count,
                         int ncomp);

/* Halo planes: pack the bottom (lo != 0) and top (hi != 0) node planes of y
 * into send = [lo plane: 3 x plane][hi plane: 3 x plane]; unpack adds the
 * neighbours' partial sums (same layout) into y's planes and, for mode 1,
 * re-applies the constraint convention there using THIS context's fixed
 * flags: fixed entries take vfix[i] (Hessian action: v, operator.py:417) or
 * cfix when vfix is NULL (diagonal: 1.0, operator.py:458); mode 0 keeps the
 * sum (gradient: 0 + 0).  nn must equal the context's node count. */
int tmop_halo_pack(tmop_ctx *ctx, int64_t nn, int64_t plane, int lo, int hi, const double *y, double *send);
int tmop_halo_unpack(tmop_ctx *ctx, int64_t nn, int64_t plane, int lo, int hi, const double *recv, int mode,
                     const double *vfix, double cfix, double *y);

/* Peer-memory halo (no NCCL on the data path): each rank exports a mailbox
 * box[2 slots][2 sides][3 x plane] doubles and two uint64 arrival counters
 * cnt[2 sides] (side 0: from the lower neighbour, side 1: from the upper),
 * and maps its neighbours' (CUDA IPC on one node; the stores travel over
 * NVLink).  Exchange k (k = 1, 2, ...) uses slot k & 1:
 *   put: this rank's bottom plane of y -> the lower neighbour's mailbox
 *        (side 1), its top plane -> the upper neighbour's (side 0); every
 *        CTA then releases one arrival at system scope on the receiver's
 *        counter (tmop_halo_p2p_arrivals(plane) arrivals per exchange)
 *   get: wait (acquire, bounded ~4 s -> *err = 1; once set, later gets
 *        return at once) until the own counters
 *        reach target = k * arrivals, then add the neighbours' partial sums
 *        into y's planes and re-apply the constraint convention (mode as
 *        tmop_halo_unpack).
 * Both run on the context stream after the local E->L; no host round trip.
 * Two slots suffice: a rank cannot start exchange k + 2 before its
 * neighbours finished reading exchange k (each get waits on the other's put). */
int tmop_halo_p2p_put(tmop_ctx *ctx, int64_t nn, int64_t plane, const double *y, double *peer_lo_box,
                      uint64_t *peer_lo_cnt, double *peer_hi_box, uint64_t *peer_hi_cnt, int slot);
int tmop_halo_p2p_get(tmop_ctx *ctx, int64_t nn, int64_t plane, double *y, const double *own_box,
                      const uint64_t *own_cnt, int lo, int hi, int slot, uint64_t target, int mode,
                      const double *vfix, double cfix, int32_t *err);
int64_t tmop_halo_p2p_arrivals(int64_t plane);

#ifdef __cplusplus
}
#endif

#endif /* TMOP_B200_H */
