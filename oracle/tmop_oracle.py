"""Vectorised numpy restatement of the reference TMOP path (CPU oracle).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

Reference = /root/reference/pkg/src/tmopbench (abbreviations as in
SURVEY.md: op = operator.py, fe = fe.py, met = metrics.py, ker =
_kernels.py, sol = solvers.py, mesh = mesh.py).

Layout conventions (identical to the reference, fe:1-14, mesh:67-105):
  * T-vectors are flat (d * n_nodes,), component-major;
  * node ids and element ids are lexicographic with x fastest;
  * element-local dof / quadrature indices are lexicographic with the
    direction-1 (x) index fastest, i.e. C-order ravels of (z, y, x);
  * restriction is (n_elements, (p+1)^d) int32.

Internally the oracle keeps per-point matrices "matrix last": arrays of
shape (Ne, Q, d, d).  `planar()` converts to the reference's planar
(d, d, Ne*Q) layout for comparisons against golden vectors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# metric ids (met:41-44 for 2/55/303; 7/302/321 are extensions, unpinned)
MU_2, MU_7, MU_55, MU_302, MU_303, MU_321 = 2, 7, 55, 302, 303, 321
TEMPLATE_METRICS = (MU_2, MU_7, MU_55, MU_303)
METRIC_DIM = {MU_2: 2, MU_7: 2, MU_55: None, MU_302: 3, MU_303: 3, MU_321: 3}

JACOBI_FLOOR = 1e-12   # sol:23
GROWTH = 1.2           # sol:24


class InvalidMesh(RuntimeError):
    """Oracle twin of InvalidMeshError (op:45-54)."""

    def __init__(self, element, point, value):
        self.element, self.point, self.value = int(element), int(point), float(value)
        super().__init__(f"det(A) = {value:.3e} at element {element} point {point}")


# ---------------------------------------------------------------------------
# 1D tables (fe:42-160)
# ---------------------------------------------------------------------------

def gll_points(n: int) -> np.ndarray:
    """n Gauss-Lobatto points on [0,1]: endpoints + roots of P'_{n-1} (fe:42-53)."""
    if n == 2:
        return np.array([0.0, 1.0])
    c = np.zeros(n)
    c[-1] = 1.0
    inner = np.sort(np.polynomial.legendre.Legendre(c).deriv().roots().real)
    return (np.concatenate(([-1.0], inner, [1.0])) + 1.0) * 0.5


def gauss_legendre(nq: int):
    """Gauss-Legendre points/weights mapped to [0,1] (fe:126-131)."""
    if not 1 <= nq <= 32:
        raise ValueError("n_q must be in [1, 32]")
    x, w = np.polynomial.legendre.leggauss(nq)
    return (x + 1.0) / 2.0, w / 2.0


def lagrange_tables(nodes: np.ndarray, pts: np.ndarray):
    """B[q,i] = l_i(pts_q), G[q,i] = l_i'(pts_q), barycentric (fe:71-111)."""
    n = len(nodes)
    diff_nodes = nodes[:, None] - nodes[None, :]
    np.fill_diagonal(diff_nodes, 1.0)
    bw = 1.0 / np.prod(diff_nodes, axis=1)
    B = np.empty((len(pts), n))
    G = np.empty((len(pts), n))
    for q, x in enumerate(pts):
        dx = x - nodes
        hit = np.nonzero(np.abs(dx) < 1e-13)[0]
        if hit.size:
            k = int(hit[0])
            B[q] = 0.0
            B[q, k] = 1.0
            gap = nodes[k] - nodes
            gap[k] = 1.0
            row = (bw / bw[k]) / gap
            row[k] = 0.0
            row[k] = -row.sum()
            G[q] = row
            continue
        inv = 1.0 / dx
        t = bw * inv
        lv = t / t.sum()
        B[q] = lv
        G[q] = lv * (inv.sum() - inv)
    return B, G


def tensor_weights(w: np.ndarray, dim: int) -> np.ndarray:
    """Tensor weights, x index fastest (fe:134-140)."""
    out = w
    for _ in range(dim - 1):
        out = np.multiply.outer(w, out)
    return out.ravel()


# ---------------------------------------------------------------------------
# Mesh (mesh:108-164)
# ---------------------------------------------------------------------------

@dataclass
class OMesh:
    dim: int
    order: int
    counts: tuple
    coords: np.ndarray        # (d, N)
    restriction: np.ndarray   # (Ne, n^d) int32
    fixed: np.ndarray         # (d, N) bool

    @property
    def n_nodes(self):
        return self.coords.shape[1]

    @property
    def n_elements(self):
        return self.restriction.shape[0]

    @property
    def n_dofs(self):
        return self.dim * self.n_nodes


def box_mesh(dim: int, counts, order: int) -> OMesh:
    """Uniform Q_p lattice of [0,1]^d with GLL nodes inside elements."""
    counts = tuple(int(c) for c in counts)
    ref = gll_points(order + 1)
    axes = []
    for c in counts:
        pts = ((np.arange(c)[:, None] + ref[None, :]) / c)[:, :order].ravel()
        axes.append(np.concatenate((pts, [1.0])))
        axes[-1][0] = 0.0
    nd = [c * order + 1 for c in counts]
    # node id = ix + nx*(iy + ny*iz); coords via broadcasting (x fastest)
    lat = np.indices(nd[::-1]).reshape(dim, -1)[::-1]      # lat[a] = index on axis a
    coords = np.stack([axes[a][lat[a]] for a in range(dim)])
    fixed = np.stack([(lat[a] == 0) | (lat[a] == nd[a] - 1) for a in range(dim)])
    # element e = ex + cx*(ey + cy*ez); local l = lx + n*(ly + n*lz)
    n = order + 1
    elat = np.indices(counts[::-1]).reshape(dim, -1)[::-1]
    llat = np.indices((n,) * dim).reshape(dim, -1)[::-1]
    strides = np.cumprod([1] + nd[:-1])
    gid = np.zeros((elat.shape[1], llat.shape[1]), dtype=np.int64)
    for a in range(dim):
        gid += (elat[a][:, None] * order + llat[a][None, :]) * strides[a]
    return OMesh(dim, order, counts, coords, gid.astype(np.int32), fixed)


def perturb(mesh: OMesh, rng: np.random.Generator, amplitude: float) -> np.ndarray:
    """Seeded jitter of free components (reference tests/oracles.py:121-131)."""
    gap = (1.0 / max(mesh.counts)) / mesh.order ** 2
    x = mesh.coords.ravel().copy()
    j = amplitude * gap * rng.uniform(-1.0, 1.0, x.shape)
    j[mesh.fixed.ravel()] = 0.0
    return x + j


# ---------------------------------------------------------------------------
# Kershaw deformation (mesh:182-251)
# ---------------------------------------------------------------------------

def _k_right(eps, x):
    return np.where(x <= 0.5, (2.0 - eps) * x, 1.0 + eps * (x - 1.0))


def _k_left(eps, x):
    return 1.0 - _k_right(eps, 1.0 - x)


def _k_step(a, b, x):
    t = np.clip(x, 0.0, 1.0)
    return a + (b - a) * (t * t * t * (t * (6.0 * t - 15.0) + 10.0))


def kershaw(epsy, epsz, x, y, z):
    layer = np.trunc(x * 6.0)
    lam = (x - layer / 6.0) * 6.0

    def blend(eps, c):
        lo, hi = _k_left(eps, c), _k_right(eps, c)
        out = hi.copy()
        out = np.where(layer == 0, lo, out)
        out = np.where((layer == 1) | (layer == 4), _k_step(lo, hi, lam), out)
        out = np.where(layer == 2, _k_step(hi, lo, lam / 2.0), out)
        out = np.where(layer == 3, _k_step(hi, lo, (1.0 + lam) / 2.0), out)
        return out

    return x.copy(), blend(epsy, y), blend(epsz, z)


# ---------------------------------------------------------------------------
# Sum-factorised contractions (fe:180-294)
# ---------------------------------------------------------------------------

def _fwd(U, mats):
    """U (..., [z,] y, x) dof tensor -> quad tensor; mats[k] acts on axis k (x=0)."""
    if len(mats) == 2:
        t = np.einsum("qj,...ji->...qi", mats[1], U)
        return np.einsum("pi,...qi->...qp", mats[0], t)
    t = np.einsum("rk,...kji->...rji", mats[2], U)
    t = np.einsum("qj,...rji->...rqi", mats[1], t)
    return np.einsum("pi,...rqi->...rqp", mats[0], t)


def _bwd(Z, mats):
    """Adjoint of _fwd."""
    if len(mats) == 2:
        t = np.einsum("pi,...qp->...qi", mats[0], Z)
        return np.einsum("qj,...qi->...ji", mats[1], t)
    t = np.einsum("pi,...rqp->...rqi", mats[0], Z)
    t = np.einsum("qj,...rqi->...rji", mats[1], t)
    return np.einsum("rk,...rji->...kji", mats[2], t)


class Discretization:
    """Mesh + 1D tables + quadrature; the oracle's view of TmopProblem's
    discretisation (op:230-250)."""

    def __init__(self, mesh: OMesh, n_quad: int):
        self.mesh = mesh
        self.d = mesh.dim
        self.n = mesh.order + 1
        self.nq = n_quad
        self.Q = n_quad ** self.d
        self.nodes = gll_points(self.n)
        self.qpts, self.qw1 = gauss_legendre(n_quad)
        self.B, self.G = lagrange_tables(self.nodes, self.qpts)
        self.wq = tensor_weights(self.qw1, self.d)

    def mats(self, direction):
        return [self.G if k == direction else self.B for k in range(self.d)]

    def gather(self, vec2):
        """(c, N) -> (c, Ne, n,..,n) for any number c of fields (fe:180-187)."""
        e = vec2[:, self.mesh.restriction]
        return e.reshape((vec2.shape[0], self.mesh.n_elements) + (self.n,) * self.d)

    def scatter(self, E):
        """(d, Ne, n^d) E-vector -> (d, N), ascending element order (fe:189-204)."""
        out = np.zeros((self.d, self.mesh.n_nodes))
        idx = self.mesh.restriction.ravel()
        for a in range(self.d):
            np.add.at(out[a], idx, E[a].reshape(-1))
        return out

    def grad_at_quad(self, vec2):
        """g[e, q, a, p] = d(vec_a)/d(xi_p) at quadrature points."""
        U = self.gather(vec2)
        Ne = self.mesh.n_elements
        g = np.empty((Ne, self.Q, self.d, self.d))
        for p in range(self.d):
            g[:, :, :, p] = _fwd(U, self.mats(p)).reshape(self.d, Ne, self.Q).transpose(1, 2, 0)
        return g

    def pull_back(self, z):
        """z[e, q, a, n] -> (d, N): sum_n (G_n-contraction)^T z[..., n], scattered."""
        Ne = self.mesh.n_elements
        acc = 0.0
        for n in range(self.d):
            zn = z[:, :, :, n].transpose(2, 0, 1).reshape((self.d, Ne) + (self.nq,) * self.d)
            acc = acc + _bwd(zn, self.mats(n))
        return self.scatter(acc.reshape(self.d, Ne, -1))

    def jacobians(self, x):
        return self.grad_at_quad(np.asarray(x, float).reshape(self.d, -1))


# ---------------------------------------------------------------------------
# Point-wise metric algebra (met:64-262, ker:20-258)
# ---------------------------------------------------------------------------

def det(A):
    if A.shape[-1] == 2:
        return A[..., 0, 0] * A[..., 1, 1] - A[..., 0, 1] * A[..., 1, 0]
    return (A[..., 0, 0] * (A[..., 1, 1] * A[..., 2, 2] - A[..., 1, 2] * A[..., 2, 1])
            - A[..., 0, 1] * (A[..., 1, 0] * A[..., 2, 2] - A[..., 1, 2] * A[..., 2, 0])
            + A[..., 0, 2] * (A[..., 1, 0] * A[..., 2, 1] - A[..., 1, 1] * A[..., 2, 0]))


def cofactor(A):
    """cof(A) so that A^{-T} = cof(A) / det(A) (met:79-97)."""
    C = np.empty_like(A)
    if A.shape[-1] == 2:
        C[..., 0, 0] = A[..., 1, 1]
        C[..., 0, 1] = -A[..., 1, 0]
        C[..., 1, 0] = -A[..., 0, 1]
        C[..., 1, 1] = A[..., 0, 0]
        return C
    for i in range(3):
        i1, i2 = (i + 1) % 3, (i + 2) % 3
        for j in range(3):
            j1, j2 = (j + 1) % 3, (j + 2) % 3
            C[..., i, j] = A[..., i1, j1] * A[..., i2, j2] - A[..., i1, j2] * A[..., i2, j1]
    return C


def frob2(A):
    return np.sum(A * A, axis=(-2, -1))


def metric_value(metric, T):
    tau = det(T)
    I1 = frob2(T)
    d = T.shape[-1]
    if metric == MU_2:
        return I1 / (2.0 * tau) - 1.0
    if metric == MU_55:
        return (tau - 1.0) ** 2
    if metric == MU_303:
        return I1 / (3.0 * np.cbrt(tau * tau)) - 1.0
    S = cofactor(T) / tau[..., None, None]
    J = frob2(S)
    if metric == MU_7:
        return I1 + J - 2.0 * d   # |T - T^{-t}|^2
    if metric == MU_302:
        return I1 * J / 9.0 - 1.0
    if metric == MU_321:
        return I1 + J - 2.0 * d
    raise ValueError(metric)


def first_coeffs(metric, tau, I1):
    """(a_t, a_s) of dmu/dT = a_t T + a_s S for template metrics (met:188-196)."""
    if metric == MU_2:
        return 1.0 / tau, -I1 / (2.0 * tau)
    if metric == MU_55:
        return np.zeros_like(tau), 2.0 * tau * (tau - 1.0)
    if metric == MU_303:
        r = 1.0 / np.cbrt(tau * tau)
        return (2.0 / 3.0) * r, -(2.0 / 9.0) * I1 * r
    if metric == MU_7:
        # mu7 = I1 (1 + tau^-2) - 4 in 2D; dI1 = 2T, d(tau^-2) = -2 tau^-2 S
        it2 = 1.0 / (tau * tau)
        return 2.0 * (1.0 + it2), -2.0 * I1 * it2
    raise ValueError(metric)


def second_coeffs(metric, tau, I1):
    """(c_id, c_ts, c_ss, c_x) of the template (met:199-210)."""
    if metric == MU_2:
        h = I1 / (2.0 * tau)
        return 1.0 / tau, -1.0 / tau, h, h
    if metric == MU_55:
        z = np.zeros_like(tau)
        return z, z, 2.0 * tau * (2.0 * tau - 1.0), -2.0 * tau * (tau - 1.0)
    if metric == MU_303:
        r = 1.0 / np.cbrt(tau * tau)
        return (2.0 / 3.0) * r, -(4.0 / 9.0) * r, (4.0 / 27.0) * I1 * r, (2.0 / 9.0) * I1 * r
    if metric == MU_7:
        # P = 2(1+t^-2) T - 2 I1 t^-2 S; dP = 2(1+t^-2) dT - 4 t^-2 (S:dT) T
        #     - 4 t^-2 (T:dT) S + 4 I1 t^-2 (S:dT) S + 2 I1 t^-2 S dT^T S
        it2 = 1.0 / (tau * tau)
        return 2.0 * (1.0 + it2), -4.0 * it2, 4.0 * I1 * it2, 2.0 * I1 * it2
    raise ValueError(metric)


def metric_first(metric, T):
    """dmu/dT (..., d, d)."""
    tau = det(T)
    S = cofactor(T) / tau[..., None, None]
    I1 = frob2(T)
    if metric in TEMPLATE_METRICS:
        at, as_ = first_coeffs(metric, tau, I1)
        return at[..., None, None] * T + as_[..., None, None] * S
    J = frob2(S)
    M = S @ np.swapaxes(S, -1, -2) @ S           # dJ/dT = -2 M
    if metric == MU_321:
        return 2.0 * T - 2.0 * M
    if metric == MU_302:
        return (2.0 * J[..., None, None] * T - 2.0 * I1[..., None, None] * M) / 9.0
    raise ValueError(metric)


def hess_action_point(metric, T, S, g, c=None):
    """z = (d^2 mu/dT^2) : g per point, T/S/g (..., d, d).  For template
    metrics `c` are the (scaled) 4 coefficients (..., 4) (ker:235-258)."""
    if metric in TEMPLATE_METRICS:
        dt = np.sum(T * g, axis=(-2, -1))
        ds = np.sum(S * g, axis=(-2, -1))
        c0, c1, c2, c3 = (c[..., k] for k in range(4))
        w1 = c1 * dt + c2 * ds
        w2 = c1 * ds
        cross = S @ np.swapaxes(g, -1, -2) @ S
        return (c0[..., None, None] * g + w1[..., None, None] * S
                + w2[..., None, None] * T + c3[..., None, None] * cross)
    St = np.swapaxes(S, -1, -2)
    M = S @ St @ S
    dS = -S @ np.swapaxes(g, -1, -2) @ S
    dM = dS @ St @ S + S @ np.swapaxes(dS, -1, -2) @ S + S @ St @ dS
    if metric == MU_321:
        return 2.0 * g - 2.0 * dM
    if metric == MU_302:
        I1 = frob2(T)[..., None, None]
        J = frob2(S)[..., None, None]
        dJ = (-2.0 * np.sum(M * g, axis=(-2, -1)))[..., None, None]
        dI1 = (2.0 * np.sum(T * g, axis=(-2, -1)))[..., None, None]
        return (2.0 * dJ * T + 2.0 * J * g - 2.0 * dI1 * M - 2.0 * I1 * dM) / 9.0
    raise ValueError(metric)


def metric_second(metric, T):
    """Full (..., d*d, d*d) Hessian, row m*d+n, col o*d+p (met:240-262)."""
    d = T.shape[-1]
    tau = det(T)
    S = cofactor(T) / tau[..., None, None]
    c = None
    if metric in TEMPLATE_METRICS:
        c = np.stack(second_coeffs(metric, tau, frob2(T)), axis=-1)
    H = np.empty(T.shape[:-2] + (d * d, d * d))
    for col in range(d * d):
        g = np.zeros_like(T)
        g[..., col // d, col % d] = 1.0
        H[..., :, col] = hess_action_point(metric, T, S, g, c).reshape(T.shape[:-2] + (d * d,))
    return H


# ---------------------------------------------------------------------------
# The operator (op:220-459)
# ---------------------------------------------------------------------------

@dataclass
class OQData:
    """Oracle Q-data: c (Ne, Q, 4) [template metrics], S, T (Ne, Q, d, d),
    w (Ne, Q) = coef * w_q [non-template metrics]."""
    metric: int
    c: np.ndarray | None
    S: np.ndarray
    T: np.ndarray
    w: np.ndarray

    def planar(self):
        """Reference layout: coeffs (4, NQ), s_mat/t_mat (d, d, NQ) (op:105-113)."""
        d = self.S.shape[-1]
        def pl(A):
            return np.moveaxis(A.reshape(-1, d, d), 0, -1)
        coeffs = None if self.c is None else self.c.reshape(-1, 4).T.copy()
        return coeffs, pl(self.S).copy(), pl(self.T).copy()


def _pt(a):
    """Broadcast a per-point (Ne, Q) factor over (Ne, Q, d, d); scalars pass."""
    a = np.asarray(a, float)
    return a[..., None, None] if a.ndim else a


class OracleProblem:
    """CPU twin of TmopProblem for ideal constant isotropic targets W = s I
    (met:293-345): only inv_scale = 1/s and det_w = s^d reach the kernels."""

    def __init__(self, mesh: OMesh, metric: int, n_quad: int, target: str = "unit",
                 h: float | None = None, spatial_weight: float = 1.0,
                 limiting: dict | None = None, size=None):
        need = METRIC_DIM[metric]
        if need is not None and need != mesh.dim:
            raise ValueError("metric/dimension mismatch")
        self.disc = Discretization(mesh, n_quad)
        self.mesh = mesh
        self.metric = metric
        self.omega = spatial_weight
        if target == "field":
            # size-field targets (EXTENSION -- no reference code: parity
            # unpinned; metrics.py:282-345 has constant W only): W_q =
            # v_q^(1/d) I, v_q = B-interpolated nodal target volume; the
            # scales become (Ne, Q) arrays (material field, fixed per point)
            D = self.disc
            U = D.gather(np.asarray(size, float)[None, :])[0]
            vq = _fwd(U, [D.B] * mesh.dim).reshape(mesh.n_elements, D.Q)
            if not np.all(vq > 0):
                raise ValueError("size field: non-positive target volume at a quadrature point")
            isq = 1.0 / np.cbrt(vq) if mesh.dim == 3 else 1.0 / np.sqrt(vq)
            self.scale = 1.0 / isq
            self.inv_scale = isq
            self.det_w = 1.0 / isq ** mesh.dim
            self.limiting = None
            return
        if target == "unit":
            scale = 1.0
        elif h is not None:
            scale = float(h)
        else:
            vol = self.volume(mesh.coords.ravel())
            scale = (vol / mesh.n_elements) ** (1.0 / mesh.dim)
        self.scale = scale
        self.inv_scale = 1.0 / scale
        self.det_w = scale ** mesh.dim
        self.limiting = limiting   # {"reference": x0, "delta": float|(N,), "weight": w}

    # -- helpers
    def _x2(self, x):
        return np.asarray(x, float).reshape(self.mesh.dim, -1)

    def volume(self, x):
        """Quadrature of det(A) (met:319-330)."""
        J = self.disc.jacobians(x)
        return float(np.sum(det(J) @ self.disc.wq))

    def _checked_T(self, x):
        J = self.disc.jacobians(x)
        dj = det(J)
        k = int(np.argmin(dj))
        if dj.flat[k] <= 0.0:
            e, q = divmod(k, self.disc.Q)
            raise InvalidMesh(e, q, dj.flat[k])
        return J * _pt(self.inv_scale)

    # -- ProblemLike
    def min_det_jacobian(self, x):
        return float(det(self.disc.jacobians(x)).min())

    def objective(self, x):
        T = self._checked_T(x)
        mu = metric_value(self.metric, T)
        if np.ndim(self.det_w):
            F = self.omega * float(np.sum((self.det_w * mu) @ self.disc.wq))
        else:
            F = self.omega * self.det_w * float(np.sum(mu @ self.disc.wq))
        if self.limiting is not None:
            F += self.limiting_value(x)
        return F

    def gradient(self, x):
        T = self._checked_T(x)
        coef = self.omega * self.det_w * self.inv_scale
        P = metric_first(self.metric, T) * _pt(coef * self.disc.wq[None, :])
        out = self.disc.pull_back(P)
        if self.limiting is not None:
            out += self._lim_grad2(self._x2(x))
        out[self.mesh.fixed] = 0.0
        return out.ravel()

    def hessian_setup(self, x):
        T = self._checked_T(x)
        tau = det(T)
        S = cofactor(T) / tau[..., None, None]
        w = (self.omega * self.det_w * self.inv_scale ** 2) * np.broadcast_to(self.disc.wq, tau.shape)
        w = np.broadcast_to(w, tau.shape)
        c = None
        if self.metric in TEMPLATE_METRICS:
            c = np.stack(second_coeffs(self.metric, tau, frob2(T)), axis=-1) * w[..., None]
        return OQData(self.metric, c, S, T, np.array(w))

    def hessian_apply(self, qd: OQData, v):
        v2 = self._x2(v)
        vin = np.where(self.mesh.fixed, 0.0, v2)
        g = self.disc.grad_at_quad(vin)
        if self.metric in TEMPLATE_METRICS:
            z = hess_action_point(self.metric, qd.T, qd.S, g, qd.c)
        else:
            z = hess_action_point(self.metric, qd.T, qd.S, g) * qd.w[..., None, None]
        out = self.disc.pull_back(z)
        if self.limiting is not None:
            out += self._lim_hess2(vin)
        out[self.mesh.fixed] = v2[self.mesh.fixed]
        return out.ravel()

    def hessian_diagonal(self, qd: OQData):
        """Exact diagonal (op:420-459): H[(a,n),(a,p)] contracted with the
        1D products M_n * M_p per axis."""
        d, D = self.mesh.dim, self.disc
        Ne = self.mesh.n_elements
        acc = 0.0
        if qd.c is None:
            H = metric_second(self.metric, qd.T) * qd.w[..., None, None]
        for n in range(d):
            for p in range(d):
                if qd.c is not None:
                    c = qd.c
                    hv = (c[..., 1, None] * (qd.S[..., :, n] * qd.T[..., :, p] + qd.T[..., :, n] * qd.S[..., :, p])
                          + (c[..., 2, None] + c[..., 3, None]) * qd.S[..., :, n] * qd.S[..., :, p])
                    if n == p:
                        hv = hv + c[..., 0, None]
                else:
                    hv = np.stack([H[..., a * d + n, a * d + p] for a in range(d)], axis=-1)
                mats = [(D.G if k == n else D.B) * (D.G if k == p else D.B) for k in range(d)]
                Z = hv.transpose(2, 0, 1).reshape((d, Ne) + (D.nq,) * d)
                acc = acc + _bwd(Z, mats)
        if self.limiting is not None:
            cq = self._lim_scale()
            Z = np.broadcast_to(cq.reshape((1, Ne) + (D.nq,) * d), (d, Ne) + (D.nq,) * d)
            acc = acc + _bwd(Z, [D.B * D.B] * d)
        out = D.scatter(acc.reshape(d, Ne, -1))
        out[self.mesh.fixed] = 1.0
        return out.ravel()

    # -- limiting term (op:463-533)
    def _lim_scale(self):
        lim, D = self.limiting, self.disc
        delta = lim.get("delta", 1.0)
        Ne = self.mesh.n_elements
        if np.ndim(delta) == 0:
            dq = np.full((Ne, D.Q), float(delta))
        else:
            U = D.gather(np.asarray(delta, float)[None, :])[0]
            dq = _fwd(U, [D.B] * self.mesh.dim).reshape(Ne, D.Q)
        base = 2.0 * lim.get("weight", 1.0) * self.det_w * D.wq[None, :]
        return base / (dq * dq)

    def _interp(self, v2):
        D = self.disc
        return _fwd(D.gather(v2), [D.B] * self.mesh.dim).reshape(self.mesh.dim, self.mesh.n_elements, D.Q)

    def limiting_value(self, x):
        disp = self._x2(x) - np.asarray(self.limiting["reference"], float).reshape(self.mesh.dim, -1)
        dq = self._interp(disp)
        return 0.5 * float(np.sum(self._lim_scale()[None] * dq * dq))

    def _lim_apply(self, u2):
        D = self.disc
        d, Ne = self.mesh.dim, self.mesh.n_elements
        Z = (self._lim_scale()[None] * self._interp(u2)).reshape((d, Ne) + (D.nq,) * d)
        return D.scatter(_bwd(Z, [D.B] * d).reshape(d, Ne, -1))

    def _lim_grad2(self, x2):
        ref = np.asarray(self.limiting["reference"], float).reshape(x2.shape)
        return self._lim_apply(x2 - ref)

    def _lim_hess2(self, vin2):
        return self._lim_apply(vin2)

    # -- full assembly matvec (op:537-589), for PA-vs-FA checks
    def fa_matvec(self, x, v):
        """Dense per-element Hessian (no sum factorisation) applied to v, with
        the same constrained-dof convention as hessian_apply."""
        D, mesh = self.disc, self.mesh
        d = mesh.dim
        T = self._checked_T(x)
        H = metric_second(self.metric, T) * _pt(self.omega * self.det_w * self.inv_scale ** 2
                                                * D.wq[None, :])
        # dense gradient tables grads[q, i, b]
        Np = D.n ** d
        eye = np.eye(Np).reshape((Np,) + (D.n,) * d)
        grads = np.stack([_fwd(eye, D.mats(b)).reshape(Np, D.Q).T for b in range(d)], axis=-1)
        v2 = self._x2(v)
        vin = np.where(mesh.fixed, 0.0, v2)
        vE = vin[:, mesh.restriction]                          # (d, Ne, Np)
        g = np.einsum("qib,aei->eqab", grads, vE)
        Hr = H.reshape(H.shape[:2] + (d, d, d, d))
        z = np.einsum("eqanbp,eqbp->eqan", Hr, g)
        yE = np.einsum("eqan,qin->aei", z, grads)
        out = D.scatter(yE)
        if self.limiting is not None:
            out += self._lim_hess2(vin)
        out[mesh.fixed] = v2[mesh.fixed]
        return out.ravel()


# ---------------------------------------------------------------------------
# Solvers (sol:83-321)
# ---------------------------------------------------------------------------

def jacobi(diag):
    diag = np.asarray(diag, float)
    if not np.all(np.isfinite(diag)):
        raise ValueError("non-finite diagonal")
    inv = 1.0 / np.maximum(np.abs(diag), JACOBI_FLOOR)
    return lambda r: inv * r


def minres(apply_op, b, max_it=50, rtol=1e-8, precond=None):
    """Paige-Saunders preconditioned MINRES from x0 = 0 (sol:93-180).
    Returns (x, iterations, rel_residual, converged, history)."""
    b = np.asarray(b, float)
    M = precond if precond is not None else (lambda r: r)
    x = np.zeros_like(b)
    r1 = b.copy()
    y = M(r1)
    beta1 = float(r1 @ y)
    if beta1 < 0:
        raise ValueError("indefinite preconditioner")
    beta1 = np.sqrt(beta1)
    if beta1 == 0.0:
        return x, 0, 0.0, True, [0.0]
    oldb, beta, dbar, epsln, sn, cs, phibar = 0.0, beta1, 0.0, 0.0, 0.0, -1.0, beta1
    w = np.zeros_like(b)
    w2 = np.zeros_like(b)
    r2 = r1.copy()
    hist = [1.0]
    it = 0
    while it < max_it:
        it += 1
        v = y / beta
        y = apply_op(v)
        if it >= 2:
            y = y - (beta / oldb) * r1
        alfa = float(v @ y)
        y = y - (alfa / beta) * r2
        r1, r2 = r2, y
        y = M(r2)
        oldb = beta
        beta2 = float(r2 @ y)
        if beta2 < 0:
            raise ValueError("indefinite preconditioner")
        beta = np.sqrt(beta2)
        oldeps = epsln
        delta = cs * dbar + sn * alfa
        gbar = sn * dbar - cs * alfa
        epsln = sn * beta
        dbar = -cs * beta
        gamma = max(np.hypot(gbar, beta), np.finfo(float).eps)
        cs, sn = gbar / gamma, beta / gamma
        phi = cs * phibar
        phibar = sn * phibar
        w1, w2 = w2, w
        w = (v - oldeps * w1 - delta * w2) / gamma
        x = x + phi * w
        if beta == 0.0:
            r = b - apply_op(x)
            ex = np.sqrt(max(float(r @ M(r)), 0.0)) / beta1
            hist.append(ex)
            if ex <= rtol:
                return x, it, ex, True, hist
            raise RuntimeError(f"MINRES breakdown at {it}")
        hist.append(phibar / beta1)
        if phibar / beta1 <= rtol:
            return x, it, hist[-1], True, hist
    return x, it, hist[-1], False, hist


def line_search(x, dx, prob, f0, g0, max_halvings=30):
    """Backtracking alpha = 1, 1/2, ... (sol:202-224)."""
    alpha = 1.0
    for _ in range(max_halvings + 1):
        xt = x - alpha * dx
        md = prob.min_det_jacobian(xt)
        if md > 0.0:
            ft = prob.objective(xt)
            if ft < GROWTH * f0:
                gt = prob.gradient(xt)
                ngt = float(np.linalg.norm(gt))
                if ngt < GROWTH * g0:
                    return alpha, xt, ft, ngt, md, gt
        alpha *= 0.5
    raise RuntimeError("line search failed")


def newton(x0, prob, rel_tol=1e-10, max_it=100, minres_max=50, minres_rtol=1e-8,
           precond=True, abs_tol=1e-12, max_halvings=30):
    """Newton + MINRES + line search (sol:263-321).  Returns (x, records,
    success, rel_grad, g0, message); records are tuples (alpha, F, |g|,
    minres_its, minres_relres, min_det)."""
    x = np.asarray(x0, float).copy()
    if prob.min_det_jacobian(x) <= 0.0:
        raise RuntimeError("initial mesh is inverted")
    g = prob.gradient(x)
    ng0 = float(np.linalg.norm(g))
    recs = []
    if ng0 <= abs_tol:
        return x, recs, True, 0.0, ng0, "initial gradient is zero"
    f, ng = prob.objective(x), ng0
    for _ in range(max_it):
        qd = prob.hessian_setup(x)
        P = jacobi(prob.hessian_diagonal(qd)) if precond else None
        try:
            dx, its, rr, _, _ = minres(lambda v: prob.hessian_apply(qd, v), g, minres_max,
                                       minres_rtol, P)
        except RuntimeError as err:
            return x, recs, False, ng / ng0, ng0, str(err)
        try:
            alpha, x, f, ng, md, g = line_search(x, dx, prob, f, ng, max_halvings)
        except RuntimeError as err:
            return x, recs, False, ng / ng0, ng0, str(err)
        recs.append((alpha, f, ng, its, rr, md))
        if ng / ng0 <= rel_tol:
            return x, recs, True, ng / ng0, ng0, "converged"
    return x, recs, False, ng / ng0, ng0, f"no convergence in {max_it} iterations"


# ---------------------------------------------------------------------------
# Yardstick accounting (fe:222-223, op:396-398)
# ---------------------------------------------------------------------------

def apply_yardstick(dim, order, nq, n_elements, n_dofs):
    """(bytes, flops) of one Hessian action in the reference's Q-data format."""
    n = order + 1
    Q = nq ** dim
    byts = 8 * (4 + 2 * dim * dim) * n_elements * Q + 4 * n_elements * n ** dim + 16 * n_dofs
    s = sum(nq ** k * n ** (dim + 1 - k) for k in range(1, dim + 1))
    flops = 2 * n_elements * (2 * dim * dim * s + (6 * dim * dim + 2 * dim ** 3) * Q)
    return byts, flops
