"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py) and against finite differences for the
metrics the reference lacks (mu_7, mu_302, mu_321: parity unpinned)."""

import numpy as np
import pytest

from conftest import golden_names, load_golden
from oracle import tmop_oracle as O


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def problem_from(g):
    mesh = O.box_mesh(int(g["dim"]), tuple(g["counts"]), int(g["order"]))
    lim = None
    if "lim_delta" in g:
        lim = dict(reference=mesh.coords.ravel().copy(), delta=float(g["lim_delta"]),
                   weight=float(g["lim_weight"]))
    return O.OracleProblem(mesh, int(g["metric"]), int(g["n_quad"]),
                           target="unit" if int(g["target"]) == 0 else "size",
                           spatial_weight=float(g["spatial_weight"]), limiting=lim)


OPS = golden_names("op")


@pytest.mark.parametrize("name", OPS)
def test_mesh_and_tables_match_reference(name):
    g = load_golden(name)
    p = problem_from(g)
    assert np.array_equal(p.mesh.restriction, g["restriction"])
    assert np.array_equal(p.mesh.fixed, g["fixed"])
    assert np.abs(p.mesh.coords - g["coords"]).max() <= 1e-15
    assert np.abs(p.disc.B - g["B"]).max() <= 1e-14
    assert np.abs(p.disc.G - g["G"]).max() <= 1e-13
    assert np.abs(p.disc.wq - g["wq"]).max() <= 1e-16
    assert p.inv_scale == pytest.approx(float(g["inv_scale"]), rel=1e-14)


@pytest.mark.parametrize("name", OPS)
def test_operator_matches_reference(name):
    g = load_golden(name)
    p = problem_from(g)
    x, v = g["x"], g["v"]
    qd = p.hessian_setup(x)
    coeffs, s, t = qd.planar()
    assert rel(coeffs, g["coeffs"]) <= 1e-13
    assert rel(s, g["s_mat"]) <= 1e-13
    assert rel(t, g["t_mat"]) <= 1e-14
    assert rel(p.hessian_apply(qd, v), g["apply"]) <= 1e-12
    assert rel(p.gradient(x), g["gradient"]) <= 1e-12
    assert p.objective(x) == pytest.approx(float(g["objective"]), rel=1e-12, abs=1e-14)
    assert rel(p.hessian_diagonal(qd), g["diagonal"]) <= 1e-12
    assert p.min_det_jacobian(x) == pytest.approx(float(g["min_det"]), rel=1e-14)


@pytest.mark.parametrize("name", OPS[:4])
def test_pa_matches_fa(name):
    g = load_golden(name)
    p = problem_from(g)
    qd = p.hessian_setup(g["x"])
    assert rel(p.hessian_apply(qd, g["v"]), p.fa_matvec(g["x"], g["v"])) <= 1e-12


def test_metric_points_match_reference():
    g = load_golden("metric_points")
    for metric, dim in [(2, 2), (55, 2), (55, 3), (303, 3)]:
        T = g[f"T_{metric}_{dim}"]
        assert rel(O.metric_value(metric, T), g[f"mu_{metric}_{dim}"]) <= 1e-13
        assert rel(O.metric_first(metric, T), g[f"P_{metric}_{dim}"]) <= 1e-13
        assert rel(O.metric_second(metric, T), g[f"H_{metric}_{dim}"]) <= 1e-13


def test_minres_matches_reference():
    g = load_golden("minres_dense")
    A, b = g["A"], g["b"]
    x, its, rr, conv, hist = O.minres(lambda v: A @ v, b, 25, 1e-10, O.jacobi(np.diag(A)))
    assert its == int(g["iterations"])
    assert rel(x, g["x"]) <= 1e-12
    assert np.allclose(hist, g["history"], rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("name", golden_names("newton"))
def test_newton_trace_matches_reference(name):
    g = load_golden(name)
    mesh = O.box_mesh(int(g["dim"]), tuple(g["counts"]), int(g["order"]))
    p = O.OracleProblem(mesh, int(g["metric"]), int(g["n_quad"]))
    x, recs, ok, relg, g0, msg = O.newton(g["x0"], p, max_it=int(g["iters"]),
                                          precond=bool(g["precond"]))
    want = g["records"]
    assert len(recs) == len(want)
    for got, ref in zip(recs, want):
        assert got[0] == ref[0]                      # alpha exact
        assert got[3] == ref[3]                      # MINRES iterations exact
        assert got[1] == pytest.approx(ref[1], rel=1e-9, abs=1e-13)
        assert got[2] == pytest.approx(ref[2], rel=1e-8, abs=1e-13)
    assert rel(x, g["x"]) <= 1e-10


def test_kershaw_matches_reference():
    g = load_golden("kershaw_6x2x2_p2")
    mesh = O.box_mesh(3, (6, 2, 2), 2)
    c = mesh.coords
    X = np.stack(O.kershaw(0.3, 0.3, c[0], c[1], c[2]))
    assert np.array_equal(mesh.restriction, g["restriction"])
    assert np.abs(X - g["coords"]).max() <= 1e-15


# ---- extension metrics (parity unpinned: FD + invariance + PA-vs-FA) -------

NEW = [(O.MU_7, 2), (O.MU_302, 3), (O.MU_321, 3), (O.MU_2, 2), (O.MU_303, 3)]


def random_valid(dim, rng):
    while True:
        t = rng.uniform(-1.5, 1.5, (dim, dim)) + np.eye(dim)
        d = np.linalg.det(t)
        if d > 1e-3:
            return t * (rng.uniform(0.1, 10.0) / d) ** (1.0 / dim)


@pytest.mark.parametrize("metric,dim", NEW)
def test_new_metric_derivatives_fd(metric, dim, rng):
    for _ in range(10):
        T = random_valid(dim, rng)
        P = O.metric_first(metric, T)
        H = O.metric_second(metric, T)
        fdP = np.empty_like(T)
        fdH = np.empty((dim * dim, dim * dim))
        for i in range(dim):
            for j in range(dim):
                e = np.zeros_like(T)
                e[i, j] = 1e-6
                fdP[i, j] = (O.metric_value(metric, T + e) - O.metric_value(metric, T - e)) / 2e-6
                e[i, j] = 1e-5
                fdH[i * dim + j] = ((O.metric_first(metric, T + e) - O.metric_first(metric, T - e)) / 2e-5).ravel()
        assert np.allclose(P, fdP, atol=1e-6 * (np.abs(fdP).max() + 1e-3))
        assert np.allclose(H, fdH, atol=1e-5 * (np.abs(fdH).max() + 1e-3))
        assert np.abs(H - H.T).max() <= 1e-11 * (np.abs(H).max() + 1)


@pytest.mark.parametrize("metric,dim", NEW)
def test_new_metric_invariances(metric, dim, rng):
    for _ in range(5):
        T = random_valid(dim, rng)
        q, r = np.linalg.qr(rng.standard_normal((dim, dim)))
        q = q @ np.diag(np.sign(np.diag(r)))
        if np.linalg.det(q) < 0:
            q[:, 0] *= -1
        mu = O.metric_value(metric, T)
        assert mu >= -1e-12
        assert O.metric_value(metric, q @ T) == pytest.approx(mu, rel=1e-11, abs=1e-12)
        if metric in (O.MU_2, O.MU_303, O.MU_302):
            assert O.metric_value(metric, 2.7 * T) == pytest.approx(mu, rel=1e-11, abs=1e-12)
    ident = np.eye(dim)
    assert abs(O.metric_value(metric, ident)) <= 1e-14


@pytest.mark.parametrize("metric,dim,order", [(O.MU_7, 2, 2), (O.MU_302, 3, 1), (O.MU_321, 3, 2)])
def test_new_metric_operator_consistency(metric, dim, order, rng):
    mesh = O.box_mesh(dim, (2,) * dim, order)
    p = O.OracleProblem(mesh, metric, order + 2)
    x = O.perturb(mesh, rng, 0.2)
    v = rng.standard_normal(x.shape)
    qd = p.hessian_setup(x)
    assert rel(p.hessian_apply(qd, v), p.fa_matvec(x, v)) <= 1e-12
    vf = np.where(mesh.fixed.ravel(), 0.0, v)
    fd = (p.gradient(x + 1e-5 * vf) - p.gradient(x - 1e-5 * vf)) / 2e-5
    assert rel(p.hessian_apply(qd, vf), fd) <= 1e-5
    gv = float(p.gradient(x) @ vf)
    fdf = (p.objective(x + 1e-6 * vf) - p.objective(x - 1e-6 * vf)) / 2e-6
    assert gv == pytest.approx(fdf, rel=1e-6)
    # diagonal = diagonal of the assembled operator (probe with unit vectors)
    diag = p.hessian_diagonal(qd)
    for k in rng.choice(mesh.n_dofs, 6, replace=False):
        e = np.zeros(mesh.n_dofs)
        e[k] = 1.0
        assert diag[k] == pytest.approx(p.hessian_apply(qd, e)[k], rel=1e-11, abs=1e-13)


def test_yardstick_matches_survey():
    # C3-p2 = 160^3, n_q = 4 -> 485 B/DOF, 1230 flop/DOF
    n_dofs = 3 * (160 * 2 + 1) ** 3
    b, f = O.apply_yardstick(3, 2, 4, 160 ** 3, n_dofs)
    assert b / n_dofs == pytest.approx(485, rel=0.01)
    assert f / n_dofs == pytest.approx(1230, rel=0.01)


@pytest.mark.parametrize("name", golden_names("limnodal"))
def test_limiting_nodal_delta_matches_reference(name):
    """Nodal delta + perturbed reference: the oracle's limiting term
    (value, raw gradient, raw action) and the full operator against the
    reference (operator.py:463-533)."""
    g = load_golden(name)
    mesh = O.box_mesh(int(g["dim"]), tuple(g["counts"]), int(g["order"]))
    lim = dict(reference=g["lim_reference"], delta=g["lim_delta_nodal"], weight=float(g["lim_weight"]))
    p = O.OracleProblem(mesh, int(g["metric"]), int(g["n_quad"]), limiting=lim)
    x, v = g["x"], g["v"]
    qd = p.hessian_setup(x)
    assert rel(p.hessian_apply(qd, v), g["apply"]) <= 1e-12
    assert rel(p.gradient(x), g["gradient"]) <= 1e-12
    assert p.objective(x) == pytest.approx(float(g["objective"]), rel=1e-12)
    assert rel(p.hessian_diagonal(qd), g["diagonal"]) <= 1e-12
    assert p.limiting_value(x) == pytest.approx(float(g["lim_value"]), rel=1e-12)
    assert rel(p._lim_grad2(p._x2(x)).ravel(), g["lim_gradient"]) <= 1e-12
    assert rel(p._lim_hess2(p._x2(v)).ravel(), g["lim_apply"]) <= 1e-12


@pytest.mark.parametrize("name", [n for n in OPS if n.startswith("op3d") and "lim" not in n])
@pytest.mark.parametrize("threads", [1, 3])
def test_cpu_port_matches_reference(name, threads):
    """oracle/tmop_cpu.c (the C/OpenMP restatement timed as a secondary CPU
    baseline by bench.py) against the reference's own apply, bitwise
    independent of the thread count."""
    from oracle.cpu_apply import CpuApply
    g = load_golden(name)
    p = problem_from(g)
    qd = p.hessian_setup(g["x"])
    y = CpuApply(p, qd, threads)(g["v"])
    assert rel(y, g["apply"]) <= 1e-12
    assert np.array_equal(y, CpuApply(p, qd, 2)(g["v"]))


# ---- size-field targets (extension: parity unpinned -- FD, PA-vs-FA and the
# constant-field limit, which IS pinned: it equals IDEAL_EQUAL_SIZE) ---------

def _shell_field(mesh, amp=0.5):
    r = np.sqrt(((mesh.coords - 0.5) ** 2).sum(axis=0))
    return (1.0 / mesh.n_elements) * (1.0 + amp * np.cos(2.0 * np.pi * r / 0.35))


@pytest.mark.parametrize("metric,dim,order", [(O.MU_321, 3, 2), (O.MU_303, 3, 1), (O.MU_302, 3, 2),
                                              (O.MU_2, 2, 2), (O.MU_7, 2, 3)])
def test_size_field_operator_consistency(metric, dim, order, rng):
    mesh = O.box_mesh(dim, (3, 2, 2)[:dim], order)
    p = O.OracleProblem(mesh, metric, order + 2, target="field", size=_shell_field(mesh))
    x = O.perturb(mesh, rng, 0.2)
    v = rng.standard_normal(x.shape)
    qd = p.hessian_setup(x)
    assert rel(p.hessian_apply(qd, v), p.fa_matvec(x, v)) <= 1e-12
    vf = np.where(mesh.fixed.ravel(), 0.0, v)
    fd = (p.gradient(x + 1e-5 * vf) - p.gradient(x - 1e-5 * vf)) / 2e-5
    assert rel(p.hessian_apply(qd, vf), fd) <= 1e-5
    gv = float(p.gradient(x) @ vf)
    fdf = (p.objective(x + 1e-6 * vf) - p.objective(x - 1e-6 * vf)) / 2e-6
    assert gv == pytest.approx(fdf, rel=1e-6)


def test_size_field_constant_equals_equal_size_target(rng):
    """eta = h^d everywhere is the reference's IDEAL_EQUAL_SIZE target with
    that h (metrics.py:333-345) -- the pinned limit of the extension."""
    mesh = O.box_mesh(3, (3, 2, 2), 2)
    h = 0.37
    pf = O.OracleProblem(mesh, O.MU_303, 4, target="field", size=np.full(mesh.n_nodes, h ** 3))
    pc = O.OracleProblem(mesh, O.MU_303, 4, target="size", h=h)
    x = O.perturb(mesh, rng, 0.2)
    v = rng.standard_normal(x.shape)
    assert pf.objective(x) == pytest.approx(pc.objective(x), rel=1e-13)
    assert rel(pf.gradient(x), pc.gradient(x)) <= 1e-13
    qf, qc = pf.hessian_setup(x), pc.hessian_setup(x)
    assert rel(pf.hessian_apply(qf, v), pc.hessian_apply(qc, v)) <= 1e-13
    assert rel(pf.hessian_diagonal(qf), pc.hessian_diagonal(qc)) <= 1e-13
