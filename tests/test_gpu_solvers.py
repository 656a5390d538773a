"""Line search / Newton behaviour on the device operator, mirroring the
reference's own solver tests (pkg/tests/test_solvers.py:123-269) case by case:
same meshes, same constructed steps, same expectations."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def P():
    import paper_2205_12721_b200 as pkg
    return pkg


def kershaw_problem(metric=None, order=1, n_quad=3):
    """test_solvers.py:117-120."""
    p = P()
    metric = p.MetricId.MU_55 if metric is None else metric
    mesh = p.apply_kershaw(p.build_cartesian(p.MeshSpec(3, 6, 2, 2, order=order)), 0.3, 0.3)
    return p.TmopProblem(mesh, p.ObjectiveConfig(metric, p.TargetSpec(p.TargetKind.IDEAL_UNIT)), n_quad)


def _start(p):
    x = p.mesh.dof_vector()
    return x, p.objective(x), float(np.linalg.norm(p.gradient(x)))


def test_full_step_accepted_when_valid(rng):
    p = kershaw_problem()
    x, f0, g0 = _start(p)
    dx = 1e-4 * rng.standard_normal(x.shape)
    ls = P().line_search(x, dx, p, f0=f0, grad_norm0=g0)
    assert ls.alpha == 1.0
    assert np.array_equal(np.asarray(ls.x), x - dx)


def test_zero_step_accepted():
    p = kershaw_problem()
    x, f0, g0 = _start(p)
    ls = P().line_search(x, np.zeros_like(x), p, f0=f0, grad_norm0=g0)
    assert ls.alpha == 1.0
    assert np.array_equal(np.asarray(ls.x), x)


def test_inverting_step_halved_once():
    p = kershaw_problem()
    x, f0, g0 = _start(p)
    interior = np.nonzero(~p.mesh.fixed_mask.any(axis=0))[0]
    node = interior[len(interior) // 2]
    dx = np.zeros_like(x)
    dx[node] = -0.15
    assert p.min_det_jacobian(x - dx) < 0
    assert p.min_det_jacobian(x - 0.5 * dx) > 0
    assert P().line_search(x, dx, p, f0=f0, grad_norm0=g0).alpha == 0.5


def test_failure_after_max_halvings():
    p = kershaw_problem()
    x, f0, g0 = _start(p)
    dx = np.zeros_like(x)
    interior = np.nonzero(~p.mesh.fixed_mask.any(axis=0))[0]
    dx[interior[0]] = -0.15 * 2.0 ** 31
    with pytest.raises(P().LineSearchError):
        P().line_search(x, dx, p, f0=f0, grad_norm0=g0, max_halvings=30)


def test_rejects_nonfinite_step():
    p = kershaw_problem()
    x = p.mesh.dof_vector()
    with pytest.raises(P().LineSearchError):
        P().line_search(x, np.full_like(x, np.nan), p, f0=1.0, grad_norm0=1.0)


class QuadraticProblem:
    """Displacement-limiting term only (test_solvers.py:178-204): exactly quadratic."""

    def __init__(self, mesh, delta=0.7):
        p = P()
        mesh.fixed_mask[:] = False
        cfg = p.ObjectiveConfig(metric=p.MetricId.MU_55, target=p.TargetSpec(p.TargetKind.IDEAL_UNIT),
                                limiting=p.LimitingConfig(reference=mesh.dof_vector(), delta=delta))
        self.base = p.TmopProblem(mesh, cfg, n_quad=mesh.order + 1)

    def objective(self, x):
        return self.base.limiting_value(x)

    def gradient(self, x):
        return self.base.limiting_gradient(x)

    def hessian_setup(self, x):
        return None

    def hessian_apply(self, qdata, v):
        return self.base.limiting_hessian_apply(v)

    def hessian_diagonal(self, qdata):
        raise NotImplementedError("run unpreconditioned")

    def min_det_jacobian(self, x):
        return 1.0


def test_zero_iterations_at_optimum():
    p = P()
    mesh = p.build_box(3, (2, 2, 2), 1)
    prob = p.TmopProblem(mesh, p.ObjectiveConfig(p.MetricId.MU_303, p.TargetSpec(p.TargetKind.IDEAL_EQUAL_SIZE)), 2)
    res = p.newton_solve(mesh.dof_vector(), prob)
    assert res.success
    assert res.trace.newton_iterations == 0
    assert np.array_equal(np.asarray(res.x), mesh.dof_vector())


def test_displaced_node_regression():
    p = P()
    mesh = p.build_box(2, (4, 4), 2)
    x2 = mesh.dof_vector().reshape(2, -1)
    interior = np.nonzero(~mesh.fixed_mask.any(axis=0))[0]
    x2[0, interior[len(interior) // 2]] += 0.05
    prob = p.TmopProblem(mesh, p.ObjectiveConfig(p.MetricId.MU_2, p.TargetSpec(p.TargetKind.IDEAL_UNIT)), 4)
    x0 = x2.ravel()
    f0 = prob.objective(x0)
    res = p.newton_solve(x0, prob, p.NewtonConfig(rel_grad_tolerance=1e-10))
    assert res.success
    assert res.trace.newton_iterations <= 20
    assert res.rel_grad <= 1e-10
    assert prob.objective(res.x) <= f0
    assert all(r.min_det > 0 for r in res.trace.records)


def test_quadratic_objective_single_iteration(rng):
    p = P()
    qp = QuadraticProblem(p.build_box(3, (2, 2, 2), 2))
    x0 = qp.base.mesh.dof_vector() + 0.05 * rng.standard_normal(qp.base.mesh.n_dofs)
    res = p.newton_solve(x0, qp, p.NewtonConfig(rel_grad_tolerance=1e-10),
                         p.MinresConfig(max_iterations=500, rel_tolerance=1e-14, preconditioned=False))
    assert res.success
    assert res.trace.newton_iterations == 1
    assert np.allclose(np.asarray(res.x), qp.base.mesh.dof_vector(), atol=1e-10)


def test_failure_reported_when_iterations_exhausted():
    p = P()
    prob = kershaw_problem()
    res = p.newton_solve(prob.mesh.dof_vector(), prob, p.NewtonConfig(rel_grad_tolerance=1e-12, max_iterations=1),
                         p.MinresConfig(max_iterations=2))
    assert not res.success
    assert res.trace.newton_iterations == 1
    assert "no convergence" in res.message


def test_initial_inverted_mesh_rejected():
    p = P()
    prob = kershaw_problem()
    x2 = prob.mesh.dof_vector().reshape(3, -1)
    conn = prob.mesh.restriction[0]
    x2[:, [conn[0], conn[1]]] = x2[:, [conn[1], conn[0]]]
    with pytest.raises(p.LineSearchError, match="inverted"):
        p.newton_solve(x2.ravel(), prob)


def test_stopping_criterion_on_success():
    p = P()
    prob = kershaw_problem(metric=p.MetricId.MU_303, order=1)
    res = p.newton_solve(prob.mesh.dof_vector(), prob, p.NewtonConfig(rel_grad_tolerance=1e-6),
                         p.MinresConfig(max_iterations=50))
    assert res.success
    assert res.rel_grad <= 1e-6
    g_final = np.linalg.norm(np.asarray(prob.gradient(res.x)))
    assert g_final <= 1e-6 * res.initial_grad_norm * (1 + 1e-9)
