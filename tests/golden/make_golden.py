"""Generate golden input/output vectors by running the REFERENCE package.

Run here (the container that has /root/reference), never on the GPU box:

    python tests/golden/make_golden.py

Imports `tmopbench` from /root/reference/pkg/src with NUMBA_CACHE_DIR pointed
at a scratch dir and bytecode writing disabled, so nothing is written into the
read-only reference tree.  Fixtures land next to this
script as compressed .npz files; tests/test_oracle.py pins the oracle against
them and the GPU tests pin the CUDA path against them.
"""

from __future__ import annotations

import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_golden_"))
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

import numpy as np  # noqa: E402

import tmopbench as tb  # noqa: E402
from oracles import perturbed_mesh_vector  # noqa: E402  (reference tests/oracles.py:121)

HERE = os.path.dirname(os.path.abspath(__file__))
SEED = 20240901  # reference tests/conftest.py:19-21


def operator_case(name, dim, counts, order, n_quad, metric, target="unit",
                  amplitude=0.2, limiting=None, spatial_weight=1.0):
    mesh = tb.build_box(dim, counts, order)
    rng = np.random.default_rng(SEED)
    x = perturbed_mesh_vector(mesh, rng, amplitude)
    v = rng.standard_normal(x.shape)
    kind = tb.TargetKind.IDEAL_UNIT if target == "unit" else tb.TargetKind.IDEAL_EQUAL_SIZE
    lim = None
    if limiting is not None:
        lim = tb.LimitingConfig(reference=mesh.dof_vector(), delta=limiting[0],
                                weight=limiting[1])
    cfg = tb.ObjectiveConfig(metric=tb.MetricId(metric), target=tb.TargetSpec(kind),
                             spatial_weight=spatial_weight, limiting=lim)
    p = tb.TmopProblem(mesh, cfg, n_quad)
    qd = p.hessian_setup(x)
    out = dict(
        dim=dim, counts=np.array(counts), order=order, n_quad=n_quad, metric=metric,
        target=0 if target == "unit" else 1, spatial_weight=spatial_weight,
        coords=mesh.coords, restriction=mesh.restriction, fixed=mesh.fixed_mask,
        B=p.em.b, G=p.em.g, wq=p.wq, inv_scale=p.targets.inv_scale, det_w=p.targets.det_w,
        x=x, v=v,
        coeffs=qd.coeffs, s_mat=qd.s_mat, t_mat=qd.t_mat,
        apply=p.hessian_apply(qd, v), gradient=p.gradient(x),
        objective=p.objective(x), diagonal=p.hessian_diagonal(qd),
        min_det=p.min_det_jacobian(x), min_det_uniform=p.min_det_jacobian(mesh.dof_vector()),
    )
    if limiting is not None:
        out.update(lim_delta=limiting[0], lim_weight=limiting[1])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    return p, x


def limiting_nodal_case(name, dim, counts, order, n_quad, metric, weight):
    """Limiting with a NODAL delta and a perturbed reference (operator.py:463-533):
    the full operator plus limiting_value / limiting_gradient /
    limiting_hessian_apply on their own."""
    mesh = tb.build_box(dim, counts, order)
    rng = np.random.default_rng(SEED + 7)
    x0 = perturbed_mesh_vector(mesh, rng, 0.1)
    delta = 0.3 + 0.2 * rng.random(mesh.n_nodes)
    x = perturbed_mesh_vector(mesh, rng, 0.2)
    v = rng.standard_normal(x.shape)
    lim = tb.LimitingConfig(reference=x0, delta=delta, weight=weight)
    cfg = tb.ObjectiveConfig(metric=tb.MetricId(metric), target=tb.TargetSpec(tb.TargetKind.IDEAL_UNIT),
                             limiting=lim)
    p = tb.TmopProblem(mesh, cfg, n_quad)
    qd = p.hessian_setup(x)
    out = dict(dim=dim, counts=np.array(counts), order=order, n_quad=n_quad, metric=metric, x=x, v=v,
               lim_reference=x0, lim_delta_nodal=delta, lim_weight=weight,
               apply=p.hessian_apply(qd, v), gradient=p.gradient(x), objective=p.objective(x),
               diagonal=p.hessian_diagonal(qd), lim_value=p.limiting_value(x), lim_gradient=p.limiting_gradient(x),
               lim_apply=p.limiting_hessian_apply(v))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def newton_case(name, dim, counts, order, n_quad, metric, iters, amplitude=0.2,
                precond=True):
    mesh = tb.build_box(dim, counts, order)
    rng = np.random.default_rng(SEED)
    x0 = perturbed_mesh_vector(mesh, rng, amplitude)
    p = tb.TmopProblem(mesh, tb.ObjectiveConfig(tb.MetricId(metric),
                                                tb.TargetSpec(tb.TargetKind.IDEAL_UNIT)),
                       n_quad)
    res = tb.newton_solve(x0, p, tb.NewtonConfig(max_iterations=iters),
                          tb.MinresConfig(preconditioned=precond))
    recs = np.array([[r.alpha, r.objective, r.grad_norm, r.minres_iterations,
                      r.minres_rel_residual, r.min_det] for r in res.trace.records])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"),
                        dim=dim, counts=np.array(counts), order=order, n_quad=n_quad,
                        metric=metric, iters=iters, precond=precond, x0=x0, x=res.x,
                        records=recs, f0=p.objective(x0), f_final=p.objective(res.x),
                        success=res.success, rel_grad=res.rel_grad,
                        initial_grad_norm=res.initial_grad_norm)


def kershaw_newton_case(name, counts, order, n_quad, iters):
    """The paper benchmark's flow at a small size (bench.py:170-245): Kershaw
    eps 0.3 mesh, mu_303 ideal shape, Jacobi-MINRES Newton, fixed iterations."""
    spec = tb.MeshSpec(dim=3, nx=counts[0], ny=counts[1], nz=counts[2], order=order)
    mesh = tb.apply_kershaw(tb.build_cartesian(spec), 0.3, 0.3)
    x0 = mesh.dof_vector()
    p = tb.TmopProblem(mesh, tb.ObjectiveConfig(tb.MetricId.MU_303, tb.TargetSpec(tb.TargetKind.IDEAL_UNIT)),
                       n_quad)
    res = tb.newton_solve(x0, p, tb.NewtonConfig(max_iterations=iters), tb.MinresConfig(preconditioned=True))
    recs = np.array([[r.alpha, r.objective, r.grad_norm, r.minres_iterations,
                      r.minres_rel_residual, r.min_det] for r in res.trace.records])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), counts=np.array(counts), order=order, n_quad=n_quad,
                        iters=iters, x0=x0, x=res.x, records=recs, f0=p.objective(x0),
                        f_final=p.objective(res.x), success=res.success)


def minres_case(name, n=40, seed=7):
    """Small dense symmetric indefinite system with Jacobi (sol:93-180)."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n))
    A = a + a.T + np.diag(np.linspace(-3, 6, n))
    b = rng.standard_normal(n)
    diag = np.diag(A).copy()
    pre = tb.jacobi_preconditioner(diag)
    r = tb.minres(lambda v: A @ v, b, tb.MinresConfig(max_iterations=25, rel_tolerance=1e-10), pre)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), A=A, b=b, x=r.x,
                        iterations=r.iterations, history=np.array(r.residual_history))


def minres_conditioned_case(name, n=200, seed=11, indefinite=True):
    """Well-conditioned system: few iterations, rounding does not amplify."""
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = rng.uniform(1.0, 4.0, n)
    if indefinite:
        lam[: n // 3] *= -1.0
    A = (q * lam) @ q.T
    A = 0.5 * (A + A.T)
    b = rng.standard_normal(n)
    pre = tb.jacobi_preconditioner(np.diag(A).copy())
    r = tb.minres(lambda v: A @ v, b, tb.MinresConfig(max_iterations=12, rel_tolerance=1e-10), pre)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), A=A, b=b, x=r.x,
                        iterations=r.iterations, history=np.array(r.residual_history))


def metric_points(name):
    rng = np.random.default_rng(SEED)
    out = {}
    for metric, dim in [(2, 2), (55, 2), (55, 3), (303, 3)]:
        ts = []
        for _ in range(12):
            t = rng.uniform(-1.5, 1.5, (dim, dim)) + np.eye(dim)
            dt = np.linalg.det(t)
            if dt <= 1e-3:
                continue
            ts.append(t * (rng.uniform(0.1, 10.0) / dt) ** (1.0 / dim))
        ts = np.stack(ts)
        out[f"T_{metric}_{dim}"] = ts
        out[f"mu_{metric}_{dim}"] = tb.metric_value(tb.MetricId(metric), ts)
        out[f"P_{metric}_{dim}"] = tb.metric_first_derivative(tb.MetricId(metric), ts)
        out[f"H_{metric}_{dim}"] = tb.metric_second_derivative(tb.MetricId(metric), ts)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def kershaw_case(name):
    mesh = tb.apply_kershaw(tb.build_cartesian(tb.MeshSpec(3, 6, 2, 2, order=2)), 0.3, 0.3)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), coords=mesh.coords,
                        restriction=mesh.restriction)


def report_case(name):
    """Reporting formats of the reference driver (bench.py:31-37, 244-330):
    VTK Lagrange-hex permutations p = 1..4, the VTK text of a small Kershaw
    mesh, and the CSV row of a RunReport with fixed values."""
    import tempfile as _tf

    from tmopbench import bench as rb
    out = {f"perm_p{p}": rb.vtk_lagrange_hex_permutation(p) for p in (1, 2, 3, 4)}
    mesh = tb.apply_kershaw(tb.build_cartesian(tb.MeshSpec(3, 6, 2, 2, order=2)), 0.3, 0.3)
    with _tf.TemporaryDirectory() as d:
        path = os.path.join(d, "m.vtk")
        rb.write_vtk(mesh, path, title="kershaw initial mesh")
        out["vtk_text"] = np.array(open(path).read())
    times = {"total": 12.5, "gradient": 0.1 / 3, "hessian_setup": 1.0 / 7, "hessian_apply": 9.87654321,
             "linesearch": 2e-5, "objective": 0.01}
    rep = rb.RunReport(nx=24, ny=24, nz=24, order=1, n_quad=9, epsy=0.3, epsz=0.3, metric=303, preconditioned=True,
                       dofs_per_component=15625, dofs_total=46875, quad_points=24 ** 3 * 729, newton_iterations=13,
                       minres_iterations=650, times=times, f_initial=43335.601057054526, f_final=-4.279e-12,
                       relgrad_final=7.68e-10, min_det_initial=3.78e-06, min_det_final=4.6296296296296e-06,
                       max_dev_uniform=8.41e-9, status="failed", success=False)
    out["csv_row"] = np.array(",".join(rep.csv_row()))
    out["csv_header"] = np.array(",".join(rb.CSV_COLUMNS))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def main():
    for p in (1, 2, 3, 4):
        for nq in sorted({p + 1, p + 2}):
            operator_case(f"op3d_p{p}_q{nq}_mu303", 3, (3, 2, 2) if p == 1 else (2, 2, 2),
                          p, nq, 303)
    operator_case("op3d_p2_q3_mu55", 3, (2, 2, 2), 2, 3, 55)
    operator_case("op3d_p2_q4_mu303_size", 3, (2, 3, 2), 2, 4, 303, target="size")
    operator_case("op3d_p3_q6_mu303", 3, (2, 2, 2), 3, 6, 303)
    operator_case("op3d_p2_q9_mu303", 3, (2, 2, 2), 2, 9, 303)
    operator_case("op3d_p1_q3_mu303_w", 3, (4, 3, 2), 1, 3, 303, spatial_weight=2.5)
    for p in (1, 2, 3):
        operator_case(f"op2d_p{p}_q{p + 2}_mu2", 2, (3, 2), p, p + 2, 2)
    operator_case("op2d_p2_q3_mu55", 2, (3, 3), 2, 3, 55)
    operator_case("op2d_p2_q3_mu55_lim", 2, (2, 2), 2, 3, 55, limiting=(0.4, 1.0))
    operator_case("op3d_p2_q3_mu55_lim", 3, (2, 2, 2), 2, 3, 55, limiting=(0.4, 1.5))
    limiting_nodal_case("limnodal3d_p2_q4_mu303", 3, (3, 2, 3), 2, 4, 303, 1.7)
    limiting_nodal_case("limnodal2d_p3_q5_mu2", 2, (3, 4), 3, 5, 2, 0.8)
    newton_case("newton_c1_2d_q2_16x16_mu2", 2, (16, 16), 2, 4, 2, iters=5)
    newton_case("newton_3d_p2_4c_mu303", 3, (4, 4, 4), 2, 4, 303, iters=3)
    newton_case("newton_3d_p1_4c_mu303_noprec", 3, (4, 4, 4), 1, 3, 303, iters=2,
                precond=False)
    kershaw_newton_case("kershawnewton_6x4x4_p2_q4", (6, 4, 4), 2, 4, 100)
    minres_case("minres_dense")
    minres_conditioned_case("minres_wellcond")
    metric_points("metric_points")
    kershaw_case("kershaw_6x2x2_p2")
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    if sys.argv[1:] == ["--only", "report"]:
        report_case("report_formats")
    else:
        main()
