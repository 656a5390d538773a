"""Reference-side drop-in: the reference's OWN solver and timing proxy
(tmopbench.newton_solve, solvers.py:263-321; tmopbench.bench.KernelTimer,
bench.py:133-168), pip-installed into baseline/_ref, driving this package's
TmopProblem through the ProblemLike protocol (solvers.py:183-189) with numpy
vectors -- exactly what a reference user gets by swapping the class.  The
trace must equal the reference-generated golden trace and this package's own
device-resident newton_solve."""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, load_golden

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def tb():
    if not os.path.isdir(os.path.join(REF, "tmopbench")):
        pytest.skip("baseline/_ref/tmopbench not installed")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tmop_test_numba_cache")
    sys.path.insert(0, REF)
    try:
        import tmopbench
    finally:
        sys.path.remove(REF)
    return tmopbench


@pytest.mark.parametrize("name", ["newton_c1_2d_q2_16x16_mu2", "newton_3d_p2_4c_mu303"])
def test_reference_newton_solve_drives_our_problem(tb, name):
    import paper_2205_12721_b200 as P
    g = load_golden(name)
    mesh = P.build_box(int(g["dim"]), tuple(int(c) for c in g["counts"]), int(g["order"]))
    prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId(int(g["metric"])),
                                                 P.TargetSpec(P.TargetKind.IDEAL_UNIT)), int(g["n_quad"]))
    timer = tb.bench.KernelTimer(prob)
    res = tb.newton_solve(g["x0"], timer, tb.NewtonConfig(max_iterations=int(g["iters"])),
                          tb.MinresConfig(preconditioned=bool(g["precond"])))
    assert isinstance(res.x, np.ndarray)
    want = g["records"]
    assert res.trace.newton_iterations == len(want)
    for rec, ref in zip(res.trace.records, want):
        assert rec.alpha == ref[0]
        assert rec.minres_iterations == int(ref[3])
        assert rec.objective == pytest.approx(ref[1], rel=1e-9, abs=1e-13)
        assert rec.grad_norm == pytest.approx(ref[2], rel=1e-8, abs=1e-13)
    assert np.linalg.norm(res.x - g["x"]) <= 1e-10 * np.linalg.norm(g["x"])
    # the KernelTimer buckets saw every ProblemLike call
    assert timer.seconds["hessian_apply"] > 0 and timer.seconds["hessian_setup"] > 0
    assert timer.seconds["objective"] > 0 and timer.seconds["gradient"] > 0
    # same trajectory as this package's device-resident solver
    own = P.newton_solve(g["x0"], prob, P.NewtonConfig(max_iterations=int(g["iters"])),
                         P.MinresConfig(preconditioned=bool(g["precond"])))
    assert [r.alpha for r in own.trace.records] == [r.alpha for r in res.trace.records]
    assert [r.minres_iterations for r in own.trace.records] == [r.minres_iterations for r in res.trace.records]
    assert np.linalg.norm(np.asarray(own.x) - res.x) <= 1e-10 * np.linalg.norm(res.x)


def test_reference_line_search_and_minres_accept_our_operator(tb, rng):
    """tmopbench.minres (solvers.py:93-180) with our hessian_apply as the
    operator closure and tmopbench.jacobi_preconditioner on our diagonal."""
    import paper_2205_12721_b200 as P
    g = load_golden("op3d_p2_q4_mu303")
    mesh = P.build_box(3, tuple(int(c) for c in g["counts"]), 2)
    prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_303, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), 4)
    qd = prob.hessian_setup(g["x"])
    pre = tb.jacobi_preconditioner(prob.hessian_diagonal(qd))
    b = prob.gradient(g["x"])
    r = tb.minres(lambda v: prob.hessian_apply(qd, v), b, tb.MinresConfig(max_iterations=30), pre)
    own = P.minres(lambda v: prob.hessian_apply(qd, v), b, P.MinresConfig(max_iterations=30),
                   P.jacobi_preconditioner(prob.hessian_diagonal(qd)))
    assert r.iterations == own.iterations
    assert np.linalg.norm(np.asarray(own.x) - r.x) <= 1e-10 * np.linalg.norm(r.x)
    ls = tb.line_search(g["x"], r.x, prob, f0=prob.objective(g["x"]), grad_norm0=float(np.linalg.norm(b)))
    assert ls.alpha > 0 and ls.min_det > 0


def test_kershaw_run_benchmark_on_gpu(tmp_path):
    """The reference driver flow (bench.py:171-241) through
    paper_2205_12721_b200.kershaw_bench.run_benchmark on the GPU: CSV row with
    the reference columns, VTK files, per-kernel buckets, and the trajectory
    of the pinned small Kershaw case (tests/golden/kershawnewton_6x4x4_p2_q4)."""
    from paper_2205_12721_b200 import kershaw_bench as KB
    g = load_golden("kershawnewton_6x4x4_p2_q4")
    cfg = KB.BenchConfig(nx=6, ny=4, nz=4, order=2, n_quad=4, csv_path=os.path.join(tmp_path, "r.csv"),
                         vtk_prefix=os.path.join(tmp_path, "m"))
    rep = KB.run_benchmark(cfg)
    assert rep.success and rep.status == "ok"
    assert abs(rep.newton_iterations - len(g["records"])) <= 3
    assert rep.max_dev_uniform <= 1e-9
    row = KB.read_csv_row(cfg.csv_path)
    assert list(row) == list(KB.CSV_COLUMNS) and row["status"] == "ok"
    assert int(row["newton_iters"]) == rep.newton_iterations
    assert rep.times["hessian_apply"] > 0 and rep.times["hessian_setup"] > 0 and rep.times["linesearch"] > 0
    assert sum(rep.times[k] for k in KB.KERNELS) <= rep.times["total"]
    for s in ("initial", "final"):
        txt = open(f"{cfg.vtk_prefix}_{s}.vtk").read()
        assert txt.count("\n72") == 6 * 4 * 4
    fused = KB.run_benchmark(KB.BenchConfig(nx=6, ny=4, nz=4, order=2, n_quad=4), fused=True)
    # (the fused MINRES step sums in another order; near convergence the
    # Newton count may move by a few, as between reference and oracle)
    assert abs(fused.newton_iterations - rep.newton_iterations) <= 3 and fused.success
