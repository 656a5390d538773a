"""Run the REFERENCE's full paper-table Kershaw solve here
on the CPU and log its progress, for BASELINE.md section 2.1.

    NUMBA_NUM_THREADS=4 python tools/ref_kershaw_full.py --order 1 --out profiles/ref_kershaw24_p1.json

Same flow as the reference CLI (`tmop-bench --nx 24 --ny 24 --nz 24 --order 1
--nq 9`, bench.py:171-241): Kershaw eps 0.3, mu_303, ideal shape, Jacobi
MINRES cap 50 / rtol 1e-8, Newton rtol 1e-10, 100 iterations.  A proxy in
front of the reference problem (the KernelTimer pattern, bench.py:133-168)
appends one line per Newton iteration (F at the iterate the Hessian is set up
at) to `<out>.log` so a multi-hour run can be watched.  Container only: it
imports /root/reference.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_refrun_"))
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import tmopbench as tb  # noqa: E402


class Logged:
    def __init__(self, problem, log):
        self.p, self.log, self.t0, self.k = problem, log, time.perf_counter(), 0

    def objective(self, x):
        return self.p.objective(x)

    def gradient(self, x):
        return self.p.gradient(x)

    def hessian_setup(self, x):
        f = self.p.objective(x)
        with open(self.log, "a") as fh:
            fh.write(json.dumps({"newton_iteration": self.k, "F": f, "wall_s": time.perf_counter() - self.t0}) + "\n")
        self.k += 1
        return self.p.hessian_setup(x)

    def hessian_diagonal(self, q):
        return self.p.hessian_diagonal(q)

    def hessian_apply(self, q, v):
        return self.p.hessian_apply(q, v)

    def min_det_jacobian(self, x):
        return self.p.min_det_jacobian(x)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--order", type=int, default=1)
    ap.add_argument("--n", type=int, default=24)
    ap.add_argument("--nq", type=int, default=9)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    spec = tb.MeshSpec(dim=3, nx=a.n, ny=a.n, nz=a.n, order=a.order)
    mesh0 = tb.build_cartesian(spec)
    uniform = mesh0.dof_vector()
    mesh = tb.apply_kershaw(mesh0, 0.3, 0.3)
    x0 = mesh.dof_vector()
    prob = tb.TmopProblem(mesh, tb.ObjectiveConfig(tb.MetricId.MU_303, tb.TargetSpec(tb.TargetKind.IDEAL_UNIT)),
                          a.nq)
    log = a.out + ".log"
    open(log, "w").close()
    t = time.perf_counter()
    status, msg = "ok", "converged"
    try:
        res = tb.newton_solve(x0, Logged(prob, log),
                              tb.NewtonConfig(rel_grad_tolerance=1e-10, max_iterations=a.iters),
                              tb.MinresConfig(max_iterations=50, rel_tolerance=1e-8, preconditioned=True))
        x, tr, msg = res.x, res.trace, res.message
        if not res.success:
            status = "failed"
    except (tb.LineSearchError, tb.InvalidMeshError, tb.MinresBreakdownError) as err:
        status, msg, x, tr = "failed", str(err), x0, None
    wall = time.perf_counter() - t
    out = {"order": a.order, "n": a.n, "n_quad": a.nq, "precond": True, "dofs": mesh.n_dofs,
           "threads": int(os.environ.get("NUMBA_NUM_THREADS", "0")) or os.cpu_count(),
           "solve_s": wall, "newton_iterations": tr.newton_iterations if tr else None,
           "minres_iterations": tr.minres_total if tr else None, "status": status, "message": msg,
           "f_initial": prob.objective(x0), "f_final": prob.objective(x),
           "max_dev_uniform": float(np.max(np.abs(x - uniform))),
           "records": [[r.alpha, r.objective, r.grad_norm, r.minres_iterations, r.minres_rel_residual, r.min_det]
                       for r in tr.records] if tr else None}
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "records"}))


if __name__ == "__main__":
    main()
