"""Paper-table Kershaw solve on one B200 (reference
bench.py:170-245 run_benchmark restated): eps_y = eps_z = 0.3, 24^3 elements,
mu_303, ideal-shape target, Newton rtol 1e-10, MINRES cap 50 / rtol 1e-8,
Jacobi preconditioner.  Prints one JSON line per order.
    python tools/kershaw_solve.py --orders 1,2 --nq 9"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_12721_b200 as P  # noqa: E402


def solve(order, n, nq, precond=True):
    spec = P.MeshSpec(dim=3, nx=n, ny=n, nz=n, order=order)
    mesh0 = P.build_cartesian(spec)
    uniform = mesh0.dof_vector()
    mesh = P.apply_kershaw(mesh0, 0.3, 0.3)
    x0 = torch.from_numpy(mesh.dof_vector()).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_303, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), nq)
    t1 = time.perf_counter()
    f0 = prob.objective(x0)
    status, msg = "ok", ""
    try:
        res = P.newton_solve(x0, prob, P.NewtonConfig(rel_grad_tolerance=1e-10, max_iterations=100),
                             P.MinresConfig(max_iterations=50, rel_tolerance=1e-8, preconditioned=precond))
        x, tr, ok, msg = res.x, res.trace, res.success, res.message
        if not ok:
            status = "failed"
    except (P.LineSearchError, P.InvalidMeshError, P.MinresBreakdownError) as err:
        status, msg, x, tr = "failed", str(err), x0, None
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    xf = x.cpu().numpy() if hasattr(x, "cpu") else x
    return {"order": order, "n": n, "n_quad": nq, "precond": precond, "dofs": mesh.n_dofs,
            "problem_build_s": t1 - t0, "solve_s": t2 - t1,
            "newton_iterations": tr.newton_iterations if tr else None,
            "minres_iterations": tr.minres_total if tr else None,
            "status": status, "message": msg, "f_initial": f0, "f_final": prob.objective(x),
            "f_per_iteration": [float(f"{r.objective:.6g}") for r in tr.records] if tr else None,
            "max_dev_uniform": float(np.max(np.abs(xf - uniform)))}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--orders", default="1,2,3,4")
    ap.add_argument("--n", type=int, default=24)
    ap.add_argument("--nq", type=int, default=9)
    ap.add_argument("--no-precond", action="store_true")
    a = ap.parse_args()
    for p in [int(s) for s in a.orders.split(",")]:
        print(json.dumps(solve(p, a.n, a.nq, not a.no_precond)), flush=True)
