"""Where a paper-table Kershaw MINRES iteration goes (24^3, n_q = 9): the
Hessian action's device time vs the wall time of a 50-iteration Jacobi-MINRES
solve, eager and as CUDA-graph replay.
    python tools/kershaw_minres_probe.py --orders 1,2,3,4"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_12721_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--orders", default="1,2,3,4")
ap.add_argument("--n", type=int, default=24)
ap.add_argument("--nq", type=int, default=9)
a = ap.parse_args()
for p in [int(s) for s in a.orders.split(",")]:
    mesh = P.apply_kershaw(P.build_cartesian(P.MeshSpec(dim=3, nx=a.n, ny=a.n, nz=a.n, order=p)), 0.3, 0.3)
    x = torch.from_numpy(mesh.dof_vector()).cuda()
    prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_303, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), a.nq)
    qd = prob.hessian_setup(x)
    g = prob.gradient(x)
    pre = P.jacobi_preconditioner(prob.hessian_diagonal(qd))
    v = torch.randn(mesh.n_dofs, dtype=torch.float64, device="cuda")
    y = torch.empty_like(v)
    for _ in range(3):
        prob.hessian_apply(qd, v, out=y)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(50):
        prob.hessian_apply(qd, v, out=y)
    e1.record(s)
    torch.cuda.synchronize()
    t_apply = e0.elapsed_time(e1) / 50
    out = {}
    for graph in (False, True):
        cfg = P.MinresConfig(max_iterations=50, rel_tolerance=1e-30, preconditioned=True, graph=graph)
        P.minres(lambda u: prob.hessian_apply(qd, u), -g, cfg, precond=pre, operator=(prob, qd))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            r = P.minres(lambda u: prob.hessian_apply(qd, u), -g, cfg, precond=pre, operator=(prob, qd))
        torch.cuda.synchronize()
        out[graph] = ((time.perf_counter() - t0) / 3 * 1e3, r.iterations)
    print(f"p={p} dofs={mesh.n_dofs} apply {t_apply:.3f} ms (device); MINRES 50 its eager {out[False][0]:.2f} ms "
          f"({out[False][0] / out[False][1]:.3f} ms/it), graph {out[True][0]:.2f} ms "
          f"({out[True][0] / out[True][1]:.3f} ms/it)", flush=True)
