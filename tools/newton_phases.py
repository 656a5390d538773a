"""Wall time of the phases of Newton iterations on the Kershaw mesh
(setup+diagonal, MINRES (cap 50), line search), device synchronised:
    python tools/newton_phases.py --order 4 --nq 9 --iters 3"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_12721_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--order", type=int, default=4)
ap.add_argument("--n", type=int, default=24)
ap.add_argument("--nq", type=int, default=9)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
mesh = P.apply_kershaw(P.build_cartesian(P.MeshSpec(dim=3, nx=a.n, ny=a.n, nz=a.n, order=a.order)), 0.3, 0.3)
prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_303, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), a.nq)
x = torch.from_numpy(mesh.dof_vector()).cuda()
g = prob.gradient(x)
f = prob.objective(x)
ng = float(torch.linalg.norm(g))
for it in range(a.iters):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    qd = prob.hessian_setup(x)
    pre = P.jacobi_preconditioner(prob.hessian_diagonal(qd), prob.ctx)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    mr = P.minres(lambda vv: prob.hessian_apply(qd, vv), g, P.MinresConfig(max_iterations=50), pre, prob.ctx,
                  operator=(prob, qd))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ls = P.line_search(x, mr.x, prob, f, ng, ctx=prob.ctx)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    x, f, ng, g = ls.x, ls.objective, ls.grad_norm, ls.gradient
    print(f"iter {it}: setup+diag {1e3 * (t1 - t0):7.2f} ms  minres({mr.iterations}) {1e3 * (t2 - t1):7.2f} ms "
          f"({1e3 * (t2 - t1) / max(mr.iterations, 1):.3f} ms/it)  line search(alpha={ls.alpha}) {1e3 * (t3 - t2):7.2f} ms")
