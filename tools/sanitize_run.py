"""Small end-to-end exercise of every device kernel for compute-sanitizer
(memcheck / racecheck / synccheck):
    compute-sanitizer --tool racecheck python tools/sanitize_run.py
3D p = 1..4 (x-line and work-item kernels, x-line diagonal, fused setup +
diagonal), 2D, size-field targets, limiting, MINRES, overlapped apply."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_12721_b200 as P  # noqa: E402
from bench import perturbed_x  # noqa: E402


def run(dim, counts, order, nq, metric, target=None, limiting=False):
    mesh = P.build_box(dim, counts, order)
    spec = target or P.TargetSpec(P.TargetKind.IDEAL_UNIT)
    lim = P.LimitingConfig(reference=mesh.dof_vector(), delta=0.4, weight=1.0) if limiting else None
    prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId(metric), spec, limiting=lim), nq)
    x = torch.from_numpy(perturbed_x(mesh)).cuda()
    v = torch.from_numpy(np.random.default_rng(1).standard_normal(mesh.n_dofs)).cuda()
    qd, diag = prob.hessian_setup_diagonal(x)
    y = prob.hessian_apply(qd, v)
    g = prob.gradient(x)
    f = prob.objective(x)
    md = prob.min_det_jacobian(x)
    prob.evaluate_trial(x)
    mr = P.minres(lambda u: prob.hessian_apply(qd, u), g, P.MinresConfig(max_iterations=6), 
                  P.jacobi_preconditioner(diag, prob.ctx), prob.ctx, operator=(prob, qd))
    torch.cuda.synchronize()
    print(dim, counts, order, nq, metric, float(y.norm()), f, md, mr.iterations, flush=True)


run(3, (5, 4, 3), 1, 3, 303)
run(3, (5, 3, 3), 2, 4, 303)
run(3, (3, 2, 3), 3, 5, 303)
run(3, (2, 2, 2), 4, 6, 303)
run(3, (3, 3, 2), 2, 4, 321)
run(3, (2, 2, 2), 2, 8, 303)
run(2, (5, 4), 2, 4, 2)
run(3, (4, 3, 3), 2, 4, 321, target=P.TargetSpec(P.TargetKind.SIZE_FIELD,
                                                 size=P.size_field(P.build_box(3, (4, 3, 3), 2))))
run(3, (3, 3, 3), 2, 4, 55, limiting=True)
os.environ["TMOP_SETUP_DIAG_FUSED"] = "1"    # (read at first call: already fixed for this process)
print("sanitize run ok")
