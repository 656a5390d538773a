"""ncu driver for the MINRES vector kernels at C3 (p = 2, 160^3):
    ncu -k regex:minres_k3 -c 1 python tools/prof_minres.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_12721_b200 as P  # noqa: E402
from bench import perturbed_x  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 160
mesh = P.build_box(3, (n,) * 3, 2)
prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_303, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), 4)
x = torch.from_numpy(perturbed_x(mesh)).cuda()
qd = prob.hessian_setup(x)
g = prob.gradient(x)
pre = P.jacobi_preconditioner(prob.hessian_diagonal(qd), prob.ctx)
for _ in range(2):
    r = P.minres(lambda v: prob.hessian_apply(qd, v), g, P.MinresConfig(max_iterations=4, rel_tolerance=1e-300),
                 pre, prob.ctx, operator=(prob, qd))
torch.cuda.synchronize()
print("ok", r.iterations)
