"""ncu driver for the diagonal kernel: python tools/prof_diag.py --order 2 --n 80"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_12721_b200 as P  # noqa: E402
from bench import perturbed_x  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--order", type=int, default=2)
ap.add_argument("--n", type=int, default=80)
a = ap.parse_args()
mesh = P.build_box(3, (a.n,) * 3, a.order)
prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_303, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), a.order + 2)
x = torch.from_numpy(perturbed_x(mesh)).cuda()
qd = prob.hessian_setup(x)
for _ in range(2):
    d = prob.hessian_diagonal(qd)
torch.cuda.synchronize()
print("ok", float(d.norm()))
