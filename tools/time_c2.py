"""C2 (32^3 Q1, n_q = 3) Hessian action, template vs non-template metric:
    python tools/time_c2.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_12721_b200 as P  # noqa: E402
from bench import perturbed_x  # noqa: E402

mesh = P.build_box(3, (32, 32, 32), 1)
x = torch.from_numpy(perturbed_x(mesh)).cuda()
v = torch.from_numpy(np.random.default_rng(1).standard_normal(mesh.n_dofs)).cuda()
for metric in (P.MetricId.MU_302, P.MetricId.MU_303, P.MetricId.MU_321):
    prob = P.TmopProblem(mesh, P.ObjectiveConfig(metric, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), 3)
    qd = prob.hessian_setup(x)
    y = torch.empty_like(v)
    for _ in range(5):
        prob.hessian_apply(qd, v, out=y)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(200):
        prob.hessian_apply(qd, v, out=y)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"{metric.name}: {e0.elapsed_time(e1) / 200 * 1e3:7.1f} us per apply", flush=True)
