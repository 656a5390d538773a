"""Device time of every operator entry point at one size (CUDA events):
    python tools/time_phases.py --order 2 --n 160"""
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
ap.add_argument("--n", type=int, default=160)
ap.add_argument("--nq", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
nq = a.nq or a.order + 2
mesh = P.build_box(3, (a.n,) * 3, a.order)
prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_303, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), nq)
x = torch.from_numpy(perturbed_x(mesh)).cuda()
v = torch.from_numpy(np.random.default_rng(1).standard_normal(mesh.n_dofs)).cuda()
qd = prob.hessian_setup(x)
y = torch.empty_like(v)
s = torch.cuda.current_stream()


def timed(name, fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"{name:18s} {e0.elapsed_time(e1) / a.reps:9.3f} ms")


print(f"p={a.order} n={a.n} nq={nq} dofs={mesh.n_dofs}")
timed("hessian_setup", lambda: prob.hessian_setup(x))
timed("hessian_apply", lambda: prob.hessian_apply(qd, v, out=y))
timed("hessian_diagonal", lambda: prob.hessian_diagonal(qd))
timed("gradient", lambda: prob.gradient(x))
timed("objective", lambda: prob.objective(x))
timed("min_det", lambda: prob.min_det_jacobian(x))
