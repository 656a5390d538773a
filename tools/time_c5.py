"""C5 pieces at 96^3 Q2 (mu_321, size-field targets): per-operator device
times and the full Newton solve of bench.c5_solve.
    python tools/time_c5.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2205_12721_b200 as P  # noqa: E402
from bench import perturbed_x  # noqa: E402

mesh = P.build_box(3, (96, 96, 96), 2)
eta = P.size_field(mesh, "shell")
prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_321, P.TargetSpec(P.TargetKind.SIZE_FIELD, size=eta)), 4)
x = torch.from_numpy(perturbed_x(mesh)).cuda()
s = torch.cuda.current_stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


qd = prob.hessian_setup(x)
v = torch.randn(mesh.n_dofs, dtype=torch.float64, device="cuda")
print("mu_321 size-field 96^3 Q2: setup %.3f  diagonal %.3f  apply %.3f  gradient %.3f ms"
      % (t(lambda: prob.hessian_setup(x)), t(lambda: prob.hessian_diagonal(qd)), t(lambda: prob.hessian_apply(qd, v)),
         t(lambda: prob.gradient(x))))
del prob, qd
torch.cuda.empty_cache()
print(bench.c5_solve())
