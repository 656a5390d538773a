"""Small driver for ncu captures of the Hessian-action kernels:
    python tools/prof_apply.py --order 2 --n 80 --reps 3
(setup once, then `reps` applies; the apply element kernel is
elem_kernel<3, p+1, n_q, 1>)."""

import argparse
import os
import sys

# one whole-mesh element launch (not the overlapped z-slab launches), so the
# capture is the kernel the roofline is quoted for
os.environ.setdefault("TMOP_OVERLAP_MIN", str(2 ** 62))

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_12721_b200 as P  # noqa: E402
from bench import perturbed_x  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--order", type=int, default=2)
ap.add_argument("--n", type=int, default=80)
ap.add_argument("--nq", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--metric", type=int, default=303)
a = ap.parse_args()
nq = a.nq or a.order + 2
mesh = P.build_box(3, (a.n,) * 3, a.order)
prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId(a.metric), P.TargetSpec(P.TargetKind.IDEAL_UNIT)), nq)
x = torch.from_numpy(perturbed_x(mesh)).cuda()
v = torch.from_numpy(np.random.default_rng(1).standard_normal(mesh.n_dofs)).cuda()
qd = prob.hessian_setup(x)
y = torch.empty_like(v)
for _ in range(a.reps):
    prob.hessian_apply(qd, v, out=y)
torch.cuda.synchronize()
print("ok", mesh.n_dofs, float(y.norm()))
