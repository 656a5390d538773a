"""End-to-end (pinned host in / out) Hessian action vs the pipeline slab
count:  python tools/time_e2e.py --order 2 --n 160 --slabs 4,8,16,32"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_12721_b200 as P  # noqa: E402
from bench import perturbed_x  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--order", type=int, default=2)
ap.add_argument("--n", type=int, default=160)
ap.add_argument("--nq", type=int, default=0)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--slabs", default="4,8,16,32")
a = ap.parse_args()
nq = a.nq or a.order + 2
mesh = P.build_box(3, (a.n,) * 3, a.order)
prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_303, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), nq)
x = torch.from_numpy(perturbed_x(mesh)).cuda()
qd = prob.hessian_setup(x)
vh = torch.from_numpy(np.random.default_rng(1).standard_normal(mesh.n_dofs)).pin_memory()
yh = torch.empty(mesh.n_dofs, dtype=torch.float64, pin_memory=True)
ref = prob.hessian_apply(qd, vh.cuda()).cpu()
for ns, ramp in [(int(s), r) for s in a.slabs.split(",") for r in (False, True)]:
    prob.pipeline_slabs, prob.pipeline_ramp = ns, ramp
    for _ in range(2):
        prob.hessian_apply(qd, vh, out=yh)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(a.steps):
        prob.hessian_apply(qd, vh, out=yh)
    torch.cuda.synchronize()
    te = (time.perf_counter() - t) / a.steps
    print(f"slabs {ns:3d} ramp {int(ramp)}: {1e3 * te:7.3f} ms  {mesh.n_dofs / te / 1e9:6.3f} GDOF/s  exact={torch.equal(yh, ref)}",
          flush=True)
