"""How sensitive is the REFERENCE's own paper-table Kershaw trajectory to
round-off?  Runs tmopbench.newton_solve (solvers.py:263-321) at 24^3, n_q=9,
p=1 for 3 Newton iterations from x0 and from x0 perturbed by one ulp on
every free coordinate, and prints the relative change of F / |grad F| /
min det per iteration (container only: imports /root/reference).

    NUMBA_NUM_THREADS=3 python tools/ref_sensitivity.py --order 1 > tests/golden/kershaw24_sensitivity_p1.json
"""
import argparse
import json
import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_sens_"))
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import tmopbench as tb  # noqa: E402


def run(order, iters, bump):
    mesh = tb.apply_kershaw(tb.build_cartesian(tb.MeshSpec(dim=3, nx=24, ny=24, nz=24, order=order)), 0.3, 0.3)
    x0 = mesh.dof_vector()
    if bump:
        free = ~mesh.fixed_mask.ravel()
        x0 = x0.copy()
        x0[free] = np.nextafter(x0[free], np.inf)
    p = tb.TmopProblem(mesh, tb.ObjectiveConfig(tb.MetricId.MU_303, tb.TargetSpec(tb.TargetKind.IDEAL_UNIT)), 9)
    res = tb.newton_solve(x0, p, tb.NewtonConfig(max_iterations=iters), tb.MinresConfig())
    return [[r.alpha, r.objective, r.grad_norm, r.minres_iterations, r.min_det] for r in res.trace.records]


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--order", type=int, default=1)
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    base, bumped = run(a.order, a.iters, False), run(a.order, a.iters, True)
    rows = [{"iteration": k + 1, "alpha": (b[0], c[0]), "minres": (b[3], c[3]), "F_rel": c[1] / b[1] - 1,
             "grad_rel": c[2] / b[2] - 1, "min_det_rel": c[4] / b[4] - 1} for k, (b, c) in enumerate(zip(base, bumped))]
    print(json.dumps({"order": a.order, "perturbation": "x0 + 1 ulp on every free coordinate", "rows": rows},
                     indent=1))
