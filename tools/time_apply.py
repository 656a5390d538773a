"""Time the Hessian action (element kernel + E->L) at one size:
    TMOP_APPLY_KERNEL=generic python tools/time_apply.py --order 2 --n 160"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--order", type=int, default=2)
ap.add_argument("--n", type=int, default=160)
ap.add_argument("--nq", type=int, default=0)
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
nq = a.nq or a.order + 2
r, _ = bench.run_order(a.order, a.n, nq, a.steps, 3, torch.device("cuda", 0))
print(f"xl={os.environ.get('TMOP_XL', '1')} lattice={os.environ.get('TMOP_LATTICE', '1')} p={a.order} n={a.n} nq={nq} dofs={r['n_dofs']} "
      f"ms={r['ms_per_step']:.3f} elem_ms={r['t_elem_ms']:.3f} gather_ms={r['t_gather_ms']:.3f} "
      f"GDOF/s={r['gdofs']:.2f}")
