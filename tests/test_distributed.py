"""World-size-2 gloo tests of the slab partition + halo exchange
(paper_2205_12721_b200/distributed.py) on CPU.  The local operator is the CPU
oracle (test infrastructure); the partition, plane sums, constraint re-fix,
owned-node dots and the distributed MINRES / Newton are the product code."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tmop_oracle as O
from paper_2205_12721_b200.distributed import (DistributedProblem, SlabPartition, dist_minres,
                                               dist_newton_solve, split_layers)

COUNTS, ORDER, NQ = (3, 2, 4), 2, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _local_oracle(part, gmesh, metric):
    lm = O.box_mesh(3, part.local_counts, ORDER)
    sl = slice(part.node_lo, part.node_hi)
    lm.coords = gmesh.coords[:, sl].copy()
    lm.fixed = gmesh.fixed[:, sl].copy()
    return O.OracleProblem(lm, metric, NQ), lm


def _worker(rank, world, port, metric, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gmesh = O.box_mesh(3, COUNTS, ORDER)
        rng = np.random.default_rng(20240901)
        x = O.perturb(gmesh, rng, 0.2)
        v = rng.standard_normal(x.shape)
        gp = O.OracleProblem(gmesh, metric, NQ)
        part = SlabPartition(COUNTS, ORDER, world, rank)
        lp, lm = _local_oracle(part, gmesh, metric)
        dp = DistributedProblem(lp, part, lm.fixed,
                                to_local=lambda t: t.numpy() if torch.is_tensor(t) else t,
                                from_local=lambda a: torch.from_numpy(np.array(a, dtype=np.float64)))
        xl = torch.from_numpy(part.local_vector(x))
        vl = torch.from_numpy(part.local_vector(v))
        out = {}
        gq = gp.hessian_setup(x)
        lq = dp.hessian_setup(xl)
        def err(local, glob):
            want = part.local_vector(glob)
            return float(np.linalg.norm(local.numpy() - want) / np.linalg.norm(want))
        out["apply"] = err(dp.hessian_apply(lq, vl), gp.hessian_apply(gq, v))
        out["grad"] = err(dp.gradient(xl), gp.gradient(x))
        out["diag"] = err(dp.hessian_diagonal(lq), gp.hessian_diagonal(gq))
        out["obj"] = abs(dp.objective(xl) - gp.objective(x)) / abs(gp.objective(x))
        out["mindet"] = abs(dp.min_det_jacobian(xl) - gp.min_det_jacobian(x))
        out["dot"] = abs(dp.dot(vl, vl) - float(v @ v)) / float(v @ v)
        # distributed MINRES vs single-process oracle MINRES (same recurrence)
        g = gp.gradient(x)
        inv = 1.0 / np.maximum(np.abs(gp.hessian_diagonal(gq)), 1e-12)
        xs, its, rr, _, _ = O.minres(lambda u: gp.hessian_apply(gq, u), g, 20, 1e-8, lambda r: inv * r)
        ld = dp.hessian_diagonal(lq)
        linv = 1.0 / ld.abs().clamp_min(1e-12)
        xd, itd, rrd, _ = dist_minres(dp, lambda u: dp.hessian_apply(lq, u), dp.gradient(xl), 20, 1e-8, linv)
        out["minres_its"] = (its, itd)
        out["minres_x"] = err(xd, xs)
        # two Newton iterations
        xn, recs, ok, msg = dist_newton_solve(dp, xl, max_iterations=2)
        xo, orecs, _, _, _, _ = O.newton(x, gp, max_it=2)
        out["newton_x"] = err(xn, xo)
        out["newton_alpha"] = ([r[0] for r in recs], [r[0] for r in orecs])
        results[rank] = out
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("metric", [O.MU_303, O.MU_321])
def test_slab_partition_matches_global_operator(metric):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, metric, results)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    for r in range(2):
        out = results[r]
        assert out["apply"] <= 1e-13, out
        assert out["grad"] <= 1e-13, out
        assert out["diag"] <= 1e-13, out
        assert out["obj"] <= 1e-13, out
        assert out["mindet"] == 0.0, out
        assert out["dot"] <= 1e-14, out
        assert out["minres_its"][0] == out["minres_its"][1], out
        assert out["minres_x"] <= 1e-10, out
        assert out["newton_alpha"][0] == out["newton_alpha"][1], out
        assert out["newton_x"] <= 1e-9, out


def test_split_layers_and_ranges():
    assert split_layers(10, 3) == [(0, 4), (4, 7), (7, 10)]
    with pytest.raises(ValueError):
        split_layers(2, 3)
    gm = O.box_mesh(3, (2, 2, 5), 2)
    parts = [SlabPartition((2, 2, 5), 2, 3, r) for r in range(3)]
    owned = sum(p.n_owned for p in parts)
    assert owned == gm.n_nodes
    for a, b in zip(parts, parts[1:]):
        assert a.node_hi - a.plane == b.node_lo          # one shared plane
    assert parts[0].elem_lo == 0 and parts[-1].elem_hi == gm.n_elements
