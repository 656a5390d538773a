"""The z-slab multi-GPU path (paper_2205_12721_b200/distributed.py) with the
REAL device operator: two ranks share the one GPU of the test box (gloo moves
the halo planes through host memory -- the NCCL transport is the only part
not exercised).  Each rank's slab operator (CUDA kernels on its local
lattice) + plane sums + all-reduces must reproduce the single-process GPU
operator on the global mesh."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

COUNTS, ORDER, NQ = (4, 3, 8), 2, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    import torch
    import torch.distributed as dist

    import paper_2205_12721_b200 as P
    from oracle import tmop_oracle as O
    from paper_2205_12721_b200.distributed import (DistributedProblem, SlabPartition, dist_minres,
                                                   dist_minres_device, dist_newton_solve)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cfg = P.ObjectiveConfig(P.MetricId.MU_303, P.TargetSpec(P.TargetKind.IDEAL_UNIT))
        gmesh = P.build_box(3, COUNTS, ORDER)
        rng = np.random.default_rng(20240901)
        x = O.perturb(O.box_mesh(3, COUNTS, ORDER), rng, 0.2)
        v = rng.standard_normal(x.shape)
        gp = P.TmopProblem(gmesh, cfg, NQ)
        part = SlabPartition(COUNTS, ORDER, world, rank)
        lmesh = part.local_mesh(gmesh)
        lp = P.TmopProblem(lmesh, cfg, NQ)
        dp = DistributedProblem(lp, part, lmesh.fixed_mask).to("cuda")
        xl = torch.from_numpy(part.local_vector(x)).cuda()
        vl = torch.from_numpy(part.local_vector(v)).cuda()
        gq, lq = gp.hessian_setup(x), dp.hessian_setup(xl)

        def err(local, glob):
            want = part.local_vector(glob)
            return float(np.linalg.norm(local.cpu().numpy() - want) / np.linalg.norm(want))

        out = {"lattice": bool(lp.lattice)}
        ya = dp.hessian_apply(lq, vl)
        out["apply"] = err(ya, gp.hessian_apply(gq, v))
        dp.overlap = True                        # boundary layers first, exchange overlapping the interior
        out["overlap_bitwise"] = bool(torch.equal(ya, dp.hessian_apply(lq, vl)))
        dp.overlap = False
        # host-resident pipelined action + device plane sums == the device path
        vpin = vl.cpu().pin_memory()
        out["host_bitwise"] = bool(torch.equal(dp.hessian_apply_host(lq, vpin), ya.cpu()))
        out["grad"] = err(dp.gradient(xl), gp.gradient(x))
        out["diag"] = err(dp.hessian_diagonal(lq), gp.hessian_diagonal(gq))
        out["obj"] = abs(dp.objective(xl) - gp.objective(x)) / abs(gp.objective(x))
        out["mindet"] = abs(dp.min_det_jacobian(xl) - gp.min_det_jacobian(x))
        out["dot"] = abs(dp.dot(vl, vl) - float(v @ v)) / float(v @ v)
        # distributed MINRES (20 its) vs the single-process device MINRES
        g = gp.gradient(x)
        pre = P.jacobi_preconditioner(gp.hessian_diagonal(gq), gp.ctx)
        mr = P.minres(lambda u: gp.hessian_apply(gq, u), g,
                      P.MinresConfig(max_iterations=20, rel_tolerance=1e-300), pre, gp.ctx)
        ld = dp.hessian_diagonal(lq)
        linv = 1.0 / ld.abs().clamp_min(1e-12)
        xd, itd, _, _ = dist_minres(dp, lambda u: dp.hessian_apply(lq, u), dp.gradient(xl), 20, 1e-300, linv)
        out["minres_its"] = (int(mr.iterations), int(itd))
        out["minres_x"] = err(xd, mr.x)
        # device-resident distributed MINRES: library phases with owned-node
        # partial dots all-reduced in between, halo pack / unpack kernels
        assert dp.device_op
        xdd, itdd, rrd, _ = dist_minres_device(dp, lq, dp.gradient(xl), 20, 1e-300, linv)
        out["dminres_its"] = int(itdd)
        out["dminres_x"] = err(xdd, mr.x)
        out["dminres_vs_eager"] = float((xdd - xd).norm() / xd.norm())
        # two Newton iterations (device MINRES inside) vs the single-GPU solver
        xn, recs, ok, msg = dist_newton_solve(dp, xl, max_iterations=2)
        own = P.newton_solve(x, gp, P.NewtonConfig(max_iterations=2), P.MinresConfig())
        out["newton_alpha"] = ([r[0] for r in recs], [r.alpha for r in own.trace.records])
        out["newton_its"] = ([r[3] for r in recs], [r.minres_iterations for r in own.trace.records])
        out["newton_x"] = err(xn, np.asarray(own.x))
        # peer-memory halo (CUDA IPC mailboxes, no NCCL / gloo on the data
        # path): same plane sums -> bitwise the same results
        dq = DistributedProblem(lp, part, lmesh.fixed_mask).to("cuda").enable_p2p()
        out["p2p_apply"] = bool(torch.equal(dq.hessian_apply(lq, vl), ya))
        out["p2p_grad"] = bool(torch.equal(dq.gradient(xl), dp.gradient(xl)))
        out["p2p_diag"] = bool(torch.equal(dq.hessian_diagonal(lq), dp.hessian_diagonal(lq)))
        xq, itq, _, _ = dist_minres_device(dq, lq, dq.gradient(xl), 20, 1e-300, linv)
        out["p2p_minres"] = bool(torch.equal(xq, xdd)) and itq == itdd
        dq.halo.check_p2p()
        dq.disable_p2p()
        # size-field targets (mu_321) over the partition vs the global operator
        eta = P.size_field(gmesh, "shell")
        cfw = P.ObjectiveConfig(P.MetricId.MU_321, P.TargetSpec(P.TargetKind.SIZE_FIELD, size=eta))
        gw = P.TmopProblem(gmesh, cfw, NQ)
        lw = P.TmopProblem(lmesh, P.ObjectiveConfig(P.MetricId.MU_321, P.TargetSpec(
            P.TargetKind.SIZE_FIELD, size=eta[part.node_lo:part.node_hi])), NQ)
        dw = DistributedProblem(lw, part, lmesh.fixed_mask).to("cuda")
        gqw, lqw = gw.hessian_setup(x), dw.hessian_setup(xl)
        out["size_apply"] = err(dw.hessian_apply(lqw, vl), gw.hessian_apply(gqw, v))
        out["size_grad"] = err(dw.gradient(xl), gw.gradient(x))
        out["size_obj"] = abs(dw.objective(xl) - gw.objective(x)) / abs(gw.objective(x))
        results[rank] = out
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_partition_with_device_operator_matches_global(world):
    """world 3: the middle rank has both neighbours (two planes per exchange)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    # (one retry on a fresh port: _free_port's port can be taken by another
    # process between its release and the rendezvous)
    for attempt in range(2):
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, results)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(900)
        if all(p.exitcode == 0 for p in procs) or attempt == 1:
            break
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    for r in range(world):
        out = results[r]
        assert out["lattice"], out
        assert out["apply"] <= 1e-13, out
        assert out["overlap_bitwise"], out
        assert out["host_bitwise"], out
        assert out["grad"] <= 1e-13, out
        assert out["diag"] <= 1e-13, out
        assert out["obj"] <= 1e-13, out
        assert out["mindet"] == 0.0, out
        assert out["dot"] <= 1e-14, out
        assert out["minres_its"][0] == out["minres_its"][1] == 20, out
        assert out["minres_x"] <= 1e-10, out
        assert out["dminres_its"] == 20, out
        assert out["dminres_x"] <= 1e-10, out
        assert out["newton_alpha"][0] == out["newton_alpha"][1], out
        assert out["newton_its"][0] == out["newton_its"][1], out
        assert out["newton_x"] <= 1e-9, out
        assert out["p2p_apply"] and out["p2p_grad"] and out["p2p_diag"] and out["p2p_minres"], out
        assert out["size_apply"] <= 1e-13 and out["size_grad"] <= 1e-13 and out["size_obj"] <= 1e-13, out


def test_bench_distributed_schema_gloo_two_ranks_matches_single_rank():
    """bench.py's multi-GPU leg as the driver launches it (torch.distributed.run,
    2 ranks) with gloo on the one GPU of the test box, against the 1-rank
    --force-dist (NCCL) line: same JSON schema, n_gpus = world size."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    common = ["--steps", "3", "--warmup", "3", "--dist-n", "16", "--no-cpu"]
    one = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "1", "--force-dist"] + common,
                         capture_output=True, text=True, timeout=900)
    assert one.returncode == 0, one.stderr[-3000:]
    two = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dist-backend", "gloo"]
                         + common, capture_output=True, text=True, timeout=900)
    assert two.returncode == 0, two.stderr[-3000:]
    l1 = json.loads([ln for ln in one.stdout.splitlines() if ln.startswith("{")][-1])
    l2 = json.loads([ln for ln in two.stdout.splitlines() if ln.startswith("{")][-1])
    assert l1["n_gpus"] == 1 and l2["n_gpus"] == 2
    assert set(l1) == set(l2)
    for k in ("headline_leg", "c4_strong", "c4_weak", "newton_iteration", "e2e", "roofline"):
        assert set(l1[k]) == set(l2[k]), k
    assert l2["halo_ms_per_step"] > 0 and l2["halo_bytes_per_neighbor"] == 3 * (16 * 2 + 1) ** 2 * 8
    assert l2["c4_strong"]["global_dofs"] == l1["c4_strong"]["global_dofs"]
    assert l2["newton_iteration"]["minres_iterations"] == 20


def test_bench_gpus_beyond_device_count_fails_loudly():
    import subprocess
    import sys

    import torch
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    n = torch.cuda.device_count() + 1
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", str(n), "--steps", "3"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "CUDA device" in r.stderr
