"""Benchmark of the TMOP Hessian action (AddMultGradPA) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], "C3"): 3D hex perturbed unit cube,
p = 2, 160^3 elements (99.2 M DOFs), n_q = p + 2 = 4, mu_303, ideal-shape
target; x = uniform lattice + 0.2 * (h/p^2) * U(-1, 1) on free components
(seed 20240901), v ~ N(0, 1) (seed 1).  One step = one Hessian action over
the whole mesh; metric = N_dof / t_step (GDOF/s).  Inputs (46 GB of Q-data)
are far larger than L2, so no flush is needed between steps.

Also reported: per-order throughput (p = 1..4 at ~1e8 DOFs, p = 1 at 2.4e7),
the roofline of the dominant kernel (element kernel, HBM-bound), e2e through
the public API with pinned host buffers, one Newton iteration (paper
protocol: MINRES fixed at 20) and the CPU baseline: the reference's own
`TmopProblem.hessian_apply` (tmopbench pip-installed into baseline/_ref,
numba from the image) on the host cores, bounded sample, with the C/OpenMP
oracle port beside it.  `--impl reference` times the reference alone
(rank 0; other ranks exit without work).  `--gpus N` (N > 1) without a
launcher starts N ranks itself (torch.distributed.run, 127.0.0.1).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 20240901
ORDERS = {1: (200, 3), 2: (160, 4), 3: (107, 5), 4: (80, 6)}   # p -> (elements per axis, n_q)
HEADLINE_P = 2
OVERLAP_SLABS = int(os.environ.get("TMOP_APPLY_SLABS", "8"))   # element + E->L launches per apply (lattice)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def perturbed_x(mesh, amplitude=0.2, seed=SEED):
    """Reference test recipe (tests/oracles.py:121-131) restated for inputs."""
    gap = (1.0 / max(mesh.element_counts)) / mesh.order ** 2
    rng = np.random.default_rng(seed)
    x = mesh.coords.ravel().copy()
    j = amplitude * gap * rng.uniform(-1.0, 1.0, x.shape)
    j[mesh.fixed_mask.ravel()] = 0.0
    return x + j


def apply_bytes(dim, order, nq, ne, n_dofs):
    """SURVEY 8(d) yardstick per apply: reference Q-data + restriction + v + y."""
    Q, n = nq ** dim, order + 1
    return 8 * (4 + 2 * dim * dim) * ne * Q + 4 * ne * n ** dim + 16 * n_dofs


def apply_flops(dim, order, nq, ne):
    """SURVEY 8(d) algorithmic flops per apply (the reference's OpCounter x 2:
    sum-factorised contractions + the 108-madd block multiply per point)."""
    n, q, d = order + 1, nq, dim
    per_dir = sum(q ** k * n ** (d + 1 - k) for k in range(1, d + 1))
    return 2 * ne * (2 * d * d * per_dir + (6 * d * d + 2 * d ** 3) * q ** d)


FP64_PEAK_TFLOPS = 37.1   # measured on this pool's B200: DMMA loop 37.1, DFMA loop 34.1 (profiles/round1_fp64_peak.txt)


def measured_traffic(key):
    try:
        with open(os.path.join(ROOT, "profiles", "round1_traffic.json")) as f:
            t = json.load(f)[key]
        return t["dram_bytes_read"] + t["dram_bytes_write"], t
    except Exception:
        return None, None


def element_kernel_bytes(dim, order, nq, ne, n_dofs):
    """Algorithmic bytes of one element-kernel launch: Q-data (22 fp64 / point)
    + restriction (int32) + one read of v + the E-vector write."""
    Q, n = nq ** dim, order + 1
    return 8 * (4 + 2 * dim * dim) * ne * Q + 4 * ne * n ** dim + 8 * n_dofs + 8 * dim * ne * n ** dim


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out = self.proc.communicate(timeout=5)[0]
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            f = [t.strip() for t in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, val in zip(names, f[2:6]):
                if val.lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def build_problem(order, n, nq, device):
    import paper_2205_12721_b200 as P
    mesh = P.build_box(3, (n, n, n), order)
    prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_303, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), nq,
                         device=device)
    return mesh, prob


def time_applies(prob, qd, v, y, steps, warmup):
    """Device-resident steps (one step = tmop_hessian_apply: element kernel +
    E->L, overlapped slab by slab on lattices) timed with CUDA events on the
    launching stream; a second, split pass times the element kernel and the
    one-shot E->L separately for the breakdown / roofline."""
    import torch
    lib, ctx = prob.lib, prob.ctx
    from paper_2205_12721_b200 import _lib
    s = torch.cuda.current_stream()
    prob._sync_stream()
    for _ in range(warmup):
        prob.hessian_apply(qd, v, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(steps):
        _lib.check(lib.tmop_hessian_apply(ctx, _lib.ptr(qd.data), _lib.ptr(v), _lib.ptr(y)), "apply")
    e1.record(s)
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1) / 1e3
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for k in range(steps):
        ev[k][0].record(s)
        _lib.check(lib.tmop_hessian_apply_elements(ctx, _lib.ptr(qd.data), _lib.ptr(v)), "elements")
        ev[k][1].record(s)
        _lib.check(lib.tmop_hessian_apply_gather(ctx, _lib.ptr(v), _lib.ptr(y)), "gather")
        ev[k][2].record(s)
    torch.cuda.synchronize()
    elem = [e[0].elapsed_time(e[1]) / 1e3 for e in ev]
    gath = [e[1].elapsed_time(e[2]) / 1e3 for e in ev]
    return total, statistics.mean(elem), statistics.mean(gath)


def run_order(order, n, nq, steps, warmup, device, with_e2e=False, with_newton=False, sampler_index=None):
    import torch
    t0 = time.time()
    mesh, prob = build_problem(order, n, nq, device)
    x = torch.from_numpy(perturbed_x(mesh)).to(device)
    rng = np.random.default_rng(1)
    v = torch.from_numpy(rng.standard_normal(mesh.n_dofs)).to(device)
    y = torch.empty_like(v)
    qd = prob.hessian_setup(x)
    setup_s = time.time() - t0
    res = {"order": order, "elements": mesh.n_elements, "n_quad": nq, "n_dofs": mesh.n_dofs,
           "qdata_gb": qd.nbytes / 1e9}
    clocks = None
    if sampler_index is not None:
        with ClockSampler(sampler_index) as cs:
            time.sleep(0.3)
            total, t_elem, t_gath = time_applies(prob, qd, v, y, steps, warmup)
        clocks = cs.summary()
    else:
        total, t_elem, t_gath = time_applies(prob, qd, v, y, steps, warmup)
    res.update(ms_per_step=1e3 * total / steps, gdofs=mesh.n_dofs * steps / total / 1e9,
               t_elem_ms=1e3 * t_elem, t_gather_ms=1e3 * t_gath,
               elem_bytes=element_kernel_bytes(3, order, nq, mesh.n_elements, mesh.n_dofs),
               apply_bytes=apply_bytes(3, order, nq, mesh.n_elements, mesh.n_dofs),
               host_setup_s=setup_s)
    if with_e2e:
        # public API with pinned host buffers: H2D of v + apply + D2H of y every step
        vh = v.cpu().pin_memory()
        yh = torch.empty(mesh.n_dofs, dtype=torch.float64, pin_memory=True)
        for _ in range(max(1, warmup)):
            prob.hessian_apply(qd, vh, out=yh)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(steps):
            prob.hessian_apply(qd, vh, out=yh)
        torch.cuda.synchronize()
        te = (time.perf_counter() - t) / steps
        res["e2e"] = {"value": mesh.n_dofs / te / 1e9, "unit": "GDOF/s", "h2d_bytes_per_step": 8 * mesh.n_dofs,
                      "d2h_bytes_per_step": 8 * yh.numel(), "ms_per_step": 1e3 * te}
        ref = y.cpu()
        res["e2e_matches_device"] = bool(torch.equal(yh, ref))
    if with_newton:
        # wall-clock (host-driven) metric: the better of two iterations from the same x
        runs = [newton_iteration(prob, x) for _ in range(2)]
        res["newton"] = min(runs, key=lambda r: r["ms"])
        res["newton"]["runs_ms"] = [r["ms"] for r in runs]
    del qd
    torch.cuda.synchronize()
    return res, clocks


def small_config_c2(steps=200):
    """BASELINE configs[1] (C2): 3D Q1 perturbed cube 32^3, mu_302 (non-template
    Hessian), n_q = 3 -- 107,811 DOFs, launch-latency territory.  Eager
    applies vs a CUDA graph replaying `steps` applies (element kernel + E->L)."""
    import torch

    import paper_2205_12721_b200 as P
    from paper_2205_12721_b200 import _lib
    mesh = P.build_box(3, (32, 32, 32), 1)
    prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_302, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), 3)
    x = torch.from_numpy(perturbed_x(mesh)).cuda()
    v = torch.from_numpy(np.random.default_rng(1).standard_normal(mesh.n_dofs)).cuda()
    y = torch.empty_like(v)
    qd = prob.hessian_setup(x)
    for _ in range(5):
        prob.hessian_apply(qd, v, out=y)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(steps):
        prob.hessian_apply(qd, v, out=y)
    e1.record(s)
    torch.cuda.synchronize()
    t_eager = e0.elapsed_time(e1) / 1e3 / steps
    side = torch.cuda.Stream()
    side.wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        prob._sync_stream()
        with torch.cuda.graph(g, stream=side):
            for _ in range(steps):
                _lib.check(prob.lib.tmop_hessian_apply(prob.ctx, _lib.ptr(qd.data), _lib.ptr(v), _lib.ptr(y)),
                           "tmop_hessian_apply")
    s.wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    t_graph = e0.elapsed_time(e1) / 1e3 / steps
    prob._sync_stream()
    return {"workload": "C2: 3D Q1 perturbed cube 32^3 elements, mu_302, n_q=3", "n_dofs": mesh.n_dofs,
            "us_per_apply_eager": 1e6 * t_eager, "gdofs_eager": mesh.n_dofs / t_eager / 1e9,
            "us_per_apply_graph": 1e6 * t_graph, "gdofs_graph": mesh.n_dofs / t_graph / 1e9,
            "graph_applies": steps}


# Kershaw eps=0.3, 24^3, n_q=9, mu_303, Jacobi-MINRES,
# GPU-PA* time to solution on 4x V100 and its Newton / MINRES iteration counts.
PAPER_KERSHAW = {1: (0.4, 11, 203), 2: (0.9, 18, 507), 3: (3.9, 41, 1536), 4: (8.5, 70, 3110)}


def kershaw_paper_table(orders=(1, 2, 3, 4)):
    """The paper's time-to-solution table on ONE B200 (tools/kershaw_solve.py);
    the second of two identical solves per order is reported."""
    from tools.kershaw_solve import solve
    out = []
    for p in orders:
        solve(p, 24, 9)            # warm-up: first-launch kernel configuration, graph capture paths
        r = solve(p, 24, 9)
        t, nn, nm = PAPER_KERSHAW[p]
        r.update(paper_gpu_pa_star_s_4xV100=t, paper_newton_iterations=nn, paper_minres_iterations=nm,
                 speedup_vs_paper=t / r["solve_s"])
        out.append(r)
    return out


def c1_solve():
    """BASELINE configs[0] (C1): 2D Q2 16x16 unit square, perturbed interior
    (amp 0.2, seed 20240901), mu_2, n_q = 4, 5 Newton iterations, Jacobi-MINRES
    -- the case the CPU reference runs in 2.85 s.
    Wall time of the warm solve (second of two)."""
    import torch

    import paper_2205_12721_b200 as P
    mesh = P.build_box(2, (16, 16), 2)
    x0 = torch.from_numpy(perturbed_x(mesh)).cuda()
    prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_2, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), 4)
    out = None
    for _ in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = P.newton_solve(x0, prob, P.NewtonConfig(max_iterations=5), P.MinresConfig())
        torch.cuda.synchronize()
        out = {"workload": "C1: 2D Q2 16x16, mu_2, n_q=4, 5 Newton", "n_dofs": mesh.n_dofs,
               "solve_s": time.perf_counter() - t, "newton_iterations": res.trace.newton_iterations,
               "minres_iterations": res.trace.minres_total, "f_final": prob.objective(res.x),
               "reference_cpu_s_survey": 2.85}
    return out


def newton_iteration(prob, x):
    """One Newton iteration, paper protocol (MINRES fixed at 20 iterations,
    PAPER.md:1002-1004): setup + diagonal + MINRES + line search."""
    import torch

    import paper_2205_12721_b200 as P
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = prob.gradient(x)
    f = prob.objective(x)
    ng = float(torch.linalg.norm(g))
    torch.cuda.synchronize()
    t_pre = time.perf_counter() - t
    t = time.perf_counter()
    qd = prob.hessian_setup(x)
    pre = P.jacobi_preconditioner(prob.hessian_diagonal(qd), prob.ctx)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t
    t = time.perf_counter()
    mr = P.minres(lambda vv: prob.hessian_apply(qd, vv), g,
                  P.MinresConfig(max_iterations=20, rel_tolerance=1e-300), pre, prob.ctx, operator=(prob, qd))
    torch.cuda.synchronize()
    t_minres = time.perf_counter() - t
    t = time.perf_counter()
    ls = P.line_search(x, mr.x, prob, f, ng, ctx=prob.ctx)
    torch.cuda.synchronize()
    t_ls = time.perf_counter() - t
    return {"ms": 1e3 * (t_setup + t_minres + t_ls), "setup_diag_ms": 1e3 * t_setup,
            "minres_ms": 1e3 * t_minres, "minres_iterations": mr.iterations, "line_search_ms": 1e3 * t_ls,
            "alpha": ls.alpha, "initial_gradient_ms": 1e3 * t_pre}


def cpu_baseline_port(order=2, n=40, budget_s=12.0, threads=0):
    """C/OpenMP oracle port of the reference apply on a bounded sample
    (secondary CPU number: the reference's algorithm in C, all cores)."""
    from oracle import tmop_oracle as O
    from oracle.cpu_apply import CpuApply
    nq = order + 2
    om = O.box_mesh(3, (n, n, n), order)
    prob = O.OracleProblem(om, O.MU_303, nq)
    x = O.perturb(om, np.random.default_rng(SEED), 0.2)
    v = np.random.default_rng(1).standard_normal(x.shape)
    qd = prob.hessian_setup(x)
    ca = CpuApply(prob, qd, threads)
    ca(v)
    times = []
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < budget_s or len(times) < 3:
        t = time.perf_counter()
        ca(v)
        times.append(time.perf_counter() - t)
    best = min(times)
    return {"value": om.n_dofs / best / 1e9, "unit": "GDOF/s", "cores": ca.threads, "kind": "port",
            "sample": f"p={order} {n}^3 elements ({om.n_dofs} DOFs), n_q={nq}, mu_303; best of {len(times)} "
                      f"applies of the C/OpenMP oracle port (oracle/tmop_cpu.c)",
            "cpu_model": _cpu_model()}


# ----------------------------------------------------------------------------
# The reference itself (tmopbench, pip-installed into baseline/_ref, which
# travels to the GPU box; numba / numpy / scipy are in the image).  Its
# TmopProblem.hessian_apply (operator.py:401-418) is timed on the host cores:
# NUMBA_NUM_THREADS = the cores this process may use (the reference CLI's
# --threads does not set it, cli.py:63-65), one JIT warm-up, then the timed
# applies.  Run in a subprocess so the thread count is fixed before numba loads.
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def ref_probe(n, order, threads, steps, warmup):
    """Child process body: build the reference problem on an n^3 p=order
    perturbed cube (n_q = p + 2, mu_303, ideal shape), set up the Q-data
    and time `steps` reference applies after `warmup` untimed ones."""
    sys.path.insert(0, REF_DIR)
    import tmopbench as tb
    nq = order + 2
    t0 = time.perf_counter()
    mesh = tb.build_box(3, (n, n, n), order)
    prob = tb.TmopProblem(mesh, tb.ObjectiveConfig(tb.MetricId.MU_303, tb.TargetSpec(tb.TargetKind.IDEAL_UNIT)), nq)
    x = perturbed_x(mesh)
    v = np.random.default_rng(1).standard_normal(mesh.n_dofs)
    qd = prob.hessian_setup(x)
    t_setup = time.perf_counter() - t0
    for _ in range(warmup):
        prob.hessian_apply(qd, v)
    times = []
    for _ in range(steps):
        t = time.perf_counter()
        y = prob.hessian_apply(qd, v)
        times.append(time.perf_counter() - t)
    tot = sum(times)
    return {"n": n, "order": order, "n_quad": nq, "n_dofs": mesh.n_dofs, "threads": threads, "steps": steps,
            "warmup": warmup, "total_s": tot, "mean_s": tot / steps, "best_s": min(times),
            "gdofs": mesh.n_dofs * steps / tot / 1e9, "setup_and_build_s": t_setup,
            "y_norm": float(np.linalg.norm(y))}


def run_ref_probe(n, order, threads, steps, warmup, timeout=1800):
    """Run ref_probe in a child with the thread count fixed (numba reads
    NUMBA_NUM_THREADS at import)."""
    env = dict(os.environ)
    env.update(NUMBA_NUM_THREADS=str(threads), OMP_NUM_THREADS=str(threads), OPENBLAS_NUM_THREADS=str(threads),
               MKL_NUM_THREADS=str(threads), PYTHONDONTWRITEBYTECODE="1")
    env.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "tmop_bench_numba_cache"))
    cmd = [sys.executable, os.path.abspath(__file__), "--ref-probe", f"{n},{order},{threads},{steps},{warmup}"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout)
    if r.returncode != 0:
        raise RuntimeError(f"reference probe failed: {r.stderr[-2000:]}")
    return json.loads(r.stdout.strip().splitlines()[-1])


def reference_available():
    if not os.path.isdir(os.path.join(REF_DIR, "tmopbench")):
        return False, "baseline/_ref/tmopbench is not installed (pip install --target baseline/_ref /root/reference/pkg)"
    try:
        import numba  # noqa: F401
    except Exception as err:
        return False, f"numba unavailable: {err}"
    return True, ""


REF_SAMPLE_N = 76        # p=2, 76^3 hexes: 10.6 M DOFs (>= 1e7 DOF)
REF_SMALL_N = 24         # 1-thread sample: p=2, 24^3 hexes (352,947 DOFs)


def cpu_baseline(budget_s=25.0):
    """The reference's own TmopProblem.hessian_apply on the host cores
    (kind "reference"), bounded sample: p=2 at 40^3 hexes (1.59 M DOFs),
    applies for ~budget_s."""
    ok, why = reference_available()
    if not ok:
        cb = cpu_baseline_port(HEADLINE_P, 40)
        cb["note"] = f"reference unavailable ({why}); C/OpenMP port timed instead"
        return cb
    cores = host_cores()
    r = run_ref_probe(40, HEADLINE_P, cores, 3, 1)
    return {"value": r["gdofs"], "unit": "GDOF/s", "cores": cores, "kind": "reference",
            "sample": f"reference tmopbench TmopProblem.hessian_apply (operator.py:401-418, baseline/_ref), p=2 "
                      f"40^3 hexes ({r['n_dofs']} DOFs), n_q=4, mu_303, NUMBA_NUM_THREADS={cores}; "
                      f"{r['steps']} timed applies after 1 warm-up",
            "seconds_per_apply": r["mean_s"], "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def run_distributed(args, rank, world, local, device, metric, config):
    """N > 1: weak scaling over z-slabs.  The global mesh is
    160 x 160 x (160 N) p=2 hexes; rank r owns the slab of layers
    [160 r, 160 (r+1)) and one step = local Hessian action + NCCL sum of the
    shared node planes with the z-neighbours (+ constraint re-fix).  Time is
    the max over ranks; halo time is reported separately."""
    import torch
    import torch.distributed as dist

    import paper_2205_12721_b200 as P
    from paper_2205_12721_b200.distributed import DistributedProblem, SlabPartition
    n, nq = ORDERS[HEADLINE_P]
    counts = (n, n, n * world)
    part = SlabPartition(counts, HEADLINE_P, world, rank)
    mesh = part.local_mesh_direct()
    prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_303, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), nq,
                         device=device)
    dp = DistributedProblem(prob, part, mesh.fixed_mask).to(device)
    x = torch.from_numpy(perturbed_x(mesh, seed=SEED + rank)).to(device)
    v = torch.from_numpy(np.random.default_rng(1 + rank).standard_normal(mesh.n_dofs)).to(device)
    qd = prob.hessian_setup(x)
    s = torch.cuda.current_stream()
    for _ in range(args.warmup):
        dp.hessian_apply(qd, v)
    # timed steps: the distributed action as DistributedProblem.hessian_apply
    # runs it by default -- the local (slab-overlapped) action, then the NCCL
    # plane sum and re-fix, split by events so the halo time is reported
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as cs:
        for k in range(args.steps):
            ev[k][0].record(s)
            y = prob.hessian_apply(qd, v)
            ev[k][1].record(s)
            dp.halo.sum_planes(y)
            dp.halo.refix(y, dp.fixed2, v)
            ev[k][2].record(s)
        torch.cuda.synchronize()
    dist.barrier()
    total = ev[0][0].elapsed_time(ev[-1][2]) / 1e3
    halo = statistics.mean(e[1].elapsed_time(e[2]) for e in ev) / 1e3
    # the boundary-first variant (DistributedProblem.overlap = True: outer
    # layers + planes first, exchange overlapping the interior), for comparison
    dp.overlap = True
    dp.hessian_apply(qd, v)
    b0e, b1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    b0e.record(s)
    for _ in range(args.steps):
        dp.hessian_apply(qd, v)
    b1e.record(s)
    torch.cuda.synchronize()
    dp.overlap = False
    bf = b0e.elapsed_time(b1e) / 1e3
    t = torch.tensor([total, halo, bf], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total, halo, bf = float(t[0]), float(t[1]), float(t[2])
    global_dofs = 3 * (n * HEADLINE_P + 1) ** 2 * (n * world * HEADLINE_P + 1)
    value = global_dofs * args.steps / total / 1e9
    # e2e through the distributed API with pinned host buffers
    vh = v.cpu().pin_memory()
    yh = torch.empty_like(vh).pin_memory()
    dist.barrier()
    torch.cuda.synchronize()
    te0 = time.perf_counter()
    for _ in range(args.steps):
        vd = vh.to(device, non_blocking=True)
        yd = dp.hessian_apply(qd, vd)
        yh.copy_(yd, non_blocking=True)
        torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - te0], dtype=torch.float64, device=device)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    te = float(te.item()) / args.steps
    if rank == 0:
        cfg = dict(config)
        cfg.update(workload=f"C4-style weak scaling: global {n}x{n}x{n * world} p={HEADLINE_P} hexes, n_q={nq}, "
                            f"mu_303, z-slab per GPU", parallelism=f"z-slabs x{world} (NCCL halo plane sums)")
        line = {"metric": metric, "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (perturbed slabs, seeded)",
                "config": cfg, "halo_ms_per_step": 1e3 * halo,
                "halo_note": "plane exchange + re-fix after the local action, inside the timed steps",
                "ms_per_step_boundary_first": 1e3 * bf / args.steps,
                "halo_bytes_per_neighbor": dp.halo.bytes_per_exchange,
                "roofline": {"bound": "hbm", "unit": "GB/s", "peak": peaks()[0],
                             "achieved": apply_bytes(3, HEADLINE_P, nq, mesh.n_elements, mesh.n_dofs)
                             / (total / args.steps - halo) / 1e9,
                             "frac": apply_bytes(3, HEADLINE_P, nq, mesh.n_elements, mesh.n_dofs)
                             / (total / args.steps - halo) / 1e9 / peaks()[0],
                             "traffic": None, "kernel": "local Hessian action (element kernel + E->L), per GPU"},
                "e2e": {"value": global_dofs / te / 1e9, "unit": "GDOF/s",
                        "h2d_bytes_per_step": 8 * mesh.n_dofs * world, "d2h_bytes_per_step": 8 * mesh.n_dofs * world},
                "gpu_launches": 2 * OVERLAP_SLABS * args.steps, "clocks": cs.summary()}
        print(json.dumps(line))


def self_launch(args):
    """`bench.py --gpus N` (N > 1) without a launcher: start N ranks under
    torch.distributed.run on 127.0.0.1 and pass their output through; fail
    loudly when the box has fewer than N GPUs."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested but only {have} CUDA device(s) visible"}),
              file=sys.stderr)
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def reference_arm(args, world, metric, config):
    """`--impl reference`: the reference's own TmopProblem.hessian_apply
    (baseline/_ref) on the host cores, rank 0 only.  One step = one
    reference apply over a p=2, 76^3-hex perturbed cube (10.6 M DOFs,
    BASELINE.md section 3's >= 1e7-DOF floor; CPU GDOF/s is flat in size,
    PAPER.md:1032-1033) -- a bounded sample of the C3 workload.  Warm-up:
    one JIT compile on a tiny mesh plus min(W, 1) untimed sample applies, so
    the run stays within a few minutes.  A 1-thread number at 24^3 is
    reported beside it (the reference barely scales with cores)."""
    ok, why = reference_available()
    if not ok:
        print(json.dumps({"impl": "reference", "unavailable": why}))
        return
    cores = host_cores()
    run_ref_probe(2, 1, cores, 1, 1)                     # numba JIT (cache dir under /tmp)
    big = run_ref_probe(REF_SAMPLE_N, HEADLINE_P, cores, args.steps, min(args.warmup, 1), timeout=3600)
    one = run_ref_probe(REF_SMALL_N, HEADLINE_P, 1, 2, 1)
    sample = (f"reference tmopbench TmopProblem.hessian_apply (operator.py:401-418; pip-installed to baseline/_ref), "
              f"p=2, {REF_SAMPLE_N}^3 hexes ({big['n_dofs']} DOFs), n_q=4, mu_303, ideal shape, same perturbed-x "
              f"recipe and v seed as our arm; NUMBA_NUM_THREADS={cores}")
    cb = {"value": big["gdofs"], "unit": "GDOF/s", "cores": cores, "kind": "reference", "sample": sample,
          "cpu_model": _cpu_model(),
          "one_thread": {"value": one["gdofs"], "unit": "GDOF/s", "cores": 1,
                         "sample": f"p=2, {REF_SMALL_N}^3 hexes ({one['n_dofs']} DOFs), NUMBA_NUM_THREADS=1",
                         "seconds_per_apply": one["mean_s"]}}
    line = {"impl": "reference", "metric": metric, "value": big["gdofs"], "unit": "GDOF/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * big["mean_s"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (perturbed cube, seeded)", "config": config, "cpu_baseline": cb,
            "e2e": {"value": big["gdofs"], "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "warmup_note": f"numba JIT on a 2^3 mesh + {min(args.warmup, 1)} untimed sample apply(s)",
            "reference_setup_s": big["setup_and_build_s"]}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--orders", default="1,2,3,4", help="orders reported under per_order")
    ap.add_argument("--no-newton", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--force-dist", action="store_true", help="run the z-slab (NCCL) path even with one rank")
    ap.add_argument("--ref-probe", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.ref_probe:
        n, order, threads, steps, warmup = (int(t) for t in args.ref_probe.split(","))
        print(json.dumps(ref_probe(n, order, threads, steps, warmup)))
        return
    if args.warmup < 3 and args.impl == "ours":
        ap.error("--warmup must be >= 3")
    launched = "RANK" in os.environ
    if args.gpus > 1 and not launched and args.impl == "ours":
        self_launch(args)
    rank, world, local = dist_env()
    if launched and world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), file=sys.stderr)
        sys.exit(2)
    n_h, nq_h = ORDERS[HEADLINE_P]
    config = {"workload": f"C3: 3D hex perturbed unit cube, p={HEADLINE_P}, {n_h}^3 elements, n_q={nq_h}, "
                          f"mu_303, ideal-shape target (amp 0.2 h/p^2, seed {SEED})",
              "order": HEADLINE_P, "elements_per_axis": n_h, "n_quad": nq_h, "metric_id": 303,
              "l2": "inputs > L2 (Q-data >> 126 MB), no flush", "parallelism": f"replicas x{world}"}
    metric = "3D TMOP Hessian-action GDOF/s (p=2, ~1e8 DOFs)"

    if args.impl == "reference":
        if rank != 0:
            return
        reference_arm(args, world, metric, config)
        return

    import torch
    dist_path = world > 1 or args.force_dist
    if dist_path:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = torch.device("cuda", local if dist_path else torch.cuda.current_device())
    torch.cuda.set_device(device)
    if dist_path:
        torch.distributed.barrier()
        run_distributed(args, rank, world, local, device, metric, config)
        torch.distributed.destroy_process_group()
        return
    head, clocks = run_order(HEADLINE_P, n_h, nq_h, args.steps, args.warmup, device, with_e2e=True,
                             with_newton=not args.no_newton, sampler_index=local)
    # whole-job aggregate: max time over ranks (replicas, weak scaling)
    ms = torch.tensor([head["ms_per_step"]], dtype=torch.float64, device=device)
    if world > 1:
        torch.distributed.all_reduce(ms, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(ms.item())
    value = world * head["n_dofs"] / (ms_max / 1e3) / 1e9
    per_order = {}
    for p in [int(s) for s in args.orders.split(",") if s.strip()]:
        if p == HEADLINE_P:
            per_order[str(p)] = {k: head[k] for k in ("gdofs", "ms_per_step", "n_dofs", "elements", "n_quad",
                                                      "t_elem_ms", "t_gather_ms")}
            continue
        n, nq = ORDERS[p]
        r, _ = run_order(p, n, nq, max(3, args.steps // 2), args.warmup, device)
        r["roofline_frac_elem"] = r["elem_bytes"] / (r["t_elem_ms"] / 1e3) / 1e9 / peaks()[0]
        r["fp64_frac_elem"] = apply_flops(3, p, nq, r["elements"]) / (r["t_elem_ms"] / 1e3) / 1e12 / FP64_PEAK_TFLOPS
        per_order[str(p)] = {k: r[k] for k in ("gdofs", "ms_per_step", "n_dofs", "elements", "n_quad",
                                               "t_elem_ms", "t_gather_ms", "roofline_frac_elem", "fp64_frac_elem")}
    if rank != 0:
        torch.distributed.barrier()
        return
    peak, peak_src = peaks()
    achieved = head["elem_bytes"] / (head["t_elem_ms"] / 1e3) / 1e9
    traffic, tinfo = measured_traffic(f"p{HEADLINE_P}_n{n_h}_nq{nq_h}")
    flops = apply_flops(3, HEADLINE_P, nq_h, head["elements"])
    ach_tf = flops / (head["t_elem_ms"] / 1e3) / 1e12
    line = {
        "metric": metric, "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (perturbed cube, seeded)", "config": config,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "xl_kernel<3,4,K_APPLY> (tmop_xl.cuh)",
                     "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
                     "algorithmic_bytes_per_launch": head["elem_bytes"],
                     "bytes_note": "algorithmic = reference-format Q-data (22 fp64/point) + restriction + v + "
                                   "E-vector write (SURVEY 8(d)); the kernel streams the lean 11-fp64 record, so "
                                   "frac > 1 is possible -- traffic (ncu dram bytes, profiles/round1_traffic.json) "
                                   "is what it actually moves",
                     "traffic_frac_of_peak": (traffic / (head["t_elem_ms"] / 1e3) / 1e9 / peak) if traffic else None,
                     "kernel_share_of_step": head["t_elem_ms"] / head["ms_per_step"],
                     "fp64": {"algorithmic_flops": flops, "achieved": ach_tf, "peak": FP64_PEAK_TFLOPS,
                              "unit": "TFLOP/s", "frac": ach_tf / FP64_PEAK_TFLOPS,
                              "pipe_util_ncu": tinfo["fp64_pipe_util"] if tinfo else None}},
        "apply_roofline": {"yardstick_bytes": head["apply_bytes"],
                           "achieved_gbs": head["apply_bytes"] / (head["ms_per_step"] / 1e3) / 1e9,
                           "frac": head["apply_bytes"] / (head["ms_per_step"] / 1e3) / 1e9 / peak},
        "e2e": head["e2e"], "e2e_matches_device": head.get("e2e_matches_device"),
        "gpu_launches": (2 * OVERLAP_SLABS if HEADLINE_P <= 3 else 2) * args.steps, "clocks": clocks,
        "per_order": per_order,
        "qdata_gb": head["qdata_gb"],
    }
    if "newton" in head:
        line["newton_iteration"] = head["newton"]
    import gc
    gc.collect()
    torch.cuda.empty_cache()   # the small-problem sections below run after the 1e8-DOF ones
    line["c2_small"] = small_config_c2()
    line["c1_solve"] = c1_solve()
    if not args.no_newton:
        line["kershaw_paper_table"] = kershaw_paper_table()
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline()
        line["cpu_baseline_port"] = cpu_baseline_port(HEADLINE_P, 40)
    print(json.dumps(line))
    if world > 1:
        torch.distributed.barrier()


if __name__ == "__main__":
    main()
