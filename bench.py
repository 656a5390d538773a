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
# NCCL communicator logging for the multi-GPU legs (read back by nccl_summary);
# set before torch loads NCCL.  %p = pid.
if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
    os.environ["NCCL_DEBUG"] = "INFO"
os.environ["NCCL_DEBUG_FILE"] = "/tmp/tmop_nccl.%p.log"

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
        with open(os.path.join(ROOT, "profiles", "round2_traffic.json")) as f:
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
        r.pop("f_per_iteration", None)   # (tools/kershaw_solve.py prints the per-iteration F)
        r.pop("problem_build_s", None)
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


def c5_solve(n=96, max_newton=60):
    """BASELINE configs[4] (C5) on one GPU: 3D Q2 hexes, shape+size metric
    mu_321 with size-adaptive targets (TargetKind.SIZE_FIELD: nodal target
    volume 'shell' field, W_q = v_q^(1/3) I), perturbed start, full Newton
    + Jacobi-MINRES (cap 50, rtol 1e-8) to rtol 1e-10 or `max_newton`
    iterations.  Reports the solve time, iteration counts, F and how far
    the element volumes moved toward their targets."""
    import torch

    import paper_2205_12721_b200 as P
    mesh = P.build_box(3, (n, n, n), 2)
    eta = P.size_field(mesh, "shell")
    prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_321, P.TargetSpec(P.TargetKind.SIZE_FIELD, size=eta)),
                         4)
    x0 = torch.from_numpy(perturbed_x(mesh)).cuda()
    f0 = prob.objective(x0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = P.newton_solve(x0, prob, P.NewtonConfig(max_iterations=max_newton), P.MinresConfig())
    torch.cuda.synchronize()
    ts = time.perf_counter() - t
    return {"workload": f"C5 (1 GPU): 3D Q2 {n}^3 hexes, mu_321, size-field targets (shell), n_q=4, "
                        f"full Newton + Jacobi-MINRES", "n_dofs": mesh.n_dofs, "solve_s": ts,
            "newton_iterations": res.trace.newton_iterations, "minres_iterations": res.trace.minres_total,
            "status": "ok" if res.success else "stopped", "message": res.message, "f_initial": f0,
            "f_final": prob.objective(res.x), "rel_grad": res.rel_grad,
            "ms_per_newton_iteration": 1e3 * ts / max(1, res.trace.newton_iterations)}


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


def _hash_unit(idx, salt):
    """Counter-based uniform(-1, 1) from global indices (splitmix64): every
    rank draws the same value for a shared node, whatever the partition."""
    with np.errstate(over="ignore"):            # modular uint64 arithmetic
        z = (idx.astype(np.uint64) + np.uint64(salt) * np.uint64(0x9E3779B97F4A7C15)) * np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(31)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(29)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 / 2 ** 53) - 1.0


def slab_inputs(part, mesh, seed=SEED):
    """x (perturbed lattice, amp 0.2 h/p^2 on free components) and v (unit
    variance) as functions of GLOBAL (component, node) ids, so the copies of
    a shared node plane on two ranks are identical."""
    nx, ny, nz = part.counts
    n_glob = (nx * part.order + 1) * (ny * part.order + 1) * (nz * part.order + 1)
    gid = (np.arange(3, dtype=np.int64)[:, None] * n_glob
           + np.arange(part.node_lo, part.node_hi, dtype=np.int64)[None, :]).ravel()
    gap = (1.0 / max(part.counts)) / part.order ** 2
    j = 0.2 * gap * _hash_unit(gid, seed)
    j[mesh.fixed_mask.ravel()] = 0.0
    x = mesh.coords.ravel() + j
    v = np.sqrt(3.0) * _hash_unit(gid, seed + 1)
    return x, v


def dist_leg(rank, world, device, counts, order, nq, steps, warmup, group=None, sampler=None, transport="nccl"):
    """One distributed Hessian-action leg over z-slabs: the
    local action (slab-overlapped element kernel + E->L) then the halo plane
    sum + constraint re-fix (library pack / NCCL send-recv / unpack), timed
    with CUDA events per step; returns the max-over-ranks times."""
    import torch
    import torch.distributed as dist

    import paper_2205_12721_b200 as P
    from paper_2205_12721_b200.distributed import DistributedProblem, SlabPartition, allreduce_
    part = SlabPartition(counts, order, world, rank)
    mesh = part.local_mesh_direct()
    prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_303, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), nq,
                         device=device)
    dp = DistributedProblem(prob, part, mesh.fixed_mask, group=group).to(device)
    if transport == "p2p":
        dp.enable_p2p()
    xh, vh_np = slab_inputs(part, mesh)
    x = torch.from_numpy(xh).to(device)
    v = torch.from_numpy(vh_np).to(device)
    qd = prob.hessian_setup(x)
    y = torch.empty_like(v)
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        dp.hessian_apply_into(qd, v, y)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    dist.barrier(group)
    torch.cuda.synchronize()
    ctx_s = sampler if sampler is not None else _NullCtx()
    with ctx_s:
        for k in range(steps):
            ev[k][0].record(s)
            prob.hessian_apply(qd, v, out=y)
            ev[k][1].record(s)
            dp.halo.sum_planes_device(y, 1, vfix=v)
            ev[k][2].record(s)
        torch.cuda.synchronize()
    dist.barrier(group)
    total = ev[0][0].elapsed_time(ev[-1][2]) / 1e3
    halo = statistics.mean(e[1].elapsed_time(e[2]) for e in ev) / 1e3
    loc = statistics.mean(e[0].elapsed_time(e[1]) for e in ev) / 1e3
    t = torch.tensor([total, halo, loc], dtype=torch.float64, device=device)
    allreduce_(t, op=dist.ReduceOp.MAX, group=group)
    total, halo, loc = (float(u) for u in t.cpu())
    nx, ny, nz = counts
    global_dofs = 3 * (nx * order + 1) * (ny * order + 1) * (nz * order + 1)
    # e2e through the distributed public API: pinned host v -> pinned host y
    # every step (DistributedProblem.hessian_apply_host: the slab-pipelined
    # H2D / action / D2H, then the plane sums on the device)
    vpin = v.cpu().pin_memory()
    ypin = torch.empty_like(vpin).pin_memory()
    dp.hessian_apply_host(qd, vpin, ypin)          # (configures the pipeline streams)
    dist.barrier(group)
    torch.cuda.synchronize()
    te0 = time.perf_counter()
    for _ in range(steps):
        dp.hessian_apply_host(qd, vpin, ypin)
        torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - te0], dtype=torch.float64, device=device)
    allreduce_(te, op=dist.ReduceOp.MAX, group=group)
    te = float(te.cpu()[0]) / steps
    out = {"counts": list(counts), "order": order, "n_quad": nq, "global_dofs": global_dofs,
           "local_dofs": mesh.n_dofs, "local_elements": mesh.n_elements, "ms_per_step": 1e3 * total / steps,
           "local_action_ms": 1e3 * loc, "halo_ms_per_step": 1e3 * halo,
           "halo_bytes_per_neighbor": dp.halo.bytes_per_exchange,
           "gdofs": global_dofs * steps / total / 1e9, "e2e_gdofs": global_dofs / te / 1e9,
           "e2e_ms_per_step": 1e3 * te, "h2d_bytes_per_step": 8 * mesh.n_dofs * world,
           "d2h_bytes_per_step": 8 * mesh.n_dofs * world,
           "elem_bytes_per_rank": element_kernel_bytes(3, order, nq, mesh.n_elements, mesh.n_dofs)}
    return out, (prob, dp, qd, x)


class _NullCtx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False

    def summary(self):
        return None


def dist_newton_iteration(dp, prob, x, group=None):
    """One distributed Newton iteration, paper protocol (MINRES fixed at 20,
    PAPER.md:1002-1004): setup + diagonal + device-resident MINRES (halo
    sums and in-stream all-reduces) + line search; wall time, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2205_12721_b200.distributed import allreduce_, dist_minres_device
    torch.cuda.synchronize()
    dist.barrier(group)
    t0 = time.perf_counter()
    g = dp.gradient(x)
    f = dp.objective(x)
    ng = float(np.sqrt(dp.dot(g, g)))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    qd = dp.hessian_setup(x)
    d = dp.hessian_diagonal(qd)
    inv = 1.0 / d.abs().clamp_min(1e-12)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dx, its, rr, _ = dist_minres_device(dp, qd, g, 20, 1e-300, inv)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    alpha = 1.0
    for _ in range(31):
        xt = x - alpha * dx
        md, ft, gt = dp.evaluate_trial(xt)          # one fused element pass per trial
        if md > 0.0 and ft < 1.2 * f and float(np.sqrt(dp.dot(gt, gt))) < 1.2 * ng:
            break
        alpha *= 0.5
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    t = torch.tensor([t4 - t1, t2 - t1, t3 - t2, t4 - t3, t1 - t0], dtype=torch.float64, device=x.device)
    allreduce_(t, op=dist.ReduceOp.MAX, group=group)
    t = [1e3 * float(u) for u in t.cpu()]
    return {"ms": t[0], "setup_diag_ms": t[1], "minres_ms": t[2], "minres_iterations": its, "line_search_ms": t[3],
            "alpha": alpha, "initial_gradient_ms": t[4]}


def dist_c5(rank, world, device, n, group=None, iters=60):
    """BASELINE configs[4] over z-slabs: Q2 mu_321 with size-field targets
    (the 'shell' target-volume field of the GLOBAL mesh), global n x n x nN
    hexes, the full distributed Newton solve (device MINRES, cap 50, rtol
    1e-8, Jacobi; Newton rtol 1e-10, at most `iters` iterations), wall time
    max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2205_12721_b200 as P
    from paper_2205_12721_b200.distributed import DistributedProblem, SlabPartition, allreduce_, dist_newton_solve
    counts = (n, n, n * world)
    part = SlabPartition(counts, 2, world, rank)
    mesh = part.local_mesh_direct()
    eta = P.size_field(mesh, "shell", n_elements=counts[0] * counts[1] * counts[2])
    prob = P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_321, P.TargetSpec(P.TargetKind.SIZE_FIELD, size=eta)),
                         4, device=device)
    dp = DistributedProblem(prob, part, mesh.fixed_mask, group=group).to(device)
    x0 = torch.from_numpy(slab_inputs(part, mesh)[0]).to(device)
    f0 = dp.objective(x0)
    dist_newton_solve(dp, x0, max_iterations=1)                 # warm-up (kernel configuration, allocator)
    torch.cuda.synchronize()
    dist.barrier(group)
    t = time.perf_counter()
    x, recs, ok, msg = dist_newton_solve(dp, x0, max_iterations=iters)
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - t], dtype=torch.float64, device=device)
    allreduce_(te, op=dist.ReduceOp.MAX, group=group)
    te = float(te.cpu()[0])
    return {"workload": f"C5 over z-slabs: global {n}x{n}x{n * world} Q2 hexes, mu_321, size-field targets (shell), "
                        f"n_q=4, full Newton (<= {iters} iterations)", "status": "ok" if ok else "stopped",
            "global_dofs": 3 * (2 * n + 1) ** 2 * (2 * n * world + 1),
            "solve_s": te, "newton_iterations": len(recs), "minres_iterations": int(sum(r[3] for r in recs)),
            "ms_per_newton_iteration": 1e3 * te / max(1, len(recs)), "f_initial": f0,
            "f_final": recs[-1][1] if recs else f0, "message": msg}


def nccl_summary():
    """Communicator lines NCCL_DEBUG=INFO wrote to NCCL_DEBUG_FILE (set in
    main() before the process group starts): init, rank count, transports
    (P2P/NVLS/NET) and channel setup."""
    path = os.environ.get("NCCL_DEBUG_FILE", "").replace("%p", str(os.getpid()))
    keys = ("Init COMPLETE", "nRanks", "NVLS", "P2P", "Channel 00", "Connected all", "Using network", "comm 0x",
            "NCCL version")
    lines = []
    try:
        for ln in open(path):
            if any(k in ln for k in keys):
                lines.append(ln.strip()[-200:])
    except Exception as err:
        lines.append(f"(no NCCL log at {path!r}: {err})")
    return lines[:30]


DIST_ORDERS = {"c3_weak": (2, 160, 4), "c4": (3, 112, 5)}   # leg -> (p, elements per axis per slab, n_q)


def run_distributed(args, rank, world, local, device, metric, config, group=None):
    """z-slab multi-GPU legs (BASELINE configs[3]):
      headline  C3 weak scaling: global 160 x 160 x (160 N) p=2 hexes, n_q=4,
                one 160-layer slab per GPU (the N=1 headline's per-GPU work);
      c4_strong Q3 (n_q=5) 112^3 total, 112/N layers per GPU;
      c4_weak   Q3 112 x 112 x (112 N), 112 layers per GPU;
      newton    one distributed Newton iteration on the headline mesh
                (MINRES fixed at 20, device resident).
    Times are CUDA events on the launching stream, max over ranks; the halo
    (pack + NCCL send/recv + unpack/re-fix) is reported per step."""
    p2, n2, q2 = DIST_ORDERS["c3_weak"]
    p3, n3, q3 = DIST_ORDERS["c4"]
    if args.dist_n:
        n2 = n3 = args.dist_n
    with ClockSampler(local) as cs:
        head, (prob, dp, qd, x) = dist_leg(rank, world, device, (n2, n2, n2 * world), p2, q2, args.steps,
                                           args.warmup, group)
    newton = None
    if not args.no_newton:
        # the better of two iterations from the same x (the first configures
        # kernels and fills the caching allocator), as the 1-GPU line does
        runs = [dist_newton_iteration(dp, prob, x, group) for _ in range(2)]
        newton = min(runs, key=lambda r: r["ms"])
        newton["runs_ms"] = [r["ms"] for r in runs]
    del prob, dp, qd, x
    import gc
    gc.collect()
    import torch
    torch.cuda.empty_cache()
    strong, _ = dist_leg(rank, world, device, (n3, n3, n3), p3, q3, args.steps, args.warmup, group)
    gc.collect()
    torch.cuda.empty_cache()
    weak, _ = dist_leg(rank, world, device, (n3, n3, n3 * world), p3, q3, args.steps, args.warmup, group)
    gc.collect()
    torch.cuda.empty_cache()
    c5 = None if args.no_newton else dist_c5(rank, world, device, args.dist_n or 96, group)
    p2p = None
    if world > 1:
        # the same headline leg with the peer-memory halo (CUDA IPC mailboxes,
        # stores over NVLink; no NCCL on the data path)
        gc.collect()
        torch.cuda.empty_cache()
        try:
            r, (prob2, dp2, _, _) = dist_leg(rank, world, device, (n2, n2, n2 * world), p2, q2, args.steps,
                                             args.warmup, group, transport="p2p")
            dp2.halo.check_p2p()
            dp2.disable_p2p()
            p2p = {k: r[k] for k in ("ms_per_step", "local_action_ms", "halo_ms_per_step", "gdofs")}
        except Exception as err:   # reported, not fatal: NCCL legs above are the measurement
            p2p = {"error": str(err)[:300]}
    if rank != 0:
        return
    peak = peaks()[0]
    t_loc = head["local_action_ms"] / 1e3
    achieved = head["elem_bytes_per_rank"] / t_loc / 1e9
    cfg = dict(config)
    cfg.update(workload=f"C3 weak scaling over z-slabs: global {n2}x{n2}x{n2 * world} p={p2} hexes, n_q={q2}, mu_303, "
                        f"one {n2}-layer slab per GPU",
               elements_per_axis=n2, parallelism=f"z-slabs x{world} (NCCL halo plane sums)",
               backend=args.dist_backend)
    line = {"metric": metric, "value": head["gdofs"], "unit": "GDOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (perturbed slabs; inputs hashed from global ids)",
            "config": cfg, "halo_ms_per_step": head["halo_ms_per_step"],
            "halo_bytes_per_neighbor": head["halo_bytes_per_neighbor"],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "kernel": "local Hessian action per GPU (element kernel + E->L, overlapped)",
                         "algorithmic_bytes_per_launch": head["elem_bytes_per_rank"]},
            "e2e": {"value": head["e2e_gdofs"], "unit": "GDOF/s", "h2d_bytes_per_step": head["h2d_bytes_per_step"],
                    "d2h_bytes_per_step": head["d2h_bytes_per_step"], "ms_per_step": head["e2e_ms_per_step"]},
            "gpu_launches": (2 * OVERLAP_SLABS + 2) * args.steps, "clocks": cs.summary(),
            "headline_leg": head, "c4_strong": strong, "c4_weak": weak, "newton_iteration": newton,
            "c5_dist": c5, "halo_p2p": p2p,
            "nccl": nccl_summary()}
    print(json.dumps(line))


def self_launch(args):
    """`bench.py --gpus N` (N > 1) without a launcher: start N ranks under
    torch.distributed.run on 127.0.0.1 and pass their output through; fail
    loudly when the box has fewer than N GPUs."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and args.dist_backend != "gloo":   # (gloo runs share cuda:0)
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
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl",
                    help="gloo: all ranks share cuda:0 (schema / correctness runs on a 1-GPU box)")
    ap.add_argument("--dist-n", type=int, default=0, help=argparse.SUPPRESS)
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
        if args.dist_backend == "gloo":
            local = 0                       # every rank on cuda:0 (schema / correctness runs)
        elif local >= torch.cuda.device_count():
            print(json.dumps({"error": f"rank {rank}: LOCAL_RANK {local} but only {torch.cuda.device_count()} "
                                       f"CUDA device(s)"}), file=sys.stderr)
            sys.exit(2)
        torch.cuda.set_device(local)
        if "RANK" not in os.environ:            # --force-dist without a launcher: a 1-rank group
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=str(port))
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
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
                                   "frac > 1 is possible -- traffic (ncu dram bytes, profiles/round2_traffic.json) "
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
        gc.collect()
        torch.cuda.empty_cache()
        line["c5_solve"] = c5_solve()
    if not args.no_newton:
        line["kershaw_paper_table"] = kershaw_paper_table()
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline()
        line["cpu_baseline_port"] = cpu_baseline_port(HEADLINE_P, 40)
    # the driver keeps the last ~3 KB of stdout: the per-order and Newton
    # sections go last so they survive in its record
    tail = ("c1_solve", "c2_small", "c5_solve", "kershaw_paper_table", "newton_iteration", "per_order")
    line = {**{k: v for k, v in line.items() if k not in tail}, **{k: line[k] for k in tail if k in line}}
    print(json.dumps(line))
    if world > 1:
        torch.distributed.barrier()


if __name__ == "__main__":
    main()
