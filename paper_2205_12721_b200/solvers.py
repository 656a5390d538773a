"""Device-resident MINRES (+ Jacobi), backtracking line search and Newton
loop; API mirrors the reference's solvers.py (solvers.py:37-321).

All vectors live in HBM as torch float64 tensors and every vector operation
is a fused libtmop_b200 kernel; MINRES keeps its scalar recurrence on the
device too (tmop_minres_state), so one iteration is: apply + 3 fused
kernels, with one 112-byte state read per `check_every` iterations.  numpy
inputs are accepted at the API edge and copied to the device once.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Protocol

import numpy as np

from . import _lib

__all__ = ["MinresConfig", "NewtonConfig", "MinresResult", "MinresBreakdownError", "LineSearchError",
           "LineSearchResult", "NewtonIterationRecord", "SolveTrace", "NewtonResult", "ProblemLike",
           "JacobiPreconditioner", "jacobi_preconditioner", "minres", "line_search", "newton_solve"]

JACOBI_FLOOR = 1e-12
GROWTH_FACTOR = 1.2


@dataclass
class MinresConfig:
    max_iterations: int = 50
    rel_tolerance: float = 1e-8
    preconditioned: bool = True
    # device state is read every k iterations (results identical for any k:
    # once converged every fused step -- element kernel included -- is a no-op)
    check_every: int = 8
    # Replay the fused TMOP iteration as a CUDA graph of 6 iterations (the
    # buffer rotation and the state parity repeat with period 6).  None / False
    # = eager launches.
    graph: bool | None = None

    def validate(self) -> None:
        if self.max_iterations < 1:
            raise ValueError("MINRES needs at least one iteration")
        if self.rel_tolerance <= 0:
            raise ValueError("MINRES tolerance must be positive")


@dataclass
class NewtonConfig:
    rel_grad_tolerance: float = 1e-10
    max_iterations: int = 100
    max_line_search_halvings: int = 30
    abs_grad_tolerance: float = 1e-12

    def validate(self) -> None:
        if self.rel_grad_tolerance <= 0:
            raise ValueError("Newton gradient tolerance must be positive")


class MinresBreakdownError(RuntimeError):
    def __init__(self, iteration: int):
        self.iteration = iteration
        super().__init__(f"MINRES breakdown (beta = 0) at iteration {iteration}")


class LineSearchError(RuntimeError):
    pass


@dataclass
class MinresResult:
    x: object
    iterations: int
    rel_residual: float
    converged: bool
    residual_history: list = field(default_factory=list)


def _torch():
    import torch
    return torch


class _VecCtx:
    """A minimal library context for vector kernels when no TmopProblem is
    at hand (generic apply_op callables)."""

    def __init__(self, device):
        torch = _torch()
        lib = _lib.load()
        ctx = C.c_void_p()
        B = np.array([0.5, 0.5, 0.5, 0.5])
        dp = C.POINTER(C.c_double)
        restr = torch.zeros(1, dtype=torch.int32, device=device)
        self._keep = restr
        _lib.check(lib.tmop_ctx_create(C.byref(ctx), 2, 1, 2, 0, 0, _lib.ptr(restr), _lib.ptr(restr),
                                       _lib.ptr(restr), _lib.ptr(restr), B.ctypes.data_as(dp),
                                       B.ctypes.data_as(dp), B.ctypes.data_as(dp), 2, 1.0, 1.0, 1.0,
                                       torch.cuda.current_stream(device).cuda_stream), "tmop_ctx_create")
        self.ctx = ctx
        self.lib = lib

    def __del__(self):
        if getattr(self, "ctx", None) is not None:
            self.lib.tmop_ctx_destroy(self.ctx)


_VEC_CTX = {}


def _ctx_for(device, problem=None):
    if problem is not None and hasattr(problem, "ctx"):
        return problem.ctx
    key = str(device)
    if key not in _VEC_CTX:
        _VEC_CTX[key] = _VecCtx(device)
    return _VEC_CTX[key].ctx


def _dev(x, device=None):
    torch = _torch()
    if type(x).__module__.startswith("torch"):
        t = x.detach()
        if t.dtype != torch.float64:
            t = t.double()
        if device is not None and t.device != device:
            t = t.to(device)
        if not t.is_cuda:
            t = t.cuda()
        return t.reshape(-1).contiguous(), False
    if not torch.cuda.is_available():
        raise _lib.TmopLibraryError("the solvers run on the GPU; no CUDA device is available")
    dev = device or torch.device("cuda", torch.cuda.current_device())
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64).reshape(-1)).to(dev), True


def _dot(ctx, a, b, out) -> float:
    _lib.check(_lib.load().tmop_dot(ctx, a.numel(), _lib.ptr(a), _lib.ptr(b), _lib.ptr(out)), "tmop_dot")
    return float(out.item())


class JacobiPreconditioner:
    """z = r / max(|diag|, 1e-12) (solvers.py:83-90); `inv` stays on the device
    and is consumed directly by the fused MINRES kernels."""

    def __init__(self, diag, ctx=None):
        torch = _torch()
        d, _ = _dev(diag)
        self.inv = torch.empty_like(d)
        flag = torch.zeros(1, dtype=torch.int32, device=d.device)
        ctx = ctx or _ctx_for(d.device)
        _lib.check(_lib.load().tmop_jacobi_inverse(ctx, d.numel(), _lib.ptr(d), JACOBI_FLOOR, _lib.ptr(self.inv),
                                                   _lib.ptr(flag)), "tmop_jacobi_inverse")
        if int(flag.item()):
            raise ValueError("preconditioner diagonal contains non-finite entries")

    def __call__(self, r):
        t, host = _dev(r, self.inv.device)
        z = self.inv * t
        return z.cpu().numpy() if host else z


def jacobi_preconditioner(diag, ctx=None) -> JacobiPreconditioner:
    return JacobiPreconditioner(diag, ctx)


_ST = np.dtype([(n, "<f8") for n in ("beta1", "beta", "oldb", "alfa", "beta2", "dbar", "epsln", "sn", "cs",
                                      "phibar", "relres", "gamma")] +
               [(n, "<i4") for n in ("itn", "done", "breakdown", "nonpd")])


def minres(apply_op: Callable, b, cfg: MinresConfig, precond=None, ctx=None, operator=None) -> MinresResult:
    """Preconditioned MINRES from x0 = 0 (solvers.py:93-180), device resident.
    See _minres_body; this wrapper guarantees the library's residual-history
    pointer never outlives the call."""
    used = []
    try:
        return _minres_body(apply_op, b, cfg, precond, ctx, operator, used)
    finally:
        for c in used:
            _lib.load().tmop_minres_set_history(c, None, 0)


def _minres_body(apply_op: Callable, b, cfg: MinresConfig, precond, ctx, operator, used) -> MinresResult:
    """Preconditioned MINRES from x0 = 0 (solvers.py:93-180), device resident.

    `apply_op` maps a device tensor to a device tensor (a numpy result is
    copied up).  `precond` is a JacobiPreconditioner (or None).  With
    `operator=(problem, qdata)` for a device TmopProblem, each iteration is one
    library call (tmop_minres_step_op: element kernel + E->L gather fused
    with the first vector update + 2 vector kernels), and apply_op is unused.
    """
    torch = _torch()
    cfg.validate()
    b, host = _dev(b)
    n = b.numel()
    dev = b.device
    ctx = ctx or _ctx_for(dev)
    lib = _lib.load()
    inv = None
    if precond is not None:
        if not isinstance(precond, JacobiPreconditioner):
            raise TypeError("device MINRES takes a JacobiPreconditioner (jacobi_preconditioner(diag))")
        inv = precond.inv
    bufs = [torch.empty_like(b) for _ in range(9)]
    x, r1, r2, z, v, w, w1, w2, spare = bufs
    if operator is not None:
        op_prob, op_qd = operator
        ctx = op_prob.ctx
    st = torch.zeros(2 * _lib.MINRES_STATE_BYTES, dtype=torch.uint8, device=dev)
    stp = st.data_ptr()
    hist_dev = torch.full((cfg.max_iterations + 1,), float("nan"), dtype=torch.float64, device=dev)
    _lib.check(lib.tmop_minres_set_history(ctx, _lib.ptr(hist_dev), cfg.max_iterations + 1),
               "tmop_minres_set_history")
    used.append(ctx)
    _lib.check(lib.tmop_minres_init(ctx, n, _lib.ptr(b), _lib.ptr(inv), _lib.ptr(x), _lib.ptr(r1), _lib.ptr(r2),
                                    _lib.ptr(z), _lib.ptr(v), _lib.ptr(w), _lib.ptr(w2), stp), "tmop_minres_init")

    def state(k):
        raw = st.cpu().numpy().view(_ST)
        return raw[k & 1]

    s0 = state(0)
    if s0["nonpd"]:
        raise ValueError("preconditioner is not positive definite")
    if s0["beta1"] == 0.0:
        xr = torch.zeros_like(b)
        return MinresResult(x=xr.cpu().numpy() if host else xr, iterations=0, rel_residual=0.0, converged=True,
                            residual_history=[0.0])
    history = [1.0]

    def _history(itn, explicit=None):
        """[1.0, relres_1, ..., relres_itn] from the device array; at a
        breakdown the last entry is the explicit residual (solvers.py:161-176)."""
        h = [1.0] + [float(v) for v in hist_dev[1:itn + 1].cpu().numpy()]
        if explicit is not None:
            h[-1] = explicit
        return h
    k = 0
    done = False
    # CUDA-graph replay is opt-in: a capture costs 5-10 ms of host time per
    # MINRES call, more than it saves on one 50-iteration solve (measured on C1
    # and the Kershaw sizes); eager launches with a state read every
    # `check_every` iterations are the default
    use_graph = operator is not None and bool(cfg.graph)
    if use_graph and cfg.max_iterations >= 7:
        # one eager iteration (configures the kernels), then 6-iteration graphs
        bufs_r = [r1, r2, spare]
        bufs_w = [w, w1, w2]

        def step(kk):
            _lib.check(lib.tmop_minres_step_op(ctx, _lib.ptr(op_qd.data), n, _lib.ptr(bufs_r[2]),
                                               _lib.ptr(bufs_r[0]), _lib.ptr(bufs_r[1]), _lib.ptr(inv), _lib.ptr(z),
                                               _lib.ptr(v), _lib.ptr(bufs_w[0]), _lib.ptr(bufs_w[1]),
                                               _lib.ptr(bufs_w[2]), _lib.ptr(x), float(cfg.rel_tolerance), stp, kk),
                       "tmop_minres_step_op")
            bufs_r[0], bufs_r[1], bufs_r[2] = bufs_r[1], bufs_r[2], bufs_r[0]
            bufs_w[1], bufs_w[2], bufs_w[0] = bufs_w[2], bufs_w[0], bufs_w[1]

        step(0)
        k = 1
        cur = torch.cuda.current_stream(dev)
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(cur)
        graph = torch.cuda.CUDAGraph()
        _lib.check(lib.tmop_ctx_set_stream(ctx, side.cuda_stream), "tmop_ctx_set_stream")
        try:
            with torch.cuda.graph(graph, stream=side):
                for j in range(6):
                    step(k + j)
        finally:
            _lib.check(lib.tmop_ctx_set_stream(ctx, cur.cuda_stream), "tmop_ctx_set_stream")
        cur.wait_stream(side)
        s_ = state(k)
        done = bool(s_["done"])
        while not done and k + 6 <= cfg.max_iterations:
            graph.replay()
            k += 6
            s_ = state(k)
            done = bool(s_["done"]) or bool(s_["breakdown"])
        r1, r2, spare = bufs_r
        w, w1, w2 = bufs_w
        del graph
        if s_["breakdown"]:
            r = b - (apply_op(x).reshape(-1))
            zz = inv * r if inv is not None else r
            explicit = np.sqrt(max(float(torch.dot(r, zz).item()), 0.0)) / float(s_["beta1"])
            if explicit <= cfg.rel_tolerance:
                return MinresResult(x=x.cpu().numpy() if host else x, iterations=int(s_["itn"]),
                                    rel_residual=explicit, converged=True,
                                    residual_history=_history(int(s_["itn"]), explicit))
            raise MinresBreakdownError(int(s_["itn"]))
    while k < cfg.max_iterations and not done:
        todo = min(cfg.check_every, cfg.max_iterations - k)
        for _ in range(todo):
            if operator is not None:
                _lib.check(lib.tmop_minres_step_op(ctx, _lib.ptr(op_qd.data), n, _lib.ptr(spare), _lib.ptr(r1),
                                                   _lib.ptr(r2), _lib.ptr(inv), _lib.ptr(z), _lib.ptr(v),
                                                   _lib.ptr(w), _lib.ptr(w1), _lib.ptr(w2), _lib.ptr(x),
                                                   float(cfg.rel_tolerance), stp, k), "tmop_minres_step_op")
                r1, r2, spare = r2, spare, r1
                w1, w2, w = w2, w, w1
                k += 1
                continue
            Av = apply_op(v)
            if not type(Av).__module__.startswith("torch"):
                Av = torch.from_numpy(np.ascontiguousarray(Av, dtype=np.float64)).to(dev)
            Av = Av.reshape(-1)
            if not Av.is_contiguous() or Av.data_ptr() in (v.data_ptr(), r1.data_ptr(), r2.data_ptr()):
                Av = Av.contiguous().clone()
            _lib.check(lib.tmop_minres_step(ctx, n, _lib.ptr(Av), _lib.ptr(r1), _lib.ptr(r2), _lib.ptr(inv),
                                            _lib.ptr(z), _lib.ptr(v), _lib.ptr(w), _lib.ptr(w1), _lib.ptr(w2),
                                            _lib.ptr(x), float(cfg.rel_tolerance), stp, k), "tmop_minres_step")
            r1, r2 = r2, Av
            w1, w2, w = w2, w, w1
            k += 1
        s = state(k)
        if s["nonpd"]:
            raise ValueError("preconditioner is not positive definite")
        its = int(s["itn"])
        done = bool(s["done"])
        if s["breakdown"]:
            # Krylov space exhausted: decide on an explicit residual (solvers.py:161-172)
            r = b - (apply_op(x).reshape(-1))
            zz = inv * r if inv is not None else r
            explicit = np.sqrt(max(float(torch.dot(r, zz).item()), 0.0)) / float(s["beta1"])
            if explicit <= cfg.rel_tolerance:
                return MinresResult(x=x.cpu().numpy() if host else x, iterations=its, rel_residual=explicit,
                                    converged=True, residual_history=_history(its, explicit))
            raise MinresBreakdownError(its)
    s = state(k)
    its = int(s["itn"])
    return MinresResult(x=x.cpu().numpy() if host else x, iterations=its, rel_residual=float(s["relres"]),
                        converged=bool(s["done"]) and float(s["relres"]) <= cfg.rel_tolerance,
                        residual_history=_history(its))


class ProblemLike(Protocol):
    def objective(self, x) -> float: ...
    def gradient(self, x): ...
    def hessian_setup(self, x): ...
    def hessian_apply(self, qdata, v): ...
    def hessian_diagonal(self, qdata): ...
    def min_det_jacobian(self, x) -> float: ...


@dataclass
class LineSearchResult:
    alpha: float
    x: object
    objective: float
    grad_norm: float
    min_det: float
    gradient: object


def _norm(ctx, t, scratch) -> float:
    return float(np.sqrt(_dot(ctx, t, t, scratch)))


def line_search(x, dx, problem: ProblemLike, f0: float, grad_norm0: float, max_halvings: int = 30,
                ctx=None) -> LineSearchResult:
    """alpha = 1, 1/2, ... until min det > 0, F < 1.2 F0 and |grad| < 1.2 |grad0|
    (all strict; solvers.py:202-224); update x - alpha dx on the device."""
    torch = _torch()
    xd, host = _dev(x)
    dxd, _ = _dev(dx, xd.device)
    ctx = ctx or _ctx_for(xd.device, problem)
    lib = _lib.load()
    scratch = torch.zeros(1, dtype=torch.float64, device=xd.device)
    fin = torch.zeros(1, dtype=torch.float64, device=xd.device)
    _lib.check(lib.tmop_dot(ctx, dxd.numel(), _lib.ptr(dxd), _lib.ptr(dxd), _lib.ptr(fin)), "tmop_dot")
    if not np.isfinite(float(fin.item())):
        raise LineSearchError("step direction contains non-finite entries")
    alpha = 1.0
    xt = torch.empty_like(xd)
    fused = getattr(problem, "evaluate_trial", None)
    for _ in range(max_halvings + 1):
        _lib.check(lib.tmop_trial_point(ctx, xd.numel(), _lib.ptr(xd), _lib.ptr(dxd), alpha, _lib.ptr(xt)),
                   "tmop_trial_point")
        if fused is not None:
            # one element pass gives min det, F and grad F; same acceptance tests
            md, ft, gt = fused(xt)
            if md > 0.0 and ft < GROWTH_FACTOR * f0:
                gtd, _ = _dev(gt, xd.device)
                ngt = _norm(ctx, gtd, scratch)
                if ngt < GROWTH_FACTOR * grad_norm0:
                    if host:
                        return LineSearchResult(alpha, xt.cpu().numpy(), ft, ngt, md, gtd.cpu().numpy())
                    return LineSearchResult(alpha, xt, ft, ngt, md, gtd)
            alpha *= 0.5
            continue
        md = problem.min_det_jacobian(xt)
        if md > 0.0:
            ft = problem.objective(xt)
            if ft < GROWTH_FACTOR * f0:
                gt = problem.gradient(xt)
                gtd, _ = _dev(gt, xd.device)
                ngt = _norm(ctx, gtd, scratch)
                if ngt < GROWTH_FACTOR * grad_norm0:
                    if host:
                        return LineSearchResult(alpha, xt.cpu().numpy(), ft, ngt, md, gtd.cpu().numpy())
                    return LineSearchResult(alpha, xt, ft, ngt, md, gtd)
        alpha *= 0.5
    raise LineSearchError(f"no acceptable step after {max_halvings} halvings "
                          f"(F0 = {f0:.6e}, |grad F0| = {grad_norm0:.6e})")


@dataclass
class NewtonIterationRecord:
    alpha: float
    objective: float
    grad_norm: float
    minres_iterations: int
    minres_rel_residual: float
    min_det: float


@dataclass
class SolveTrace:
    records: list = field(default_factory=list)

    def append(self, record: NewtonIterationRecord) -> None:
        self.records.append(record)

    @property
    def newton_iterations(self) -> int:
        return len(self.records)

    @property
    def minres_total(self) -> int:
        return sum(r.minres_iterations for r in self.records)


@dataclass
class NewtonResult:
    x: object
    trace: SolveTrace
    success: bool
    rel_grad: float
    initial_grad_norm: float
    message: str = "converged"


def newton_solve(x0, problem: ProblemLike, newton_cfg: NewtonConfig | None = None,
                 minres_cfg: MinresConfig | None = None) -> NewtonResult:
    """Newton + MINRES + line search (solvers.py:263-321), device resident.
    The Hessian quadrature data is rebuilt at every accepted iterate."""
    torch = _torch()
    newton_cfg = newton_cfg or NewtonConfig()
    minres_cfg = minres_cfg or MinresConfig()
    newton_cfg.validate()
    minres_cfg.validate()
    x, host = _dev(x0, getattr(problem, "device", None))
    ctx = _ctx_for(x.device, problem)
    scratch = torch.zeros(1, dtype=torch.float64, device=x.device)

    def ret(xv, trace, ok, rg, g0, msg="converged"):
        return NewtonResult(x=xv.cpu().numpy() if host else xv, trace=trace, success=ok, rel_grad=rg,
                            initial_grad_norm=g0, message=msg)

    md0 = problem.min_det_jacobian(x)
    if md0 <= 0.0:
        raise LineSearchError(f"initial mesh is inverted (min det A = {md0:.3e})")
    trace = SolveTrace()
    g, _ = _dev(problem.gradient(x), x.device)
    ng0 = _norm(ctx, g, scratch)
    if ng0 <= newton_cfg.abs_grad_tolerance:
        return ret(x.clone(), trace, True, 0.0, ng0, "initial gradient is zero")
    x = x.clone()
    f = problem.objective(x)
    ng = ng0
    qdata = None
    for _ in range(newton_cfg.max_iterations):
        qdata = None
        precond = None
        setup_diag = getattr(problem, "hessian_setup_diagonal", None)
        if minres_cfg.preconditioned and setup_diag is not None:
            # setup + diagonal from one element pass (records never re-read)
            qdata, diag = setup_diag(x)
            precond = jacobi_preconditioner(diag, ctx)
        else:
            qdata = problem.hessian_setup(x)
            if minres_cfg.preconditioned:
                precond = jacobi_preconditioner(problem.hessian_diagonal(qdata), ctx)
        fused = (problem, qdata) if getattr(problem, "supports_fused_minres", False) else None
        try:
            mr = minres(lambda v: problem.hessian_apply(qdata, v), g, minres_cfg, precond, ctx, operator=fused)
        except MinresBreakdownError as err:
            return ret(x, trace, False, ng / ng0, ng0, str(err))
        try:
            ls = line_search(x, mr.x, problem, f0=f, grad_norm0=ng,
                             max_halvings=newton_cfg.max_line_search_halvings, ctx=ctx)
        except LineSearchError as err:
            return ret(x, trace, False, ng / ng0, ng0, str(err))
        x, f, ng = ls.x, ls.objective, ls.grad_norm
        g = ls.gradient
        trace.append(NewtonIterationRecord(alpha=ls.alpha, objective=f, grad_norm=ng,
                                           minres_iterations=mr.iterations,
                                           minres_rel_residual=mr.rel_residual, min_det=ls.min_det))
        if ng / ng0 <= newton_cfg.rel_grad_tolerance:
            return ret(x, trace, True, ng / ng0, ng0)
    return ret(x, trace, False, ng / ng0, ng0, f"no convergence in {newton_cfg.max_iterations} iterations")
