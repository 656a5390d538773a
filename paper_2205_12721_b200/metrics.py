"""Metric ids, pointwise metric evaluation (on the GPU) and target
construction.  API mirrors metrics.py of the reference (metrics.py:41-345).

Template metrics share the Hessian skeleton (metrics.py:7-13)

    c_id I + c_ts (S (x) T + T (x) S) + c_ss S (x) S + c_x S_mp S_on,  S = T^{-T}.

mu_2, mu_55, mu_303 follow the reference; mu_7 (2D) fits the
same template; mu_302 and mu_321 (3D, MFEM numbering) do not and have
their own Hessian action.  Pointwise evaluation runs
in the library's `tmop_metric_eval` kernel -- there is no CPU path.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum

import numpy as np

__all__ = ["MetricId", "MetricEval", "TargetKind", "TargetSpec", "TargetData", "metric_dim",
           "check_metric_dim", "metric_value", "metric_first_derivative", "metric_second_derivative",
           "evaluate", "build_targets", "is_template_metric"]


class MetricId(IntEnum):
    MU_2 = 2        # 2D shape            (metrics.py:42)
    MU_7 = 7        # 2D shape, |T - T^{-t}|^2        [extension]
    MU_55 = 55      # size, 2D and 3D     (metrics.py:43)
    MU_302 = 302    # 3D shape, |T|^2 |T^{-1}|^2 / 9 - 1             [extension]
    MU_303 = 303    # 3D shape            (metrics.py:44)
    MU_321 = 321    # 3D shape+size, |T|^2 + |T^{-1}|^2 - 6         [extension]


_DIM = {MetricId.MU_2: 2, MetricId.MU_7: 2, MetricId.MU_55: None, MetricId.MU_302: 3,
        MetricId.MU_303: 3, MetricId.MU_321: 3}


def metric_dim(metric) -> int | None:
    return _DIM[MetricId(metric)]


def check_metric_dim(metric, dim: int) -> None:
    need = metric_dim(metric)
    if need is not None and need != dim:
        raise ValueError(f"{MetricId(metric).name} requires dim={need}, got dim={dim}")


def is_template_metric(metric) -> bool:
    return MetricId(metric) in (MetricId.MU_2, MetricId.MU_7, MetricId.MU_55, MetricId.MU_303)


def _eval(metric, t, want):
    import torch

    from . import _lib
    t = np.asarray(t, dtype=float)
    if t.ndim < 2 or t.shape[-1] != t.shape[-2] or t.shape[-1] not in (2, 3):
        raise ValueError(f"expected (..., d, d) with d in (2, 3), got shape {t.shape}")
    d = t.shape[-1]
    check_metric_dim(metric, d)
    batch = t.shape[:-2]
    flat = t.reshape(-1, d, d)
    if np.any(np.linalg.det(flat) <= 0.0):
        raise ValueError("metric evaluated at a matrix with nonpositive determinant")
    if not torch.cuda.is_available():
        raise _lib.TmopLibraryError("metric evaluation runs on the GPU; no CUDA device is available")
    n = flat.shape[0]
    dev = torch.device("cuda", torch.cuda.current_device())
    T = torch.from_numpy(np.ascontiguousarray(flat)).to(dev)
    mu = torch.empty(n, dtype=torch.float64, device=dev) if "mu" in want else None
    P = torch.empty((n, d, d), dtype=torch.float64, device=dev) if "P" in want else None
    H = torch.empty((n, d * d, d * d), dtype=torch.float64, device=dev) if "H" in want else None
    lib = _lib.load()
    _lib.check(lib.tmop_metric_eval(int(metric), d, n, _lib.ptr(T), _lib.ptr(mu), _lib.ptr(P), _lib.ptr(H)),
               "tmop_metric_eval")
    out = {}
    if mu is not None:
        m = mu.cpu().numpy().reshape(batch)
        out["mu"] = float(m) if m.ndim == 0 else m
    if P is not None:
        out["P"] = P.cpu().numpy().reshape(batch + (d, d))
    if H is not None:
        out["H"] = H.cpu().numpy().reshape(batch + (d * d, d * d))
    return out


def metric_value(metric, t):
    return _eval(metric, t, ("mu",))["mu"]


def metric_first_derivative(metric, t) -> np.ndarray:
    return _eval(metric, t, ("P",))["P"]


def metric_second_derivative(metric, t) -> np.ndarray:
    """Hessian (..., d*d, d*d), row m*d+n, column o*d+p (metrics.py:240-262)."""
    return _eval(metric, t, ("H",))["H"]


@dataclass(frozen=True)
class MetricEval:
    value: float
    first: np.ndarray
    second: np.ndarray


def evaluate(metric, t) -> MetricEval:
    t = np.asarray(t, dtype=float)
    if t.ndim != 2:
        raise ValueError("evaluate() takes a single (d, d) matrix")
    r = _eval(metric, t, ("mu", "P", "H"))
    return MetricEval(value=float(r["mu"]), first=r["P"], second=r["H"])


class TargetKind(IntEnum):
    IDEAL_UNIT = 0
    IDEAL_EQUAL_SIZE = 1
    # EXTENSION (BASELINE configs[4], "size-adaptive targets"; the reference
    # has constant isotropic W only, metrics.py:282-345): W(x_q) = v_q^(1/d) I
    # with v_q the nodal target volume field TargetSpec.size interpolated to
    # the quadrature points (material field: fixed per point while x moves)
    SIZE_FIELD = 2


@dataclass(frozen=True)
class TargetSpec:
    kind: TargetKind
    h: float | None = None
    size: object = None     # SIZE_FIELD: nodal target element volume (n_nodes,)


@dataclass(frozen=True)
class TargetData:
    """Constant isotropic target W = scale * I (metrics.py:293-316)."""
    dim: int
    scale: float

    @property
    def det_w(self) -> float:
        return self.scale ** self.dim

    @property
    def inv_scale(self) -> float:
        return 1.0 / self.scale

    def w_matrix(self) -> np.ndarray:
        return self.scale * np.eye(self.dim)

    def w_inv_matrix(self) -> np.ndarray:
        return self.inv_scale * np.eye(self.dim)


def build_targets(mesh, spec: TargetSpec, rule, volume: float | None = None) -> TargetData:
    """W = I, or W = h I with h = (vol / Ne)^(1/d) from the quadrature volume
    of the mesh (metrics.py:333-345); the volume is integrated on the GPU."""
    if spec.kind is TargetKind.IDEAL_UNIT or spec.kind is TargetKind.SIZE_FIELD:
        # SIZE_FIELD: the per-point scales live on the device (tmop_ctx_set_size_field)
        return TargetData(dim=mesh.dim, scale=1.0)
    if spec.h is not None:
        if spec.h <= 0:
            raise ValueError(f"target size h must be positive, got {spec.h}")
        return TargetData(dim=mesh.dim, scale=float(spec.h))
    if volume is None:
        from .operator import mesh_volume
        volume = mesh_volume(mesh, rule)
    if volume <= 0:
        raise ValueError(f"mesh volume must be positive, got {volume}")
    return TargetData(dim=mesh.dim, scale=(volume / mesh.n_elements) ** (1.0 / mesh.dim))


def size_field(mesh, kind: str = "shell", amplitude: float = 0.5, n_elements: int | None = None):
    """Synthetic nodal target-volume fields for the size-adaptive runs
    (BASELINE configs[4]): the uniform element volume 1/Ne of the unit box
    modulated by 1 + a*f(x) with mean(f) ~ 0, so the total target volume
    stays near the box volume (the boundary nodes only slide tangentially).
      shell: f = cos(2 pi r / r0) of the distance to the box centre (a
             refined spherical shell, the usual adaptivity demo);
      sine:  f = prod_k sin(2 pi x_k).
    n_elements: the GLOBAL element count when `mesh` is one slab of a
    partition (the field is a function of position only)."""
    x = np.asarray(mesh.coords, dtype=float)
    base = 1.0 / (n_elements or mesh.n_elements)
    if kind == "shell":
        r = np.sqrt(((x - 0.5) ** 2).sum(axis=0))
        f = np.cos(2.0 * np.pi * r / 0.35)
    elif kind == "sine":
        f = np.prod(np.sin(2.0 * np.pi * x), axis=0)
    else:
        raise ValueError(f"unknown size field {kind!r}")
    return base * (1.0 + amplitude * f)
