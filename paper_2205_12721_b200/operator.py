"""Device TMOP operator: the reference `TmopProblem` API (operator.py:220-459)
backed by the sm_100a kernels of libtmop_b200.so.

Every method accepts numpy arrays or torch tensors.  numpy in -> numpy out
(host buffers, explicit H2D / D2H copies: the drop-in path); torch CUDA in ->
torch CUDA out (device-resident path used by the solvers).  There is no CPU
implementation: without the library or a CUDA device every call raises.
"""

from __future__ import annotations

import os

from dataclasses import dataclass

import numpy as np

from . import _lib
from .fe import Basis1D, OpCounter, build_eval_matrices, gauss_legendre_1d, tensor_weights
from .mesh import Mesh
from .metrics import (MetricId, TargetData, TargetKind, TargetSpec, build_targets, check_metric_dim,
                      is_template_metric)

__all__ = ["InvalidMeshError", "LimitingConfig", "ObjectiveConfig", "HessQData", "TmopProblem",
           "DeviceMesh", "mesh_volume"]


class InvalidMeshError(RuntimeError):
    """Nonpositive Jacobian determinant at a quadrature point (operator.py:45-54)."""

    def __init__(self, element: int, point: int, value: float):
        self.element = element
        self.point = point
        self.value = value
        super().__init__(f"nonpositive det(A) = {value:.3e} in element {element}, quadrature point {point}")


@dataclass
class LimitingConfig:
    """Penalty |x - x0|^2 / delta^2 (operator.py:57-76)."""
    reference: np.ndarray
    delta: float | np.ndarray = 1.0
    weight: float = 1.0

    def validate(self, n_dofs: int) -> None:
        if np.shape(self.reference) != (n_dofs,):
            raise ValueError(f"limiting reference has shape {np.shape(self.reference)}, expected ({n_dofs},)")
        if np.any(np.asarray(self.delta) <= 0):
            raise ValueError("limiting delta must be positive everywhere")
        if self.weight <= 0:
            raise ValueError(f"limiting weight must be positive, got {self.weight}")


@dataclass
class ObjectiveConfig:
    metric: MetricId
    target: TargetSpec
    spatial_weight: float = 1.0
    limiting: LimitingConfig | None = None

    def validate(self) -> None:
        if self.spatial_weight <= 0:
            raise ValueError(f"spatial weight must be positive, got {self.spatial_weight}")


def _torch():
    import torch
    return torch


class DeviceMesh:
    """Mesh arrays resident in HBM: restriction (int32), per-node fixed flags
    (uint8, bit a = component a constrained) and the L->E transpose map
    (int64 offsets, uint32 E-indices e*Np+l sorted by node, then element) that
    makes the E->L sum deterministic in np.add.at order (fe.py:189-204)."""

    def __init__(self, mesh: Mesh, device):
        torch = _torch()
        self.device = device
        self.n_nodes = mesh.n_nodes
        self.n_elements = mesh.n_elements
        restr = torch.from_numpy(np.ascontiguousarray(mesh.restriction, dtype=np.int32)).to(device)
        self.restriction = restr
        # padded to a multiple of 4 bytes: the element kernels fetch the
        # aligned 32-bit word holding fixed[node] (tmop_b200.h, ctx_create)
        flags = np.zeros((mesh.n_nodes + 3) // 4 * 4, dtype=np.uint8)
        for a in range(mesh.dim):
            flags[:mesh.n_nodes] |= (mesh.fixed_mask[a].astype(np.uint8) << a)
        self.fixed = torch.from_numpy(flags).to(device)
        self.fixed_mask = torch.from_numpy(np.ascontiguousarray(mesh.fixed_mask.ravel())).to(device)
        flat = restr.reshape(-1).to(torch.int64)
        order = torch.sort(flat, stable=True).indices   # ascending node, then ascending (e, l)
        counts = torch.bincount(flat, minlength=mesh.n_nodes)
        self.l2e_offsets = torch.zeros(mesh.n_nodes + 1, dtype=torch.int64, device=device)
        self.l2e_offsets[1:] = torch.cumsum(counts, 0)
        # uint32 storage (torch has no uint32 arithmetic needs here; int32 view
        # is reinterpreted by the kernel)
        self.l2e_index = order.to(torch.int32)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


@dataclass
class HessQData:
    """Partially assembled Hessian on the device (operator.py:91-138).

    `data` is the lean element-blocked record (n_elements, stride) float64:
    per point T (d*d), k0, itau = 1/det T (include/tmop_b200.h) -- d^2 + 2
    doubles per point instead of the reference's 4 + 2 d^2.  The reference's
    planar arrays `coeffs`, `s_mat`, `t_mat` and `block(e, q)` are
    materialised on demand by a device kernel (tmop_qdata_to_reference).
    """
    data: object
    dim: int
    n_quad_total: int
    template: bool
    host: bool = False          # built from a numpy x: diagonal() answers in numpy
    _expand: object = None      # callable(data) -> (fields_ref, NQ) device tensor
    _ref: object = None

    @property
    def fields(self) -> int:
        return self.dim * self.dim + 2

    @property
    def nbytes(self) -> int:
        return self.data.numel() * self.data.element_size()

    @property
    def n_elements(self) -> int:
        return self.data.shape[0]

    @property
    def bytes_per_element(self) -> int:
        return self.nbytes // max(self.n_elements, 1)

    @property
    def reference_nbytes(self) -> int:
        """Bytes of the same data in the reference's HessQData format."""
        f = (4 if self.template else 1) + 2 * self.dim * self.dim
        return 8 * f * self.n_quad_total * self.n_elements

    def _planar(self):
        if self._ref is None:
            self._ref = self._expand(self.data).cpu().numpy()
        return self._ref

    @property
    def coeffs(self) -> np.ndarray:
        if not self.template:
            raise AttributeError("mu_302 / mu_321 carry a point weight, not template coefficients")
        return self._planar()[:4]

    @property
    def s_mat(self) -> np.ndarray:
        o, d = (4 if self.template else 1), self.dim
        return self._planar()[o:o + d * d].reshape(d, d, -1)

    @property
    def t_mat(self) -> np.ndarray:
        d = self.dim
        o = (4 if self.template else 1) + d * d
        return self._planar()[o:o + d * d].reshape(d, d, -1)

    def block(self, element: int, point: int) -> np.ndarray:
        """Full (d^2 x d^2) block at (element, point) (operator.py:127-138)."""
        if not self.template:
            raise NotImplementedError("block() reconstruction is defined for template metrics")
        d = self.dim
        k = element * self.n_quad_total + point
        c_id, c_ts, c_ss, c_x = self.coeffs[:, k]
        sv = self.s_mat[:, :, k].ravel()
        tv = self.t_mat[:, :, k].ravel()
        full = c_id * np.eye(d * d)
        full += c_ts * (np.outer(sv, tv) + np.outer(tv, sv))
        full += c_ss * np.outer(sv, sv)
        s = sv.reshape(d, d)
        full += c_x * np.einsum("mp,on->mnop", s, s).reshape(d * d, d * d)
        return full


class TmopProblem:
    """Mesh + objective + quadrature on one GPU; the six `ProblemLike`
    methods (solvers.py:183-189) run as sm_100a kernels.

    `counter` accumulates the reference's multiply-add accounting
    analytically; `batch_quad_points` only sets the element batching used to
    report InvalidMeshError exactly like the reference (operator.py:267-272)
    -- the kernels themselves stream all elements in one launch.
    """

    def __init__(self, mesh: Mesh, config: ObjectiveConfig, n_quad: int,
                 counter: OpCounter | None = None, batch_quad_points: int = 2_000_000,
                 device=None):
        torch = _torch()
        config.validate()
        check_metric_dim(config.metric, mesh.dim)
        if not torch.cuda.is_available():
            raise _lib.TmopLibraryError("TmopProblem needs a CUDA device (sm_100a); none is available")
        self.lib = _lib.load()
        self.mesh = mesh
        self.config = config
        self.basis = Basis1D.gauss_lobatto(mesh.order)
        self.rule = gauss_legendre_1d(n_quad)
        self.em = build_eval_matrices(self.basis, self.rule)
        self.wq = tensor_weights(self.rule, mesh.dim)
        self.counter = counter
        d = mesh.dim
        self.n_quad = n_quad
        self.n_quad_total = n_quad ** d
        self._qshape = (n_quad,) * d
        self.batch_elements = max(1, batch_quad_points // self.n_quad_total)
        if config.limiting is not None:
            config.limiting.validate(mesh.n_dofs)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.dmesh = DeviceMesh(mesh, self.device)
        self._stream = None
        ctx = _lib.C.c_void_p()
        B = np.ascontiguousarray(self.em.b, dtype=np.float64)
        G = np.ascontiguousarray(self.em.g, dtype=np.float64)
        w1 = np.ascontiguousarray(self.rule.weights, dtype=np.float64)
        dp = _lib.C.POINTER(_lib.C.c_double)
        stream = torch.cuda.current_stream(self.device)
        _lib.check(self.lib.tmop_ctx_create(
            _lib.C.byref(ctx), d, mesh.order, n_quad, mesh.n_elements, mesh.n_nodes,
            _lib.ptr(self.dmesh.restriction), _lib.ptr(self.dmesh.fixed), _lib.ptr(self.dmesh.l2e_offsets),
            _lib.ptr(self.dmesh.l2e_index), B.ctypes.data_as(dp), G.ctypes.data_as(dp), w1.ctypes.data_as(dp),
            int(config.metric), 1.0, 1.0, float(config.spatial_weight), stream.cuda_stream), "tmop_ctx_create")
        self._ctx = ctx
        self._stream = stream.cuda_stream
        self._status = torch.zeros(2, dtype=torch.float64, device=self.device)
        self._scalar = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.template = is_template_metric(config.metric)
        self.qdata_fields = self.lib.tmop_qdata_fields(ctx)
        self.qdata_stride = int(self.lib.tmop_qdata_stride(ctx))
        if config.target.kind == TargetKind.SIZE_FIELD:
            self.targets = build_targets(mesh, config.target, self.rule)
            self._set_size_field(config.target.size)
        elif config.target.kind != 0 and config.target.h is None:
            vol = self.volume(mesh.coords.ravel())
            self.targets: TargetData = build_targets(mesh, config.target, self.rule, volume=vol)
        else:
            self.targets = build_targets(mesh, config.target, self.rule)
        if config.target.kind != TargetKind.SIZE_FIELD:
            _lib.check(self.lib.tmop_ctx_set_target(ctx, self.targets.inv_scale, self.targets.det_w),
                       "tmop_ctx_set_target")
        self._lim = None
        if config.limiting is not None:
            # device copies owned here; the context keeps the pointers (operator.py:463-486)
            lim = config.limiting
            x0 = torch.from_numpy(np.ascontiguousarray(lim.reference, dtype=np.float64)).to(self.device)
            dn = None
            if np.ndim(lim.delta) != 0:
                dn = torch.from_numpy(np.ascontiguousarray(lim.delta, dtype=np.float64).reshape(-1)).to(self.device)
                if dn.numel() != mesh.n_nodes:
                    raise ValueError(f"nodal limiting delta needs {mesh.n_nodes} values, got {dn.numel()}")
            self._lim = (x0, dn)
            _lib.check(self.lib.tmop_ctx_set_limiting(
                ctx, _lib.ptr(x0), _lib.ptr(dn) if dn is not None else None,
                float(lim.delta) if dn is None else 0.0, float(lim.weight)), "tmop_ctx_set_limiting")
        # box lattices (build_box / Kershaw): verified on the device, then the
        # E->L gathers enumerate node copies arithmetically
        acc = _lib.C.c_int(0)
        if d == 3 and getattr(mesh, "element_counts", None) is not None and os.environ.get("TMOP_LATTICE", "1") != "0":
            nx, ny, nz = (int(c) for c in mesh.element_counts)
            _lib.check(self.lib.tmop_ctx_set_lattice(ctx, nx, ny, nz, _lib.C.byref(acc)), "tmop_ctx_set_lattice")
        self.lattice = bool(acc.value)

    def _set_size_field(self, size):
        """Size-field targets (TargetKind.SIZE_FIELD, an extension): upload
        the nodal target volume, compute the per-point 1/s_q on the device."""
        torch = _torch()
        if size is None:
            raise ValueError("TargetKind.SIZE_FIELD needs TargetSpec.size (nodal target volume)")
        eta = torch.as_tensor(np.ascontiguousarray(size, dtype=np.float64) if not _is_torch(size) else size,
                              dtype=torch.float64).reshape(-1).to(self.device)
        if eta.numel() != self.mesh.n_nodes:
            raise ValueError(f"size field needs {self.mesh.n_nodes} nodal values, got {eta.numel()}")
        self._size = eta
        self._sync_stream()
        _lib.check(self.lib.tmop_ctx_set_size_field(self._ctx, _lib.ptr(eta)), "tmop_ctx_set_size_field")
        n = self.mesh.n_elements * self.n_quad_total
        ptr = self.lib.tmop_ctx_point_scale(self._ctx)
        ts = torch.zeros(n, dtype=torch.float64, device=self.device)
        _lib.check(self.lib.tmop_axpby(self._ctx, n, 1.0, ptr, 0.0, _lib.ptr(ts)), "tmop_axpby")
        if not bool(torch.isfinite(ts).all()):
            raise ValueError("size field: the interpolated target volume is not positive at some quadrature point")
        self.point_inv_scale = ts

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx is not None and getattr(self, "lib", None) is not None:
            self.lib.tmop_ctx_destroy(ctx)
            self._ctx = None

    # ------------------------------------------------------------ helpers
    @property
    def n_dofs(self) -> int:
        return self.mesh.n_dofs

    def _sync_stream(self):
        torch = _torch()
        s = torch.cuda.current_stream(self.device).cuda_stream
        if s != self._stream:
            _lib.check(self.lib.tmop_ctx_set_stream(self._ctx, s), "tmop_ctx_set_stream")
            self._stream = s

    def _in(self, x):
        """(device float64 contiguous tensor, origin) with origin False for a
        device tensor, "numpy" for numpy input and "torch" for a host torch
        tensor (pinned host tensors are copied asynchronously)."""
        torch = _torch()
        if _is_torch(x):
            t = x.detach()
            origin = False if t.is_cuda else "torch"
            if t.device != self.device or t.dtype != torch.float64:
                t = t.to(device=self.device, dtype=torch.float64, non_blocking=True)
            t = t.reshape(-1).contiguous()
        else:
            t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64).reshape(-1)).to(self.device)
            origin = "numpy"
        if t.numel() != self.mesh.n_dofs:
            raise ValueError(f"expected a T-vector of length {self.mesh.n_dofs}, got {t.numel()}")
        self._sync_stream()
        return t, origin

    def _out(self, t, origin, out=None):
        """Return the device result `t` in the caller's currency.  A host torch
        `out` (ideally pinned) receives an asynchronous D2H copy."""
        torch = _torch()
        if out is not None and not out.is_cuda:
            out.view(-1).copy_(t, non_blocking=True)
            torch.cuda.current_stream(self.device).synchronize()
            return out
        if not origin:
            return t
        if origin == "numpy":
            return t.cpu().numpy()
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return h

    @staticmethod
    def _dev_out(out, like):
        torch = _torch()
        return out if (out is not None and out.is_cuda) else torch.empty_like(like)

    def _det(self):
        st = self._status.cpu().numpy()
        return float(st[0]), int(st[1:2].view(np.int64)[0])

    def _raise_if_inverted(self, x, min_det):
        if min_det > 0.0:
            return
        # exact emulation of the reference's batched check (operator.py:267-272)
        torch = _torch()
        ne = self.mesh.n_elements
        emin = torch.empty(ne, dtype=torch.float64, device=self.device)
        earg = torch.empty(ne, dtype=torch.int32, device=self.device)
        _lib.check(self.lib.tmop_element_min_det(self._ctx, _lib.ptr(x), _lib.ptr(emin), _lib.ptr(earg)),
                   "tmop_element_min_det")
        em = emin.cpu().numpy()
        ea = earg.cpu().numpy()
        for lo in range(0, ne, self.batch_elements):
            hi = min(lo + self.batch_elements, ne)
            k = int(np.argmin(em[lo:hi]))
            if em[lo + k] <= 0.0:
                raise InvalidMeshError(lo + k, int(ea[lo + k]), float(em[lo + k]))
        raise InvalidMeshError(0, 0, min_det)

    def _count(self, kind: str) -> None:
        if self.counter is None:
            return
        d, n, q = self.mesh.dim, self.mesh.order + 1, self.n_quad
        ne, Q = self.mesh.n_elements, self.n_quad_total
        per_dir = sum(q ** k * n ** (d + 1 - k) for k in range(1, d + 1))
        contr = d * d * per_dir * ne          # one d x d set of d-axis contractions
        if kind == "apply":
            self.counter.add(2 * contr + ne * Q * (6 * d * d + 2 * d ** 3))
        elif kind in ("gradient",):
            self.counter.add(2 * contr)
        elif kind in ("setup", "objective", "min_det"):
            self.counter.add(contr)

    # ----------------------------------------------------------- ProblemLike
    def volume(self, x) -> float:
        xt, _ = self._in(x)
        _lib.check(self.lib.tmop_volume(self._ctx, _lib.ptr(xt), _lib.ptr(self._scalar)), "tmop_volume")
        return float(self._scalar.item())

    def min_det_jacobian(self, x) -> float:
        xt, _ = self._in(x)
        _lib.check(self.lib.tmop_min_det(self._ctx, _lib.ptr(xt), _lib.ptr(self._status)), "tmop_min_det")
        self._count("min_det")
        return self._det()[0]

    def objective(self, x) -> float:
        """F(x); raises InvalidMeshError at the first nonpositive det(A)."""
        xt, _ = self._in(x)
        _lib.check(self.lib.tmop_objective(self._ctx, _lib.ptr(xt), _lib.ptr(self._scalar),
                                           _lib.ptr(self._status)), "tmop_objective")
        self._count("objective")
        md, _ = self._det()
        self._raise_if_inverted(xt, md)
        return float(self._scalar.item())

    def gradient(self, x, out=None):
        torch = _torch()
        xt, host = self._in(x)
        g = self._dev_out(out, xt)
        _lib.check(self.lib.tmop_gradient(self._ctx, _lib.ptr(xt), _lib.ptr(g), _lib.ptr(self._status)),
                   "tmop_gradient")
        self._count("gradient")
        md, _ = self._det()
        self._raise_if_inverted(xt, md)
        return self._out(g, host, out)

    def evaluate_trial(self, x):
        """(min det A, F, grad F) at a line-search trial point from ONE element
        pass (tmop_gradient_energy) instead of three (solvers.py:210-216).
        F and grad F are None when the mesh is inverted there -- the
        reference evaluates neither in that case -- so nothing is raised."""
        torch = _torch()
        xt, host = self._in(x)
        g = torch.empty_like(xt)
        _lib.check(self.lib.tmop_gradient_energy(self._ctx, _lib.ptr(xt), _lib.ptr(g), _lib.ptr(self._scalar),
                                                 _lib.ptr(self._status)), "tmop_gradient_energy")
        self._count("gradient")
        md, _ = self._det()
        if not md > 0.0:
            return md, None, None
        return md, float(self._scalar.item()), self._out(g, host)

    def hessian_setup(self, x) -> HessQData:
        torch = _torch()
        xt, host = self._in(x)
        qd = torch.empty((self.mesh.n_elements, self.qdata_stride), dtype=torch.float64, device=self.device)
        _lib.check(self.lib.tmop_hessian_setup(self._ctx, _lib.ptr(xt), _lib.ptr(qd), _lib.ptr(self._status)),
                   "tmop_hessian_setup")
        self._count("setup")
        md, _ = self._det()
        self._raise_if_inverted(xt, md)
        return HessQData(data=qd, dim=self.mesh.dim, n_quad_total=self.n_quad_total, template=self.template,
                         host=host, _expand=self._expand_qdata)

    def hessian_setup_diagonal(self, x):
        """hessian_setup(x) and hessian_diagonal of the result from one element
        pass (tmop_hessian_setup_diagonal; 3D p <= 3, template metrics);
        returns (qdata, diagonal).  newton_solve uses it when the Jacobi
        preconditioner is on (solvers.py:292-295)."""
        torch = _torch()
        xt, host = self._in(x)
        qd = torch.empty((self.mesh.n_elements, self.qdata_stride), dtype=torch.float64, device=self.device)
        d = torch.empty_like(xt)
        _lib.check(self.lib.tmop_hessian_setup_diagonal(self._ctx, _lib.ptr(xt), _lib.ptr(qd), _lib.ptr(d),
                                                        _lib.ptr(self._status)), "tmop_hessian_setup_diagonal")
        self._count("setup")
        md, _ = self._det()
        self._raise_if_inverted(xt, md)
        qdata = HessQData(data=qd, dim=self.mesh.dim, n_quad_total=self.n_quad_total, template=self.template,
                          host=host, _expand=self._expand_qdata)
        return qdata, self._out(d, host)

    def _expand_qdata(self, data):
        torch = _torch()
        nf = self.lib.tmop_qdata_reference_fields(self._ctx)
        out = torch.empty((nf, self.mesh.n_elements * self.n_quad_total), dtype=torch.float64, device=self.device)
        self._sync_stream()
        _lib.check(self.lib.tmop_qdata_to_reference(self._ctx, _lib.ptr(data), _lib.ptr(out)),
                   "tmop_qdata_to_reference")
        return out

    def hessian_apply(self, qdata: HessQData, v, out=None):
        """Action of the Hessian frozen at the setup positions; constrained
        inputs are treated as zero, constrained outputs return v
        (operator.py:401-418)."""
        torch = _torch()
        if (self.lattice and _is_torch(v) and not v.is_cuda and v.is_pinned() and v.dtype == torch.float64
                and v.is_contiguous() and v.numel() == self.mesh.n_dofs
                and (out is None or (not out.is_cuda and out.is_contiguous() and out.dtype == torch.float64))
                and self.pipeline_slabs > 1 and self._lim is None):
            return self._apply_host_pipelined(qdata, v, out)
        vt, host = self._in(v)
        y = self._dev_out(out, vt)
        _lib.check(self.lib.tmop_hessian_apply(self._ctx, _lib.ptr(qdata.data), _lib.ptr(vt), _lib.ptr(y)),
                   "tmop_hessian_apply")
        self._count("apply")
        return self._out(y, host, out)

    def hessian_apply_boundary_first(self, qdata: HessQData, v, on_planes):
        """Hessian action of a z-slab for the multi-GPU path:
        the first and last element layers and the two outer node planes are
        computed first, then `on_planes(y)` is called (the caller starts the
        halo exchange of those planes, which then overlaps the rest), then
        the interior elements and nodes.  Returns (y, on_planes' result);
        y is bitwise the one-shot hessian_apply.  Device tensors, box
        lattices without the limiting term; otherwise the one-shot apply."""
        torch = _torch()
        m = self.mesh
        if not (self.lattice and _is_torch(v) and v.is_cuda and self._lim is None and m.dim == 3):
            y = self.hessian_apply(qdata, v)
            return y, on_planes(y)
        nx, ny, _ = m.element_counts
        p = m.order
        layer, ne, nn = nx * ny, m.n_elements, m.n_nodes
        plane = (nx * p + 1) * (ny * p + 1)
        vt, _ = self._in(v)
        y = torch.empty_like(vt)
        self._sync_stream()
        a1 = min(ne, -(-layer // 16) * 16)              # range starts stay multiples of 16
        b0 = max(a1, (ne - layer) // 16 * 16)
        ctx, qp, vp = self._ctx, _lib.ptr(qdata.data), _lib.ptr(vt)
        self.last_launches = 0

        def elems(e0, e1):
            if e1 > e0:
                _lib.check(self.lib.tmop_hessian_apply_elements_range(ctx, qp, vp, e0, e1),
                           "tmop_hessian_apply_elements_range")
                self.last_launches += 1

        def nodes(n0, n1):
            if n1 > n0:
                _lib.check(self.lib.tmop_hessian_apply_gather_range(ctx, vp, _lib.ptr(y), n0, n1),
                           "tmop_hessian_apply_gather_range")
                self.last_launches += 1

        elems(0, a1)
        elems(b0, ne)
        nodes(0, min(plane, nn))
        nodes(max(plane, nn - plane), nn)
        handle = on_planes(y)
        # interior: element slabs on the caller's stream, the E->L sum of the
        # node layers each slab completes on a second stream behind it
        main = torch.cuda.current_stream(self.device)
        aux = getattr(self, "_aux", None)
        if aux is None:
            aux = self._aux = torch.cuda.Stream(self.device)
        ns = max(1, min(self.pipeline_slabs // 2, (b0 - a1) // max(layer, 1)))
        zs = [a1 + ((b0 - a1) * k // ns) // layer * layer for k in range(ns)] + [b0]
        cuts = sorted(set([a1] + [z // 16 * 16 for z in zs[1:-1] if a1 < z // 16 * 16 < b0] + [b0]))
        done, top = plane, max(plane, nn - plane)
        for k in range(len(cuts) - 1):
            elems(cuts[k], cuts[k + 1])
            fin = top if k == len(cuts) - 2 else min(top, (cuts[k + 1] // layer) * p * plane)
            if fin > done:
                aux.wait_stream(main)
                with torch.cuda.stream(aux):
                    self._sync_stream()
                    nodes(done, fin)
                self._sync_stream()
                done = fin
        main.wait_stream(aux)
        y.record_stream(aux)
        nodes(done, top)   # (no interior slab: the remaining node layers, all elements done)
        self._count("apply")
        return y, handle

    # Host-resident Hessian action, pipelined slab by slab over z-layers of
    # the box lattice: the H2D copy of slab k+1's new node planes, the element
    # kernel + E->L of slab k and the D2H copy of the finished node planes of
    # slab k-1 run on three streams (PCIe is full duplex), so the end-to-end
    # time approaches max(H2D, D2H, compute) instead of their sum.  Bitwise
    # identical to the one-shot apply.
    pipeline_slabs = int(os.environ.get("TMOP_PIPE_SLABS", "16"))
    pipeline_ramp = os.environ.get("TMOP_PIPE_RAMP", "1") != "0"

    def _apply_host_pipelined(self, qdata: HessQData, vh, out):
        torch = _torch()
        m = self.mesh
        nx, ny, nz = m.element_counts
        p = m.order
        NX, NY = nx * p + 1, ny * p + 1
        nn, ne, layer = m.n_nodes, m.n_elements, nx * ny
        if out is None:
            out = torch.empty(m.n_dofs, dtype=torch.float64, pin_memory=True)
        pipe = getattr(self, "_pipe", None)
        if pipe is None:
            pipe = self._pipe = (torch.cuda.Stream(self.device), torch.cuda.Stream(self.device),
                                 torch.cuda.Stream(self.device))
        h2d, comp, d2h = pipe
        caller = torch.cuda.current_stream(self.device)
        vt = torch.empty(m.n_dofs, dtype=torch.float64, device=self.device)
        y = torch.empty_like(vt)
        for s_ in pipe:
            s_.wait_stream(caller)

        def node_lo(e):
            ex, ey, ez = e % nx, (e // nx) % ny, e // layer
            return ex * p + NX * (ey * p + NY * ez * p)

        def node_hi(e):   # last node of element e, + 1
            ex, ey, ez = e % nx, (e // nx) % ny, e // layer
            return (ex * p + p) + NX * ((ey * p + p) + NY * (ez * p + p)) + 1

        # slab sizes ramp up and down (1/4, 1/2, 1, ..., 1, 1/2, 1/4): the
        # first H2D and the last D2H are not overlapped, so they are kept short
        ns = min(self.pipeline_slabs, nz)
        w = [1.0] * ns
        if self.pipeline_ramp and ns >= 8:
            w[0] = w[-1] = 0.25
            w[1] = w[-2] = 0.5
        cum = np.concatenate([[0.0], np.cumsum(w)]) / sum(w)
        zs = sorted(set(int(round(c * nz)) for c in cum[:-1]))
        # several ramp points can round to the same z layer (nz < ~4 ns): the
        # set() above drops them, so walk the bounds actually produced
        bounds = [z * layer // 16 * 16 for z in zs] + [ne]
        copied, done = 0, 0
        for k in range(len(bounds) - 1):
            e0, e1 = bounds[k], bounds[k + 1]
            if e1 <= e0:
                continue
            hi = node_hi(e1 - 1)
            with torch.cuda.stream(h2d):
                if hi > copied:
                    self._sync_stream()
                    _lib.check(self.lib.tmop_copy_components(self._ctx, _lib.ptr(vt), _lib.ptr(vh), nn, copied,
                                                             hi - copied, 3), "tmop_copy_components")
                    copied = hi
            comp.wait_stream(h2d)
            fin = nn if e1 == ne else (e1 // layer) * p * NX * NY
            with torch.cuda.stream(comp):
                self._sync_stream()
                _lib.check(self.lib.tmop_hessian_apply_elements_range(
                    self._ctx, _lib.ptr(qdata.data), _lib.ptr(vt), e0, e1), "tmop_hessian_apply_elements_range")
                if fin > done:
                    _lib.check(self.lib.tmop_hessian_apply_gather_range(
                        self._ctx, _lib.ptr(vt), _lib.ptr(y), done, fin), "tmop_hessian_apply_gather_range")
            d2h.wait_stream(comp)
            if fin > done:
                with torch.cuda.stream(d2h):
                    self._sync_stream()
                    _lib.check(self.lib.tmop_copy_components(self._ctx, _lib.ptr(out), _lib.ptr(y), nn, done,
                                                             fin - done, 3), "tmop_copy_components")
                done = fin
        d2h.synchronize()
        vt.record_stream(comp)
        y.record_stream(d2h)
        self._count("apply")
        return out

    def hessian_diagonal(self, qdata: HessQData, out=None):
        torch = _torch()
        self._sync_stream()
        y = torch.empty(self.mesh.n_dofs, dtype=torch.float64, device=self.device) if out is None else out
        _lib.check(self.lib.tmop_hessian_diagonal(self._ctx, _lib.ptr(qdata.data), _lib.ptr(y)),
                   "tmop_hessian_diagonal")
        return self._out(y, qdata.host)

    # ------------------------------------------------ limiting term alone
    def _need_lim(self):
        if self._lim is None:
            raise ValueError("the objective has no limiting term (ObjectiveConfig.limiting is None)")

    def limiting_value(self, x) -> float:
        """1/2 sum_q c_q |B(x - x0)|^2 (operator.py:488-495)."""
        self._need_lim()
        xt, _ = self._in(x)
        _lib.check(self.lib.tmop_limiting_value(self._ctx, _lib.ptr(xt), _lib.ptr(self._scalar)), "tmop_limiting_value")
        return float(self._scalar.item())

    def limiting_gradient(self, x):
        """B^T (c_q B(x - x0)), no constraint handling (operator.py:497-512)."""
        self._need_lim()
        xt, host = self._in(x)
        y = _torch().empty_like(xt)
        _lib.check(self.lib.tmop_limiting_gradient(self._ctx, _lib.ptr(xt), _lib.ptr(y)), "tmop_limiting_gradient")
        return self._out(y, host)

    def limiting_hessian_apply(self, v):
        """B^T (c_q B v), no constraint handling (operator.py:514-533)."""
        self._need_lim()
        vt, host = self._in(v)
        y = _torch().empty_like(vt)
        _lib.check(self.lib.tmop_limiting_apply(self._ctx, _lib.ptr(vt), _lib.ptr(y)), "tmop_limiting_apply")
        return self._out(y, host)

    def set_apply_overlap(self, slabs: int, min_elements: int = 0) -> None:
        """Slab-overlapped action on lattices (tmop_ctx_set_apply_overlap):
        `slabs` z-slabs (1 = one-shot) for meshes of >= min_elements."""
        _lib.check(self.lib.tmop_ctx_set_apply_overlap(self._ctx, int(slabs), int(min_elements)),
                   "tmop_ctx_set_apply_overlap")

    # ---------------------------------------------------------- raw C-ABI
    @property
    def ctx(self):
        return self._ctx

    # newton_solve may run MINRES iterations as single fused library calls
    supports_fused_minres = True


def mesh_volume(mesh: Mesh, rule, coords=None) -> float:
    """Quadrature volume of the mesh image (metrics.py:319-330), on the GPU."""
    from .metrics import MetricId, TargetKind, TargetSpec
    metric = MetricId.MU_2 if mesh.dim == 2 else MetricId.MU_303
    p = TmopProblem(mesh, ObjectiveConfig(metric, TargetSpec(TargetKind.IDEAL_UNIT)), rule.n_points)
    x = mesh.coords.ravel() if coords is None else np.asarray(coords, dtype=float).ravel()
    return p.volume(x)
