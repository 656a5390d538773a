"""ctypes binding of libtmop_b200.so (C ABI declared in include/tmop_b200.h).

The product path has no fallback: if the shared library is missing or no
CUDA device is present, every operator call raises.  Build the library with
`python -m paper_2205_12721_b200.build` (or `__graft_entry__.build()`).
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TMOP_LIB", os.path.join(_HERE, "libtmop_b200.so"))

TMOP_OK = 0


class TmopLibraryError(RuntimeError):
    """The native library is missing or a C-ABI call failed."""


class DetStatus(C.Structure):
    _fields_ = [("min_det", C.c_double), ("argmin", C.c_int64)]


class MinresState(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("beta1", "beta", "oldb", "alfa", "beta2", "dbar", "epsln", "sn",
                                            "cs", "phibar", "relres", "gamma")] + \
               [(n, C.c_int32) for n in ("itn", "done", "breakdown", "nonpd")]


MINRES_STATE_BYTES = C.sizeof(MinresState)
DET_STATUS_BYTES = C.sizeof(DetStatus)

_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double
_INT = C.c_int

_SIGS = {
    "tmop_ctx_create": [C.POINTER(_P), _INT, _INT, _INT, _I64, _I64, _P, _P, _P, _P,
                        C.POINTER(_D), C.POINTER(_D), C.POINTER(_D), _INT, _D, _D, _D, _P],
    "tmop_ctx_destroy": [_P],
    "tmop_ctx_set_stream": [_P, _P],
    "tmop_ctx_set_apply_overlap": [_P, _INT, _I64],
    "tmop_ctx_set_target": [_P, _D, _D],
    "tmop_ctx_set_size_field": [_P, _P],
    "tmop_ctx_point_scale": [_P],
    "tmop_ctx_set_lattice": [_P, _INT, _INT, _INT, _P],
    "tmop_hessian_apply_elements_range": [_P, _P, _P, _I64, _I64],
    "tmop_hessian_apply_gather_range": [_P, _P, _P, _I64, _I64],
    "tmop_qdata_fields": [_P],
    "tmop_qdata_stride": [_P],
    "tmop_qdata_size": [_P],
    "tmop_qdata_reference_fields": [_P],
    "tmop_qdata_to_reference": [_P, _P, _P],
    "tmop_ctx_set_limiting": [_P, _P, _P, _D, _D],
    "tmop_limiting_value": [_P, _P, _P],
    "tmop_limiting_gradient": [_P, _P, _P],
    "tmop_limiting_apply": [_P, _P, _P],
    "tmop_hessian_setup": [_P, _P, _P, _P],
    "tmop_hessian_setup_diagonal": [_P, _P, _P, _P, _P],
    "tmop_hessian_apply": [_P, _P, _P, _P],
    "tmop_hessian_apply_elements": [_P, _P, _P],
    "tmop_hessian_apply_gather": [_P, _P, _P],
    "tmop_hessian_diagonal": [_P, _P, _P],
    "tmop_gradient": [_P, _P, _P, _P],
    "tmop_gradient_energy": [_P, _P, _P, _P, _P],
    "tmop_objective": [_P, _P, _P, _P],
    "tmop_min_det": [_P, _P, _P],
    "tmop_element_min_det": [_P, _P, _P, _P],
    "tmop_volume": [_P, _P, _P],
    "tmop_metric_eval": [_INT, _INT, _I64, _P, _P, _P, _P],
    "tmop_dot": [_P, _I64, _P, _P, _P],
    "tmop_axpby": [_P, _I64, _D, _P, _D, _P],
    "tmop_trial_point": [_P, _I64, _P, _P, _D, _P],
    "tmop_jacobi_inverse": [_P, _I64, _P, _D, _P, _P],
    "tmop_minres_init": [_P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "tmop_minres_step": [_P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _D, _P, _INT],
    "tmop_minres_set_history": [_P, _P, _INT],
    "tmop_minres_step_op": [_P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _D, _P, _INT],
    "tmop_minres_dist_init_a": [_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "tmop_minres_dist_init_b": [_P, _I64, _P, _P, _P, _P],
    "tmop_minres_dist_k1": [_P, _I64, _I64, _I64, _P, _P, _P, _P, _INT, _P],
    "tmop_minres_dist_k2": [_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _INT, _P],
    "tmop_minres_dist_k3": [_P, _I64, _P, _P, _P, _P, _P, _P, _D, _P, _INT, _P],
    "tmop_copy_components": [_P, _P, _P, _I64, _I64, _I64, _INT],
    "tmop_halo_pack": [_P, _I64, _I64, _INT, _INT, _P, _P],
    "tmop_halo_unpack": [_P, _I64, _I64, _INT, _INT, _P, _INT, _P, _D, _P],
    "tmop_halo_p2p_put": [_P, _I64, _I64, _P, _P, _P, _P, _P, _INT],
    "tmop_halo_p2p_get": [_P, _I64, _I64, _P, _P, _P, _INT, _INT, _INT, C.c_uint64, _INT, _P, _D, _P],
    "tmop_halo_p2p_arrivals": [_I64],
    "tmop_last_error": [],
}
_RESTYPES = {"tmop_qdata_size": _I64, "tmop_qdata_stride": _I64, "tmop_last_error": C.c_char_p,
             "tmop_ctx_point_scale": _P, "tmop_halo_p2p_arrivals": _I64}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: str | None = None):
    """Load the library (once).  Raises TmopLibraryError if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise TmopLibraryError(
            f"{p} not found: build it with `python -m paper_2205_12721_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(p)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, _INT)
    if path is None:
        _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != TMOP_OK:
        msg = load().tmop_last_error()
        raise TmopLibraryError(f"{what} failed (code {rc}): {msg.decode() if msg else ''}")


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()
