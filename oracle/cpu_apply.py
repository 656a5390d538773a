"""ctypes driver of oracle/lib/libtmop_oracle.so (C/OpenMP restatement of
the reference Hessian action) -- TEST INFRASTRUCTURE / CPU BASELINE ONLY."""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "lib", "libtmop_oracle.so")
_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-C", HERE], check=True, capture_output=True)
        _lib = C.CDLL(LIB)
        p = C.c_void_p
        _lib.oracle_hessian_apply3d.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64] + [p] * 12 + [C.c_int]
        _lib.oracle_hessian_apply3d.restype = C.c_int
        _lib.oracle_max_threads.restype = C.c_int
    return _lib


class CpuApply:
    """Precomputes the planar Q-data / node map once; `__call__(v)` runs the
    multi-threaded C apply."""

    def __init__(self, prob, qd, nthreads: int = 0):
        m = prob.mesh
        assert m.dim == 3
        self.n1, self.nq = prob.disc.n, prob.disc.nq
        self.ne, self.nn = m.n_elements, m.n_nodes
        self.restr = np.ascontiguousarray(m.restriction, dtype=np.int32)
        flags = np.zeros(m.n_nodes, dtype=np.uint8)
        for a in range(3):
            flags |= m.fixed[a].astype(np.uint8) << a
        self.fixed = flags
        self.B = np.ascontiguousarray(prob.disc.B)
        self.G = np.ascontiguousarray(prob.disc.G)
        c, s, t = qd.planar()
        self.c, self.s, self.t = (np.ascontiguousarray(a) for a in (c, s, t))
        flat = self.restr.ravel()
        order = np.argsort(flat, kind="stable")
        self.idx = order.astype(np.uint32)
        self.off = np.zeros(m.n_nodes + 1, dtype=np.int64)
        self.off[1:] = np.cumsum(np.bincount(flat, minlength=m.n_nodes))
        self.E = np.empty(self.ne * 3 * self.n1 ** 3)
        self.nthreads = nthreads
        self.lib = load()

    @property
    def threads(self) -> int:
        return self.nthreads or self.lib.oracle_max_threads()

    def __call__(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        y = np.empty_like(v)
        P = lambda a: a.ctypes.data  # noqa: E731
        rc = self.lib.oracle_hessian_apply3d(self.n1, self.nq, self.ne, self.nn, P(self.restr), P(self.fixed),
                                             P(self.B), P(self.G), P(self.c), P(self.s), P(self.t), P(v), P(y),
                                             P(self.off), P(self.idx), P(self.E), self.nthreads)
        if rc:
            raise RuntimeError("oracle_hessian_apply3d failed")
        return y
