"""1D Lagrange bases on Gauss-Lobatto nodes and Gauss-Legendre rules
(host-side setup; the tables are uploaded once into the kernels' constant
bank).  API mirrors the reference's fe.py (fe.py:42-177).

Conventions (fe.py:1-14): dof / quadrature tensors are lexicographic with
the direction-1 (x) index fastest.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["Basis1D", "QuadRule1D", "EvalMatrices", "OpCounter", "gauss_lobatto_points",
           "gauss_legendre_1d", "tensor_weights", "build_eval_matrices"]

_HIT = 1e-13


def gauss_lobatto_points(n: int) -> np.ndarray:
    """n >= 2 Gauss-Lobatto points on [0, 1] (endpoints and the roots of
    P'_{n-1}) -- fe.py:42-53."""
    if n < 2:
        raise ValueError(f"need at least 2 points, got {n}")
    if n == 2:
        return np.array([0.0, 1.0])
    leg = np.polynomial.legendre.Legendre(np.eye(n)[-1])
    inner = np.sort(leg.deriv().roots().real)
    return (np.concatenate(([-1.0], inner, [1.0])) + 1.0) / 2.0


@dataclass(frozen=True)
class QuadRule1D:
    points: np.ndarray
    weights: np.ndarray

    @property
    def n_points(self) -> int:
        return len(self.points)


def gauss_legendre_1d(n_q: int) -> QuadRule1D:
    """n_q-point Gauss-Legendre rule on [0, 1] (fe.py:126-131)."""
    if not 1 <= n_q <= 32:
        raise ValueError(f"n_q must be in [1, 32], got {n_q}")
    x, w = np.polynomial.legendre.leggauss(n_q)
    return QuadRule1D(points=(x + 1.0) / 2.0, weights=w / 2.0)


def tensor_weights(rule: QuadRule1D, dim: int) -> np.ndarray:
    """Flattened tensor-product weights, x fastest (fe.py:134-140)."""
    out = rule.weights
    for _ in range(dim - 1):
        out = np.multiply.outer(rule.weights, out)
    return np.ravel(out)


@dataclass(frozen=True)
class Basis1D:
    """Lagrange basis of degree `order` on increasing nodes in [0, 1]."""
    order: int
    nodes: np.ndarray

    @classmethod
    def gauss_lobatto(cls, order: int) -> "Basis1D":
        return cls(order, gauss_lobatto_points(order + 1))

    @property
    def n_nodes(self) -> int:
        return self.order + 1

    def _weights(self) -> np.ndarray:
        d = self.nodes[:, None] - self.nodes[None, :]
        np.fill_diagonal(d, 1.0)
        return 1.0 / d.prod(axis=1)

    def _tables(self, x):
        """(values, derivatives) at points x, barycentric form; rows whose
        point coincides with a node use the exact node formulas
        (fe.py:76-111)."""
        x = np.atleast_1d(np.asarray(x, dtype=float))
        bw = self._weights()
        diff = x[:, None] - self.nodes[None, :]
        hit = np.abs(diff) < _HIT
        safe = np.where(hit, 1.0, diff)
        tv = bw[None, :] / safe                       # values: w_i / (x - x_i)
        vals = tv / tv.sum(axis=1, keepdims=True)
        inv = 1.0 / safe                              # derivatives: l_i (sum_j inv_j - inv_i)
        td = bw[None, :] * inv
        ders = (td / td.sum(axis=1, keepdims=True)) * (inv.sum(axis=1, keepdims=True) - inv)
        for r in np.flatnonzero(hit.any(axis=1)):
            k = int(np.argmax(hit[r]))
            vals[r] = 0.0
            vals[r, k] = 1.0
            gap = self.nodes[k] - self.nodes
            gap[k] = 1.0
            row = (bw / bw[k]) / gap
            row[k] = 0.0
            row[k] = -row.sum()
            ders[r] = row
        return vals, ders

    def eval_values(self, x) -> np.ndarray:
        return self._tables(x)[0]

    def eval_derivs(self, x) -> np.ndarray:
        return self._tables(x)[1]


@dataclass(frozen=True)
class EvalMatrices:
    """B[q, i] = l_i(chi_q), G[q, i] = l_i'(chi_q), each (n_q, n_i)."""
    b: np.ndarray
    g: np.ndarray

    @property
    def n_quad(self) -> int:
        return self.b.shape[0]

    @property
    def n_dofs(self) -> int:
        return self.b.shape[1]


def build_eval_matrices(basis: Basis1D, rule: QuadRule1D) -> EvalMatrices:
    b, g = basis._tables(rule.points)
    return EvalMatrices(b=b, g=g)


@dataclass
class OpCounter:
    """Multiply-add counter with the reference's accounting (fe.py:163-177,
    222-223; operator.py:396-398).  The device kernels do not count at run
    time; TmopProblem adds the analytic per-call counts."""
    madds: int = 0

    def add(self, n: int) -> None:
        self.madds += int(n)

    def reset(self) -> None:
        self.madds = 0
