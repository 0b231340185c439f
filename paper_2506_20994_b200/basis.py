"""GLL basis for the host side of the product path (setup, not hot path).

Builds the Gauss-Lobatto-Legendre nodes, weights and differentiation matrix
the caller passes through the ABI's six matrix slots.  Same rule as the
reference's ``mdg.sem.gll_basis`` (/root/reference/pkg/src/mdg/sem.py:182-236)
and ``operator_matrices`` (sem.py:288-297): interior nodes are roots of
L_N' found by Newton iteration on the left half and mirrored;
w = 2/(N(N+1) L_N(x)^2); D[i][j] = L_N(x_i)/(L_N(x_j)(x_i-x_j)), corners
-+N(N+1)/4.  tests/test_basis.py pins it bit-for-bit to the reference's
values (tests/golden/gll.json).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import RangeError

LX_MIN, LX_MAX = 2, 16


@dataclass(frozen=True)
class Basis:
    lx: int
    points: np.ndarray
    weights: np.ndarray
    deriv: np.ndarray

    def operator_matrices(self) -> tuple[np.ndarray, np.ndarray]:
        """(stage-1 slot matrix, stage-2 slot matrix) = (D^T, D)."""
        return np.ascontiguousarray(self.deriv.T), np.ascontiguousarray(self.deriv)


def _leg(n: int, x: np.ndarray):
    p_prev = np.ones_like(x)
    if n == 0:
        return p_prev, np.zeros_like(x)
    p, d = x.copy(), np.ones_like(x)
    for k in range(2, n + 1):
        p_next = ((2 * k - 1) * x * p - (k - 1) * p_prev) / k
        d = x * d + k * p
        p_prev, p = p, p_next
    return p, d


def gll_basis(lx: int) -> Basis:
    if not isinstance(lx, (int, np.integer)) or not (LX_MIN <= lx <= LX_MAX):
        raise RangeError(f"lx must be an integer in [{LX_MIN}, {LX_MAX}], got {lx!r}")
    n = lx - 1
    pts = np.empty(lx)
    pts[0], pts[-1] = -1.0, 1.0
    if lx % 2:
        pts[lx // 2] = 0.0
    half_step = 0.5 * np.pi / n
    for q in range(1, (lx - 2) // 2 + 1):
        x = np.asarray(-np.cos(np.pi * q / n))
        for _ in range(100):
            p, d = _leg(n, x)
            dd = (2.0 * x * d - n * (n + 1) * p) / (1.0 - x * x)
            step = float(np.clip(d / dd, -half_step, half_step))
            x = x - step
            if abs(step) < 1e-16:
                break
        pts[q] = float(x)
        pts[lx - 1 - q] = -float(x)
    vals, _ = _leg(n, pts)
    w = 2.0 / (n * (n + 1) * vals * vals)
    dm = np.zeros((lx, lx))
    for i in range(lx):
        for j in range(lx):
            if i != j:
                dm[i, j] = (vals[i] / vals[j]) / (pts[i] - pts[j])
    dm[0, 0] = -n * (n + 1) / 4.0
    dm[-1, -1] = n * (n + 1) / 4.0
    return Basis(lx, pts, w, dm)
