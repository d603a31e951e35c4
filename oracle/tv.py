"""Regulariser lambda*phi(D x) and its gradient, fp64.  TEST INFRASTRUCTURE ONLY.

D: forward finite differences (Sec. IV-A), circular within the
facet's estimate block (S:323 example [1,2,4] -> [1,2,-3]) or
Neumann (last difference = 0) when boundary == 1.
phi (per-pixel isotropic 2-vector norm g = (Dy x, Dx x)):
  kind 0 (default, BASELINE.json "smoothed TV"): phi(g) = sqrt(|g|^2+eps^2) - eps,
         psi(g) = grad phi = g / sqrt(|g|^2 + eps^2)
  kind 1 (paper's Huber, delta = eps): phi = |g|^2/2 if
         |g| <= delta else delta(|g| - delta/2); psi = g * min(1, delta/|g|)
"""
from __future__ import annotations

import numpy as np


def D(x: np.ndarray, boundary: int = 0):
    """Returns (dy, dx): dy[p,q] = x[p+1,q] - x[p,q], dx[p,q] = x[p,q+1] - x[p,q]."""
    dy = np.roll(x, -1, axis=0) - x
    dx = np.roll(x, -1, axis=1) - x
    if boundary == 1:
        dy[-1, :] = 0.0
        dx[:, -1] = 0.0
    return dy, dx


def Dt(vy: np.ndarray, vx: np.ndarray, boundary: int = 0) -> np.ndarray:
    """Adjoint of D: (D^T v)[p] = v[p-1] - v[p] per component (circular), with the
    rows/cols that D zeroes dropped for Neumann."""
    if boundary == 1:
        vy = vy.copy()
        vx = vx.copy()
        vy[-1, :] = 0.0
        vx[:, -1] = 0.0
    return (np.roll(vy, 1, axis=0) - vy) + (np.roll(vx, 1, axis=1) - vx)


def phi(dy: np.ndarray, dx: np.ndarray, eps: float, kind: int = 0) -> np.ndarray:
    t2 = dy * dy + dx * dx
    if kind == 0:
        return np.sqrt(t2 + eps * eps) - eps
    t = np.sqrt(t2)
    return np.where(t <= eps, 0.5 * t2, eps * (t - 0.5 * eps))


def psi(dy: np.ndarray, dx: np.ndarray, eps: float, kind: int = 0):
    t2 = dy * dy + dx * dx
    if kind == 0:
        s = 1.0 / np.sqrt(t2 + eps * eps)
    else:
        t = np.sqrt(t2)
        s = np.where(t <= eps, 1.0, eps / np.where(t > 0, t, 1.0))
    return dy * s, dx * s


def value(x: np.ndarray, eps: float, kind: int = 0, boundary: int = 0) -> float:
    dy, dx = D(x, boundary)
    return float(phi(dy, dx, eps, kind).sum())


def grad(x: np.ndarray, eps: float, kind: int = 0, boundary: int = 0) -> np.ndarray:
    """D^T psi(D x): gradient of sum phi(D x)."""
    dy, dx = D(x, boundary)
    py, px = psi(dy, dx, eps, kind)
    return Dt(py, px, boundary)


def lipschitz_psi(eps: float, kind: int = 0) -> float:
    """Lipschitz constant of psi: 1/eps for smoothed TV, 1 for Huber."""
    return 1.0 / eps if kind == 0 else 1.0
