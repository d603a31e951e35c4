"""Bound-constrained limited-memory variable-metric minimiser (VMLM-B family),
fp64, step by step.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:287 names VMLM-B (Thiebaut 2002), "a variant of the standard L-BFGS-B
... the only parameter step-length ... estimated by line-search methods
satisfying Wolfe's conditions", and PAPER.md:290 its use as the Local-Solver:
warm-started at x_i^(k), 10 inner iterations at the first outer iteration and
10 more at every next one.  The paper gives no further detail (SPEC.md local-
solver module: "VMLM-B is proprietary in detail"), so both sides implement this
reading (V1-V6), in this order:

  V1  bound x >= 0; the iterate is projected after every step
  V2  free set F = {i : x_i > 0 or g_i < 0}; the active set is frozen
  V3  direction d = -H g on F by the L-BFGS two-loop recursion over the last
      m = 5 pairs (s, y), every inner product restricted to F; H0 = <s,y>/<y,y>
      of the newest pair, or h0 (the fixed projected-gradient step tau, A4')
      without pairs; if <g, d> >= 0 the memory is dropped and d = -h0 g_F
  V4  projected backtracking line search t = 1, 1/2, 1/4, ... (at most 10
      trials: the first step is the projected-gradient step and later ones are
      quasi-Newton, so more halvings only happen at the rounding floor): accept
      the first t with f(P(x + t d)) <= f(x) + c1 <g, P(x + t d) - x>, c1 = 1e-4 (the sufficient-decrease half of the Wolfe conditions; the
      curvature half is not enforced on a projected path); no acceptable t ends
      the solve (line-search stall, the iterate is kept)
  V5  pair (s, y) = (x+ - x, g+ - g) stored iff <s, y> > 1e-12 |s| |y| (oldest dropped)
  V6  stop after the iteration budget, or when |P(x - g) - x|_inf <= gtol
"""
from __future__ import annotations

import dataclasses
from typing import Callable, List, Tuple

import numpy as np

C1 = 1e-4
MAX_LS = 10


@dataclasses.dataclass
class Report:
    iterations: int
    f: float
    pg_norm: float
    reason: str          # "budget" | "converged" | "stall"
    evaluations: int


def _pgnorm(x, g):
    return float(np.abs(np.maximum(x - g, 0.0) - x).max()) if x.size else 0.0


def minimize(fg: Callable[[np.ndarray], Tuple[float, np.ndarray]], x0: np.ndarray, h0: float, m: int = 5,
             max_iter: int = 10, gtol: float = 0.0) -> Tuple[np.ndarray, Report]:
    """Minimise f over x >= 0 from x0 (V1-V6); fg(x) -> (f, grad f)."""
    x = np.maximum(np.asarray(x0, np.float64), 0.0)
    f, g = fg(x)
    if not np.isfinite(f):
        raise FloatingPointError("non-finite objective at x0")
    S: List[np.ndarray] = []
    Y: List[np.ndarray] = []
    R: List[float] = []
    nev = 1
    it = 0
    reason = "budget"
    while it < max_iter:
        if gtol > 0 and _pgnorm(x, g) <= gtol:
            reason = "converged"
            break
        free = (x > 0) | (g < 0)                                           # V2
        q = np.where(free, g, 0.0)                                         # V3 two-loop
        alphas = []
        for s, y, rho in zip(reversed(S), reversed(Y), reversed(R)):
            a = rho * float(np.dot(np.where(free, s, 0.0).ravel(), q.ravel()))
            q = q - a * np.where(free, y, 0.0)
            alphas.append(a)
        if S:
            sy = float(np.dot(S[-1].ravel(), Y[-1].ravel()))
            yy = float(np.dot(Y[-1].ravel(), Y[-1].ravel()))
            r = (sy / yy) * q
        else:
            r = h0 * q
        for s, y, rho, a in zip(S, Y, R, reversed(alphas)):
            b = rho * float(np.dot(np.where(free, y, 0.0).ravel(), r.ravel()))
            r = r + (a - b) * np.where(free, s, 0.0)
        d = -np.where(free, r, 0.0)
        if float(np.dot(g.ravel(), d.ravel())) >= 0.0:                    # not a descent direction
            S, Y, R = [], [], []
            d = -h0 * np.where(free, g, 0.0)
        t = 1.0                                                            # V4
        accepted = False
        for _ in range(MAX_LS):
            xn = np.maximum(x + t * d, 0.0)
            fn, gn = fg(xn)
            nev += 1
            if fn <= f + C1 * float(np.dot(g.ravel(), (xn - x).ravel())):
                accepted = True
                break
            t *= 0.5
        if not accepted:
            reason = "stall"
            break
        s = xn - x                                                         # V5
        y = gn - g
        sy = float(np.dot(s.ravel(), y.ravel()))
        if sy > 1e-12 * float(np.linalg.norm(s)) * float(np.linalg.norm(y)):
            S.append(s)
            Y.append(y)
            R.append(1.0 / sy)
            if len(S) > m:
                S.pop(0)
                Y.pop(0)
                R.pop(0)
        x, f, g = xn, fn, gn
        it += 1
    return x, Report(it, float(f), _pgnorm(x, g), reason, nev)
