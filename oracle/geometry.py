"""Facet geometry: index sets P_f, observed blocks O_f, consensus weights.

TEST INFRASTRUCTURE ONLY.  Follows the readings of SURVEY §8c:
  A12  overlap O is measured between OBSERVED blocks; facet bounds
       b_k = floor(k M / F); O_f = [b_f - O/2, b_{f+1} + O/2) clipped to [0, M);
       P_f = O_f dilated by c on each side, i.e. estimate [lo, hi + P - 1)
       (the "extra boundary pixels" of Fig. 1).
  A13  consensus weights omega^F: on the band [s, e) shared by facets f and f+1
       omega_{f+1}(t) = (t - s + 0.5)/(e - s), omega_f = 1 - omega_{f+1}; 1
       elsewhere; 2-D weight = product (ramp of Fig. 1 / Fig. 3(e)).
  A28  8-neighbour topology (pixels can lie in 4 blocks).
Index sets P_f of PAPER.md:118; P_l^- = {f : l in P_f} of PAPER.md:168.
"""
from __future__ import annotations

import dataclasses
from typing import List, Tuple

import numpy as np


@dataclasses.dataclass(frozen=True)
class AxisFacet:
    o_lo: int   # observed block [o_lo, o_hi)
    o_hi: int
    e_lo: int   # estimate block [e_lo, e_hi) = [o_lo, o_hi + P - 1)
    e_hi: int


def axis_plan(M: int, F: int, O: int, P: int) -> List[AxisFacet]:
    if F < 1 or O < 0 or O % 2:
        raise ValueError("F >= 1 and even O >= 0 required")
    b = [(k * M) // F for k in range(F + 1)]
    out = []
    for k in range(F):
        lo = 0 if k == 0 else max(0, b[k] - O // 2)
        hi = M if k == F - 1 else min(M, b[k + 1] + O // 2)
        out.append(AxisFacet(lo, hi, lo, hi + P - 1))
    for k in range(1, F - 1):   # bands of non-adjacent facets must not overlap
        if out[k - 1].e_hi > out[k + 1].e_lo:
            raise ValueError("facet core smaller than estimate overlap: a pixel would be in >2 facets per axis")
    return out


def axis_weight(plan: List[AxisFacet], k: int) -> np.ndarray:
    """omega^F along one axis for facet k over its estimate block (fp64)."""
    f = plan[k]
    n = f.e_hi - f.e_lo
    w = np.ones(n)
    t = np.arange(f.e_lo, f.e_hi, dtype=np.float64)
    if k > 0:                               # band with the previous facet: ramp up
        s, e = f.e_lo, plan[k - 1].e_hi
        m = t < e
        w[m] = (t[m] - s + 0.5) / (e - s)
    if k < len(plan) - 1:                   # band with the next facet: ramp down
        s, e = plan[k + 1].e_lo, f.e_hi
        m = t >= s
        w[m] = 1.0 - (t[m] - s + 0.5) / (e - s)
    return w


@dataclasses.dataclass(frozen=True)
class Facet:
    id: int
    fy: int
    fx: int
    oy: Tuple[int, int]     # observed rows [lo, hi)
    ox: Tuple[int, int]
    ey: Tuple[int, int]     # estimate rows [lo, hi)
    ex: Tuple[int, int]
    wy: np.ndarray          # omega^F along rows (fp64)
    wx: np.ndarray

    @property
    def shape(self):
        return (self.ey[1] - self.ey[0], self.ex[1] - self.ex[0])

    @property
    def oshape(self):
        return (self.oy[1] - self.oy[0], self.ox[1] - self.ox[0])

    def omega(self) -> np.ndarray:
        return self.wy[:, None] * self.wx[None, :]


def plan(Ny: int, Nx: int, P: int, Fy: int, Fx: int, O: int) -> List[Facet]:
    My, Mx = Ny - P + 1, Nx - P + 1
    py = axis_plan(My, Fy, O, P)
    px = axis_plan(Mx, Fx, O, P)
    facets = []
    for a in range(Fy):
        for b in range(Fx):
            facets.append(Facet(a * Fx + b, a, b, (py[a].o_lo, py[a].o_hi), (px[b].o_lo, px[b].o_hi),
                                (py[a].e_lo, py[a].e_hi), (px[b].e_lo, px[b].e_hi),
                                axis_weight(py, a), axis_weight(px, b)))
    return facets


def neighbours(facets: List[Facet]):
    """Pairs (f, g), f < g, whose estimate blocks intersect, with the rectangle."""
    out = []
    for f in facets:
        for g in facets:
            if g.id <= f.id:
                continue
            y0, y1 = max(f.ey[0], g.ey[0]), min(f.ey[1], g.ey[1])
            x0, x1 = max(f.ex[0], g.ex[0]), min(f.ex[1], g.ex[1])
            if y0 < y1 and x0 < x1:
                out.append((f.id, g.id, (y0, y1, x0, x1)))
    return out
