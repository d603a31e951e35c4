"""Distributed Douglas-Rachford deblurring (Algorithm 1), fp64, step by step.

TEST INFRASTRUCTURE ONLY.  Follows, in the paper's order and notation:
  f_i(x_i) = 1/2 |y_i - H_i x_i|^2_{W_i} + lambda phi(D_i x_i) + iota_{>=0}
  x_i^{k+1} = Prox_{V_i^{-1}, f_i}(u_i^k)
  zbar(l)   = sum_{i in P_l^-} alpha_i(l)(2 x_i - u_i) / sum alpha_i(l)      PAPER.md:201 (Lemma 1, :169-175)
  u_i(l)   += rho (zbar(l) - x_i(l))
  alpha_i   = gamma * omega_i
with the readings of SURVEY §8c:
  A3/R2  Local-Solver = K_in fixed-step projected-gradient steps on
         f_i(w) + 1/2 |w - u_i|^2_{alpha_i}, warm-started at x_i
  A4     step tau: see default_tau (A4' in DESIGN.md)
  A6     x^0 = u^0 = max(0, y edge-replicated into the c-wide margin)|P_f
  A7     image = sum_f omega^F_f x_f
  A8/A9  consensus divides by the computed sum of weights, facets in ascending id
  A20    every facet uses its full W_i (no multiplicity division)
  A22    objective = sum_f [data_f + lambda reg_f] at the current x (+ max |x_i - x_j|)
Independent baseline (NEXT-3): every facet runs the Local-Solver on
  its own f_i with alpha = 0 (gamma := 0, also in tau) and no consensus; image as A7.
Operator modes (NEXT-2):
  0  H_i = the global PSF-interpolation H restricted to facet i (R1);
     omega_i = the A13 ramps (partition of unity on every band)
  1  per-node: facet (a, b) holds PSF h_i, i = a G_x + b,
     and H_i = C_i calH_i is the valid convolution with h_i alone; omega_i = the
     interpolation weights wy[a] (x) wx[b] of that PSF on the facet's estimate block;
     the image is sum_i omega_i x_i / sum_i omega_i (the weights need not sum to 1
     on a facet union)
"""
from __future__ import annotations

import dataclasses
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import geometry, tv, vmlmb
from .operators import Operator


# --------------------------------------------------------------------------
# generic D-R driver over explicit windows (used by the deblurring problem and,
# unchanged, by the exact-arithmetic hand trace of tests/test_oracle_driver.py)
# --------------------------------------------------------------------------
def consensus(shape: Tuple[int, int], windows: Sequence[Tuple[slice, slice]], omegas: Sequence[np.ndarray],
              x: Sequence[np.ndarray], u: Sequence[np.ndarray], rho) -> List[np.ndarray]:
    """Lemma 1 applied to v_i = 2x_i - u_i, then the relaxed
    dual update.  Returns the new u_i."""
    num = np.zeros(shape, dtype=np.asarray(x[0]).dtype)
    den = np.zeros(shape, dtype=np.asarray(omegas[0]).dtype)
    for win, om, xi, ui in zip(windows, omegas, x, u):       # ascending facet id (A9)
        num[win] = num[win] + om * (2 * xi - ui)
        den[win] = den[win] + om
    zbar = np.empty_like(num)
    m = den != 0
    zbar[m] = num[m] / den[m]
    return [ui + rho * (zbar[win] - xi) for win, xi, ui in zip(windows, x, u)]


def dr_iteration(shape, windows, omegas, x, u, local_prox: Callable, rho):
    """One full distributed iteration of Algorithm 1."""
    x_new = [local_prox(i, x[i], u[i]) for i in range(len(windows))]    # Local-Solver, in parallel
    u_new = consensus(shape, windows, omegas, x_new, u, rho)             # synchronise, average, update
    return x_new, u_new


# --------------------------------------------------------------------------
# the deblurring instance
# --------------------------------------------------------------------------
def default_tau(psfs, wy, wx, w_max: float, lam: float, eps: float, reg_kind: int, gamma: float) -> float:
    """A4': tau = 1 / L with L an upper bound of the Lipschitz
    constant of the local gradient:
      |H|^2 <= (max row sum)(max col sum) (Schur), with
        row sums <= S_w * sum_{a,b} max_k |h_k[a,b]|,
        col sums <= S_w * max_k sum_{a,b} |h_k[a,b]|,
        S_w = max_r sum_p |wy[p,r]| * max_c sum_q |wx[q,c]|
      |D|^2 <= 8, Lip(psi) = 1/eps (smoothed TV) or 1 (Huber), max alpha = gamma.
    """
    h = np.abs(np.asarray(psfs, dtype=np.float64))
    S = np.abs(np.asarray(wy, np.float64)).sum(0).max() * np.abs(np.asarray(wx, np.float64)).sum(0).max()
    a_row = h.max(axis=0).sum()
    a_col = h.sum(axis=(1, 2)).max()
    L = w_max * S * S * a_row * a_col + lam * 8.0 * tv.lipschitz_psi(eps, reg_kind) + gamma
    return 1.0 / L


@dataclasses.dataclass
class Params:
    lam: float
    eps: float
    gamma: float
    rho: float
    reg_kind: int = 0
    tv_boundary: int = 0
    inner_steps: int = 1
    local_solver: int = 0        # 0: K_in projected-gradient steps (R2); 1: VMLM-B (V1-V6, vmlmb.py)
    inner_increment: int = 0     # VMLM-B budget at outer iteration k: inner_steps + k * inner_increment


class Deblur:
    """Oracle state for one problem: per-facet x_f, u_f (fp64)."""

    def __init__(self, psfs, wy, wx, y, w, Fy: int, Fx: int, overlap: int, params: Params,
                 tau: Optional[float] = None, x0: Optional[np.ndarray] = None, operator_mode: int = 0,
                 independent: bool = False):
        self.op = Operator(psfs, wy, wx)
        self.independent = bool(independent)
        if self.independent:      # the paper's independent baseline: alpha = 0, no consensus
            params = dataclasses.replace(params, gamma=0.0)
        self.prm = params
        self.operator_mode = int(operator_mode)
        self.y = np.asarray(y, np.float64)
        self.w = np.broadcast_to(np.asarray(w, np.float64), self.y.shape)
        assert self.y.shape == (self.op.My, self.op.Mx)
        self.facets = geometry.plan(self.op.Ny, self.op.Nx, self.op.P, Fy, Fx, overlap)
        self.windows = [(slice(*f.ey), slice(*f.ex)) for f in self.facets]
        self.owin = [(slice(*f.oy), slice(*f.ox)) for f in self.facets]
        if self.operator_mode == 0:
            self.omegas = [f.omega() for f in self.facets]
            self.ops = [self.op] * len(self.facets)
        else:
            # per-node: facet grid = PSF grid; facet (a, b) blurs with PSF a*G_x + b only
            assert (Fy, Fx) == (self.op.gy, self.op.gx), "per-node mode needs facet grid == PSF grid"
            wy64 = np.asarray(wy, np.float64)
            wx64 = np.asarray(wx, np.float64)
            self.omegas = [np.outer(wy64[f.fy, f.ey[0]:f.ey[1]], wx64[f.fx, f.ex[0]:f.ex[1]]) for f in self.facets]
            ones_y = np.ones((1, self.op.Ny))
            ones_x = np.ones((1, self.op.Nx))
            self.ops = [Operator(np.asarray(psfs)[f.fy * self.op.gx + f.fx][None], ones_y, ones_x)
                        for f in self.facets]
        self.tau = default_tau(psfs, wy, wx, float(self.w.max()), params.lam, params.eps,
                               params.reg_kind, params.gamma) if tau is None else float(tau)
        if x0 is None:                                   # A6
            c = self.op.c
            x0 = np.maximum(0.0, np.pad(self.y, c, mode="edge"))
        x0 = np.asarray(x0, np.float64)
        self.x = [x0[win].copy() for win in self.windows]
        self.u = [x0[win].copy() for win in self.windows]
        self.k = 0                                        # outer iteration counter (VMLM-B budget)

    @property
    def shape(self):
        return (self.op.Ny, self.op.Nx)

    # ---- local objective pieces ----------------------------
    def residual(self, i: int, xi: np.ndarray) -> np.ndarray:
        """r = W_i (H_i x_i - y_i) on O_i."""
        f = self.facets[i]
        hx = self.ops[i].H_window(xi, f.ey[0], f.ex[0])
        return self.w[self.owin[i]] * (hx - self.y[self.owin[i]])

    def local_grad(self, i: int, xi: np.ndarray, ui: np.ndarray) -> np.ndarray:
        """grad of f_i(w) + 1/2|w - u_i|^2_{alpha_i} without the indicator."""
        f = self.facets[i]
        p = self.prm
        r = self.residual(i, xi)
        g = self.ops[i].HT_window(r, f.ey[0], f.ex[0])
        g = g + p.lam * tv.grad(xi, p.eps, p.reg_kind, p.tv_boundary)
        g = g + p.gamma * self.omegas[i] * (xi - ui)
        return g

    def local_value_grad(self, i: int, w: np.ndarray, ui: np.ndarray):
        """f_i(w) + 1/2 |w - u_i|^2_{alpha_i} (without the indicator) and its gradient."""
        f = self.facets[i]
        p = self.prm
        d = self.ops[i].H_window(w, f.ey[0], f.ex[0]) - self.y[self.owin[i]]
        wd = self.w[self.owin[i]] * d
        al = p.gamma * self.omegas[i]
        val = 0.5 * float((wd * d).sum()) + p.lam * tv.value(w, p.eps, p.reg_kind, p.tv_boundary) \
            + 0.5 * float((al * (w - ui) ** 2).sum())
        g = self.ops[i].HT_window(wd, f.ey[0], f.ex[0]) + p.lam * tv.grad(w, p.eps, p.reg_kind, p.tv_boundary) \
            + al * (w - ui)
        return val, g

    def local_prox(self, i: int, xi: np.ndarray, ui: np.ndarray) -> np.ndarray:
        """Local-Solver (R2): K_in projected-gradient steps, warm start at x_i; or
        VMLM-B with budget inner_steps + k inner_increment."""
        if self.prm.local_solver == 1:
            budget = self.prm.inner_steps + self.k * self.prm.inner_increment
            x, _ = vmlmb.minimize(lambda w: self.local_value_grad(i, w, ui), xi, h0=self.tau, m=5,
                                  max_iter=budget)
            return x
        for _ in range(self.prm.inner_steps):
            xi = np.maximum(0.0, xi - self.tau * self.local_grad(i, xi, ui))
        return xi

    # ---- Algorithm 1 ------------------------------------------------------
    def iterate(self, n: int = 1):
        for _ in range(n):
            if self.independent:
                self.x = [self.local_prox(i, self.x[i], self.u[i]) for i in range(len(self.windows))]
            else:
                self.x, self.u = dr_iteration(self.shape, self.windows, self.omegas, self.x, self.u,
                                              self.local_prox, self.prm.rho)
            self.k += 1
        return self

    # ---- diagnostics ------------------------------------------------------
    def objective(self):
        """(total, data, reg, consensus_maxdiff) at the current x (A22)."""
        p = self.prm
        data = 0.0
        reg = 0.0
        for i, f in enumerate(self.facets):
            hx = self.ops[i].H_window(self.x[i], f.ey[0], f.ex[0])
            d = hx - self.y[self.owin[i]]
            data += 0.5 * float((self.w[self.owin[i]] * d * d).sum())
            reg += p.lam * tv.value(self.x[i], p.eps, p.reg_kind, p.tv_boundary)
        hi = np.full(self.shape, -np.inf)
        lo = np.full(self.shape, np.inf)
        cnt = np.zeros(self.shape, np.int64)
        for win, xi in zip(self.windows, self.x):
            hi[win] = np.maximum(hi[win], xi)
            lo[win] = np.minimum(lo[win], xi)
            cnt[win] += 1
        m = cnt >= 2
        maxdiff = float((hi[m] - lo[m]).max()) if m.any() else 0.0
        return data + reg, data, reg, maxdiff

    def image(self) -> np.ndarray:
        """x_hat = sum_f omega^F_f x_f (A7)."""
        out = np.zeros(self.shape)
        den = np.zeros(self.shape)
        for win, om, xi in zip(self.windows, self.omegas, self.x):
            out[win] += om * xi
            den[win] += om
        return out if self.operator_mode == 0 else out / den

    def state(self):
        """Concatenated facets in planner (ascending id) order: (x, u)."""
        return (np.concatenate([a.ravel() for a in self.x]), np.concatenate([a.ravel() for a in self.u]))


def from_problem(pb, tau: Optional[float] = None, **over) -> Deblur:
    """Build the oracle for a synth.Problem (inputs used verbatim, fp32 -> fp64)."""
    prm = Params(lam=pb.lam, eps=pb.eps, gamma=pb.gamma, rho=pb.rho, reg_kind=pb.reg_kind,
                 tv_boundary=pb.tv_boundary, inner_steps=pb.inner_steps,
                 local_solver=getattr(pb, "local_solver", 0), inner_increment=getattr(pb, "inner_increment", 0))
    for k, v in over.items():
        setattr(prm, k, v)
    w = pb.noise_w if pb.noise_w is not None else np.float64(np.float32(pb.noise_w_scalar))
    return Deblur(pb.psfs, pb.wy, pb.wx, pb.y, w, pb.fy, pb.fx, pb.overlap, prm, tau=tau, x0=pb.x0,
                  operator_mode=getattr(pb, "operator_mode", 0), independent=bool(getattr(pb, "independent", 0)))
