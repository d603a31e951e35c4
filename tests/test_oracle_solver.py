"""Pins for oracle/geometry.py and oracle/solver.py (CPU, -m "not gpu").

  geometry   union of O_f = observed domain, overlap widths, partition of unity,
             neighbour counts
  Lemma 1    brute-force minimiser of sum alpha_i (w - v_i)^2; golden examples;
             gamma invariance; consistent state is a fixed point
  driver     exact rational trace of the two-pixel problem -> (c1+c2)/2
  gradient   analytic local gradient vs central differences of the local cost
             evaluated with the dense paper-matrix A_f
  iterate    1 facet, rho = 1 == centralized projected gradient on Eq. (3)
             (dense A; BASELINE.json "a single facet must equal the centralized
             solve"); 2x2 facets converge to argmin_{x>=0} sum_f f_f(R_f x)
             (scipy L-BFGS-B on the consensus-reduced objective, PAPER.md:125,
             :160); exact-rational full-path trace (fractions)
  objective  zero at the noiseless truth; Eq. (3) value for one facet; additive
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.optimize

import synth
from oracle import geometry, solver, tv
from oracle.solver import Deblur, Params
from tests.dense_ref import dense_H

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ----------------------------------------------------------------- geometry
@pytest.mark.parametrize("N,P,F,O", [(1024, 31, 2, 64), (4096, 63, 4, 128), (300, 15, 3, 20), (64, 5, 5, 0)])
def test_axis_plan_invariants(N, P, F, O):
    M = N - P + 1
    pl = geometry.axis_plan(M, F, O, P)
    assert pl[0].o_lo == 0 and pl[-1].o_hi == M
    for a, b in zip(pl, pl[1:]):
        assert a.o_hi - b.o_lo == O                      # observed overlap O (A12)
        assert a.e_hi - b.e_lo == O + P - 1              # estimate band B = O + P - 1
    total = np.zeros(N)
    for k, f in enumerate(pl):
        w = geometry.axis_weight(pl, k)
        assert np.all(w > 0) and np.all(w <= 1)
        total[f.e_lo:f.e_hi] += w
    np.testing.assert_allclose(total, 1.0, rtol=0, atol=1e-15)


def test_neighbour_counts():
    f22 = geometry.plan(200, 200, 5, 2, 2, 8)
    assert len(geometry.neighbours(f22)) == 6               # 4 edges + 2 diagonals
    f33 = geometry.plan(300, 300, 5, 3, 3, 8)
    nb = geometry.neighbours(f33)
    assert sum(1 for a, b, _ in nb if 4 in (a, b)) == 8     # centre facet: 8-neighbourhood (A28)
    om = np.zeros((300, 300))
    for f in f33:
        om[slice(*f.ey), slice(*f.ex)] += f.omega()
    np.testing.assert_allclose(om, 1.0, atol=1e-15)


def test_planner_rejects_triple_overlap():
    with pytest.raises(ValueError):
        geometry.axis_plan(100, 5, 16, 9)                  # core 20 < O + P - 1 = 24


# ----------------------------------------------------------------- Lemma 1
def test_consensus_golden():
    for key in ("consensus_equal_weights", "consensus_unequal_weights"):
        g = GOLD[key]
        x = [np.array([[v]]) for v in g["values"]]
        om = [np.array([[w]]) for w in g["weights"]]
        win = [(slice(0, 1), slice(0, 1))] * len(x)
        # with u = x, v = 2x - u = x, and rho = 1: u_new = zbar
        u_new = solver.consensus((1, 1), win, om, x, x, 1.0)
        for un in u_new:
            assert un[0, 0] == pytest.approx(g["zbar"], rel=1e-15)


def test_lemma1_bruteforce_and_gamma_invariance():
    rng = np.random.default_rng(0)
    for _ in range(200):
        m = rng.integers(2, 5)
        alpha = rng.uniform(0.05, 1.0, m)
        v = rng.normal(0, 3, m)
        res = scipy.optimize.minimize_scalar(lambda w: float((alpha * (w - v) ** 2).sum()),
                                             bracket=(v.min() - 1, v.max() + 1), method="golden", tol=1e-12)
        x = [np.array([[vi]]) for vi in v]
        win = [(slice(0, 1), slice(0, 1))] * m
        for gamma in (1e-3, 1.0, 4000.0):
            u_new = solver.consensus((1, 1), win, [np.array([[gamma * a]]) for a in alpha], x, x, 1.0)
            assert u_new[0][0, 0] == pytest.approx(res.x, abs=1e-7)


def test_consistent_state_is_fixed_point():
    fac = geometry.plan(60, 60, 5, 2, 2, 6)
    rng = np.random.default_rng(1)
    xg = rng.uniform(0, 1, (60, 60))
    win = [(slice(*f.ey), slice(*f.ex)) for f in fac]
    x = [xg[w].copy() for w in win]
    u_new = solver.consensus((60, 60), win, [f.omega() for f in fac], x, [a.copy() for a in x], 1.0)
    for a, b in zip(u_new, x):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-15)


# ------------------------------------------------------------------ driver
def test_two_pixel_exact_trace():
    """two 1-pixel blocks sharing the pixel, f_i(w) = (w - c_i)^2/2,
    omega = (1/2, 1/2), rho = 1, exact prox; rational arithmetic throughout."""
    g = GOLD["two_pixel_fixed_point"]
    c = [Fraction(v).limit_denominator() for v in g["c"]]
    gamma = Fraction(3)
    om = [np.array([[Fraction(1, 2)]], dtype=object)] * 2
    win = [(slice(0, 1), slice(0, 1))] * 2

    def prox(i, xi, ui):     # argmin (w-c)^2/2 + alpha/2 (w-u)^2 = (c + alpha u)/(1 + alpha)
        a = gamma * om[i][0, 0]
        return np.array([[(c[i] + a * ui[0, 0]) / (1 + a)]], dtype=object)

    x = [np.array([[Fraction(0)]], dtype=object)] * 2
    u = [np.array([[Fraction(0)]], dtype=object)] * 2
    # hand recursion (equal weights): x_i = (c_i + a u_i)/(1+a); zbar = mean(2x - u); u_i += zbar - x_i
    hu = [Fraction(0), Fraction(0)]
    a = gamma / 2
    for _ in range(10):
        x, u = solver.dr_iteration((1, 1), win, om, x, u, prox, Fraction(1))
        hx = [(c[i] + a * hu[i]) / (1 + a) for i in range(2)]
        zb = ((2 * hx[0] - hu[0]) + (2 * hx[1] - hu[1])) / 2
        hu = [hu[i] + zb - hx[i] for i in range(2)]
        assert [x[0][0, 0], x[1][0, 0]] == hx and [u[0][0, 0], u[1][0, 0]] == hu
    for _ in range(200):
        x, u = solver.dr_iteration((1, 1), win, om, x, u, prox, Fraction(1))
    for xi in x:
        assert abs(float(xi[0, 0]) - g["fixed_point"]) < 1e-12


# ------------------------------------------------------------ tiny problems
def tiny(n=24, P=5, G=2, F=(2, 2), O=4, lam=0.0, eps=1e-3, gamma=2.0, seed=0, kind=0, bnd=0, w_arr=True):
    rng = np.random.default_rng(seed)
    psfs = rng.uniform(0, 1, (G * G, P, P))
    psfs /= psfs.sum(axis=(1, 2), keepdims=True)
    wy, wx = synth.hat_weights(n, G), synth.hat_weights(n, G)
    M = n - P + 1
    y = rng.uniform(0.1, 1.0, (M, M))
    w = rng.uniform(0.5, 2.0, (M, M)) if w_arr else 1.0
    prm = Params(lam=lam, eps=eps, gamma=gamma, rho=1.0, reg_kind=kind, tv_boundary=bnd)
    return psfs, wy, wx, y, w, prm, F, O


def test_local_gradient_matches_fd_of_dense_cost():
    psfs, wy, wx, y, w, prm, F, O = tiny(lam=0.05, eps=0.2, seed=3)
    d = Deblur(psfs, wy, wx, y, w, *F, O, prm)
    A = dense_H(psfs, wy, wx)
    n = 24
    M = y.shape[0]
    rng = np.random.default_rng(4)
    for i, f in enumerate(d.facets):
        rows = [a * M + b for a in range(*f.oy) for b in range(*f.ox)]
        cols = [a * n + b for a in range(*f.ey) for b in range(*f.ex)]
        Af = A[np.ix_(rows, cols)]
        yf, wf = y[slice(*f.oy), slice(*f.ox)].ravel(), np.broadcast_to(w, y.shape)[slice(*f.oy), slice(*f.ox)].ravel()
        al = prm.gamma * f.omega()
        u = rng.uniform(0, 1, f.shape)

        def cost(xv):
            res = Af @ xv.ravel() - yf
            return 0.5 * (wf * res * res).sum() + prm.lam * tv.value(xv, prm.eps) + 0.5 * (al * (xv - u) ** 2).sum()

        x = rng.uniform(0, 1, f.shape)
        gr = d.local_grad(i, x, u)
        for _ in range(8):
            a, b = rng.integers(0, f.shape[0]), rng.integers(0, f.shape[1])
            e = np.zeros_like(x)
            e[a, b] = 1e-6
            fd = (cost(x + e) - cost(x - e)) / 2e-6
            assert fd == pytest.approx(gr[a, b], rel=1e-6, abs=1e-8)


@pytest.mark.parametrize("kind,bnd", [(0, 0), (1, 0), (0, 1)])
def test_local_value_grad_pinned(kind, bnd):
    """local_value_grad (the function whose value drives VMLM-B's Armijo test,
    reading V4) against things other than itself: its value equals the prox
    objective f_i(w) + 1/2 |w - u_i|^2_alpha built from the
    dense matrix of the paper's operator form; its gradient equals central
    differences of its own value and the projected-gradient path's local_grad.
    A dropped 1/2 (data or prox term) or a lost lambda fails the value check."""
    psfs, wy, wx, y, w, prm, F, O = tiny(lam=0.05, eps=0.2, seed=5, kind=kind, bnd=bnd, w_arr=True)
    d = Deblur(psfs, wy, wx, y, w, *F, O, prm)
    A = dense_H(psfs, wy, wx)
    n = 24
    M = y.shape[0]
    rng = np.random.default_rng(6)
    for i, f in enumerate(d.facets):
        rows = [a * M + b for a in range(*f.oy) for b in range(*f.ox)]
        cols = [a * n + b for a in range(*f.ey) for b in range(*f.ex)]
        Af = A[np.ix_(rows, cols)]
        yf = y[slice(*f.oy), slice(*f.ox)].ravel()
        wf = np.broadcast_to(w, y.shape)[slice(*f.oy), slice(*f.ox)].ravel()
        al = prm.gamma * f.omega()
        u = rng.uniform(0, 1, f.shape)
        x = rng.uniform(0, 1, f.shape)
        res = Af @ x.ravel() - yf
        # TV term summed per pixel from the closed-form phi of A1 (smoothed TV) or the
        # paper's Huber on forward differences (circular or Neumann)
        if bnd == 0:
            dy, dx = np.roll(x, -1, 0) - x, np.roll(x, -1, 1) - x
        else:
            dy, dx = np.zeros_like(x), np.zeros_like(x)
            dy[:-1] = x[1:] - x[:-1]
            dx[:, :-1] = x[:, 1:] - x[:, :-1]
        t = np.sqrt(dy ** 2 + dx ** 2)
        if kind == 0:
            reg = (np.sqrt(t ** 2 + prm.eps ** 2) - prm.eps).sum()
        else:
            reg = np.where(t <= prm.eps, 0.5 * t ** 2, prm.eps * (t - 0.5 * prm.eps)).sum()
        want = 0.5 * (wf * res * res).sum() + prm.lam * reg + 0.5 * (al * (x - u) ** 2).sum()
        val, g = d.local_value_grad(i, x, u)
        assert val == pytest.approx(want, rel=1e-12)
        np.testing.assert_allclose(g, d.local_grad(i, x, u), rtol=1e-12, atol=1e-12)
        for _ in range(8):
            a, b = rng.integers(0, f.shape[0]), rng.integers(0, f.shape[1])
            e = np.zeros_like(x)
            e[a, b] = 1e-6
            fd = (d.local_value_grad(i, x + e, u)[0] - d.local_value_grad(i, x - e, u)[0]) / 2e-6
            assert fd == pytest.approx(g[a, b], rel=1e-6, abs=1e-8)


def test_noiseless_truth_is_stationary():
    """lambda = 0, alpha = 0, y = H x* -> residual 0, gradient 0, objective 0."""
    psfs, wy, wx, _, _, prm, F, O = tiny(gamma=0.0)
    A = dense_H(psfs, wy, wx)
    xs = np.random.default_rng(9).uniform(0, 1, (24, 24))
    y = (A @ xs.ravel()).reshape(20, 20)
    d = Deblur(psfs, wy, wx, y, 1.0, *F, O, prm, x0=xs)
    for i in range(len(d.facets)):
        assert np.abs(d.local_grad(i, d.x[i], d.u[i])).max() < 1e-13
    tot, data, reg, md = d.objective()
    assert abs(tot) < 1e-25 and md == 0.0


def test_single_facet_equals_centralized_pg():
    """1 facet, rho = 1: u^{k+1} = x^{k+1}, so each iteration is one projected
    gradient step on Eq. (3) (dense A, independent of oracle.c)."""
    psfs, wy, wx, y, w, prm, _, _ = tiny(lam=0.03, eps=0.1, gamma=1.5, seed=5)
    d = Deblur(psfs, wy, wx, y, w, 1, 1, 0, prm)
    A = dense_H(psfs, wy, wx)
    x = np.maximum(0, np.pad(y, 2, mode="edge"))
    u = x.copy()
    for k in range(25):
        g = (A.T @ (w.ravel() * (A @ x.ravel() - y.ravel()))).reshape(x.shape)
        g += prm.lam * tv.grad(x, prm.eps) + prm.gamma * (x - u)
        x = np.maximum(0, x - d.tau * g)
        u = x.copy() if k >= 0 else u
    d.iterate(25)
    np.testing.assert_allclose(d.x[0], x, rtol=0, atol=1e-12)
    np.testing.assert_allclose(d.u[0], x, rtol=0, atol=1e-12)


def test_fixed_point_is_consensus_minimiser():
    """D-R fixed point = argmin_{x >= 0} sum_f f_f(R_f x).
    Tikhonov-like regulariser (Huber, delta large) keeps the toy well posed."""
    psfs, wy, wx, y, w, prm, F, O = tiny(lam=0.05, eps=1e3, gamma=1.0, seed=7, kind=1)
    d = Deblur(psfs, wy, wx, y, w, *F, O, prm)
    A = dense_H(psfs, wy, wx)
    n, M = 24, 20
    blocks = []
    for f in d.facets:
        rows = [a * M + b for a in range(*f.oy) for b in range(*f.ox)]
        cols = [a * n + b for a in range(*f.ey) for b in range(*f.ex)]
        blocks.append((f, A[np.ix_(rows, cols)], y[slice(*f.oy), slice(*f.ox)].ravel(),
                       np.broadcast_to(w, y.shape)[slice(*f.oy), slice(*f.ox)].ravel()))

    def F_and_grad(xv):
        X = xv.reshape(n, n)
        val, G = 0.0, np.zeros((n, n))
        for f, Af, yf, wf in blocks:
            xf = X[slice(*f.ey), slice(*f.ex)]
            res = Af @ xf.ravel() - yf
            val += 0.5 * (wf * res * res).sum() + prm.lam * tv.value(xf, prm.eps, 1)
            G[slice(*f.ey), slice(*f.ex)] += (Af.T @ (wf * res)).reshape(xf.shape) + prm.lam * tv.grad(xf, prm.eps, 1)
        return val, G.ravel()

    res = scipy.optimize.minimize(F_and_grad, np.full(n * n, 0.5), jac=True, method="L-BFGS-B",
                                  bounds=[(0, None)] * (n * n), options=dict(maxiter=20000, ftol=1e-16, gtol=1e-12))
    xstar = res.x.reshape(n, n)
    d.iterate(6000)
    assert d.objective()[3] < 1e-8
    np.testing.assert_allclose(d.image(), xstar, rtol=0, atol=1e-6)


def test_exact_rational_full_path():
    """Every operation rational (lambda = 0, rational taps / weights / tau):
    the fp64 oracle matches an exact Fraction evaluation of the same iteration
    (dense A as H) to ~1e-14 after 4 iterations."""
    n, P, G = 12, 3, 2
    rng = np.random.default_rng(13)
    psfs = rng.integers(1, 5, (G * G, P, P)).astype(np.float64)
    psfs /= psfs.sum(axis=(1, 2), keepdims=True)     # binary-exact? not required: Fraction(float) is exact
    wy, wx = synth.hat_weights(n, G), synth.hat_weights(n, G)
    M = n - P + 1
    y = rng.integers(0, 9, (M, M)).astype(np.float64)
    w = rng.integers(1, 4, (M, M)).astype(np.float64) / 4
    prm = Params(lam=0.0, eps=1.0, gamma=0.5, rho=1.0)
    tau = 1.0 / 64
    d = Deblur(psfs, wy, wx, y, w, 2, 2, 2, prm, tau=tau)
    Fr = np.vectorize(Fraction, otypes=[object])
    A = dense_H(Fr(psfs), Fr(wy), Fr(wx), dtype=object)
    yq, wq = Fr(y), Fr(w)
    blocks = []
    for f in d.facets:
        rows = [a * M + b for a in range(*f.oy) for b in range(*f.ox)]
        cols = [a * n + b for a in range(*f.ey) for b in range(*f.ex)]
        blocks.append((A[np.ix_(rows, cols)], yq[slice(*f.oy), slice(*f.ox)].ravel(),
                       wq[slice(*f.oy), slice(*f.ox)].ravel()))
    om = [Fr(f.omega()) for f in d.facets]
    tq, gq = Fraction(tau), Fraction(prm.gamma)
    x = [Fr(a) for a in d.x]
    u = [Fr(a) for a in d.u]

    def prox(i, xi, ui):
        Af, yf, wf = blocks[i]
        r = wf * (Af.dot(xi.ravel()) - yf)
        g = Af.T.dot(r).reshape(xi.shape) + gq * om[i] * (xi - ui)
        z = xi - tq * g
        return np.vectorize(lambda v: v if v > 0 else Fraction(0), otypes=[object])(z)

    for _ in range(4):
        x, u = solver.dr_iteration((n, n), d.windows, om, x, u, prox, Fraction(1))
    d.iterate(4)
    for a, b in zip(d.x, x):
        np.testing.assert_allclose(a, b.astype(np.float64), rtol=0, atol=1e-13)
    for a, b in zip(d.u, u):
        np.testing.assert_allclose(a, b.astype(np.float64), rtol=0, atol=1e-13)


# --------------------------------------------------------------- objective
def test_objective_single_facet_is_eq3_and_additive():
    psfs, wy, wx, y, w, prm, F, O = tiny(lam=0.02, eps=0.05, seed=21)
    A = dense_H(psfs, wy, wx)
    x0 = np.random.default_rng(1).uniform(0, 1, (24, 24))
    d1 = Deblur(psfs, wy, wx, y, w, 1, 1, 0, prm, x0=x0)
    res = A @ x0.ravel() - y.ravel()
    eq3 = 0.5 * (w.ravel() * res * res).sum() + prm.lam * tv.value(x0, prm.eps)
    assert d1.objective()[0] == pytest.approx(eq3, rel=1e-12)
    d4 = Deblur(psfs, wy, wx, y, w, *F, O, prm, x0=x0)
    tot, data, reg, md = d4.objective()
    parts = 0.0
    for f in d4.facets:
        r = d4.op.H_window(x0[slice(*f.ey), slice(*f.ex)], f.ey[0], f.ex[0]) - y[slice(*f.oy), slice(*f.ox)]
        parts += 0.5 * (w[slice(*f.oy), slice(*f.ox)] * r * r).sum()
        parts += prm.lam * tv.value(x0[slice(*f.ey), slice(*f.ex)], prm.eps)
    assert tot == pytest.approx(parts, rel=1e-12) and md == 0.0


def test_nonnegativity_and_zero_data():
    psfs, wy, wx, y, w, prm, F, O = tiny(lam=0.1, seed=2)
    d = Deblur(psfs, wy, wx, y - 0.8, w, *F, O, prm)
    for _ in range(5):
        d.iterate(1)
        assert min(a.min() for a in d.x) >= 0.0
    z = Deblur(psfs, wy, wx, 0 * y, w, *F, O, prm, x0=np.zeros((24, 24)))
    z.iterate(5)
    assert max(np.abs(a).max() for a in z.x) == 0.0 and max(np.abs(a).max() for a in z.u) == 0.0


def test_default_tau_bounds_dense_norm():
    psfs, wy, wx, y, w, prm, F, O = tiny(seed=4)
    A = dense_H(psfs, wy, wx)
    L_true = float(np.max(w)) * np.linalg.norm(A, 2) ** 2 + prm.gamma
    tau = solver.default_tau(psfs, wy, wx, float(np.max(w)), prm.lam, prm.eps, prm.reg_kind, prm.gamma)
    assert 1.0 / tau >= L_true * (1 - 1e-12)
