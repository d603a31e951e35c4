"""Pins for oracle/vmlmb.py (the VMLM-B reading V1-V6) and its use
as the Local-Solver, CPU only.

  closed forms  1/2|x - c|^2 with x >= 0 -> max(c, 0) (KKT), in one iteration
                with h0 = 1 (SPEC local-solver examples, bound version)
  textbook      2-D Rosenbrock -> (1, 1) within 1e-6 in <= 200 iterations
  brute force   random strictly convex quadratic, x >= 0, 6 variables: the
                minimiser equals the best of all 2^6 active-set KKT solutions
  invariants    feasibility and monotone descent of every accepted iterate
  Local-Solver  the VMLM-B prox of a deblurring facet converges to the same
                unique minimiser as many projected-gradient steps (R2)
"""
import itertools

import numpy as np

import synth
from oracle import from_problem, vmlmb


def test_projection_of_a_quadratic():
    c = np.array([1.5, -2.0, 0.3, -0.1, 4.0])
    x, rep = vmlmb.minimize(lambda x: (0.5 * float(((x - c) ** 2).sum()), x - c), np.ones(5), h0=1.0, max_iter=3)
    np.testing.assert_allclose(x, np.maximum(c, 0), rtol=0, atol=1e-12)
    assert rep.iterations <= 3


def test_rosenbrock():
    def fg(z):
        a, b = z
        f = (1 - a) ** 2 + 100 * (b - a * a) ** 2
        g = np.array([-2 * (1 - a) - 400 * a * (b - a * a), 200 * (b - a * a)])
        return f, g
    x, rep = vmlmb.minimize(fg, np.array([-1.2, 1.0]), h0=1e-3, max_iter=200, gtol=1e-10)
    np.testing.assert_allclose(x, [1.0, 1.0], rtol=0, atol=1e-6)


def test_nonnegative_quadratic_vs_active_set_enumeration():
    rng = np.random.default_rng(3)
    for trial in range(5):
        n = 6
        A = rng.standard_normal((n, n))
        Q = A @ A.T + 0.5 * np.eye(n)
        b = rng.standard_normal(n) * 2
        fg = lambda x: (0.5 * float(x @ Q @ x) - float(b @ x), Q @ x - b)
        best, bestf = None, np.inf
        for act in itertools.product([0, 1], repeat=n):          # 1 = held at the bound 0
            free = [i for i in range(n) if not act[i]]
            x = np.zeros(n)
            if free:
                x[free] = np.linalg.solve(Q[np.ix_(free, free)], b[free])
            g = Q @ x - b
            if np.all(x >= -1e-12) and all(g[i] >= -1e-10 for i in range(n) if act[i]):
                fx = fg(x)[0]
                if fx < bestf:
                    best, bestf = x, fx
        x, rep = vmlmb.minimize(fg, np.ones(n), h0=1.0 / np.linalg.eigvalsh(Q).max(), max_iter=500, gtol=1e-13)
        np.testing.assert_allclose(x, best, rtol=0, atol=1e-8)


def test_feasible_monotone_descent():
    pb = synth.make_config(2, n=160, facets=(1, 1), overlap=0)
    o = from_problem(pb)
    u = o.u[0]
    seen = []

    def fg(w):
        assert np.all(w >= 0)
        val, g = o.local_value_grad(0, w, u)
        seen.append(val)
        return val, g
    x, rep = vmlmb.minimize(fg, o.x[0], h0=o.tau, max_iter=15)
    accepted = [seen[0]]
    for v in seen[1:]:
        if v <= accepted[-1]:
            accepted.append(v)
    assert rep.reason in ("budget", "converged") and len(accepted) >= rep.iterations
    assert rep.f < seen[0]


def test_local_solver_reaches_the_pg_minimiser():
    """The facet prox min_{w >= 0} f_i(w) + 1/2|w - u|^2_alpha is strictly convex:
    VMLM-B and (many) projected-gradient steps reach the same point."""
    pb = synth.make_config(1, n=40, facets=(1, 1), overlap=0)
    pb.lam = 0.05
    pb.eps = 0.05
    o = from_problem(pb)
    u = o.u[0] + 0.01
    x_vm, rep = vmlmb.minimize(lambda w: o.local_value_grad(0, w, u), o.x[0], h0=o.tau, max_iter=200)
    x_pg = o.x[0].copy()
    for _ in range(1500):
        x_pg = np.maximum(0.0, x_pg - o.tau * o.local_value_grad(0, x_pg, u)[1])
    assert rep.evaluations < 400                       # converges, then stalls at the rounding floor
    assert np.linalg.norm(x_vm - x_pg) <= 1e-8 * np.linalg.norm(x_pg)


def test_dr_with_vmlmb_budget_schedule():
    """Algorithm 1 with VMLM-B Local-Solvers (budget 10 + 10 k)
    decreases the objective faster than one projected-gradient step per iteration."""
    pb = synth.make_config(2, n=120, facets=(2, 2), overlap=10)
    pb.local_solver, pb.inner_steps, pb.inner_increment = 1, 10, 10
    a = from_problem(pb)
    a.iterate(3)
    pb.local_solver, pb.inner_steps, pb.inner_increment = 0, 1, 0
    b = from_problem(pb)
    b.iterate(3)
    assert a.objective()[0] < b.objective()[0]
