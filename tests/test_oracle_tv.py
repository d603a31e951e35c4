"""Pins for oracle/tv.py: closed forms (tests/golden), adjointness, FD gradients."""
import json
import os

import numpy as np
import pytest

from oracle import tv

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_finite_diff_golden():
    g = GOLD["finite_diff_circular"]
    x = np.array([g["x_row"]], dtype=np.float64)
    dy, dx = tv.D(x)
    np.testing.assert_array_equal(dx[0], g["dx_row"])
    np.testing.assert_array_equal(dy, 0.0 * x)   # one row: circular vertical difference vanishes


@pytest.mark.parametrize("key", ["huber_branch_boundary", "huber_linear_branch"])
def test_huber_golden(key):
    g = GOLD[key]
    dy, dx = np.array([[g["g"][0]]]), np.array([[g["g"][1]]])
    assert tv.phi(dy, dx, g["delta"], kind=1)[0, 0] == pytest.approx(g["phi"], rel=1e-15)


def test_smoothed_tv_zero():
    z = np.zeros((3, 3))
    assert tv.phi(z, z, 1e-3, 0).max() == 0.0
    py, px = tv.psi(z, z, 1e-3, 0)
    assert np.all(py == 0) and np.all(px == 0)
    # large-gradient limit: phi -> |g| - eps
    big = np.array([[1e3]])
    assert tv.phi(big, 0 * big, 1e-3, 0)[0, 0] == pytest.approx(1e3 - 1e-3, rel=1e-12)


@pytest.mark.parametrize("boundary", [0, 1])
def test_D_adjoint(boundary):
    rng = np.random.default_rng(boundary)
    x = rng.standard_normal((7, 9))
    vy, vx = rng.standard_normal((7, 9)), rng.standard_normal((7, 9))
    dy, dx = tv.D(x, boundary)
    lhs = (dy * vy).sum() + (dx * vx).sum()
    rhs = (x * tv.Dt(vy, vx, boundary)).sum()
    assert abs(lhs - rhs) < 1e-12


def test_D_norm_bound():
    """|D|^2 <= 8 (used by the step bound A4'): power iteration on D^T D."""
    rng = np.random.default_rng(0)
    x = rng.standard_normal((16, 16))
    for _ in range(300):
        x = tv.Dt(*tv.D(x))
        x /= np.linalg.norm(x)
    lam = np.linalg.norm(tv.Dt(*tv.D(x)))
    assert lam <= 8.0 + 1e-9 and lam > 7.5


@pytest.mark.parametrize("kind,eps,boundary", [(0, 1e-3, 0), (0, 0.3, 1), (1, 0.5, 0), (1, 2.0, 1)])
def test_tv_gradient_fd(kind, eps, boundary):
    rng = np.random.default_rng(kind * 10 + boundary)
    x = rng.uniform(0, 1, (6, 7))
    g = tv.grad(x, eps, kind, boundary)
    h = 1e-6
    for _ in range(12):
        i, j = rng.integers(0, 6), rng.integers(0, 7)
        e = np.zeros_like(x)
        e[i, j] = h
        fd = (tv.value(x + e, eps, kind, boundary) - tv.value(x - e, eps, kind, boundary)) / (2 * h)
        assert fd == pytest.approx(g[i, j], rel=1e-5, abs=1e-7)


def test_psi_lipschitz():
    rng = np.random.default_rng(2)
    for kind, eps in [(0, 1e-3), (1, 0.7)]:
        a = rng.standard_normal((2, 500)) * 0.01
        b = a + rng.standard_normal((2, 500)) * 1e-4
        pa, pb = np.array(tv.psi(a[0], a[1], eps, kind)), np.array(tv.psi(b[0], b[1], eps, kind))
        ratio = np.linalg.norm(pa - pb, axis=0) / np.linalg.norm(a - b, axis=0)
        assert ratio.max() <= tv.lipschitz_psi(eps, kind) * (1 + 1e-9)
