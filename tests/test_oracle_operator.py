"""Pins for the oracle's H / H^T (CPU, -m "not gpu").

Each pin ties oracle.c to something other than itself:
  * the paper's matrix form (dense circulant construction, tests/dense_ref.py)
  * a library routine (scipy.signal.convolve2d 'valid') for identical PSFs
  * the identity for delta PSFs, constants for unit-sum PSFs
  * the FFT route of PAPER.md:109 (numpy.fft circular convolution + chop)
  * the adjoint identity <Hx, r> = <x, H^T r>
  * the facet restriction of SURVEY R1 (window == rows/cols of the dense A)
"""
import numpy as np
import pytest
import scipy.signal

import synth
from oracle import Operator
from tests.dense_ref import dense_H


def rand_inputs(rng, ny, nx, P, gy, gx, nonneg=True):
    psfs = rng.uniform(0.0 if nonneg else -1.0, 1.0, (gy * gx, P, P))
    psfs /= psfs.sum(axis=(1, 2), keepdims=True)
    wy = synth.hat_weights(ny, gy)
    wx = synth.hat_weights(nx, gx)
    return psfs, wy, wx


CASES = [(9, 9, 3, 1, 1), (12, 11, 3, 2, 2), (14, 13, 5, 2, 3), (17, 15, 7, 3, 2), (20, 24, 5, 4, 4)]


@pytest.mark.parametrize("ny,nx,P,gy,gx", CASES)
def test_H_matches_dense_paper_matrix(ny, nx, P, gy, gx):
    """PAPER.md:107/109 matrix form vs the direct sum, and H^T = A^T."""
    rng = np.random.default_rng(ny * 100 + nx)
    psfs, wy, wx = rand_inputs(rng, ny, nx, P, gy, gx, nonneg=False)
    op = Operator(psfs, wy, wx)
    A = dense_H(psfs, wy, wx)
    x = rng.standard_normal((ny, nx))
    r = rng.standard_normal((ny - P + 1, nx - P + 1))
    np.testing.assert_allclose(op.H(x).ravel(), A @ x.ravel(), rtol=0, atol=1e-13)
    np.testing.assert_allclose(op.HT(r).ravel(), A.T @ r.ravel(), rtol=0, atol=1e-13)


@pytest.mark.parametrize("P,G", [(3, 1), (5, 2), (15, 3), (31, 2)])
def test_identical_psfs_reduce_to_convolve2d(P, G):
    """Identical PSFs + partition-of-unity weights -> plain valid convolution
    (S:202), checked against scipy.signal.convolve2d(mode='valid')."""
    rng = np.random.default_rng(P)
    n = 3 * P + 7
    h = rng.uniform(0, 1, (P, P))
    h /= h.sum()
    psfs = np.repeat(h[None], G * G, axis=0)
    op = Operator(psfs, synth.hat_weights(n, G), synth.hat_weights(n, G))
    x = rng.uniform(0, 1, (n, n))
    ref = scipy.signal.convolve2d(x, h, mode="valid")
    np.testing.assert_allclose(op.H(x), ref, rtol=1e-13, atol=1e-14)
    # adjoint of valid convolution = full correlation (convolve2d with the flipped kernel)
    r = rng.standard_normal(ref.shape)
    np.testing.assert_allclose(op.HT(r), scipy.signal.convolve2d(r, h[::-1, ::-1], mode="full"),
                               rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("P,G", [(3, 2), (7, 3), (15, 2)])
def test_delta_psfs_are_crop(P, G):
    """Delta PSFs -> H x = x[c:N-c, c:N-c]; H^T r embeds r."""
    n = 40
    c = (P - 1) // 2
    psfs = np.zeros((G * G, P, P))
    psfs[:, c, c] = 1.0
    op = Operator(psfs, synth.hat_weights(n, G), synth.hat_weights(n, G))
    x = np.random.default_rng(1).uniform(0, 1, (n, n))
    np.testing.assert_allclose(op.H(x), x[c:n - c, c:n - c], rtol=0, atol=1e-15)
    r = x[c:n - c, c:n - c]
    g = op.HT(r)
    assert np.all(g[:c] == 0) and np.all(g[:, :c] == 0)
    np.testing.assert_allclose(g[c:n - c, c:n - c], r, rtol=0, atol=1e-15)


def test_unit_sum_psfs_preserve_constants():
    """Identical unit-sum PSFs map a constant image to the same constant;
    H^T 1 <= 1 for non-negative unit-sum PSFs."""
    rng = np.random.default_rng(5)
    P, G, n = 9, 3, 50
    h = rng.uniform(0, 1, (P, P))
    h /= h.sum()
    op = Operator(np.repeat(h[None], G * G, 0), synth.hat_weights(n, G), synth.hat_weights(n, G))
    np.testing.assert_allclose(op.H(np.full((n, n), 3.25)), 3.25, rtol=1e-14)
    psfs, wy, wx = rand_inputs(rng, n, n, P, G, G)
    op2 = Operator(psfs, wy, wx)
    assert op2.HT(np.ones((op2.My, op2.Mx))).max() <= 1 + 1e-14


def test_fft_route_of_paper():
    """H_i = C_i calH_i evaluated in the Fourier domain (circular
    convolution by FFT, then chop to the valid region) equals the direct sum."""
    rng = np.random.default_rng(11)
    ny, nx, P, gy, gx = 64, 48, 15, 3, 2
    psfs, wy, wx = rand_inputs(rng, ny, nx, P, gy, gx)
    x = rng.uniform(0, 1, (ny, nx))
    c = (P - 1) // 2
    acc = np.zeros((ny, nx))
    for p in range(gy):
        for q in range(gx):
            emb = np.zeros((ny, nx))
            emb[:P, :P] = psfs[p * gx + q]
            emb = np.roll(emb, (-c, -c), axis=(0, 1))       # centre the PSF at (0, 0)
            xw = np.outer(wy[p], wx[q]) * x
            acc += np.real(np.fft.ifft2(np.fft.fft2(xw) * np.fft.fft2(emb)))
    ref = acc[c:ny - c, c:nx - c]
    np.testing.assert_allclose(Operator(psfs, wy, wx).H(x), ref, rtol=0, atol=1e-13)


@pytest.mark.parametrize("P,G", [(5, 2), (15, 3), (31, 4)])
def test_adjoint_identity(P, G):
    rng = np.random.default_rng(P * 7 + G)
    n = 2 * P + 37
    psfs, wy, wx = rand_inputs(rng, n, n + 5, P, G, G, nonneg=False)
    op = Operator(psfs, wy, wx)
    x = rng.standard_normal((n, n + 5))
    r = rng.standard_normal((op.My, op.Mx))
    lhs = float((op.H(x) * r).sum())
    rhs = float((x * op.HT(r)).sum())
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)


def test_window_is_restriction_of_dense():
    """H_f = rows O_f, cols P_f of the global A; H_f^T = its transpose."""
    rng = np.random.default_rng(3)
    ny, nx, P, gy, gx = 19, 21, 5, 3, 3
    psfs, wy, wx = rand_inputs(rng, ny, nx, P, gy, gx, nonneg=False)
    op = Operator(psfs, wy, wx)
    A = dense_H(psfs, wy, wx)
    My, Mx = op.My, op.Mx
    for (oy0, oy1, ox0, ox1) in [(0, 7, 2, 11), (4, My, 0, Mx), (6, 9, 5, 6)]:
        ey0, ey1, ex0, ex1 = oy0, oy1 + P - 1, ox0, ox1 + P - 1
        rows = [i * Mx + j for i in range(oy0, oy1) for j in range(ox0, ox1)]
        cols = [p * nx + q for p in range(ey0, ey1) for q in range(ex0, ex1)]
        Af = A[np.ix_(rows, cols)]
        xf = rng.standard_normal((ey1 - ey0, ex1 - ex0))
        rf = rng.standard_normal((oy1 - oy0, ox1 - ox0))
        np.testing.assert_allclose(op.H_window(xf, ey0, ex0).ravel(), Af @ xf.ravel(), atol=1e-13, rtol=0)
        np.testing.assert_allclose(op.HT_window(rf, ey0, ex0).ravel(), Af.T @ rf.ravel(), atol=1e-13, rtol=0)


def test_points_match_full():
    rng = np.random.default_rng(8)
    n, P, G = 70, 15, 3
    psfs, wy, wx = rand_inputs(rng, n, n, P, G, G)
    op = Operator(psfs, wy, wx)
    x = rng.uniform(0, 1, (n, n))
    r = rng.standard_normal((op.My, op.Mx))
    hx, g = op.H(x), op.HT(r)
    oi, oj = rng.integers(0, op.My, 50), rng.integers(0, op.Mx, 50)
    np.testing.assert_allclose(op.H_points(x, oi, oj), hx[oi, oj], rtol=1e-13, atol=1e-14)
    ei, ej = rng.integers(0, n, 50), rng.integers(0, n, 50)
    np.testing.assert_allclose(op.HT_points(r, ei, ej), g[ei, ej], rtol=1e-12, atol=1e-13)
