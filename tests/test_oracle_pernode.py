"""Pins for the oracle's per-node operator mode (DESIGN.md §2,
operator_mode 1): the paper's node model, PAPER.md:109 (H_i = C_i calH_i, the
valid convolution with the node's own PSF h_i), :118 (one PSF and one block per
node), :206 (alpha_i = gamma omega_i with omega_i the interpolation weights).

  operator    H_i = scipy.signal.convolve2d(x_i, h_i, "valid"), H_i^T r =
              correlate2d(r, h_i, "full")  (library routines, independent of oracle.c)
  weights     omega_i = wy[a] (x) wx[b] on the facet's estimate block; every
              estimate pixel has a positive weight sum; the blend of a
              consistent state returns it exactly
  special     one node (G = F = 1): identical to operator mode 0 (one PSF, unit
              weights) step by step
  fixed pt.   the D-R fixed point equals argmin_{x >= 0} sum_i f_i(R_i x) with the
              per-node dense operators (scipy L-BFGS-B)
and of the independent baseline (NEXT-3): one facet = Algorithm 1
with gamma = 0; on several facets every facet equals its own one-facet problem.
"""
import numpy as np
import scipy.optimize
import scipy.signal

import synth
from oracle import tv
from oracle.solver import Deblur, Params
from tests.dense_ref import dense_H


def tiny_nodes(n=30, P=5, G=3, lam=0.0, eps=1e-3, gamma=2.0, seed=0, kind=0, O=None):
    rng = np.random.default_rng(seed)
    psfs = rng.uniform(0, 1, (G * G, P, P))
    psfs /= psfs.sum(axis=(1, 2), keepdims=True)
    wy, wx = synth.hat_weights(n, G), synth.hat_weights(n, G)
    M = n - P + 1
    y = rng.uniform(0.1, 1.0, (M, M))
    w = rng.uniform(0.5, 2.0, (M, M))
    if O is None:
        O = max(0, M // G - (P - 1))
        O -= O % 2
    prm = Params(lam=lam, eps=eps, gamma=gamma, rho=1.0, reg_kind=kind)
    return psfs, wy, wx, y, w, prm, O


def test_per_node_operator_is_valid_convolution():
    psfs, wy, wx, y, w, prm, O = tiny_nodes(n=40, P=7, G=3, seed=1)
    d = Deblur(psfs, wy, wx, y, w, 3, 3, O, prm, operator_mode=1)
    rng = np.random.default_rng(2)
    for i, f in enumerate(d.facets):
        h = psfs[f.fy * 3 + f.fx]
        xf = rng.uniform(0, 1, f.shape)
        np.testing.assert_allclose(d.ops[i].H_window(xf, f.ey[0], f.ex[0]),
                                   scipy.signal.convolve2d(xf, h, mode="valid"), rtol=0, atol=1e-13)
        r = rng.standard_normal(f.oshape)
        np.testing.assert_allclose(d.ops[i].HT_window(r, f.oy[0], f.ox[0]),
                                   scipy.signal.correlate2d(r, h, mode="full"), rtol=0, atol=1e-13)


def test_per_node_weights_and_consistent_blend():
    psfs, wy, wx, y, w, prm, O = tiny_nodes(n=40, P=7, G=3, seed=3)
    d = Deblur(psfs, wy, wx, y, w, 3, 3, O, prm, operator_mode=1)
    den = np.zeros(d.shape)
    for f, om in zip(d.facets, d.omegas):
        np.testing.assert_array_equal(om, np.outer(wy[f.fy, f.ey[0]:f.ey[1]], wx[f.fx, f.ex[0]:f.ex[1]]))
        den[f.ey[0]:f.ey[1], f.ex[0]:f.ex[1]] += om
    assert den.min() > 0                                    # P:201 divides by it
    X = np.random.default_rng(4).uniform(0, 1, d.shape)
    d.x = [X[win].copy() for win in d.windows]
    np.testing.assert_allclose(d.image(), X, rtol=1e-14, atol=0)


def test_single_node_equals_mode0_single_psf():
    psfs, wy, wx, y, w, prm, _ = tiny_nodes(n=24, P=5, G=1, lam=0.05, eps=0.2, seed=5)
    a = Deblur(psfs, wy, wx, y, w, 1, 1, 0, prm, operator_mode=0)
    b = Deblur(psfs, wy, wx, y, w, 1, 1, 0, prm, operator_mode=1)
    a.iterate(7)
    b.iterate(7)
    np.testing.assert_array_equal(a.x[0], b.x[0])
    np.testing.assert_array_equal(a.u[0], b.u[0])
    assert a.objective() == b.objective()


def test_per_node_fixed_point_is_consensus_minimiser():
    """D-R fixed point = argmin_{x >= 0} sum_i f_i(R_i x) with the per-node dense
    operators (circulant rows, dense_ref) -- the alpha_i = gamma omega_i weights
    shape the path, not the fixed point."""
    n, P, G = 24, 5, 2
    psfs, wy, wx, y, w, prm, O = tiny_nodes(n=n, P=P, G=G, lam=0.05, eps=1e3, gamma=1.0, seed=7, kind=1)
    d = Deblur(psfs, wy, wx, y, w, G, G, O, prm, operator_mode=1)
    M = n - P + 1
    ones = np.ones((1, n))
    blocks = []
    for f in d.facets:
        A = dense_H(psfs[f.fy * G + f.fx][None], ones, ones)
        rows = [a * M + b for a in range(*f.oy) for b in range(*f.ox)]
        cols = [a * n + b for a in range(*f.ey) for b in range(*f.ex)]
        blocks.append((f, A[np.ix_(rows, cols)], y[slice(*f.oy), slice(*f.ox)].ravel(),
                       w[slice(*f.oy), slice(*f.ox)].ravel()))

    def F_and_grad(xv):
        X = xv.reshape(n, n)
        val, Gr = 0.0, np.zeros((n, n))
        for f, Af, yf, wf in blocks:
            xf = X[slice(*f.ey), slice(*f.ex)]
            res = Af @ xf.ravel() - yf
            val += 0.5 * (wf * res * res).sum() + prm.lam * tv.value(xf, prm.eps, 1)
            Gr[slice(*f.ey), slice(*f.ex)] += (Af.T @ (wf * res)).reshape(xf.shape) + prm.lam * tv.grad(xf, prm.eps, 1)
        return val, Gr.ravel()

    res = scipy.optimize.minimize(F_and_grad, np.full(n * n, 0.5), jac=True, method="L-BFGS-B",
                                  bounds=[(0, None)] * (n * n), options=dict(maxiter=20000, ftol=1e-16, gtol=1e-12))
    xstar = res.x.reshape(n, n)
    d.iterate(6000)
    assert d.objective()[3] < 1e-8
    np.testing.assert_allclose(d.image(), xstar, rtol=0, atol=1e-6)


def test_per_node_synth_geometry():
    """synth.per_node: F = G, every estimate pixel in <= 2 facets per axis, blocks
    spanning about three grid points."""
    pb = synth.per_node(synth.make_config(2, n=300))
    assert (pb.fy, pb.fx) == (pb.gy, pb.gx) and pb.operator_mode == 1
    from oracle import geometry
    pl = geometry.axis_plan(pb.my, pb.fy, pb.overlap, pb.P)
    for k in range(1, len(pl) - 1):
        assert pl[k - 1].e_hi <= pl[k + 1].e_lo
    cell = pb.ny / pb.gy
    assert all((f.e_hi - f.e_lo) > 1.5 * cell for f in pl[1:-1])


# --------------------------------------------------------- independent baseline (NEXT-3)
def test_independent_single_facet_equals_dr_with_gamma0():
    """One facet: the independent baseline (alpha = 0, no consensus) is Algorithm 1
    with gamma = 0 step by step (the prox term vanishes, u never enters)."""
    psfs, wy, wx, y, w, prm, _ = tiny_nodes(n=24, P=5, G=2, lam=0.05, eps=0.2, seed=11)
    import dataclasses
    a = Deblur(psfs, wy, wx, y, w, 1, 1, 0, dataclasses.replace(prm, gamma=0.0))
    b = Deblur(psfs, wy, wx, y, w, 1, 1, 0, prm, independent=True)
    assert a.tau == b.tau
    a.iterate(6)
    b.iterate(6)
    np.testing.assert_array_equal(a.x[0], b.x[0])


def test_independent_facets_are_separate_problems():
    """Independent baseline on 2x2 facets: facet i's iterates equal a one-facet
    problem on facet i's own data (its observed block, the weights restricted
    to its estimate block) -- the blocks never talk."""
    psfs, wy, wx, y, w, prm, _ = tiny_nodes(n=40, P=5, G=2, lam=0.05, eps=0.2, seed=12)
    d = Deblur(psfs, wy, wx, y, w, 2, 2, 6, prm, independent=True)
    d.iterate(5)
    for i, f in enumerate(d.facets):
        s = Deblur(psfs, wy[:, f.ey[0]:f.ey[1]], wx[:, f.ex[0]:f.ex[1]], y[f.oy[0]:f.oy[1], f.ox[0]:f.ox[1]],
                   w[f.oy[0]:f.oy[1], f.ox[0]:f.ox[1]], 1, 1, 0, prm, tau=d.tau,
                   x0=np.maximum(0.0, np.pad(y, 2, mode="edge"))[f.ey[0]:f.ey[1], f.ex[0]:f.ex[1]],   # A6
                   independent=True)
        s.iterate(5)
        np.testing.assert_allclose(d.x[i], s.x[0], rtol=0, atol=1e-13)
