"""Independent dense-matrix construction of the paper's blur operator (tests only).

Builds y = R sum_k Z_k H_k W_k C_k x literally as matrices on
tiny images, with H_k = C'_k calH_k, calH_k the 2-D CIRCULAR convolution
matrix of h_k ("circular convolution matrices formed from PSFs
h_i" followed by "chopping operators, which restrict the convolution results
to the valid regions").  This route shares nothing with oracle.c's direct sum:
it never forms the valid-region index arithmetic, it selects rows of circulant
matrices instead.  Any dtype (float64 or object/Fraction) works.
"""
from __future__ import annotations

import numpy as np


def circulant2d(h: np.ndarray, ny: int, nx: int, dtype=np.float64) -> np.ndarray:
    """Matrix of x -> h (*) x with circular boundary, PSF centre at (c, c):
    (calH x)(u, v) = sum_{a,b} h[a,b] x((u - a + c) mod ny, (v - b + c) mod nx)."""
    P = h.shape[0]
    c = (P - 1) // 2
    n = ny * nx
    A = np.zeros((n, n), dtype=dtype)
    if dtype == object:
        A[:] = 0
    for u in range(ny):
        for v in range(nx):
            row = u * nx + v
            for a in range(P):
                for b in range(P):
                    s = ((u - a + c) % ny) * nx + ((v - b + c) % nx)
                    A[row, s] = A[row, s] + h[a, b]
    return A


def dense_H(psfs: np.ndarray, wy: np.ndarray, wx: np.ndarray, dtype=np.float64) -> np.ndarray:
    """A = R sum_k calH_k diag(omega_k), omega_k = wy[p] (x) wx[q], R = valid chop."""
    K, P, _ = psfs.shape
    gy, ny = wy.shape
    gx, nx = wx.shape
    c = (P - 1) // 2
    n = ny * nx
    S = np.zeros((n, n), dtype=dtype)
    if dtype == object:
        S[:] = 0
    for p in range(gy):
        for q in range(gx):
            om = np.outer(wy[p], wx[q]).ravel()
            Ck = circulant2d(psfs[p * gx + q], ny, nx, dtype)
            S = S + Ck * om[None, :]          # calH_k W_k
    rows = [u * nx + v for u in range(c, ny - c) for v in range(c, nx - c)]   # R: sensor = valid region
    return S[rows]
