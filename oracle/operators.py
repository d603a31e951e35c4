"""Blur operator H (PSF interpolation) and adjoint H^T in fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Thin wrappers around the
direct double sums of oracle.c; the window forms are the facet-local H_f of
SURVEY R1 (rows = observed block O_f, columns = estimate block P_f).
"""
from __future__ import annotations

import numpy as np

from . import _clib


class Operator:
    """H for an N_y x N_x scene with a G_y x G_x grid of P x P PSFs.

    psfs [G_y*G_x, P, P] (k = p*G_x + q), wy [G_y, N_y], wx [G_x, N_x]; every
    input is promoted to fp64 once (the fp32 values the GPU also receives).
    """

    def __init__(self, psfs, wy, wx):
        self.psfs = np.ascontiguousarray(psfs, dtype=np.float64)
        self.wy = np.ascontiguousarray(wy, dtype=np.float64)
        self.wx = np.ascontiguousarray(wx, dtype=np.float64)
        self.K, self.P, P2 = self.psfs.shape
        assert self.P == P2 and self.P % 2 == 1
        self.gy, self.Ny = self.wy.shape
        self.gx, self.Nx = self.wx.shape
        assert self.K == self.gy * self.gx
        self.c = (self.P - 1) // 2
        self.My = self.Ny - self.P + 1
        self.Mx = self.Nx - self.P + 1

    def _common(self):
        return (self.Ny, self.Nx, self.P, self.gy, self.gx,
                _clib.dptr(self.psfs), _clib.dptr(self.wy), _clib.dptr(self.wx))

    # --- facet-local forms -------------------------------------------------
    def H_window(self, x_win: np.ndarray, e0y: int, e0x: int) -> np.ndarray:
        """H_f x_f: x_win is the estimate block at global origin (e0y, e0x);
        returns the observed block (rows e0y.., cols e0x.. in observed coords)."""
        x = np.ascontiguousarray(x_win, dtype=np.float64)
        ny, nx = x.shape
        out = np.zeros((ny - self.P + 1, nx - self.P + 1))
        _clib.lib().orc_H_window(*self._common(), e0y, e0x, ny, nx, _clib.dptr(x), _clib.dptr(out))
        return out

    def HT_window(self, r_win: np.ndarray, e0y: int, e0x: int) -> np.ndarray:
        """H_f^T r_f: r_win is the observed block at global observed origin
        (e0y, e0x) (zero outside it); returns the estimate block."""
        r = np.ascontiguousarray(r_win, dtype=np.float64)
        my, mx = r.shape
        ny, nx = my + self.P - 1, mx + self.P - 1
        g = np.zeros((ny, nx))
        _clib.lib().orc_HT_window(*self._common(), e0y, e0x, ny, nx, _clib.dptr(r), _clib.dptr(g))
        return g

    # --- global forms ------------------------------------------------------
    def H(self, x: np.ndarray) -> np.ndarray:
        assert x.shape == (self.Ny, self.Nx)
        return self.H_window(x, 0, 0)

    def HT(self, r: np.ndarray) -> np.ndarray:
        assert r.shape == (self.My, self.Mx)
        return self.HT_window(r, 0, 0)

    def H_points(self, x: np.ndarray, oi, oj) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        oi = np.ascontiguousarray(oi, dtype=np.int64)
        oj = np.ascontiguousarray(oj, dtype=np.int64)
        out = np.zeros(len(oi))
        _clib.lib().orc_H_points(*self._common(), _clib.dptr(x), len(oi), _clib.lptr(oi), _clib.lptr(oj),
                                 _clib.dptr(out))
        return out

    def HT_points(self, r: np.ndarray, ei, ej) -> np.ndarray:
        r = np.ascontiguousarray(r, dtype=np.float64)
        ei = np.ascontiguousarray(ei, dtype=np.int64)
        ej = np.ascontiguousarray(ej, dtype=np.int64)
        out = np.zeros(len(ei))
        _clib.lib().orc_HT_points(*self._common(), _clib.dptr(r), len(ei), _clib.lptr(ei), _clib.lptr(ej),
                                  _clib.dptr(out))
        return out
