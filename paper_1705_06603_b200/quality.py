"""Image-quality metrics of the paper's evaluation (Sec. IV-C): SNR in dB
and SSIM.  Host-side numpy on finished images (not part of the iteration's hot path).

The paper names both metrics but defines neither.  Readings:
  snr(ref, est)  = 10 log10(|ref|^2 / |ref - est|^2); est == ref -> the capped value 300 dB
  ssim(ref, est) = mean SSIM (Wang et al. 2004) with an 11 x 11 Gaussian window of
                   sigma 1.5, K1 = 0.01, K2 = 0.03 and the given dynamic range L,
                   C1 = (K1 L)^2, C2 = (K2 L)^2; windows are the 'valid' 11 x 11 placements
                   (no padding), so a constant image pair gives the closed-form luminance term.
"""
from __future__ import annotations

import math

import numpy as np

SNR_CAP_DB = 300.0


def snr(ref, est) -> float:
    ref = np.asarray(ref, np.float64)
    est = np.asarray(est, np.float64)
    if ref.shape != est.shape:
        raise ValueError(f"shape mismatch {ref.shape} vs {est.shape}")
    sig = float((ref * ref).sum())
    if sig == 0.0:
        raise ValueError("all-zero reference")
    err = float(((ref - est) ** 2).sum())
    if err == 0.0:
        return SNR_CAP_DB
    return min(SNR_CAP_DB, 10.0 * math.log10(sig / err))


def _gauss_window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    t = np.arange(size, dtype=np.float64) - (size - 1) / 2.0
    g = np.exp(-0.5 * (t / sigma) ** 2)
    g /= g.sum()
    return np.outer(g, g)


def _filter_valid(z: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Weighted mean of z over every valid window placement (separable: rows then cols)."""
    g = w.sum(axis=1)                       # the 1-D Gaussian (w is its outer product)
    k = g.size
    rows = sum(g[i] * z[i:z.shape[0] - k + 1 + i, :] for i in range(k))
    return sum(g[j] * rows[:, j:rows.shape[1] - k + 1 + j] for j in range(k))


def ssim(ref, est, dynamic_range: float, size: int = 11, sigma: float = 1.5, k1: float = 0.01,
         k2: float = 0.03) -> float:
    a = np.asarray(ref, np.float64)
    b = np.asarray(est, np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch {a.shape} vs {b.shape}")
    if not dynamic_range > 0:
        raise ValueError("dynamic_range must be > 0")
    if min(a.shape) < size:
        raise ValueError(f"images smaller than the {size} x {size} window")
    w = _gauss_window(size, sigma)
    c1, c2 = (k1 * dynamic_range) ** 2, (k2 * dynamic_range) ** 2
    ma, mb = _filter_valid(a, w), _filter_valid(b, w)
    va = _filter_valid(a * a, w) - ma * ma
    vb = _filter_valid(b * b, w) - mb * mb
    cab = _filter_valid(a * b, w) - ma * mb
    s = ((2 * ma * mb + c1) * (2 * cab + c2)) / ((ma * ma + mb * mb + c1) * (va + vb + c2))
    return float(s.mean())
