"""Pins of the SNR / SSIM evaluation metrics (readings SPEC S:583-598):
closed forms, constructed ratios, invariants and a per-window brute force."""
import math

import numpy as np
import pytest

from paper_1705_06603_b200 import quality as Q


def test_snr_closed_forms():
    rng = np.random.default_rng(0)
    ref = rng.uniform(0.1, 2.0, (40, 30))
    assert Q.snr(ref, ref) == Q.SNR_CAP_DB                         # est == ref: capped
    assert Q.snr(ref, np.zeros_like(ref)) == pytest.approx(0.0, abs=1e-12)   # error energy = signal energy
    n = rng.standard_normal(ref.shape)
    n *= math.sqrt((ref ** 2).sum() / 10.0 / (n ** 2).sum())      # |n|^2 = |ref|^2 / 10
    assert Q.snr(ref, ref + n) == pytest.approx(10.0, abs=1e-9)
    assert Q.snr(3.7 * ref, 3.7 * (ref + n)) == pytest.approx(Q.snr(ref, ref + n), abs=1e-12)
    with pytest.raises(ValueError):
        Q.snr(ref, ref[:, :-1])
    with pytest.raises(ValueError):
        Q.snr(np.zeros((4, 4)), np.ones((4, 4)))


def _ssim_brute(a, b, L, size=11, sigma=1.5):
    """Wang et al. 2004 evaluated window by window with the explicit 2-D weights."""
    t = np.arange(size) - (size - 1) / 2.0
    g = np.exp(-0.5 * (t / sigma) ** 2)
    w = np.outer(g, g)
    w /= w.sum()
    c1, c2 = (0.01 * L) ** 2, (0.03 * L) ** 2
    vals = []
    for i in range(a.shape[0] - size + 1):
        for j in range(a.shape[1] - size + 1):
            pa, pb = a[i:i + size, j:j + size], b[i:i + size, j:j + size]
            ma, mb = (w * pa).sum(), (w * pb).sum()
            va, vb = (w * (pa - ma) ** 2).sum(), (w * (pb - mb) ** 2).sum()
            cab = (w * (pa - ma) * (pb - mb)).sum()
            vals.append(((2 * ma * mb + c1) * (2 * cab + c2)) / ((ma * ma + mb * mb + c1) * (va + vb + c2)))
    return float(np.mean(vals))


def test_ssim_matches_per_window_brute_force():
    rng = np.random.default_rng(1)
    a = rng.uniform(0, 100, (17, 23))
    b = a + rng.normal(0, 10, a.shape)
    assert Q.ssim(a, b, 100.0) == pytest.approx(_ssim_brute(a, b, 100.0), rel=1e-10)


def test_ssim_invariants_and_constant_closed_form():
    rng = np.random.default_rng(2)
    a = rng.uniform(0, 1, (32, 32))
    b = np.clip(a + rng.normal(0, 0.1, a.shape), 0, None)
    assert Q.ssim(a, a, 1.0) == 1.0
    assert Q.ssim(a, b, 1.0) == pytest.approx(Q.ssim(b, a, 1.0), abs=1e-12)
    assert Q.ssim(a, 0.8 * a + 0.1, 1.0) < 1.0
    c, d, L = 40.0, 7.0, 255.0
    C1 = (0.01 * L) ** 2
    want = (2 * c * (c + d) + C1) / (c * c + (c + d) ** 2 + C1)        # luminance term; contrast/structure -> 1
    got = Q.ssim(np.full((16, 16), c), np.full((16, 16), c + d), L)
    assert got == pytest.approx(want, rel=1e-9)
    with pytest.raises(ValueError):
        Q.ssim(a, a, 0.0)
