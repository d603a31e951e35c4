"""GPU edge cases vs the fp64 oracle, both conv paths: degenerate PSF size, unmeasured
pixels (W = 0), relaxed D-R (rho != 1) with several inner
steps, zero overlap, an image smaller than one tile, and the c5 facet geometry (8x8
facets, P = 127) shrunk to an oracle-friendly size."""
import numpy as np
import pytest

import synth
from oracle import Operator, from_problem
from paper_1705_06603_b200 import deblur as D
from tests.test_gpu_parity import IT_TOL, OBJ_TOL, H_TOL, check_pair, rel_l2, run_pair

pytestmark = pytest.mark.gpu
PATHS = [D.CONV_DIRECT, D.CONV_FFT]
IDS = ["direct", "fft"]


def small(P, n, G, facets, O, seed=0, **kw):
    pb = synth.make_problem(name="edge", n=n, P=P, G=G, psf="gauss_axis", sources=max(1, n * n // 300), galaxies=0,
                            noise=("gauss", 0.01), facets=facets, overlap=O, iters=5, seed=seed, **kw)
    return pb


@pytest.mark.parametrize("path", PATHS, ids=IDS)
def test_P1_iterate(path):
    pb = small(1, 96, 3, (2, 2), 8)
    check_pair(run_pair(pb, 6, path))


@pytest.mark.parametrize("path", PATHS, ids=IDS)
def test_unmeasured_pixels(path):
    """W = 0 on a block of unmeasured pixels and a dead column."""
    pb = small(15, 200, 2, (2, 2), 24)
    w = np.full((pb.my, pb.mx), np.float32(1e4))
    w[40:70, 100:150] = 0
    w[:, 7] = 0
    pb.noise_w = w.astype(np.float32)
    check_pair(run_pair(pb, 8, path))


@pytest.mark.parametrize("path", PATHS, ids=IDS)
def test_relaxed_rho_inner_steps(path):
    pb = small(7, 160, 2, (2, 3), 20)
    pb.rho = 1.5
    check_pair(run_pair(pb, 6, path, inner_steps=3))


@pytest.mark.parametrize("path", PATHS, ids=IDS)
def test_zero_overlap(path):
    """O = 0: estimate blocks still share a (P-1)-wide band (A12)."""
    pb = small(9, 180, 3, (3, 3), 0)
    check_pair(run_pair(pb, 6, path))


@pytest.mark.parametrize("path", PATHS, ids=IDS)
def test_image_smaller_than_a_tile(path):
    pb = small(5, 24, 1, (1, 1), 0)
    check_pair(run_pair(pb, 5, path))


@pytest.mark.parametrize("path", PATHS, ids=IDS)
def test_c5_geometry_shrunk(path):
    """8x8 facets with the c5 PSF family (P = 127, elliptical Moffat grid), shrunk so
    the oracle finishes: facet cores just above O + P - 1."""
    n = 8 * 256 + 126                     # facet core 256 >= O + P - 1 = 254; O >= P - 1 for apply_HT
    pb = synth.make_config(5, n=n, overlap=128)
    op = Operator(pb.psfs, pb.wy, pb.wx)
    rng = np.random.default_rng(5)
    x = (0.05 + 0.5 * rng.random((pb.ny, pb.nx))).astype(np.float32)
    r = rng.standard_normal((pb.my, pb.mx)).astype(np.float32)
    with D.Deblur.from_problem(pb, conv_path=path) as dev:
        hx = dev.apply_H(x)
        g = dev.apply_HT(r)
    oi, oj = rng.integers(0, pb.my, 1500), rng.integers(0, pb.mx, 1500)
    assert rel_l2(hx[oi, oj], op.H_points(x, oi, oj)) <= H_TOL
    ei, ej = rng.integers(0, pb.ny, 1500), rng.integers(0, pb.nx, 1500)
    assert rel_l2(g[ei, ej], op.HT_points(r, ei, ej)) <= H_TOL


def test_fft_and_direct_iterates_agree_at_scale():
    """c3 at full size (4096^2, 2x4 facets, per-pixel W), 5 iterations: the two
    independent GPU operator implementations agree to the iterate bar."""
    pb = synth.make_config(3)
    out = []
    for path in PATHS:
        with D.Deblur.from_problem(pb, conv_path=path) as dev:
            dev.iterate(5)
            out.append((dev.get_state()[0], dev.objective()))
    assert rel_l2(out[0][0], out[1][0]) <= IT_TOL
    for i in range(3):
        assert abs(out[0][1][i] - out[1][1][i]) <= OBJ_TOL * abs(out[1][1][i])


def test_c_abi_from_plain_c():
    """examples/c_demo.c drives create / apply_H / reset / objective / iterate / get_image /
    destroy from C (no Python binding): it exits 0 when the objective fell."""
    import os
    import subprocess
    import __graft_entry__ as g
    exe = g.build_c_demo()
    r = subprocess.run([exe, "10"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "objective" in r.stdout and "SNR" in r.stdout
