"""Full-size GPU parity against stored fp64 oracle results (tests/golden/*.npz).

The golden files are written by tools/make_golden.py, which calls only oracle/ and
synth/ (never the CUDA path): Algorithm 1 from the A6 start at the
BASELINE geometry, with the objective of Eq. (4) (A22) at every iterate
and x_f / u_f at sampled state entries of every pixel class (single-owner interior,
facet borders where the circular D wraps, 2-facet edge bands and 4-facet corner bands
where Lemma 1 acts), plus the blended image (A7) at sampled pixels.

  c3  4096^2, 8x8 PSFs P = 63, 2x4 facets, per-pixel W: the BASELINE 100 iterations
  c4  16384^2, 16x16 PSFs P = 63, 4x2 facets: a 2-iteration prefix with the objective at
      every iterate, and the BASELINE 50 iterations with files at 10, 20, 30, 40 and the
      objective at every 5th iterate (the fp64 oracle needs ~4.5 min per iteration on 8
      host cores); every c*_it*.npz present is tested

The GPU runs in bench.py's launch configuration (AUTO = FFT path, CUDA-graph replay
of deblur_iterate) and, separately, through deblur_iterate_traced for the objective
history.  Bars (BASELINE north_star): iterate rel-L2 <= 1e-3, objective <= 1e-4.
"""
import os

import numpy as np
import pytest

import synth
from tests.fullsize import full_config
from paper_1705_06603_b200 import deblur as D

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
IT_TOL = 1e-3
OBJ_TOL = 1e-4


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def pixel_class(pb, idx):
    """Class of each state entry: 'border' (2 px from the facet edge, where the
    circular D wraps), else 'single' / 'edge' / 'corner' by the number of facets
    containing the pixel (1 / 2 / >= 3)."""
    from oracle import geometry
    fac = geometry.plan(pb.ny, pb.nx, pb.P, pb.fy, pb.fx, pb.overlap)
    sizes = [(f.ey[1] - f.ey[0]) * (f.ex[1] - f.ex[0]) for f in fac]
    offs = np.cumsum([0] + sizes)
    fi = np.searchsorted(offs, idx, side="right") - 1
    out = np.empty(idx.size, object)
    for i, f in enumerate(fac):
        m = fi == i
        w = f.ex[1] - f.ex[0]
        loc = idx[m] - offs[i]
        ly, lx = loc // w, loc % w
        gy, gx = f.ey[0] + ly, f.ex[0] + lx
        cnt = np.zeros(loc.size, np.int64)
        for h in fac:
            cnt += (gy >= h.ey[0]) & (gy < h.ey[1]) & (gx >= h.ex[0]) & (gx < h.ex[1])
        border = (ly < 2) | (ly >= f.ey[1] - f.ey[0] - 2) | (lx < 2) | (lx >= w - 2)
        c = np.where(cnt == 1, "single", np.where(cnt == 2, "edge", "corner")).astype(object)
        c[border] = "border"
        out[m] = c
    return out


def load(name):
    path = os.path.join(GOLDEN, name + ".npz")
    assert os.path.exists(path), f"missing golden file {path} (tools/make_golden.py)"
    return np.load(path)


GOLDEN_RUNS = sorted((f[:-4] for f in os.listdir(GOLDEN) if f.startswith("c") and "_it" in f and f.endswith(".npz")),
                     key=lambda n: (int(n[1:n.index("_")]), int(n[n.index("_it") + 3:])))


def test_golden_runs_present():
    assert {"c3_it100", "c4_it2"} <= set(GOLDEN_RUNS), GOLDEN_RUNS


@pytest.mark.parametrize("name", GOLDEN_RUNS)
def test_full_size_against_golden(name):
    g = load(name)
    k, iters = int(g["config"]), int(g["iters"])
    pb = full_config(k)
    assert synth.input_hash(pb) == str(g["input_hash"]), "inputs differ from the ones the golden file was made from"
    tau = float(g["tau"])
    trace_ref = g["trace"]                                   # [iters + 1, 4] at x^(0..iters); NaN rows not evaluated
    with D.Deblur.from_problem(pb, tau=tau) as dev:
        assert dev.conv_path == D.CONV_FFT                   # the bench's AUTO choice
        dev.iterate(iters)                                   # graph replay, as bench.py times it
        xs, us = dev.get_state()
        obj_end = dev.objective()
        img = dev.get_image()
    idx = g["idx"]
    ex, eu = rel_l2(xs[idx], g["x"]), rel_l2(us[idx], g["u"])
    assert ex <= IT_TOL and eu <= IT_TOL, (ex, eu)
    # every sampled class on its own (the band classes are where consensus acts)
    cls = pixel_class(pb, idx)
    for c in ("single", "edge", "corner", "border"):
        m = cls == c
        assert m.sum() >= 1000, (c, m.sum())
        ec, uc = rel_l2(xs[idx[m]], g["x"][m]), rel_l2(us[idx[m]], g["u"][m])
        assert ec <= IT_TOL and uc <= IT_TOL, (c, ec, uc)
    assert rel_l2(img[g["img_i"], g["img_j"]], g["img"]) <= IT_TOL
    for i in range(3):
        assert abs(obj_end[i] - trace_ref[iters, i]) <= OBJ_TOL * abs(trace_ref[iters, i]), (i, obj_end[i])
    with D.Deblur.from_problem(pb, tau=tau) as dev:
        tr = dev.iterate_traced(iters)
        xt, _ = dev.get_state()
    np.testing.assert_array_equal(xt, xs)                    # the traced run is the same run
    for it in range(iters):
        if np.isnan(trace_ref[it, 0]):
            continue
        for i in range(3):
            assert abs(tr[it, i] - trace_ref[it, i]) <= OBJ_TOL * abs(trace_ref[it, i]), (it, i, tr[it, i])
        assert abs(tr[it, 3] - trace_ref[it, 3]) <= IT_TOL * max(1.0, np.abs(g["x"]).max())
    assert trace_ref[iters, 0] < trace_ref[0, 0]             # the run makes progress


def test_c5_objective_at_start_against_golden():
    """c5 (32768^2, 32x32 PSFs of 127^2, 8x8 facets) at full size: Eq. (4) at the A6 start
    against the oracle's facet-by-facet evaluation (tools/make_golden.py --objective-only;
    a full c5 oracle iteration does not fit the host's memory, the iterate at c5 is checked
    at sampled interior and band pixels in test_gpu_fullsize.py)."""
    g = load("c5_obj0")
    pb = full_config(5)
    assert synth.input_hash(pb) == str(g["input_hash"])
    with D.Deblur.from_problem(pb) as dev:
        obj = dev.objective()
    ref = g["trace"][0]
    for i in range(3):
        assert abs(obj[i] - ref[i]) <= OBJ_TOL * abs(ref[i]), (i, obj[i], ref[i])
    assert obj[3] == 0.0                                     # every facet starts from the same x0
