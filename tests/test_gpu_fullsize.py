"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (AUTO path = FFT, CUDA-graph replay of deblur_iterate), on sampled outputs
the fp64 oracle evaluates one by one.

One full distributed iteration from a seeded state (set_state) is checked at
sampled *single-owner* estimate pixels lying at least 2c+2 pixels inside their
facet's estimate block.  There the Local-Solver step (Alg. 1, PAPER.md:226-229,
rows a1-a4 of SURVEY §8a) and the single-owner dual update (Lemma 1 with one
term, A8) depend only on a (4c+1)^2 neighbourhood of x and on u at the pixel:

    r  = W (H x - y) on observed rows/cols [p - 2c, p]     (oracle H_window)
    g  = (H^T r)(p)                                         (oracle HT_window)
    t  = (D^T psi(D x))(p)                                  (oracle tv.grad on a crop)
    x+ = max(0, x - tau (g + lambda t + gamma (x - u)))     (omega^F = 1)
    u+ = u + rho (x+ - u)

so the oracle recomputes x+ and u+ there exactly (fp64) without a full-size
solve.  Band pixels (2- and 4-facet, facet borders) take every facet's own step and
Lemma 1 (test_iterate_full_size_band_pixels).  One iteration is launched eagerly;
test_graph_replay_equals_eager_full_size ties it to the CUDA-graph replay bench.py
times (bitwise).  tests/test_gpu_golden.py holds the multi-iteration full-size runs.
"""
import numpy as np
import pytest

import synth
from tests.fullsize import full_config
from oracle import Operator, geometry, solver, tv
from paper_1705_06603_b200 import deblur as D

pytestmark = pytest.mark.gpu

IT_TOL = 1e-3            # BASELINE north_star: iterate within rel-L2 1e-3
H_TOL = 1e-5


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _state(pb, facets, seed):
    """x = max(0, edge-padded y) + small positive noise, u = x + noise: a state
    near the data so that x+ is mostly unclipped and the prox term is active."""
    rng = np.random.default_rng(seed)
    c = (pb.P - 1) // 2
    base = np.maximum(0.0, np.pad(pb.y, c, mode="edge")).astype(np.float32)
    X = base + (0.002 * rng.random(base.shape, dtype=np.float32))
    U = X + (0.002 * rng.standard_normal(base.shape, dtype=np.float32))
    xs = np.concatenate([X[f.ey[0]:f.ey[1], f.ex[0]:f.ex[1]].ravel() for f in facets])
    us = np.concatenate([U[f.ey[0]:f.ey[1], f.ex[0]:f.ex[1]].ravel() for f in facets])
    return X, U, xs, us


def _single_owner_samples(pb, facets, count, rng):
    """(facet index, local row, local col) of single-owner pixels >= 2c+2 inside."""
    c = (pb.P - 1) // 2
    m = 2 * c + 2
    out = []
    while len(out) < count:
        i = int(rng.integers(len(facets)))
        f = facets[i]
        ly = int(rng.integers(m, f.ey[1] - f.ey[0] - m))
        lx = int(rng.integers(m, f.ex[1] - f.ex[0] - m))
        gy, gx = f.ey[0] + ly, f.ex[0] + lx
        n_own = sum(1 for g in facets if g.ey[0] <= gy < g.ey[1] and g.ex[0] <= gx < g.ex[1])
        if n_own == 1:
            out.append((i, ly, lx))
    return out


def _oracle_update(pb, op, X, U, tau, gy, gx):
    """x+ and u+ at global estimate pixel (gy, gx) (single owner, interior)."""
    c = op.c
    xw = X[gy - 2 * c:gy + 2 * c + 1, gx - 2 * c:gx + 2 * c + 1].astype(np.float64)
    hx = op.H_window(xw, gy - 2 * c, gx - 2 * c)                         # observed [p-2c, p]
    yw = pb.y[gy - 2 * c:gy + 1, gx - 2 * c:gx + 1].astype(np.float64)
    w = (pb.noise_w[gy - 2 * c:gy + 1, gx - 2 * c:gx + 1].astype(np.float64) if pb.noise_w is not None
         else np.float64(np.float32(pb.noise_w_scalar)))
    r = w * (hx - yw)
    g = op.HT_window(r, gy - 2 * c, gx - 2 * c)[2 * c, 2 * c]
    xc = X[gy - 2:gy + 3, gx - 2:gx + 3].astype(np.float64)
    t = tv.grad(xc, pb.eps, pb.reg_kind, pb.tv_boundary)[2, 2]
    x0 = float(X[gy, gx])
    u0 = float(U[gy, gx])
    xp = max(0.0, x0 - tau * (g + pb.lam * t + pb.gamma * (x0 - u0)))
    return xp, u0 + pb.rho * (xp - u0)


@pytest.mark.parametrize("k,count", [(4, 24), (5, 12)], ids=["c4", "c5"])
def test_iterate_full_size_sampled(k, count):
    pb = full_config(k)
    facets = geometry.plan(pb.ny, pb.nx, pb.P, pb.fy, pb.fx, pb.overlap)
    w_max = float(pb.noise_w.max()) if pb.noise_w is not None else float(np.float32(pb.noise_w_scalar))
    tau = solver.default_tau(pb.psfs, pb.wy, pb.wx, w_max, pb.lam, pb.eps, pb.reg_kind, pb.gamma)
    X, U, xs, us = _state(pb, facets, seed=100 + k)
    with D.Deblur.from_problem(pb, tau=tau) as dev:
        assert dev.conv_path == D.CONV_FFT                       # the bench's AUTO choice at P >= 7
        dev.set_state(xs, us)
        dev.iterate(1)                                           # eager; == graph replay (test below)
        xg, ug = dev.get_state()
    del xs, us
    rng = np.random.default_rng(k)
    samples = _single_owner_samples(pb, facets, count, rng)
    offs = np.cumsum([0] + [(f.ey[1] - f.ey[0]) * (f.ex[1] - f.ex[0]) for f in facets])
    op = Operator(pb.psfs, pb.wy, pb.wx)
    got_x, got_u, ref_x, ref_u = [], [], [], []
    for i, ly, lx in samples:
        f = facets[i]
        o = offs[i] + ly * (f.ex[1] - f.ex[0]) + lx
        got_x.append(xg[o])
        got_u.append(ug[o])
        xp, up = _oracle_update(pb, op, X, U, tau, f.ey[0] + ly, f.ex[0] + lx)
        ref_x.append(xp)
        ref_u.append(up)
    assert np.count_nonzero(ref_x) >= len(ref_x) // 2           # the step is not all clipped
    assert rel_l2(got_x, ref_x) <= IT_TOL, rel_l2(got_x, ref_x)
    assert rel_l2(got_u, ref_u) <= IT_TOL, rel_l2(got_u, ref_u)


def _band_samples(pb, facets, count, rng):
    """Global estimate pixels shared by >= 2 facets: half on 4-facet corner bands,
    half on 2-facet edge bands, some on a facet's first/last row or column (where
    the circular D of A2 wraps around that facet)."""
    out = []
    fac_by = {(f.fy, f.fx): f for f in facets}
    while len(out) < count:
        f = facets[int(rng.integers(len(facets)))]
        right = fac_by.get((f.fy, f.fx + 1))
        down = fac_by.get((f.fy + 1, f.fx))
        if right is None or down is None:
            continue
        kind = len(out) % 3
        ys = (down.ey[0], f.ey[1])                     # rows of the band with the facet below
        xs = (right.ex[0], f.ex[1])                    # columns of the band with the facet right
        if kind == 0:                                  # 4-facet corner band
            gy, gx = int(rng.integers(*ys)), int(rng.integers(*xs))
        elif kind == 1:                                # edge band with the facet below
            gy, gx = int(rng.integers(*ys)), int(rng.integers(f.ex[0] + 4, right.ex[0]))
        else:                                          # facet border row / column inside a band
            gy = int(rng.choice([down.ey[0], f.ey[1] - 1]))
            gx = int(rng.integers(f.ex[0] + 4, right.ex[0]))
        out.append((gy, gx))
    return out


def _oracle_band_update(pb, op, facets, X, U, tau, gy, gx):
    """x+_f and u+_f at global estimate pixel l = (gy, gx) for every facet f containing
    it: the Local-Solver step of each facet from its own data (r_f = 0 outside O_f,
    circular D on P_f, prox weight gamma omega^F_f; Alg. 1, R1, A2) and
    the consensus of Lemma 1 (A8/A9, ascending facet id)."""
    c = op.c
    y0, x0 = max(0, gy - 2 * c), max(0, gx - 2 * c)
    y1, x1 = min(pb.my, gy + 1), min(pb.mx, gx + 1)            # observed rows/cols seeing l
    hx = op.H_window(X[y0:y1 + 2 * c, x0:x1 + 2 * c].astype(np.float64), y0, x0)
    yw = pb.y[y0:y1, x0:x1].astype(np.float64)
    w = (pb.noise_w[y0:y1, x0:x1].astype(np.float64) if pb.noise_w is not None
         else np.float64(np.float32(pb.noise_w_scalar)))
    r_all = w * (hx - yw)
    res = []
    for f in facets:
        if not (f.ey[0] <= gy < f.ey[1] and f.ex[0] <= gx < f.ex[1]):
            continue
        r = r_all.copy()                                       # r_f: zero outside O_f
        ii = np.arange(y0, y1)[:, None]
        jj = np.arange(x0, x1)[None, :]
        r[~((ii >= f.oy[0]) & (ii < f.oy[1]) & (jj >= f.ox[0]) & (jj < f.ox[1]))] = 0.0
        g = op.HT_window(r, y0, x0)[gy - y0, gx - x0]
        ly, lx = gy - f.ey[0], gx - f.ex[0]
        ny, nx = f.shape
        rows = (np.arange(ly - 2, ly + 3) % ny) + f.ey[0]      # circular D within the facet
        cols = (np.arange(lx - 2, lx + 3) % nx) + f.ex[0]
        t = tv.grad(X[np.ix_(rows, cols)].astype(np.float64), pb.eps, pb.reg_kind, pb.tv_boundary)[2, 2]
        om = float(f.wy[ly] * f.wx[lx])
        xv, uv = float(X[gy, gx]), float(U[gy, gx])
        xp = max(0.0, xv - tau * (g + pb.lam * t + pb.gamma * om * (xv - uv)))
        res.append((f.id, om, xp, uv))
    num = sum(om * (2 * xp - uv) for _, om, xp, uv in res)     # ascending facet id
    den = sum(om for _, om, _, _ in res)
    zbar = num / den
    return [(fid, xp, uv + pb.rho * (zbar - xp)) for fid, _, xp, uv in res]


@pytest.mark.parametrize("k,count", [(4, 18), (5, 12)], ids=["c4", "c5"])
def test_iterate_full_size_band_pixels(k, count):
    """One full distributed iteration at BASELINE size at band pixels (shared by 2 or 4
    facets, including facet-border rows where D wraps): x+ of every facet containing the
    pixel from its own facet-local data, then Lemma 1 and the dual update, against the
    GPU state in bench.py's launch configuration."""
    pb = full_config(k)
    facets = geometry.plan(pb.ny, pb.nx, pb.P, pb.fy, pb.fx, pb.overlap)
    w_max = float(pb.noise_w.max()) if pb.noise_w is not None else float(np.float32(pb.noise_w_scalar))
    tau = solver.default_tau(pb.psfs, pb.wy, pb.wx, w_max, pb.lam, pb.eps, pb.reg_kind, pb.gamma)
    X, U, xs, us = _state(pb, facets, seed=200 + k)
    with D.Deblur.from_problem(pb, tau=tau) as dev:
        dev.set_state(xs, us)
        dev.iterate(1)                                   # eager; == graph replay (test below)
        xg, ug = dev.get_state()
    del xs, us
    rng = np.random.default_rng(300 + k)
    pix = _band_samples(pb, facets, count, rng)
    offs = np.cumsum([0] + [(f.ey[1] - f.ey[0]) * (f.ex[1] - f.ex[0]) for f in facets])
    op = Operator(pb.psfs, pb.wy, pb.wx)
    got_x, got_u, ref_x, ref_u, nshared = [], [], [], [], []
    for gy, gx in pix:
        out = _oracle_band_update(pb, op, facets, X, U, tau, gy, gx)
        nshared.append(len(out))
        for fid, xp, up in out:
            f = facets[fid]
            o = offs[fid] + (gy - f.ey[0]) * (f.ex[1] - f.ex[0]) + (gx - f.ex[0])
            got_x.append(xg[o])
            got_u.append(ug[o])
            ref_x.append(xp)
            ref_u.append(up)
    assert min(nshared) >= 2 and max(nshared) == 4
    assert rel_l2(got_x, ref_x) <= IT_TOL, rel_l2(got_x, ref_x)
    assert rel_l2(got_u, ref_u) <= IT_TOL, rel_l2(got_u, ref_u)


@pytest.mark.parametrize("count", [20000])
def test_apply_c5_sampled(count):
    """c5 (32768^2, 32x32 grid of 127x127 PSFs, 8x8 facets) H / H^T on one GPU,
    sampled pixels including facet seams and image borders."""
    pb = full_config(5)
    rng = np.random.default_rng(55)
    x = (0.05 + rng.random((pb.ny, pb.nx), dtype=np.float32) * 0.5).astype(np.float32)
    op = Operator(pb.psfs, pb.wy, pb.wx)
    with D.Deblur.from_problem(pb) as dev:
        hx = dev.apply_H(x)
        oi, oj = rng.integers(0, pb.my, count), rng.integers(0, pb.mx, count)
        oi[:6] = [0, pb.my - 1, 0, pb.my // 8, pb.my // 2, pb.my - 2]
        ref = op.H_points(x, oi, oj)
        assert rel_l2(hx[oi, oj], ref) <= H_TOL
        del hx, x
        r = rng.standard_normal((pb.my, pb.mx), dtype=np.float32)
        g = dev.apply_HT(r)
    ei, ej = rng.integers(0, pb.ny, count), rng.integers(0, pb.nx, count)
    ei[:4] = [0, pb.ny - 1, 63, pb.ny - 64]
    ref = op.HT_points(r, ei, ej)
    assert rel_l2(g[ei, ej], ref) <= H_TOL


def test_paper_shaped_c6_apply_sampled():
    """c6, the paper's shift-variant experiment shape: 1151 x 1407,
    9 x 9 Gaussian PSFs of 201 x 201 (FFT path, S = 512, T = 312); 2 x 2 facets
    with overlap P - 1 = 200 (the owner-computes apply_HT needs O >= P - 1, §8b);
    H / H^T on sampled pixels including facet seams and the image borders."""
    pb = synth.make_config(6, facets=(2, 2), overlap=200)
    rng = np.random.default_rng(66)
    x = (6000.0 * rng.random((pb.ny, pb.nx))).astype(np.float32)
    r = rng.standard_normal((pb.my, pb.mx)).astype(np.float32)
    op = Operator(pb.psfs, pb.wy, pb.wx)
    with D.Deblur.from_problem(pb) as dev:
        assert dev.conv_path == D.CONV_FFT
        hx = dev.apply_H(x)
        g = dev.apply_HT(r)
    oi, oj = rng.integers(0, pb.my, 1500), rng.integers(0, pb.mx, 1500)
    oi[:4] = [0, pb.my - 1, pb.my // 3, 2 * pb.my // 3]
    assert rel_l2(hx[oi, oj], op.H_points(x, oi, oj)) <= H_TOL
    ei, ej = rng.integers(0, pb.ny, 1500), rng.integers(0, pb.nx, 1500)
    ei[:4] = [0, pb.ny - 1, 100, pb.ny - 101]
    assert rel_l2(g[ei, ej], op.HT_points(r, ei, ej)) <= H_TOL


def test_paper_shaped_c6_iterate_small():
    """c6 parameters (Huber delta = 100, lambda = 0.002, gamma = 0.001, 6000-photon
    scale, P = 201) on a 400 x 489 crop of the geometry: 2 iterations vs the oracle."""
    from oracle import from_problem
    pb = synth.make_config(6, n=400, facets=(1, 1), overlap=0)
    orc = from_problem(pb)
    with D.Deblur.from_problem(pb, tau=orc.tau) as dev:
        dev.iterate(2)
        xs, us = dev.get_state()
        obj = dev.objective()
    orc.iterate(2)
    xr, ur = orc.state()
    assert rel_l2(xs, xr) <= IT_TOL
    assert rel_l2(us, ur) <= IT_TOL
    ro = orc.objective()
    for i in range(3):
        assert abs(obj[i] - ro[i]) <= 1e-4 * abs(ro[i]), (i, obj[i], ro[i])


@pytest.mark.parametrize("k", [4, 5])
def test_graph_replay_equals_eager_full_size(k, monkeypatch):
    """The CUDA-graph replay of deblur_iterate (bench.py's launch configuration) and
    eager launches give bitwise identical states at full size."""
    pb = full_config(k)
    facets = geometry.plan(pb.ny, pb.nx, pb.P, pb.fy, pb.fx, pb.overlap)
    _, _, xs, us = _state(pb, facets, seed=400 + k)
    with D.Deblur.from_problem(pb) as dev:
        dev.set_state(xs, us)
        dev.iterate(2)
        xa, ua = dev.get_state()
    monkeypatch.setenv("DEBLUR_NO_GRAPHS", "1")
    with D.Deblur.from_problem(pb) as dev:
        dev.set_state(xs, us)
        dev.iterate(2)
        xb, ub = dev.get_state()
    np.testing.assert_array_equal(xa, xb)
    np.testing.assert_array_equal(ua, ub)


def test_long_run_c4_stable():
    """200 full distributed iterations at c4 (four times the BASELINE count): every
    objective finite, the objective falls from the A6 start, the iterate stays >= 0 and
    the facets keep agreeing on their shared pixels (consensus max-difference bounded)."""
    pb = full_config(4)
    with D.Deblur.from_problem(pb) as dev:
        tr = dev.iterate_traced(200)
        x, _ = dev.get_state()
        end = dev.objective()
    assert np.all(np.isfinite(tr)) and np.all(np.isfinite(end))
    assert end[0] < tr[0, 0] and tr[-1, 0] < tr[0, 0]
    assert float(x.min()) >= 0.0
    assert end[3] < 1.0 and np.max(tr[:, 3]) < 1.0
