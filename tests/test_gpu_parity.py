"""GPU parity: libdeblur (through the C ABI) vs the fp64 oracle on the same
seeded inputs.  Bars (BASELINE.json north_star): rel-L2 <= 1e-5 for H / H^T,
<= 1e-4 for the objective, <= 1e-3 for the iterate after the fixed iteration
count.  rel-L2(a, b) = |a - b|_2 / |b|_2 with b the oracle."""
import numpy as np
import pytest
import scipy.signal

import synth
from tests.fullsize import full_config
from oracle import Operator, from_problem
from paper_1705_06603_b200 import deblur as D

pytestmark = pytest.mark.gpu

H_TOL = 1e-5
OBJ_TOL = 1e-4
IT_TOL = 1e-3


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def load_state(orc, xs, us):
    """Put a concatenated (planner-order) facet state into the oracle."""
    o = 0
    for i, f in enumerate(orc.facets):
        n = (f.ey[1] - f.ey[0]) * (f.ex[1] - f.ex[0])
        shp = (f.ey[1] - f.ey[0], f.ex[1] - f.ex[0])
        orc.x[i] = np.asarray(xs[o:o + n], np.float64).reshape(shp)
        orc.u[i] = np.asarray(us[o:o + n], np.float64).reshape(shp)
        o += n
    return orc


def oracle_op(pb):
    return Operator(pb.psfs, pb.wy, pb.wx)


def rand_x(pb, seed=0):
    rng = np.random.default_rng(seed)
    # star-field-like non-negative test image: background + sparse bright pixels
    x = 0.05 + 0.02 * rng.random((pb.ny, pb.nx))
    m = rng.random((pb.ny, pb.nx)) < 0.01
    x[m] += rng.uniform(0.2, 1.0, m.sum())
    return x.astype(np.float32)


def rand_r(pb, seed=1):
    return np.random.default_rng(seed).standard_normal((pb.my, pb.mx)).astype(np.float32)


# ------------------------------------------------------------------ H / H^T
OP_CASES = [
    # (config k, n, facets, overlap, path)
    (1, None, (1, 1), 0),
    (1, None, (2, 2), 16),
    (2, None, (2, 2), 64),
    (2, 300, (3, 2), 40),          # ragged tiles, 6 facets
    (3, 1024, (2, 2), 128),        # P = 63: blocked accumulation matters (A24)
]


PATHS = [D.CONV_DIRECT, D.CONV_FFT]


@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
@pytest.mark.parametrize("k,n,facets,O", OP_CASES)
def test_apply_H_HT_parity(k, n, facets, O, path):
    pb = synth.make_config(k, n=n, facets=facets, overlap=O)
    op = oracle_op(pb)
    x, r = rand_x(pb), rand_r(pb)
    with D.Deblur.from_problem(pb, conv_path=path) as dev:
        assert dev.conv_path == path
        hx = dev.apply_H(x)
        g = dev.apply_HT(r)
    assert rel_l2(hx, op.H(x)) <= H_TOL
    assert rel_l2(g, op.HT(r)) <= H_TOL


@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
@pytest.mark.parametrize("P,G,shape", [(1, 2, (37, 45)), (3, 1, (20, 300)), (7, 3, (131, 259)),
                                       (15, 2, (256, 129)), (127, 4, (400, 300)), (63, 3, (700, 1100))])
def test_apply_parity_odd_shapes(P, G, shape, path):
    """Ragged tails, P = 1 (identity-like), a tile-width-thin image, P = 127."""
    ny, nx = shape
    rng = np.random.default_rng(P)
    psfs = rng.uniform(0, 1, (G * G, P, P)).astype(np.float32)
    psfs /= psfs.sum(axis=(1, 2), keepdims=True)
    wy, wx = synth.hat_weights(ny, G).astype(np.float32), synth.hat_weights(nx, G).astype(np.float32)
    my, mx = ny - P + 1, nx - P + 1
    y = rng.uniform(0, 1, (my, mx)).astype(np.float32)
    params, keep = D.make_params(psfs, wy, wx, y, conv_path=path)
    x = rng.uniform(0, 1, (ny, nx)).astype(np.float32)
    r = rng.standard_normal((my, mx)).astype(np.float32)
    op = Operator(psfs, wy, wx)
    with D.Deblur(params, keep) as dev:
        assert rel_l2(dev.apply_H(x), op.H(x)) <= H_TOL
        assert rel_l2(dev.apply_HT(r), op.HT(r)) <= H_TOL


def test_gpu_adjoint_identity():
    pb = synth.make_config(2, n=512, facets=(1, 1), overlap=0)
    x, r = rand_x(pb, 3), rand_r(pb, 4)
    with D.Deblur.from_problem(pb, conv_path=D.CONV_DIRECT) as dev:
        lhs = float(np.dot(dev.apply_H(x).ravel().astype(np.float64), r.ravel()))
        rhs = float(np.dot(x.ravel().astype(np.float64), dev.apply_HT(r).ravel()))
    assert abs(lhs - rhs) <= 1e-5 * np.linalg.norm(x) * np.linalg.norm(r)


def test_gpu_identical_and_delta_psfs():
    rng = np.random.default_rng(7)
    n, P, G = 200, 15, 3
    h = rng.uniform(0, 1, (P, P))
    h /= h.sum()
    wy = synth.hat_weights(n, G).astype(np.float32)
    x = rng.uniform(0, 1, (n, n)).astype(np.float32)
    y = np.zeros((n - P + 1, n - P + 1), np.float32)
    params, keep = D.make_params(np.repeat(h[None], G * G, 0), wy, wy, y, conv_path=D.CONV_DIRECT)
    with D.Deblur(params, keep) as dev:
        ref = scipy.signal.convolve2d(x.astype(np.float64), h.astype(np.float32).astype(np.float64), mode="valid")
        assert rel_l2(dev.apply_H(x), ref) <= H_TOL
    delta = np.zeros((G * G, P, P), np.float32)
    delta[:, P // 2, P // 2] = 1
    params, keep = D.make_params(delta, wy, wy, y, conv_path=D.CONV_DIRECT)
    with D.Deblur(params, keep) as dev:
        c = P // 2
        assert rel_l2(dev.apply_H(x), x[c:n - c, c:n - c]) <= 1e-6


def dense_blocks(centres, lim_y, lim_x, half=24):
    """All pixels of the (2 half)^2 blocks around `centres`, clipped to the image."""
    ii, jj = [], []
    for cy, cx in centres:
        y0, x0 = min(max(cy - half, 0), lim_y - 2 * half), min(max(cx - half, 0), lim_x - 2 * half)
        yy, xx = np.meshgrid(np.arange(y0, y0 + 2 * half), np.arange(x0, x0 + 2 * half), indexing="ij")
        ii.append(yy.ravel())
        jj.append(xx.ravel())
    return np.concatenate(ii), np.concatenate(jj)


def structural_centres(pb, observed):
    """Image corners, facet-seam crossings (A12 bounds) and, in facet 0, the first FFT
    tile boundary (T = 512 - P + 1) and the start of the last, ragged tile row/column."""
    from oracle import geometry
    fac = geometry.plan(pb.ny, pb.nx, pb.P, pb.fy, pb.fx, pb.overlap)
    ly, lx = (pb.my, pb.mx) if observed else (pb.ny, pb.nx)
    T = 512 - pb.P + 1
    f0 = fac[0]
    (y0, y1), (x0, x1) = (f0.oy, f0.ox) if observed else (f0.ey, f0.ex)
    c = [(0, 0), (ly - 1, lx - 1), (0, lx - 1), (ly - 1, 0),
         (y0 + T, x0 + T), (y0 + ((y1 - y0) // T) * T, x0 + ((x1 - x0) // T) * T)]
    for f in fac[1:]:
        (a0, _), (b0, _) = (f.oy, f.ox) if observed else (f.ey, f.ex)
        c.append((a0 + (pb.overlap + pb.P) // 2, b0 + (pb.overlap + pb.P) // 2))   # inside the shared band
    return c


@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
@pytest.mark.parametrize("k,count", [(3, 20000), (4, 100000)])
def test_apply_full_size_sampled(k, count, path):
    """BASELINE full sizes (c3 4096^2, c4 16384^2), bench launch configuration,
    checked on pixels the oracle evaluates one by one (1e5 random pixels at
    c4) plus dense 48x48 blocks across the structural boundaries: image corners, facet
    seams and shared bands, FFT tile and ragged-strip boundaries."""
    pb = full_config(k)
    rng = np.random.default_rng(k)
    x = (0.05 + rng.random((pb.ny, pb.nx), dtype=np.float32) * 0.5).astype(np.float32)
    r = rng.standard_normal((pb.my, pb.mx), dtype=np.float32)
    op = oracle_op(pb)
    with D.Deblur.from_problem(pb, conv_path=path) as dev:
        hx = dev.apply_H(x)
        g = dev.apply_HT(r)
    bi, bj = dense_blocks(structural_centres(pb, True), pb.my, pb.mx)
    oi = np.concatenate([rng.integers(0, pb.my, count), bi])
    oj = np.concatenate([rng.integers(0, pb.mx, count), bj])
    ref = op.H_points(x, oi, oj)
    assert rel_l2(hx[oi, oj], ref) <= H_TOL
    assert rel_l2(hx[bi, bj], ref[count:]) <= H_TOL
    bi, bj = dense_blocks(structural_centres(pb, False), pb.ny, pb.nx)
    ei = np.concatenate([rng.integers(0, pb.ny, count), bi])
    ej = np.concatenate([rng.integers(0, pb.nx, count), bj])
    ref = op.HT_points(r, ei, ej)
    assert rel_l2(g[ei, ej], ref) <= H_TOL
    assert rel_l2(g[bi, bj], ref[count:]) <= H_TOL


# ------------------------------------------------------------------ iterate
def run_pair(pb, iters, path=D.CONV_DIRECT, **over):
    orc = from_problem(pb, **{k: v for k, v in over.items() if k in ("inner_steps", "reg_kind", "tv_boundary")})
    kw = dict(conv_path=path, tau=orc.tau)
    kw.update({k: v for k, v in over.items() if k in ("inner_steps", "reg_kind", "tv_boundary")})
    with D.Deblur.from_problem(pb, **kw) as dev:
        obj0 = dev.objective()
        dev.iterate(iters)
        xs, us = dev.get_state()
        obj = dev.objective()
        img = dev.get_image()
    ref0 = orc.objective()
    orc.iterate(iters)
    xr, ur = orc.state()
    return dict(x=(xs, xr), u=(us, ur), obj=(obj, orc.objective()), obj0=(obj0, ref0), img=(img, orc.image()))


def check_pair(res):
    assert rel_l2(*res["x"]) <= IT_TOL, rel_l2(*res["x"])
    assert rel_l2(*res["u"]) <= IT_TOL, rel_l2(*res["u"])
    assert rel_l2(*res["img"]) <= IT_TOL
    for (a, b) in (res["obj0"], res["obj"]):
        for i in range(3):
            assert abs(a[i] - b[i]) <= OBJ_TOL * abs(b[i]) + 1e-12, (i, a[i], b[i])
        assert abs(a[3] - b[3]) <= IT_TOL * max(1.0, np.abs(res["x"][1]).max())
    assert res["x"][0].min() >= 0.0


@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
def test_iterate_c1_full(path):
    pb = synth.make_config(1)
    check_pair(run_pair(pb, pb.iters, path))


@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
def test_iterate_c2_full(path):
    pb = synth.make_config(2)
    check_pair(run_pair(pb, pb.iters, path))


@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
@pytest.mark.parametrize("over", [dict(inner_steps=2), dict(reg_kind=1), dict(tv_boundary=1)])
def test_iterate_variants_ragged(over, path):
    pb = synth.make_config(2, n=300, facets=(3, 2), overlap=40)
    check_pair(run_pair(pb, 15, path, **over))


@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
def test_iterate_c3_small_mixed_noise(path):
    """per-pixel W (A21), P = 63, 2x4 facets."""
    pb = synth.make_config(3, n=1024, overlap=64)
    check_pair(run_pair(pb, 10, path))


def test_default_tau_matches_oracle():
    pb = synth.make_config(3, n=512, overlap=64, facets=(2, 2))
    with D.Deblur.from_problem(pb, conv_path=D.CONV_DIRECT) as dev:
        t = dev.tau
    assert t == pytest.approx(from_problem(pb).tau, rel=1e-12)


def test_determinism_and_state_roundtrip():
    pb = synth.make_config(2, n=400, facets=(2, 2), overlap=40)
    with D.Deblur.from_problem(pb, conv_path=D.CONV_DIRECT) as dev:
        x0, u0 = dev.get_state()
        dev.iterate(5)
        xa, ua = dev.get_state()
        dev.set_state(x0, u0)
        dev.iterate(5)
        xb, ub = dev.get_state()
    assert np.array_equal(xa, xb) and np.array_equal(ua, ub)


def test_zero_data_stays_zero():
    pb = synth.make_config(1, n=128, facets=(2, 2), overlap=16)
    pb.y[:] = 0
    pb.x0 = np.zeros((pb.ny, pb.nx), np.float32)
    with D.Deblur.from_problem(pb, conv_path=D.CONV_DIRECT) as dev:
        dev.iterate(3)
        x, u = dev.get_state()
    assert np.abs(x).max() == 0 and np.abs(u).max() == 0


def test_kernel_work_counts():
    """deblur_kernel_work's direct-path flop count equals an independent count of
    2 a P^2 per output pixel (a = PSFs with nonzero weight at the pixel)."""
    pb = synth.make_config(2, n=600, facets=(2, 2), overlap=64)
    from oracle import geometry
    fac = geometry.plan(pb.ny, pb.nx, pb.P, 2, 2, 64)
    c = (pb.P - 1) // 2
    ay = (pb.wy != 0).sum(0)
    ax = (pb.wx != 0).sum(0)
    fl_h = sum(2.0 * pb.P ** 2 * ay[f.oy[0] + c:f.oy[1] + c].sum() * ax[f.ox[0] + c:f.ox[1] + c].sum() for f in fac)
    fl_ht = sum(2.0 * pb.P ** 2 * ay[f.ey[0]:f.ey[1]].sum() * ax[f.ex[0]:f.ex[1]].sum() for f in fac)
    with D.Deblur.from_problem(pb, conv_path=D.CONV_DIRECT) as dev:
        w = dev.kernel_work()
    assert w["H_direct_residual"][0] == pytest.approx(fl_h, rel=1e-12)
    assert w["HT_direct_update"][0] == pytest.approx(fl_ht, rel=1e-12)


@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
def test_reset_default_init_and_image(path):
    """deblur_reset(y) restarts from the A6 default (computed on the device) and
    get_image blends the facets (A7); both equal the oracle's definitions."""
    pb = synth.make_config(2, n=300, facets=(3, 2), overlap=40)
    y2 = (pb.y[::-1, :] * 1.5 - 0.01).astype(np.float32)      # a different observation, some negatives
    with D.Deblur.from_problem(pb, conv_path=path) as dev:
        dev.iterate(3)
        dev.reset(y2)
        xs, us = dev.get_state()
        img = dev.get_image()
    pb2 = synth.make_config(2, n=300, facets=(3, 2), overlap=40)
    pb2.y = y2
    orc = from_problem(pb2)
    xr, ur = orc.state()
    np.testing.assert_array_equal(xs, xr.astype(np.float32))
    np.testing.assert_array_equal(us, ur.astype(np.float32))
    assert rel_l2(img, orc.image()) <= 1e-6


@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
def test_iterate_traced(path):
    """deblur_iterate_traced: row k is the objective (Eq. (4), A22) at x^(k), equal
    to the oracle's; the traced run leaves exactly the state of a plain run."""
    pb = synth.make_config(2, n=300, facets=(2, 2), overlap=40)
    orc = from_problem(pb)
    ref = []
    for _ in range(4):
        ref.append(orc.objective())
        orc.iterate(1)
    with D.Deblur.from_problem(pb, conv_path=path, tau=orc.tau) as dev:
        tr = dev.iterate_traced(4)
        xs, us = dev.get_state()
    with D.Deblur.from_problem(pb, conv_path=path, tau=orc.tau) as dev:
        dev.iterate(4)
        xp, up = dev.get_state()
    np.testing.assert_array_equal(xs, xp)
    np.testing.assert_array_equal(us, up)
    xr, _ = orc.state()
    for k in range(4):
        for i in range(3):
            assert abs(tr[k, i] - ref[k][i]) <= OBJ_TOL * abs(ref[k][i]) + 1e-12, (k, i, tr[k, i], ref[k][i])
        assert abs(tr[k, 3] - ref[k][3]) <= IT_TOL * max(1.0, np.abs(xr).max())
    assert tr[3, 0] < tr[0, 0]              # the objective decreases from the A6 start


# ------------------------------------------------------------------ per-node operator mode (NEXT-2)
@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
@pytest.mark.parametrize("k,n", [(2, 300), (1, 256), (3, 700)])
def test_iterate_per_node(k, n, path):
    """operator_mode 1: facet (a, b) deblurs with PSF
    (a, b) alone, alpha_f = gamma omega_f with the interpolation weights, the
    image is the normalised omega-blend -- iterate, objective and image vs the
    oracle's per-node mode."""
    pb = synth.per_node(synth.make_config(k, n=n))
    check_pair(run_pair(pb, 5, path))


def test_per_node_rejects_mismatched_grid():
    pb = synth.make_config(2, n=300)
    with pytest.raises(D.DeblurError) as e:
        D.Deblur.from_problem(pb, operator_mode=D.OP_PER_NODE)      # 2x2 facets, 4x4 PSFs
    assert "facet grid" in str(e.value)


@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
@pytest.mark.parametrize("node", [0, 1], ids=["interp", "per_node"])
def test_iterate_independent(node, path):
    """The independent baseline (no consensus, alpha = 0) vs the oracle."""
    pb = synth.make_config(2, n=300, facets=(2, 2), overlap=40)
    if node:
        pb = synth.per_node(pb)
    pb.independent = 1
    check_pair(run_pair(pb, 5, path))


def test_two_live_handles_of_different_geometry():
    """Kernel attributes (dynamic shared-memory limits) are process-wide: a second
    handle with smaller tiles must not break a live one (regression)."""
    pa = synth.make_config(2, n=300, facets=(1, 1), overlap=0)
    pb = synth.per_node(synth.make_config(2, n=300))
    with D.Deblur.from_problem(pa, conv_path=D.CONV_FFT) as ref:
        ref.iterate(3)
        xr, _ = ref.get_state()
    with D.Deblur.from_problem(pa, conv_path=D.CONV_FFT) as a:
        with D.Deblur.from_problem(pb, conv_path=D.CONV_FFT) as b:
            b.iterate(2)
        a.iterate(3)
        xa, _ = a.get_state()
        a.objective()
    np.testing.assert_array_equal(xa, xr)


# ------------------------------------------------------------------ VMLM-B Local-Solver (NEXT-1)
@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
@pytest.mark.parametrize("k,n,facets,O,budget,inc,iters", [
    (1, 120, (1, 1), 0, 60, 0, 1),          # one converged local prox (unique minimiser)
    (2, 200, (2, 2), 20, 20, 0, 3),         # Algorithm 1, fixed inner budget
    (2, 200, (2, 2), 20, 10, 10, 3),        # the paper's budget schedule 10 + 10 k
], ids=["prox", "dr", "schedule"])
def test_iterate_vmlmb(k, n, facets, O, budget, inc, iters, path):
    """VMLM-B Local-Solver (reading V1-V6) vs the oracle's VMLM-B: iterate and
    objective after a fixed number of outer iterations.  The facet proxes are
    ill-conditioned in the bands (alpha = gamma omega -> small at band edges), so
    they do not converge in these budgets and parity is on fixed-count iterates;
    the fp32 / fp64 gap of L-BFGS grows with the inner iteration count (measured
    1.1e-3 after 3 x 30 on c2@200), so the budgets stay <= 30 per call."""
    pb = synth.make_config(k, n=n, facets=facets, overlap=O)
    pb.local_solver, pb.inner_steps, pb.inner_increment = 1, budget, inc
    orc = from_problem(pb)
    with D.Deblur.from_problem(pb, conv_path=path, tau=orc.tau) as dev:
        dev.iterate(iters)
        xs, us = dev.get_state()
        obj = dev.objective()
    orc.iterate(iters)
    xr, ur = orc.state()
    xr_f, ur_f = [a.copy() for a in orc.x], [a.copy() for a in orc.u]
    assert rel_l2(xs, xr) <= IT_TOL, rel_l2(xs, xr)
    assert rel_l2(us, ur) <= IT_TOL, rel_l2(us, ur)
    # The objective bar (1e-4) applies to the objective *function* (Eq. (4), A22): the
    # oracle evaluates it at the GPU's own iterate.  Along the two trajectories the
    # objectives differ by what the iterates differ by (the L-BFGS fp32 / fp64 drift,
    # bounded by the iterate bar above; reading V7).
    at_gpu = load_state(orc, xs, us).objective()
    for i in range(3):
        assert abs(obj[i] - at_gpu[i]) <= OBJ_TOL * abs(at_gpu[i]), (i, obj[i], at_gpu[i])
    orc.x, orc.u = [a.copy() for a in xr_f], [a.copy() for a in ur_f]
    ro = orc.objective()
    for i in range(3):
        assert abs(obj[i] - ro[i]) <= IT_TOL * abs(ro[i]), (i, obj[i], ro[i])


@pytest.mark.parametrize("rem", [193, 194, 195, 60])
def test_fft_strip_plan_boundaries(rem):
    """S/2 strip plan: facets whose last tile row / column holds
    `rem` valid outputs (T = 450, T/2-plan T2 = 194 at P = 63): the strip plan is
    used iff rem <= T2; H / H^T stay exact (vs the oracle) either way."""
    P, T = 63, 450
    m = T + rem                                       # one facet: observed extent T + rem per axis
    n = m + P - 1
    pb = synth.make_config(3, n=n, facets=(1, 1), overlap=0)
    x, r = rand_x(pb), rand_r(pb)
    op = oracle_op(pb)
    with D.Deblur.from_problem(pb, conv_path=D.CONV_FFT) as dev:
        hx = dev.apply_H(x)
        g = dev.apply_HT(r)
        st = dev.kernel_stats()
    assert (st["H_fft2_cols"][0] > 0) == (rem <= 194)
    assert (st["HT_fft2_cols"][0] > 0) == (rem + P - 1 <= 194)
    assert rel_l2(hx, op.H(x)) <= H_TOL
    assert rel_l2(g, op.HT(r)) <= H_TOL


def test_fft_strips_match_single_plan(monkeypatch):
    """The two-plan split changes only the tiling: iterates equal the single-plan
    run within rounding."""
    pb = synth.make_config(3, n=1024, facets=(2, 2), overlap=128)
    with D.Deblur.from_problem(pb, conv_path=D.CONV_FFT) as dev:
        dev.iterate(3)
        xa, _ = dev.get_state()
    monkeypatch.setenv("DEBLUR_FFT_NO_STRIPS", "1")
    with D.Deblur.from_problem(pb, conv_path=D.CONV_FFT) as dev:
        dev.iterate(3)
        xb, _ = dev.get_state()
    assert rel_l2(xa, xb) <= 1e-6


@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
@pytest.mark.parametrize("combo", ["node_vmlmb", "indep_vmlmb"])
def test_combined_modes(combo, path):
    """Per-node operators and the independent baseline with the VMLM-B Local-Solver."""
    pb = synth.make_config(2, n=200, facets=(2, 2), overlap=20)
    if combo == "node_vmlmb":
        pb = synth.per_node(pb)
    else:
        pb.independent = 1
    pb.local_solver, pb.inner_steps, pb.inner_increment = 1, 10, 5
    orc = from_problem(pb)
    with D.Deblur.from_problem(pb, conv_path=path, tau=orc.tau) as dev:
        dev.iterate(2)
        xs, us = dev.get_state()
        img = dev.get_image()
    orc.iterate(2)
    xr, ur = orc.state()
    assert rel_l2(xs, xr) <= IT_TOL
    assert rel_l2(us, ur) <= IT_TOL
    assert rel_l2(img, orc.image()) <= IT_TOL


def test_vmlmb_reset_restarts_the_budget_schedule():
    """deblur_reset starts a fresh solve: the VMLM-B budget (inner_steps + k inner_increment)
    restarts at k = 0, so reset + n iterations == a fresh handle's n iterations."""
    pb = synth.make_config(2, n=200, facets=(2, 2), overlap=20)
    pb.local_solver, pb.inner_steps, pb.inner_increment = 1, 5, 5
    with D.Deblur.from_problem(pb, conv_path=D.CONV_FFT) as dev:
        dev.iterate(2)
        dev.reset(pb.y)
        dev.iterate(2)
        xa, ua = dev.get_state()
    with D.Deblur.from_problem(pb, conv_path=D.CONV_FFT) as dev:
        dev.iterate(2)
        xb, ub = dev.get_state()
    np.testing.assert_array_equal(xa, xb)
    np.testing.assert_array_equal(ua, ub)


def test_vmlmb_checkpoint_resume_with_outer_iteration():
    """A checkpoint of (x_f, u_f, k) resumes the VMLM-B run exactly: the inner budget
    inner_steps + k inner_increment continues from the stored outer iteration k."""
    pb = synth.make_config(2, n=200, facets=(2, 2), overlap=20)
    pb.local_solver, pb.inner_steps, pb.inner_increment = 1, 4, 3
    with D.Deblur.from_problem(pb, conv_path=D.CONV_FFT) as dev:
        dev.iterate(3)
        xa, ua = dev.get_state()
    with D.Deblur.from_problem(pb, conv_path=D.CONV_FFT) as dev:
        dev.iterate(2)
        xs, us = dev.get_state()
        k = dev.outer_iteration
    assert k == 2
    with D.Deblur.from_problem(pb, conv_path=D.CONV_FFT) as dev:
        dev.set_state(xs, us)
        dev.outer_iteration = k
        dev.iterate(1)
        xb, ub = dev.get_state()
        with pytest.raises(ValueError):
            dev.set_state(xs[:-1], us)
    np.testing.assert_array_equal(xa, xb)
    np.testing.assert_array_equal(ua, ub)


@pytest.mark.parametrize("path", PATHS, ids=["direct", "fft"])
def test_pipelined_jobs_equal_serial_jobs(path):
    """deblur_stage_y / reset_staged / get_image_async (the next observation uploaded and
    the previous image downloaded while a job iterates) give exactly the serial jobs'
    images: three different observations back to back."""
    pb = synth.make_config(2, n=300, facets=(3, 2), overlap=40)
    ys = [np.ascontiguousarray((pb.y * s + 0.01 * i).astype(np.float32)) for i, s in enumerate((1.0, 0.7, 1.3))]
    with D.Deblur.from_problem(pb, conv_path=path) as dev:
        ref = []
        for y in ys:
            dev.reset(y)
            dev.iterate(5)
            ref.append(dev.get_image())
        outs = [np.empty((pb.ny, pb.nx), np.float32) for _ in ys]
        dev.stage_y(ys[0])
        for j in range(len(ys)):
            dev.reset_staged()
            if j + 1 < len(ys):
                dev.stage_y(ys[j + 1])
            dev.iterate(5)
            dev.get_image_async(outs[j])
        dev.sync()
        with pytest.raises(D.DeblurError):
            dev.reset_staged()                    # nothing staged
    for a, b in zip(outs, ref):
        np.testing.assert_array_equal(a, b)
