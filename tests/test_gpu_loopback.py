"""The multi-rank exchange path on one GPU (loopback transport, params.loopback_world).

With loopback_world = V the library assigns the facets to V virtual ranks with the
same GPU-grid planner as a world-V run; every band shared by facets of different
virtual ranks goes through the real multi-rank code: the pack of each message into
its send buffer, the transport into the matching receive buffer (a device copy in
place of ncclSend/ncclRecv) and the consensus kernel reading the receive buffers
through its remote-neighbour views.  Algorithm 1's consensus sums in ascending facet
id (A9), so the result must be BITWISE equal to the single-rank run for every V
("bit-identical" backends), with CUDA graphs on and off.
"""
import numpy as np
import pytest

import synth
from oracle import from_problem
from paper_1705_06603_b200 import deblur as D
from tests.fullsize import full_config

pytestmark = pytest.mark.gpu


def run(pb, iters, V, path, **over):
    with D.Deblur.from_problem(pb, conv_path=path, loopback_world=V, **over) as dev:
        dev.iterate(iters)
        x, u = dev.get_state()
        obj = dev.objective()
        img = dev.get_image()
        st = dev.kernel_stats()
    return x, u, np.array(obj), img, st


CASES = [
    # (config, n, facets, overlap, virtual world sizes)
    (2, None, (2, 2), 64, (2, 4)),          # c2 geometry, full size
    (3, 1024, (2, 4), 128, (2, 4, 8)),      # c3 facet grid (BASELINE GPU sweep 1/2/4/8)
    (2, 300, (3, 2), 40, (2, 3, 6)),        # ragged 3x2 grid, a 3-way split
]


@pytest.mark.parametrize("graphs", [True, False], ids=["graphs", "eager"])
@pytest.mark.parametrize("path", [D.CONV_FFT, D.CONV_DIRECT], ids=["fft", "direct"])
@pytest.mark.parametrize("k,n,facets,O,worlds", CASES)
def test_loopback_bitwise_equal(k, n, facets, O, worlds, path, graphs, monkeypatch):
    if not graphs:
        monkeypatch.setenv("DEBLUR_NO_GRAPHS", "1")
    pb = synth.make_config(k, n=n, facets=facets, overlap=O)
    tau = from_problem(pb).tau
    x1, u1, o1, i1, _ = run(pb, 6, 0, path, tau=tau)
    for V in worlds:
        xv, uv, ov, iv, st = run(pb, 6, V, path, tau=tau)
        assert st["halo_exchange"][0] > 0                        # the exchange path ran
        np.testing.assert_array_equal(xv, x1)
        np.testing.assert_array_equal(uv, u1)
        np.testing.assert_array_equal(ov, o1)
        np.testing.assert_array_equal(iv, i1)


def test_loopback_c4_full_size_gpu_sweep():
    """BASELINE's 1 -> 8 GPU sweep on c4 (16384^2, 4x2 facets) through the loopback transport,
    in the launch configuration bench.py times (FFT path, graph replay): the facet states and
    the objective after 3 iterations (both graph parities) are bitwise those of the
    single-rank run for 2, 4 and 8 virtual ranks."""
    pb = full_config(4)
    ref = None
    for V in (0, 2, 4, 8):
        with D.Deblur.from_problem(pb, loopback_world=V) as dev:
            assert dev.conv_path == D.CONV_FFT
            dev.iterate(3)
            x, u = dev.get_state()
            obj = np.array(dev.objective())
            n_x = dev.kernel_stats()["halo_exchange"][0]
        if V == 0:
            ref = (x, u, obj)
            continue
        assert n_x > 0
        np.testing.assert_array_equal(x, ref[0])
        np.testing.assert_array_equal(u, ref[1])
        np.testing.assert_array_equal(obj, ref[2])
        del x, u


def test_loopback_vmlmb_and_traced():
    """VMLM-B Local-Solver (eager, host decisions) and the traced objective over the
    loopback transport: bitwise equal to the single-rank run."""
    pb = synth.make_config(2, n=300, facets=(2, 2), overlap=40)
    pb.local_solver, pb.inner_steps, pb.inner_increment = 1, 5, 5
    out = []
    for V in (0, 4):
        with D.Deblur.from_problem(pb, conv_path=D.CONV_FFT, loopback_world=V) as dev:
            tr = dev.iterate_traced(3)
            x, u = dev.get_state()
        out.append((tr, x, u))
    for a, b in zip(out[0], out[1]):
        np.testing.assert_array_equal(a, b)


def test_loopback_matches_oracle():
    """The loopback run is also an oracle-parity run (c2 geometry, 20 iterations)."""
    pb = synth.make_config(2, facets=(2, 2), overlap=64)
    orc = from_problem(pb)
    with D.Deblur.from_problem(pb, tau=orc.tau, loopback_world=4) as dev:
        dev.iterate(20)
        xs, us = dev.get_state()
    orc.iterate(20)
    xr, ur = orc.state()
    assert np.linalg.norm(xs - xr) / np.linalg.norm(xr) <= 1e-3
    assert np.linalg.norm(us - ur) / np.linalg.norm(ur) <= 1e-3


@pytest.mark.parametrize("V", [4, 16])
def test_loopback_per_node_and_independent(V):
    """Per-node operators (16 facets = the 4x4 PSF grid, nearly every pixel shared by 4
    facets) and the independent baseline (no exchange at all) over the loopback transport."""
    base = synth.per_node(synth.make_config(2, n=300))
    for pb in (base, synth.make_config(2, n=300, facets=(4, 4), overlap=20)):
        if pb is not base:
            pb.independent = 1
        x1, u1, o1, i1, _ = run(pb, 4, 0, D.CONV_FFT)
        xv, uv, ov, iv, _ = run(pb, 4, V, D.CONV_FFT)
        np.testing.assert_array_equal(xv, x1)
        np.testing.assert_array_equal(uv, u1)
        np.testing.assert_array_equal(ov, o1)
        np.testing.assert_array_equal(iv, i1)
