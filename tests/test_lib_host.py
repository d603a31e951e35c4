"""Host-side checks of libdeblur (no GPU): the C ABI loads and exports every
symbol include/deblur.h declares; the planner agrees with the oracle's
independent geometry; validation errors name their argument; without an
sm_100 device deblur_create fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

import synth
from oracle import geometry
from paper_1705_06603_b200 import deblur as D

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "deblur.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(deblur_[a-z_0-9A-Z]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = D.lib()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert sorted(D.EXPORTED) == names


def small_params(**over):
    pb = synth.make_config(2, n=256, facets=(2, 3), overlap=32)
    kw = dict(facet_gy=2, facet_gx=3, overlap=32)
    kw.update(over)
    return D.problem_params(pb, **kw) + (pb,)


@pytest.mark.parametrize("fy,fx,O,world", [(2, 3, 32, 1), (2, 2, 32, 2), (2, 3, 32, 6), (1, 1, 0, 1), (3, 1, 20, 3)])
def test_planner_matches_oracle_geometry(fy, fx, O, world):
    params, keep, pb = small_params(facet_gy=fy, facet_gx=fx, overlap=O, world=world, rank=0,
                                    nccl_id_bytes=b"\0" * 128 if world > 1 else None)
    boxes, owner = D.plan_facets(params)
    fac = geometry.plan(pb.ny, pb.nx, pb.P, fy, fx, O)
    assert len(fac) == len(boxes)
    for f, b in zip(fac, boxes):
        assert tuple(b) == (*f.oy, *f.ox, *f.ey, *f.ex)
    assert sorted(set(owner.tolist())) == list(range(world))


def test_planner_messages_are_pairwise_consistent():
    params, keep, pb = small_params(facet_gy=2, facet_gx=2, overlap=32, world=4, nccl_id_bytes=b"\0" * 128)
    boxes, owner = D.plan_facets(params)
    sent = {}
    for r in range(4):
        for m in D.plan_messages(params, r):
            peer, s, d, y0, y1, x0, x1, nbytes = m.tolist()
            assert owner[s] == r and owner[d] == peer and peer != r
            assert nbytes == (y1 - y0) * (x1 - x0) * 4
            sent[(s, d)] = (y0, y1, x0, x1)
    fac = geometry.plan(pb.ny, pb.nx, pb.P, 2, 2, 32)
    expect = {}
    for a, b, (y0, y1, x0, x1) in geometry.neighbours(fac):
        expect[(a, b)] = expect[(b, a)] = (y0, y1, x0, x1)
    assert sent == expect          # every cross-rank neighbour pair, both directions (8-neighbour, A28)


@pytest.mark.parametrize("field,value,needle", [("rho", 2.0, "rho"), ("eps", 0.0, "eps"), ("overlap", 3, "overlap"),
                                                ("inner_steps", 0, "inner_steps"), ("psf_size", 4, "psf_size"),
                                                ("world", 5, "world"), ("operator_mode", 2, "operator_mode"),
                                                ("operator_mode", 1, "facet grid"), ("independent", 3, "independent"),
                                                ("local_solver", 2, "local_solver"),
                                                ("inner_increment", -1, "inner_increment"),
                                                ("loopback_world", -1, "loopback_world"),
                                                ("abi_version", 1, "abi_version")])
def test_validation_names_argument(field, value, needle):
    params, keep, pb = small_params()
    setattr(params, field, value)
    if field == "world":
        params.nccl_id = ctypes.cast(ctypes.create_string_buffer(128), ctypes.c_void_p)
    with pytest.raises(D.DeblurError) as ei:
        D.plan_facets(params)
    assert needle in str(ei.value)


def test_triple_overlap_rejected():
    params, keep, pb = small_params(facet_gy=1, facet_gx=8, overlap=32)
    with pytest.raises(D.DeblurError) as ei:
        D.plan_facets(params)
    assert ei.value.status == -2


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    params, keep, pb = small_params()
    with pytest.raises(D.DeblurError) as ei:
        D.Deblur(params, keep)
    assert ei.value.status == -4       # DEBLUR_ECUDA, never a silent CPU path


def test_loopback_world_validation():
    """loopback_world (the one-process multi-rank path) must factor into a GPU grid of
    the facet grid, and needs world == 1; both are checked before any device work."""
    params, keep, pb = small_params(loopback_world=5)          # 2 x 3 facets: no 5-rank grid
    with pytest.raises(D.DeblurError) as ei:
        D.Deblur(params, keep)
    assert ei.value.status == -2 and "loopback_world" in str(ei.value)
    params, keep, pb = small_params(loopback_world=2, world=2, nccl_id_bytes=b"\0" * 128)
    with pytest.raises(D.DeblurError) as ei:
        D.plan_facets(params)
    assert "loopback_world" in str(ei.value)
