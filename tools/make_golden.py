"""Write full-size oracle golden files for the GPU parity tests (tests/golden/).

TEST INFRASTRUCTURE.  Calls only oracle/ (the fp64 reference) and synth/ (the
seeded inputs); nothing here touches the CUDA path, so every stored value is the
oracle's.  For BASELINE config k it runs Algorithm 1 (readings of
DESIGN.md §2) from the A6 start for `iters` outer iterations at the BASELINE
geometry and stores

  * the input hash (synth.input_hash) the values belong to, and the step tau (A4');
  * the objective of Eq. (4) (A22) at x^(0..iters): total, data, reg,
    consensus max-difference;
  * x_f and u_f (fp64) at sampled entries of the concatenated facet state (planner
    order) covering every pixel class: single-owner interior, facet borders (where the
    circular D of A2 wraps), 2-facet edge bands and 4-facet corner bands (Lemma 1,
    PAPER.md:169-175);
  * the blended image x_hat = sum_f omega^F_f x_f (A7) at sampled global pixels.

Usage:  python tools/make_golden.py 3 100      (c3, 100 iterations: ~2 h on 8 cores)
        python tools/make_golden.py 4 2        (c4, a stated 2-iteration prefix)
        python tools/make_golden.py 4 50 --checkpoints 10,20,30,40 --objective-every 5
                                               (c4, the BASELINE 50 iterations, a file every 10)
        python tools/make_golden.py 5 0 --objective-only
                                               (c5: Eq. (4) at the A6 start, facet by facet; a full
                                                c5 oracle iteration needs > 62 GB of host memory)
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import from_problem, geometry  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pixel_classes(facets):
    """Per facet: boolean masks (local) of the sampled classes."""
    out = []
    for f in facets:
        ny, nx = f.ey[1] - f.ey[0], f.ex[1] - f.ex[0]
        cnt = np.zeros((ny, nx), np.int32)
        for g in facets:
            y0, y1 = max(f.ey[0], g.ey[0]), min(f.ey[1], g.ey[1])
            x0, x1 = max(f.ex[0], g.ex[0]), min(f.ex[1], g.ex[1])
            if y0 < y1 and x0 < x1:
                cnt[y0 - f.ey[0]:y1 - f.ey[0], x0 - f.ex[0]:x1 - f.ex[0]] += 1
        border = np.zeros((ny, nx), bool)
        border[:2, :] = border[-2:, :] = True
        border[:, :2] = border[:, -2:] = True
        out.append(dict(single=(cnt == 1) & ~border, edge=cnt == 2, corner=cnt >= 3, border=border))
    return out


def sample_state(facets, rng, n_random, n_per_class):
    """Indices into the concatenated state: n_random uniform + n_per_class from each
    class (edge band, corner band, facet border), spread over the facets."""
    sizes = [(f.ey[1] - f.ey[0]) * (f.ex[1] - f.ex[0]) for f in facets]
    offs = np.cumsum([0] + sizes)
    idx = [rng.integers(0, offs[-1], n_random)]
    cls = pixel_classes(facets)
    for name in ("edge", "corner", "border"):
        per = []
        for i, c in enumerate(cls):
            flat = np.flatnonzero(c[name].ravel())
            if flat.size:
                per.append(offs[i] + flat)
        if not per:
            continue
        allc = np.concatenate(per)
        idx.append(allc[rng.integers(0, allc.size, n_per_class)])
    idx = np.unique(np.concatenate(idx))
    return idx.astype(np.int64)


def objective_only(a):
    """Eq. (4) (A22) at x^(0) = u^(0) = the A6 start, per facet with the oracle's own
    pieces: data_f = 1/2 sum_{O_f} W (H_f x_f - y)^2 (Operator.H_window), reg_f = sum phi(D x_f)
    (tv.value, circular per facet); the facets agree at the start, so the consensus
    max-difference is 0."""
    from oracle import Operator, tv
    t0 = time.time()
    pb = synth.make_config(a.k)
    h = synth.input_hash(pb)
    facets = geometry.plan(pb.ny, pb.nx, pb.P, pb.fy, pb.fx, pb.overlap)
    op = Operator(pb.psfs, pb.wy, pb.wx)
    c = op.c
    y = pb.y
    w_s = np.float64(np.float32(pb.noise_w_scalar))
    data = np.zeros(len(facets))
    reg = np.zeros(len(facets))
    for i, f in enumerate(facets):
        # x0 restricted to P_f: max(0, y edge-replicated into the c-wide margin) (A6)
        rows = np.clip(np.arange(f.ey[0], f.ey[1]) - c, 0, pb.my - 1)
        cols = np.clip(np.arange(f.ex[0], f.ex[1]) - c, 0, pb.mx - 1)
        xf = np.maximum(0.0, y[np.ix_(rows, cols)].astype(np.float64))
        d = op.H_window(xf, f.ey[0], f.ex[0]) - y[f.oy[0]:f.oy[1], f.ox[0]:f.ox[1]].astype(np.float64)
        w = pb.noise_w[f.oy[0]:f.oy[1], f.ox[0]:f.ox[1]].astype(np.float64) if pb.noise_w is not None else w_s
        data[i] = 0.5 * float((w * d * d).sum())
        reg[i] = tv.value(xf, pb.eps, pb.reg_kind, pb.tv_boundary)
        print(f"  facet {i}: data {data[i]:.9e} reg {reg[i]:.9e} ({time.time() - t0:.0f} s)", flush=True)
    tot_d, tot_r = float(data.sum()), float(pb.lam * reg.sum())
    out = a.out or os.path.join(GOLDEN, f"c{a.k}_obj0.npz")
    np.savez_compressed(out, config=a.k, iters=0, input_hash=h, trace=np.array([[tot_d + tot_r, tot_d, tot_r, 0.0]]),
                        made_by="tools/make_golden.py --objective-only (oracle/ + synth/ only)")
    print(f"wrote {out}: objective {tot_d + tot_r:.12e} ({time.time() - t0:.0f} s)", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("k", type=int)
    ap.add_argument("iters", type=int)
    ap.add_argument("--n-random", type=int, default=60000)
    ap.add_argument("--n-class", type=int, default=20000)
    ap.add_argument("--out", default=None)
    ap.add_argument("--checkpoints", default="",
                    help="comma-separated iteration counts at which a golden file is also written")
    ap.add_argument("--objective-every", type=int, default=1,
                    help="evaluate Eq. (4) at every n-th iterate (and at each checkpoint)")
    ap.add_argument("--objective-only", action="store_true",
                    help="only Eq. (4) at the A6 start, evaluated facet by facet (no global arrays)")
    a = ap.parse_args()
    if a.objective_only:
        return objective_only(a)

    t0 = time.time()
    pb = synth.make_config(a.k)
    h = synth.input_hash(pb)
    orc = from_problem(pb)
    facets = geometry.plan(pb.ny, pb.nx, pb.P, pb.fy, pb.fx, pb.overlap)
    print(f"c{a.k}: inputs {h[:16]}, tau {orc.tau!r}, {len(facets)} facets, setup {time.time() - t0:.0f} s",
          flush=True)
    rng = np.random.default_rng(20000 + a.k)
    idx = sample_state(facets, rng, a.n_random, a.n_class)
    gi = rng.integers(0, pb.ny, 20000)
    gj = rng.integers(0, pb.nx, 20000)
    # a file per checkpoint (the last one = iters); the objective at every `objective_every`-th
    # iterate and at each checkpoint, NaN rows elsewhere (the test skips them)
    checkpoints = sorted({int(c) for c in a.checkpoints.split(",") if c} | {a.iters}) if a.checkpoints else [a.iters]
    trace = np.full((a.iters + 1, 4), np.nan)
    for it in range(a.iters + 1):
        to = 0.0
        if it % a.objective_every == 0 or it in checkpoints:
            t = time.time()
            trace[it] = orc.objective()
            to = time.time() - t
        if it in checkpoints:
            xs, us = orc.state()
            img = orc.image()
            out = (a.out if (a.out and it == a.iters) else
                   os.path.join(GOLDEN, f"c{a.k}_it{it}.npz"))
            np.savez_compressed(out, config=a.k, iters=it, input_hash=h, tau=orc.tau, trace=trace[:it + 1],
                                idx=idx, x=xs[idx], u=us[idx], img_i=gi, img_j=gj, img=img[gi, gj],
                                made_by="tools/make_golden.py (oracle/ + synth/ only)")
            del xs, us, img
            print(f"wrote {out}: {idx.size} state samples, {time.time() - t0:.0f} s total", flush=True)
        if it < a.iters:
            t = time.time()
            orc.iterate(1)
            print(f"  it {it}: objective {trace[it, 0]:.9e} ({to:.0f} s), iterate {time.time() - t:.0f} s",
                  flush=True)

if __name__ == "__main__":
    main()
