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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("k", type=int)
    ap.add_argument("iters", type=int)
    ap.add_argument("--n-random", type=int, default=60000)
    ap.add_argument("--n-class", type=int, default=20000)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()

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
    trace = np.zeros((a.iters + 1, 4))
    for it in range(a.iters + 1):
        t = time.time()
        trace[it] = orc.objective()
        to = time.time() - t
        if it < a.iters:
            t = time.time()
            orc.iterate(1)
            print(f"  it {it}: objective {trace[it, 0]:.9e} ({to:.0f} s), iterate {time.time() - t:.0f} s",
                  flush=True)
    xs, us = orc.state()
    img = orc.image()
    out = a.out or os.path.join(GOLDEN, f"c{a.k}_it{a.iters}.npz")
    np.savez_compressed(out, config=a.k, iters=a.iters, input_hash=h, tau=orc.tau, trace=trace,
                        idx=idx, x=xs[idx], u=us[idx], img_i=gi, img_j=gj, img=img[gi, gj],
                        made_by="tools/make_golden.py (oracle/ + synth/ only)")
    print(f"wrote {out}: {idx.size} state samples, {time.time() - t0:.0f} s total", flush=True)


if __name__ == "__main__":
    main()
