"""Deblurring quality of the three methods the paper compares (PAPER.md:266,
:296-301) on a synthetic star field with a known truth:

  centralized  one facet, Algorithm 1 degenerates to the Local-Solver on Eq. (3)
  proposed     the facet grid of the config, consensus on the overlaps (Algorithm 1)
  independent  the same facets, no consensus, alpha = 0, omega-blend (deblur independent=1)

The observation is y = H x_true + n with H the library's own forward operator
(deblur_apply_H of a one-facet handle: the PSF-interpolation model) and Gaussian
noise of the config's sigma.  Each method runs the same number of iterations from
the A6 start; reported: SNR = 10 log10(|x|^2 / |x_hat - x|^2), SSIM (Gaussian
window 11 / 1.5, data range of x_true), and the global Eq. (3)+TV objective of the
merged image (evaluated with a one-facet handle).  The paper's qualitative finding
is proposed ~ centralized > independent.  GPU only; results -> stdout (JSON lines).

  python tools/quality.py [--config 2] [--n 1024] [--iters 400] [--operator-mode 0]
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import sys

import numpy as np
import scipy.ndimage

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1705_06603_b200 import deblur as D  # noqa: E402


def snr_db(xh, x):
    return 10.0 * math.log10(float((x ** 2).sum()) / float(((xh - x) ** 2).sum()))


def ssim(a, b, rng_):
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    f = lambda z: scipy.ndimage.gaussian_filter(z, 1.5, truncate=3.5)   # 11-tap window
    c1, c2 = (0.01 * rng_) ** 2, (0.03 * rng_) ** 2
    ma, mb = f(a), f(b)
    va, vb, cab = f(a * a) - ma * ma, f(b * b) - mb * mb, f(a * b) - ma * mb
    s = ((2 * ma * mb + c1) * (2 * cab + c2)) / ((ma * ma + mb * mb + c1) * (va + vb + c2))
    return float(s.mean())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--iters", type=int, default=400)
    ap.add_argument("--operator-mode", type=int, default=0)
    ap.add_argument("--seed", type=int, default=77)
    args = ap.parse_args()
    pb = synth.make_config(args.config, n=args.n)
    if args.operator_mode == 1:
        pb = synth.per_node(pb)
    n = pb.ny
    src = synth.CONFIGS[args.config]["sources"] * (n / synth.CONFIGS[args.config]["n"]) ** 2
    x_true = synth.render_scene(n, max(1, int(src)), args.seed).astype(np.float32)
    sigma = synth.CONFIGS[args.config]["noise"][1]
    one = dataclasses.replace(pb, fy=1, fx=1, overlap=0, operator_mode=0, independent=0)
    with D.Deblur.from_problem(one) as dev:
        y_clean = dev.apply_H(x_true)
    rng = np.random.default_rng(args.seed)
    y = (y_clean + sigma * rng.standard_normal(y_clean.shape)).astype(np.float32)
    methods = {
        "centralized": dataclasses.replace(one, y=y),
        "proposed": dataclasses.replace(pb, y=y, independent=0),
        "independent": dataclasses.replace(pb, y=y, independent=1),
    }
    out = {}
    with D.Deblur.from_problem(dataclasses.replace(one, y=y)) as judge:
        for name, p in methods.items():
            with D.Deblur.from_problem(p) as dev:
                dev.iterate(args.iters)
                img = dev.get_image()
                obj_local = dev.objective()
            judge.set_state(img.ravel(), img.ravel())
            tot, data, reg, _ = judge.objective()
            out[name] = dict(snr_db=round(snr_db(img, x_true), 3), ssim=round(ssim(img, x_true, float(x_true.max() - x_true.min())), 4),
                             objective_global=tot, data=data, reg=reg, consensus_maxdiff=obj_local[3],
                             facets=f"{p.fy}x{p.fx}", overlap=p.overlap)
            print(json.dumps({"method": name, **out[name]}), flush=True)
    print(json.dumps({"config": f"c{args.config}", "n": n, "iters": args.iters, "operator_mode": args.operator_mode,
                      "summary": {k: v["snr_db"] for k, v in out.items()}}))


if __name__ == "__main__":
    main()
