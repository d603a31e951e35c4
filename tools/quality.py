"""Deblurring quality of the three methods the paper compares (PAPER.md:266,
:296-301) on a synthetic star field with a known truth:

  centralized  one facet, no prox term (alpha = 0): the Local-Solver minimises Eq. (3)
  proposed     the facet grid of the config, consensus on the overlaps (Algorithm 1)
  independent  the same facets, no consensus, alpha = 0, omega-blend (deblur independent=1)

Solvers (--solver): vmlmb (default, the paper's setting P:287-290): centralized and
independent run VMLM-B for --budget inner iterations (the paper: up to 1000), the
proposed method --outer outer iterations (25) with the 10 + 10k inner schedule;
pg: every method runs --iters fixed-step projected-gradient steps (the north-star path).

The observation is y = H x_true + n with H the library's own forward operator
(deblur_apply_H of a one-facet handle: the PSF-interpolation model) and Gaussian
noise of the config's sigma.  Each method runs the same number of iterations from
the A6 start; reported: SNR and SSIM (paper_1705_06603_b200/quality.py, data range of
x_true), and the global Eq. (3)+TV objective of the merged image (one-facet handle).  The paper's qualitative finding
is proposed ~ centralized > independent.  GPU only; results -> stdout (JSON lines).

The paper compares the methods over "different values of lambda in a sufficiently large
range": --lambdas runs every method at every value and reports each method's best.

  python tools/quality.py [--config 2] [--n 1024] [--solver vmlmb] [--operator-mode 0]
                          [--lambdas 0.001,0.01,0.1,1]
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1705_06603_b200 import deblur as D  # noqa: E402
from paper_1705_06603_b200.quality import snr, ssim  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--solver", choices=["vmlmb", "pg"], default="vmlmb")
    ap.add_argument("--iters", type=int, default=400, help="pg: steps of every method")
    ap.add_argument("--budget", type=int, default=1000, help="vmlmb: centralized / independent inner iterations")
    ap.add_argument("--outer", type=int, default=25, help="vmlmb: proposed outer iterations (10 + 10k inner)")
    ap.add_argument("--operator-mode", type=int, default=0)
    ap.add_argument("--seed", type=int, default=77)
    ap.add_argument("--lambdas", default=None, help="comma-separated lambda sweep (default: the config's lambda)")
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
    lams = [float(v) for v in args.lambdas.split(",")] if args.lambdas else [pb.lam]
    best = {}
    for lam in lams:
        res = run_methods(args, pb, one, y, x_true, lam)
        for name, r in res.items():
            if name not in best or r["snr_db"] > best[name]["snr_db"]:
                best[name] = dict(r, lam=lam)
    print(json.dumps({"config": f"c{args.config}", "n": n, "solver": args.solver, "iters": args.iters,
                      "budget": args.budget, "outer": args.outer, "operator_mode": args.operator_mode,
                      "lambdas": lams,
                      "best": {k: {"snr_db": v["snr_db"], "ssim": v["ssim"], "lam": v["lam"]} for k, v in best.items()}}))


def run_methods(args, pb, one, y, x_true, lam):
    one = dataclasses.replace(one, lam=lam)
    pb = dataclasses.replace(pb, lam=lam)
    if args.solver == "pg":
        methods = {
            "centralized": (dataclasses.replace(one, y=y, independent=1), args.iters),
            "proposed": (dataclasses.replace(pb, y=y, independent=0), args.iters),
            "independent": (dataclasses.replace(pb, y=y, independent=1), args.iters),
        }
    else:       # VMLM-B; 25 outer iterations of 10 + 10k for the proposed method
        vm = dict(local_solver=1, inner_increment=0, inner_steps=args.budget)
        methods = {
            "centralized": (dataclasses.replace(one, y=y, independent=1, **vm), 1),
            "proposed": (dataclasses.replace(pb, y=y, independent=0, local_solver=1, inner_steps=10,
                                             inner_increment=10), args.outer),
            "independent": (dataclasses.replace(pb, y=y, independent=1, **vm), 1),
        }
    out = {}
    with D.Deblur.from_problem(dataclasses.replace(one, y=y)) as judge:
        for name, (p, iters) in methods.items():
            with D.Deblur.from_problem(p) as dev:
                dev.iterate(iters)
                img = dev.get_image()
                obj_local = dev.objective()
            judge.set_state(img.ravel(), img.ravel())
            tot, data, reg, _ = judge.objective()
            out[name] = dict(snr_db=round(snr(x_true, img), 3), ssim=round(ssim(x_true, img, float(x_true.max() - x_true.min())), 4),
                             objective_global=tot, data=data, reg=reg, consensus_maxdiff=obj_local[3],
                             facets=f"{p.fy}x{p.fx}", overlap=p.overlap)
            print(json.dumps({"method": name, "lam": lam, **out[name]}), flush=True)
    return out


if __name__ == "__main__":
    main()
