#!/usr/bin/env python
"""Measure the direct-vs-FFT crossover in P (SURVEY §8d "Sweep"): 4096^2 scene,
8x8 PSF grid of random non-negative unit-sum PSFs, 1 facet; for each P time one
Local-Solver step's operator kernels with CUDA events inside libdeblur
(deblur_set_profiling): direct = K1 + K2 (K2 includes the fused update),
FFT = the six FFT passes + the update kernel.  Prints one JSON line per (P, path)
and a summary line with the crossover."""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_1705_06603_b200 import deblur as D  # noqa: E402

OPS = {D.CONV_DIRECT: ("H_direct_residual", "HT_direct_update"),
       D.CONV_FFT: ("H_fft_rows", "H_fft_cols", "H_fft_rows_inv", "HT_fft_rows", "HT_fft_cols", "HT_fft_rows_inv",
                    "update_from_g")}


def problem(n, P, G, seed=0):
    rng = np.random.default_rng(seed + P)
    psfs = rng.uniform(0, 1, (G * G, P, P)).astype(np.float32)
    psfs /= psfs.sum(axis=(1, 2), keepdims=True)
    w = synth.hat_weights(n, G).astype(np.float32)
    y = rng.uniform(0, 1, (n - P + 1, n - P + 1)).astype(np.float32)
    return psfs, w, y


def time_path(psfs, w, y, path, steps):
    params, keep = D.make_params(psfs, w, w, y, noise_w_scalar=1e4, lam=0.01, eps=1e-3, gamma=4000.0,
                                 conv_path=path)
    with D.Deblur(params, keep) as dev:
        dev.iterate(2)
        dev.set_profiling(True)
        dev.reset_stats()
        dev.iterate(steps)
        st = dev.kernel_stats()
    return sum(st[k][1] for k in OPS[path]) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--G", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--P", type=str, default="7,11,15,21,31,47,63,95,127")
    args = ap.parse_args()
    res = {}
    for P in [int(v) for v in args.P.split(",")]:
        psfs, w, y = problem(args.n, P, args.G)
        for path, name in ((D.CONV_DIRECT, "direct"), (D.CONV_FFT, "fft")):
            ms = time_path(psfs, w, y, path, args.steps)
            mpix = args.n * args.n / (ms / 1e3) / 1e6
            res[(P, name)] = ms
            print(json.dumps({"P": P, "path": name, "ms_per_step": round(ms, 4), "mpix_iter_s": round(mpix, 1)}),
                  flush=True)
    cross = None
    for P in sorted({p for p, _ in res}):
        if res[(P, "fft")] < res[(P, "direct")]:
            cross = P
            break
    print(json.dumps({"summary": "crossover", "first_P_where_fft_wins": cross,
                      "n": args.n, "G": args.G}), flush=True)


if __name__ == "__main__":
    main()
