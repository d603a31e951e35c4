"""Cost model of FFT tile placement against the PSF grid (SURVEY §7 "tile <-> PSF-cell
alignment"), on the real facet geometry of a config.

Per tile, the column pass runs one length-S DFT per active (p, q) plus one more (H: the
inverse; H^T: the forward of R), the row passes n_q + 1 real transforms; a tile's cost is
proportional to S^2 log2 S times those counts.  The active hats of a tile are the
interpolation weights wy_p / wx_q that are nonzero on its window (H: the S-wide input
window, the hats multiply x before blurring; H^T: the T-wide output range, they multiply
after correlating; A16).  Placements compared:

  uniform   the library's tiling: tiles every T from the facet origin, S = 512 (T = 450)
  aligned   the same S, tiles restarted at every grid-centre line so that no window
            straddles one where possible (the remainder of each cell period becomes a
            short tile)
  S576      H^T only, S = 576 = 2^6 3^2, T = 514 >= 512 = half a cell: every output
            range inside one half-cell (exactly 2 hats per axis)

Prints relative column-pass and row-pass work per iteration (uniform = 1).

  python tools/tile_alignment.py [--config 4]
"""
from __future__ import annotations

import argparse
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1705_06603_b200 import deblur as D  # noqa: E402


def nz_count(w, a, b):
    a, b = max(0, a), min(w.shape[1], b)
    return int((w[:, a:b] != 0).any(axis=1).sum()) if b > a else 0


def axis_tiles(e0, n_out, T, S, w, ht, centres, mode):
    """[(n_hats, S_used)] of the tiles covering n_out outputs of an axis whose estimate
    block starts at e0."""
    out, y = [], 0
    while y < n_out:
        t = min(T, n_out - y)
        if mode == "aligned":
            a = e0 + y
            nxt = [c for c in centres if c > a]
            if nxt:
                lim = nxt[0] - a if ht else nxt[0] - a - (S - T)      # keep the window left of the centre
                if 0 < lim < t and lim >= T // 4:
                    t = lim
        a, b = (e0 + y, e0 + y + t) if ht else (e0 + y, e0 + y + t + (S - T))
        out.append((nz_count(w, a, b), S))
        y += t
    return out


def cost(tiles_y, tiles_x, S_ref):
    col = row = 0.0
    for ny, sy in tiles_y:
        for nx, sx in tiles_x:
            s = sy
            unit = (s * s * math.log2(s)) / (S_ref * S_ref * math.log2(S_ref))
            col += (ny * nx + 1) * unit
            row += (nx + 1) * unit
    return col, row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    a = ap.parse_args()
    pb = synth.make_config(a.config)
    params, keep = D.problem_params(pb)
    boxes, _ = D.plan_facets(params)
    P = pb.P
    G = pb.gy
    L = pb.ny / G
    centres = [int(round((k + 0.5) * L)) for k in range(G)]
    res = {}
    for name, S, ht_only in (("uniform", 512, False), ("aligned", 512, False), ("S576", 576, True)):
        T = S - P + 1
        tot = {"H": [0.0, 0.0], "HT": [0.0, 0.0]}
        for b in boxes:
            oy0, oy1, ox0, ox1, ey0, ey1, ex0, ex1 = (int(v) for v in b)
            for op, ht in (("H", False), ("HT", True)):
                if ht_only and not ht:
                    continue
                mode = "aligned" if name in ("aligned", "S576") else "uniform"
                ny_out, nx_out = (ey1 - ey0, ex1 - ex0) if ht else (oy1 - oy0, ox1 - ox0)
                ty = axis_tiles(ey0, ny_out, T, S, pb.wy, ht, centres, mode)
                tx = axis_tiles(ex0, nx_out, T, S, pb.wx, ht, centres, mode)
                c, r = cost(ty, tx, 512)
                tot[op][0] += c
                tot[op][1] += r
        res[name] = tot
    base = res["uniform"]
    for name, tot in res.items():
        parts = []
        for op in ("H", "HT"):
            if tot[op][0] == 0:
                continue
            parts.append(f"{op}: columns {tot[op][0] / base[op][0]:.3f}, rows {tot[op][1] / base[op][1]:.3f}")
        print(f"{name:8s} " + "; ".join(parts))


if __name__ == "__main__":
    main()
