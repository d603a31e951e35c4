"""Print how far the GPU path is from the stored full-size oracle runs (tests/golden/):
rel-L2 of x / u per pixel class, of the image samples, and the largest relative objective
difference along the trace (graph-replay run for the state, traced run for the history).
GPU only; the bars themselves are asserted by tests/test_gpu_golden.py.

  python tools/golden_report.py c3_it100 [c4_it2 ...]
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import synth  # noqa: E402
from paper_1705_06603_b200 import deblur as D  # noqa: E402
from test_gpu_golden import load, pixel_class, rel_l2  # noqa: E402


def report(name):
    g = load(name)
    k, iters = int(g["config"]), int(g["iters"])
    pb = synth.make_config(k)
    same = synth.input_hash(pb) == str(g["input_hash"])
    out = {"golden": name, "inputs_match": same}
    with D.Deblur.from_problem(pb, tau=float(g["tau"])) as dev:
        dev.iterate(iters)
        xs, us = dev.get_state()
        img = dev.get_image()
        obj_end = dev.objective()
    with D.Deblur.from_problem(pb, tau=float(g["tau"])) as dev:
        tr = dev.iterate_traced(iters)
    idx = g["idx"]
    cls = pixel_class(pb, idx)
    out["x_rel_l2"] = rel_l2(xs[idx], g["x"])
    out["u_rel_l2"] = rel_l2(us[idx], g["u"])
    for c in ("single", "edge", "corner", "border"):
        m = cls == c
        out[f"x_rel_l2_{c}"] = rel_l2(xs[idx[m]], g["x"][m])
        out[f"n_{c}"] = int(m.sum())
    out["img_rel_l2"] = rel_l2(img[g["img_i"], g["img_j"]], g["img"])
    ref = g["trace"]
    dev_tr = np.vstack([tr[:, :3], np.array(obj_end[:3])[None]])
    out["objective_max_rel"] = float(np.nanmax(np.abs(dev_tr - ref[:, :3]) / np.abs(ref[:, :3])))
    out["objective_first_last"] = [float(ref[0, 0]), float(ref[-1, 0])]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:]:
        report(n)
