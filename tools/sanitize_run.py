"""Small exercise of every kernel family for compute-sanitizer runs (memcheck /
racecheck / synccheck): direct and FFT paths (with the S/2 strip plan), per-node
operators, the independent baseline, VMLM-B, objective, traced iterations, apply,
image.  Not a test by itself (tools/; run under compute-sanitizer on the GPU)."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import synth  # noqa: E402
from paper_1705_06603_b200 import deblur as D  # noqa: E402

cases = []
pb = synth.make_config(3, n=700, facets=(2, 2), overlap=64)          # P = 63: S = 512 + strips
cases.append(("c3-fft", pb, dict(conv_path=D.CONV_FFT)))
cases.append(("c3-direct", synth.make_config(2, n=200, facets=(2, 2), overlap=20), dict(conv_path=D.CONV_DIRECT)))
pn = synth.per_node(synth.make_config(2, n=300))
cases.append(("node-fft", pn, dict(conv_path=D.CONV_FFT)))
pv = synth.make_config(2, n=200, facets=(2, 2), overlap=20)
pv.local_solver, pv.inner_steps, pv.inner_increment = 1, 4, 2
cases.append(("vmlmb-fft", pv, dict(conv_path=D.CONV_FFT)))
cases.append(("vmlmb-direct", pv, dict(conv_path=D.CONV_DIRECT)))
pi = synth.make_config(2, n=200, facets=(2, 2), overlap=20)
pi.independent = 1
cases.append(("indep", pi, dict(conv_path=D.CONV_FFT)))
for name, p, kw in cases:
    with D.Deblur.from_problem(p, **kw) as dev:
        x = np.random.default_rng(0).random((p.ny, p.nx), dtype=np.float32)
        dev.apply_H(x)
        if p.fy * p.fx == 1 or p.overlap >= p.P - 1:
            dev.apply_HT(np.random.default_rng(1).standard_normal((p.my, p.mx)).astype(np.float32))
        dev.iterate(2)
        dev.iterate_traced(1)
        dev.objective()
        dev.get_image()
    print(name, "ok", flush=True)
