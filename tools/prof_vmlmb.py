"""ncu driver: c4 with the VMLM-B Local-Solver (10 inner), n outer iterations, eager launches."""
import dataclasses
import sys
sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1705_06603_b200 import deblur as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
pb = dataclasses.replace(synth.make_config(4), local_solver=1, inner_steps=10, inner_increment=0)
with D.Deblur.from_problem(pb) as dev:
    dev.iterate(n)
print("done")
