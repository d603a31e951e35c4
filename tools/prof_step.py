"""Minimal driver for ncu captures: create config k (default c4) and run n
iterations (eager launches when DEBLUR_NO_GRAPHS=1).  Not a benchmark."""
import sys
sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1705_06603_b200 import deblur as D  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pb = synth.make_config(k)
with D.Deblur.from_problem(pb) as dev:
    dev.iterate(n)
    dev.synchronize() if hasattr(dev, "synchronize") else None
print("done")
