#!/bin/bash
# one build -> measure iteration on the GPU box: FFT parity tests + c4 bench (no CPU leg)
# usage: tools/gpu_iter.sh TAG [extra pytest -k expr]
TAG=${1:-iter}
K=${2:-fft}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "$K" 2>&1 | tail -4
timeout 300 python bench.py --no-cpu > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python - "$TAG" <<'PY'
import json,sys
t=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/{t}_bench.json").read().strip().splitlines()[-1])
except Exception as e:
    print("bench failed", e); print(open(f"gpurun_out/{t}_bench.err").read()[-2000:]); sys.exit(0)
print("value", d["value"], "ms/step", d["ms_per_step"], "e2e", d["e2e"]["value"], "clocks", d["clocks"])
for k,v in d["kernels"].items(): print(f"  {k:18s} {v['ms_per_launch']:8.4f} ms  share {v['share']:.3f}  {v['achieved']} {v['unit']} frac {v['frac']}")
PY
