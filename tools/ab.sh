#!/bin/bash
# A/B: run the c4 bench (no CPU leg) for the default build and each named variant
# (paper_1705_06603_b200/libdeblur_<v>.so built with _build.py --variant v -D...).
for v in "" "$@"; do
  DEBLUR_LIB_VARIANT=${v:+libdeblur_$v.so} timeout 300 python bench.py --no-cpu --steps 10 > gpurun_out/ab_${v:-base}.json 2>gpurun_out/ab_${v:-base}.err
  python - "${v:-base}" <<'PY'
import json,sys
t=sys.argv[1]
try: d=json.loads(open(f"gpurun_out/ab_{t}.json").read().strip().splitlines()[-1])
except Exception as e: print(t,"FAILED",open(f"gpurun_out/ab_{t}.err").read()[-800:]); sys.exit(0)
print(f"== {t}: {d['value']:.1f} Mpix-it/s  {d['ms_per_step']:.3f} ms/step")
for k,v in d["kernels"].items(): print(f"   {k:18s} {v['ms_per_launch']:8.4f} ms")
PY
done
