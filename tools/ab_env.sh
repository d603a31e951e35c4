#!/bin/bash
# A/B over environment settings on the c4 bench (no CPU leg):
#   tools/ab_env.sh TAG "" "DEBLUR_FFT_SIZE=256" ...   (each argument one env assignment list)
TAG=$1; shift
i=0
for e in "$@"; do
  env $e timeout 300 python bench.py --no-cpu --steps 10 ${BENCH_ARGS} > gpurun_out/${TAG}_$i.json 2>gpurun_out/${TAG}_$i.err
  python - "${TAG}_$i" "$e" <<'PY'
import json,sys
t=sys.argv[1]
try: d=json.loads(open(f"gpurun_out/{t}.json").read().strip().splitlines()[-1])
except Exception as e: print(t,"FAILED",open(f"gpurun_out/{t}.err").read()[-800:]); sys.exit(0)
print(f"== [{sys.argv[2]}] {d['value']:.1f} Mpix-it/s  {d['ms_per_step']:.3f} ms/step")
for k,v in d["kernels"].items(): print(f"   {k:18s} {v['ms_per_launch']:8.4f} ms")
PY
  i=$((i+1))
done
