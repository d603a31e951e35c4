#!/bin/bash
# A/B of the VMLM-B Local-Solver bench (c4, 10 inner iterations) for the default build and variants
for v in "" "$@"; do
  DEBLUR_LIB_VARIANT=${v:+libdeblur_$v.so} timeout 600 python bench.py --no-cpu --local-solver vmlmb --inner 10 --steps 2 > gpurun_out/abvm_${v:-base}.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/abvm_${v:-base}.json').read().strip().splitlines()[-1])
print('${v:-base}', d['value'], d['ms_per_step'], {k: v['ms_per_launch'] for k, v in d['kernels'].items() if 'vmlmb' in k})"
done
