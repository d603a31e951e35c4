for v in "" "$@"; do DEBLUR_LIB_VARIANT=${v:+libdeblur_$v.so} timeout 300 python bench.py --no-cpu --steps 10 --operator-mode 1 > gpurun_out/pn_${v:-base}.json 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/pn_${v:-base}.json').read().strip().splitlines()[-1]); print('${v:-base}', d['value'], d['ms_per_step'], d['kernels']['consensus']['ms_per_launch'])"; done
