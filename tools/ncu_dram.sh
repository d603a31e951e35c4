#!/bin/bash
# DRAM bytes and duration of the column-pass launches of one eager c4 iteration, per
# library variant (default build and each named variant).  usage: tools/ncu_dram.sh [variant ...]
for v in "" "$@"; do
  echo "== ${v:-base}"
  DEBLUR_NO_GRAPHS=1 DEBLUR_LIB_VARIANT=${v:+libdeblur_$v.so} timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k_cols_tm --launch-skip 2 -c 2 --csv python tools/prof_step.py 4 2 2>/dev/null \
    | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>14 and 'k_cols_tm' in r[4]]
for r in rows: print('  ', r[8], r[-3], r[-2], r[-1])
"
done
