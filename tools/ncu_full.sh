#!/bin/bash
# ncu --set full of one steady-state iteration's FFT-path kernels (c4), eager launches.
# usage: tools/ncu_full.sh TAG [regex] [skip] [count]
TAG=${1:-full}; RE=${2:-"k_cols|k_rows|k_update"}; SKIP=${3:-17}; CNT=${4:-13}
mkdir -p gpurun_out
DEBLUR_NO_GRAPHS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$RE" \
  --launch-skip $SKIP -c $CNT -o gpurun_out/${TAG} -f python tools/prof_step.py 4 3 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${TAG}_ncu.log
