#!/bin/bash
# Round validation on the GPU box: c4 bench (with the CPU leg), the ncu launch list of the
# same command, the ncu --set full capture of one iteration (tools/ncu_full.sh) and its
# per-launch DRAM traffic, then the c5 / per-node c4 / c6 bench lines.
# usage: TAG=r2a bash tools/validate_round.sh   (outputs in gpurun_out/)
set -x
TAG=${TAG:-r2}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; tail -c 600 gpurun_out/${TAG}_c4.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu_list.log 2>&1; echo "list rc=$?"
bash tools/ncu_full.sh ${TAG}
python tools/traffic_from_ncu.py gpurun_out/${TAG}.ncu-rep gpurun_out/${TAG}_traffic.json > /dev/null 2>&1; echo "traffic rc=$?"
[ -n "$QUICK" ] && exit 0
for k in 1 2 3; do
  timeout 600 python bench.py --config $k --steps 40 --no-cpu > gpurun_out/${TAG}_c$k.json 2> gpurun_out/${TAG}_c$k.err; tail -c 200 gpurun_out/${TAG}_c$k.json
done
timeout 600 python bench.py --loopback 8 --no-cpu > gpurun_out/${TAG}_c4_loop8.json 2> gpurun_out/${TAG}_c4_loop8.err; tail -c 200 gpurun_out/${TAG}_c4_loop8.json
timeout 600 python bench.py --config 5 --steps 3 --no-cpu > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; tail -c 300 gpurun_out/${TAG}_c5.json
timeout 600 python bench.py --operator-mode 1 --no-cpu > gpurun_out/${TAG}_c4_pernode.json 2> gpurun_out/${TAG}_c4_pernode.err; tail -c 300 gpurun_out/${TAG}_c4_pernode.json
timeout 900 python bench.py --config 6 --steps 3 --no-cpu > gpurun_out/${TAG}_c6.json 2> gpurun_out/${TAG}_c6.err; tail -c 300 gpurun_out/${TAG}_c6.json
