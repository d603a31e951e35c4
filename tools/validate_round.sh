#!/bin/bash
# Round validation on the GPU box: c4 bench (with the CPU leg), the ncu launch list of the
# same command, the ncu --set full capture of one iteration (tools/ncu_full.sh), and the c5 /
# per-node c4 / c6 bench lines.  usage: bash tools/validate_round.sh   (outputs in gpurun_out/)
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/${TAG:-r1o}_c4.json 2> gpurun_out/${TAG:-r1o}_c4.err; tail -c 600 gpurun_out/${TAG:-r1o}_c4.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG:-r1o}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${TAG:-r1o}_ncu_list.log 2>&1; echo "list rc=$?"
bash tools/ncu_full.sh ${TAG:-r1o}
timeout 600 python bench.py --config 5 --steps 3 --no-cpu > gpurun_out/${TAG:-r1o}_c5.json 2> gpurun_out/${TAG:-r1o}_c5.err; tail -c 300 gpurun_out/${TAG:-r1o}_c5.json
timeout 600 python bench.py --operator-mode 1 --no-cpu > gpurun_out/${TAG:-r1o}_c4_pernode.json 2> gpurun_out/${TAG:-r1o}_c4_pernode.err; tail -c 300 gpurun_out/${TAG:-r1o}_c4_pernode.json
timeout 900 python bench.py --config 6 --steps 3 --no-cpu > gpurun_out/${TAG:-r1o}_c6.json 2> gpurun_out/${TAG:-r1o}_c6.err; tail -c 300 gpurun_out/${TAG:-r1o}_c6.json
