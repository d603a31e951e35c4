set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./tools/ffma_peak > gpurun_out/ffma_peak.json; cat gpurun_out/ffma_peak.json
./tools/ffma_peak > gpurun_out/ffma_peak2.json; cat gpurun_out/ffma_peak2.json
python -c "
import synth
for k in (1,2,3,4):
    print(k, synth.input_hash(synth.make_config(k)), flush=True)
" > gpurun_out/hash.txt 2>&1; cat gpurun_out/hash.txt
lscpu | grep -i 'model name'; nproc
