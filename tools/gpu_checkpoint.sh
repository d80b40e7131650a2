#!/bin/bash
# Round checkpoint: full bench line (e2e + cpu baseline + clocks), the ncu launch
# list of the same command, and one ncu --set full capture of one step's 1-D
# tile kernels + pool2d kernels.  Usage: bash tools/gpu_checkpoint.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.csv
python bench.py --cells-out gpurun_out/cells_full_$TAG.json > gpurun_out/bench_full_$TAG.json 2> gpurun_out/bench_full_$TAG.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu-launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"slide1d_tma_kernel|pool2d_vec|conv_tc" -s 18 -c 18 -o gpurun_out/prof_full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu-full rc=$?"
