#!/bin/bash
# ncu evidence for round 2: the launch list of one bench command (cold cache,
# serialised: compare shares) and a full capture of the named kernels.
# Usage: NCU_K=regex bash tools/gpu_prof_r2.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-cfg5 --cell-reps 2"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control all \
    -s 54 -c 400 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_list_$TAG.log 2>&1; echo "ncu list rc=$?"
if [ -n "$NCU_K" ]; then
ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -s ${NCU_S:-0} -c ${NCU_C:-3} \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
fi
