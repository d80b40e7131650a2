#!/bin/bash
# ncu capture of one step's 1-D tile kernels (after a plain run of the same command)
TAG=${1:-prof}
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${NCU:-slide1d_tma_kernel}" -s ${SKIP:-14} -c ${COUNT:-14} -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
