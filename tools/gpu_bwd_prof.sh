#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --workload backward --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_bwd.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCUK:-conv_filter_grad_kernel|pool_max_backward_tile|pool2d_backward_fixed}" -s 0 -c ${NCUC:-8} -o gpurun_out/prof_bwd $CMD > gpurun_out/ncu_bwd.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_bwd.log
