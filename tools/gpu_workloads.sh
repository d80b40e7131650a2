#!/bin/bash
# Per-cell timing of the widening workloads (no e2e / CPU legs).  Usage: bash tools/gpu_workloads.sh TAG [workloads...]
TAG=${1:-wl}; shift
WLS=${@:-backward conv2d affine mc winspec stride cfg1}
mkdir -p gpurun_out
for w in $WLS; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu-baseline \
    --cells-out gpurun_out/cells_${TAG}_$w.json > gpurun_out/bench_${TAG}_$w.json 2> gpurun_out/bench_${TAG}_$w.err
  echo "== $w rc=$?"; python tools/cells_print.py gpurun_out/cells_${TAG}_$w.json 2>&1 | grep -v "^roofline\|^verify"
done
