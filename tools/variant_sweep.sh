#!/bin/bash
# Build libss variants with different compile-time knobs and time one workload
# with each (kernel-only bench).  Usage: VARIANTS="A B" WL=cfg3 bash tools/variant_sweep.sh
for v in $VARIANTS; do
  NVCC_EXTRA="$v" python -c "
import os, paper_2305_16513_b200.build as b
b.FLAGS = b.FLAGS + os.environ['NVCC_EXTRA'].split(',')
b.build_libss(force=True)" > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  python bench.py --workload ${WL:-cfg3} --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --cells-out gpurun_out/sweep.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/sweep.json'))
print('$v', ' '.join(f\"{c['cell']}={c['avg_ms']*1e3:.1f}\" for c in d['cells']))"
done
