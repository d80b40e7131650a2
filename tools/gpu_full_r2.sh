#!/bin/bash
# Round-2 checkpoint: full GPU test suite, default bench line, reference arm, widening workloads.
TAG=${1:-r2c}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/smi_$TAG.csv 2>&1 &
SMI=$!
timeout 900 python bench.py --cells-out gpurun_out/cells_full_$TAG.json > gpurun_out/bench_full_$TAG.json 2> gpurun_out/bench_full_$TAG.err; echo "bench rc=$?"
kill $SMI 2>/dev/null
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
python tools/cells_print.py gpurun_out/cells_full_$TAG.json
bash tools/gpu_workloads.sh $TAG backward conv2d affine mc winspec stride cfg1 | grep -E "==|value"
