#!/bin/bash
# Round-2 GPU iteration: the multi-rank bench test, the default bench line, and
# (NCU=1) the ncu launch list of the same command.  Usage: bash tools/gpu_r2.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_sched_gpu.py -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 900 python bench.py --cells-out gpurun_out/cells_$TAG.json > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_$TAG.err
python tools/cells_print.py gpurun_out/cells_$TAG.json
