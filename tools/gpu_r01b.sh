#!/bin/bash
# Re-entry check: full GPU parity suite, smoke, default bench, affine/winspec workloads.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_b.csv
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_b.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_b.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_b.log
timeout 600 python bench.py --cells-out gpurun_out/cells_b.json > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; echo "bench rc=$?"; cat gpurun_out/bench_b.json | head -c 3000
for wl in affine winspec; do
timeout 300 python bench.py --workload $wl --no-e2e --no-cpu-baseline --cells-out gpurun_out/cells_$wl.json > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; echo "$wl rc=$?"
done
