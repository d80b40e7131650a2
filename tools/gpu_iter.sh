#!/bin/bash
# One GPU iteration: parity tests, a kernel-only bench, and an ncu capture of the
# 1-D tile kernels.  Usage (under gpurun): bash tools/gpu_iter.sh TAG [pytest-args]
TAG=${1:-iter}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
python bench.py --no-e2e --no-cpu-baseline --cells-out gpurun_out/cells_$TAG.json > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - << PY
import json
d=json.load(open("gpurun_out/cells_$TAG.json"))
print("value", d["line"]["value"], "GElem/s  hbm", d["line"]["hbm_gbs"], "GB/s ms/step", d["line"]["ms_per_step"])
for c in d["cells"]: print(f"{c['cell']:18s} {c['avg_ms']*1e3:8.1f} us {c['gbs']:7.0f} GB/s frac {c['frac_hbm']:.3f} fma {c.get('fma_frac','')}")
PY
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
if [ -n "$NCU" ]; then
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s 18 -c 18 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
fi
