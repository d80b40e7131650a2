#!/bin/bash
# A/B per-cell timing of two library builds over bench workloads, interleaved on one box: place the
# builds as paper_2305_16513_b200/libss_old.so and libss_new.so first.  Usage: bash tools/ab_cells.sh wl...
cd ${GRAFT_REPO_ROOT:-.}
D=paper_2305_16513_b200
mkdir -p gpurun_out
for w in ${@:-suite}; do
  for v in old new old new; do
    cp $D/libss_$v.so $D/libss.so
    timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu-baseline \
      --cells-out gpurun_out/ab_${w}_$v.json > /dev/null 2>&1
    python - "$w" "$v" <<'PY'
import json, sys
w, v = sys.argv[1], sys.argv[2]
d = json.load(open(f"gpurun_out/ab_{w}_{v}.json"))
print(v, " ".join(f"{c['cell']}={c['avg_ms'] * 1e3:.1f}" for c in d["cells"]))
PY
  done
done
cp $D/libss_new.so $D/libss.so
