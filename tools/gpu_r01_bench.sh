set -x
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
python bench.py --cells-out gpurun_out/cells_r01.json > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo bench rc=$?
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"slide1d_tma|pool2d_kernel" -s 18 -c 18 -o gpurun_out/prof_r01 $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
ls -la gpurun_out
