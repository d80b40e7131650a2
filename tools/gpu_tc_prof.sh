#!/bin/bash
mkdir -p gpurun_out
export SS_CONV_TC_MIN_K=1 KS=63 REPS=1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_tc -c 1 -o gpurun_out/prof_tc1 python tests/tc_conv_check.py time > gpurun_out/ncu_tc1.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_tc1.log
