#!/bin/bash
# tensor-core conv: parity (forced onto the TC path) then timing per NC
mkdir -p gpurun_out
SS_CONV_TC_MIN_K=1 timeout 300 python tests/tc_conv_check.py parity > gpurun_out/tc_parity.log 2>&1; echo "parity rc=$?"; tail -4 gpurun_out/tc_parity.log
for nc in 64 32; do echo "NC=$nc"; SS_CONV_TC_NC=$nc SS_CONV_TC_MIN_K=1 timeout 120 python tests/tc_conv_check.py time 2>&1 | tail -3; done
echo "FFMA2 (TC off)"; SS_CONV_TC_MIN_K=0 timeout 120 python tests/tc_conv_check.py time 2>&1 | tail -3
