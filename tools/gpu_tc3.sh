#!/bin/bash
SS_CONV_TC_MIN_K=1 timeout 300 python tests/tc_conv_check.py parity > gpurun_out/tc_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/tc_parity.log
for lo in 2 3 4; do echo "LO=$lo"; SS_CONV_TC_LO=$lo SS_CONV_TC_MIN_K=1 timeout 120 python tests/tc_conv_check.py time 2>&1 | tail -3; done
SS_CONV_TC_MIN_K=1 SS_CONV_TC_TRACE=1 timeout 120 python tests/tc_conv_check.py trace 2>&1 | sed -n 1,14p
