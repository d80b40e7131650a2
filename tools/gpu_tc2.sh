#!/bin/bash
for lo in 4 8 12 16; do echo "LO=$lo"; SS_CONV_TC_LO=$lo SS_CONV_TC_MIN_K=1 KS=63 timeout 120 python tests/tc_conv_check.py time 2>&1 | tail -1; done
SS_CONV_TC_LO=12 SS_CONV_TC_MIN_K=1 SS_CONV_TC_TRACE=1 timeout 120 python tests/tc_conv_check.py trace 2>&1 | sed -n 1,16p
SS_CONV_TC_LO=12 SS_CONV_TC_MIN_K=1 SS_CONV_TC_TRACE=1 timeout 120 python tests/tc_conv_check.py trace 2>&1 | tail -1
