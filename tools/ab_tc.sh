#!/bin/bash
# A/B timing of two library builds on the tensor-core conv (k = 63, config-3 shape), interleaved on
# one box: place the builds as paper_2305_16513_b200/libss_old.so and libss_new.so first.
cd ${GRAFT_REPO_ROOT:-.}
D=paper_2305_16513_b200
for r in 1 2 3; do
  for v in old new; do cp $D/libss_$v.so $D/libss.so; echo -n "$v: "; KS=${KS:-63} REPS=12 python tests/tc_conv_check.py time 2>&1 | tail -1; done
done
cp $D/libss_new.so $D/libss.so
