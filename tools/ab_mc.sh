#!/bin/bash
# A/B timing of two library builds on the multi-channel conv shapes (tools/mc_prof.py), interleaved on one
# box: place the builds as paper_2305_16513_b200/libss_old.so and libss_new.so first.
cd ${GRAFT_REPO_ROOT:-.}
D=paper_2305_16513_b200
for r in 1 2; do
  for v in old new; do
    cp $D/libss_$v.so $D/libss.so
    for m in ${MODES:-1d9 2d dx2d}; do echo -n "$v "; python tools/mc_prof.py $m 3 2>&1 | tail -1; done
  done
done
cp $D/libss_new.so $D/libss.so
