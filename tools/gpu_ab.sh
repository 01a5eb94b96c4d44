#!/bin/bash
# same-box A/B: tools/_ab/libsf_base.so (tools/ab_build.sh) against the in-tree build
mkdir -p gpurun_out; O=gpurun_out/ab.log; : > $O
B=tools/_ab/libsf_base.so
CASES=${CASES:-"cfg5 16 cfg5 4 cfg5 64 cfg4 16 cfg2 8"}
for rep in 1 2; do
  echo "-- base" >> $O; SF_LIB_OVERRIDE=$B timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
  echo "-- new" >> $O; timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
done
