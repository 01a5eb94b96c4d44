#!/bin/bash
# same-box A/B of one library: tools/_ab/libsf_$AB.so vs the in-tree build
mkdir -p gpurun_out; O=gpurun_out/ab_$AB.log; : > $O
CASES=${CASES:-"cfg5 16 cfg5 4 cfg5 24 cfg4 16 cfg2 8"}
for rep in 1 2; do
  echo "-- $AB" >> $O; SF_LIB_OVERRIDE=tools/_ab/libsf_$AB.so timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
  echo "-- in-tree" >> $O; timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
done
cat $O
