#!/bin/bash
# same-box A/B: tools/_ab/libsf_$AB.so against the in-tree build (timings + bitwise outputs)
mkdir -p gpurun_out; AB=${AB:-base}; O=gpurun_out/ab_$AB.log; : > $O
B=tools/_ab/libsf_$AB.so
CASES=${CASES:-"cfg5 16 cfg5 4 cfg5 24 cfg4 16 cfg2 8"}
[ -n "$BITWISE" ] && timeout 600 python tools/ab_bitwise.py $B >> $O 2>&1
for rep in 1 2; do
  echo "-- $AB" >> $O; SF_LIB_OVERRIDE=$B timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
  echo "-- in-tree" >> $O; timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
done
cat $O
