#!/bin/bash
# same-box A/B of several prebuilt libraries: LIBS="tools/_ab/libsf_x.so ..." CASES="cfg5 16 ..."
mkdir -p gpurun_out; O=gpurun_out/abn.log; : > $O
for rep in 1 2; do
  echo "-- in-tree" >> $O; timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
  for L in $LIBS; do echo "-- $L" >> $O; SF_LIB_OVERRIDE=$L timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1; done
done
