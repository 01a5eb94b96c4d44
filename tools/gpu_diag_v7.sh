#!/bin/bash
# v7 role isolation: in-tree build vs diag1 (consumers skip their work) vs diag2 (producers skip theirs)
mkdir -p gpurun_out; O=gpurun_out/diag_v7.log; : > $O
CASES="cfg5 16 cfg5 4 cfg5 24 cfg2 8"
for rep in 1 2; do
  echo "-- base" >> $O; timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
  [ -f tools/_ab/libsf_diag1.so ] && echo "-- diag1 (producers alone)" >> $O && SF_LIB_OVERRIDE=tools/_ab/libsf_diag1.so timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
  [ -f tools/_ab/libsf_diag2.so ] && echo "-- diag2 (consumers alone)" >> $O && SF_LIB_OVERRIDE=tools/_ab/libsf_diag2.so timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
done
cat $O
