#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/v7w3.log; : > $O
C="cfg5 64 cfg5 48 cfg5 32 cfg5 25"
for rep in 1 2; do
  echo "-- v7w UNR=8 (in-tree)" >> $O; SF_VARIANT=v7w timeout 300 python tools/time_cfg.py $C >> $O 2>&1
  echo "-- v7w UNR=4" >> $O; SF_LIB_OVERRIDE=tools/_ab/libsf_u4.so SF_VARIANT=v7w timeout 300 python tools/time_cfg.py $C >> $O 2>&1
done
cat $O
