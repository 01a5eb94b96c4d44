#!/bin/bash
# default dispatch against SF_VARIANT=$V on the same box
mkdir -p gpurun_out; O=gpurun_out/var_$V.log; : > $O
CASES=${CASES:-"cfg5 16 cfg5 4 cfg5 24"}
for rep in 1 2; do
  echo "-- $V" >> $O; SF_VARIANT=$V timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
  echo "-- default" >> $O; timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
done
cat $O
