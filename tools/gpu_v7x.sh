#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/v7x2.log; : > $O
for x in 1 2 3 4; do
  for v in v7 v7m; do
    echo "-- $v X=$x" >> $O
    SF_V7_X=$x SF_VARIANT=$v timeout 300 python tools/time_cfg.py cfg5 16 cfg5 4 >> $O 2>&1
  done
done
