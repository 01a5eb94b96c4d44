#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/ab.log; : > $O
B=tools/_ab/libsf_base.so
for rep in 1 2; do
  SF_LIB_OVERRIDE=$B timeout 300 python tools/time_cfg.py cfg5 16 cfg5 64 cfg4 16 >> $O 2>&1
  echo "-- new maxseg32" >> $O
  SF_V5_MAXSEG=32 timeout 300 python tools/time_cfg.py cfg5 16 cfg5 64 cfg4 16 >> $O 2>&1
  echo "-- new maxseg1000" >> $O
  SF_V5_MAXSEG=1000 timeout 300 python tools/time_cfg.py cfg5 16 cfg5 64 >> $O 2>&1
  echo "-- new v5m maxseg1000" >> $O
  SF_VARIANT=v5m SF_V5_MAXSEG=1000 timeout 300 python tools/time_cfg.py cfg5 16 cfg4 16 >> $O 2>&1
  echo "-- base v5m" >> $O
  SF_LIB_OVERRIDE=$B SF_VARIANT=v5m timeout 300 python tools/time_cfg.py cfg5 16 cfg4 16 >> $O 2>&1
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv >> $O
