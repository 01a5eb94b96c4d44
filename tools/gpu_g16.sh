#!/bin/bash
# same-box A/B of the G = 16 wide kernel (in-tree) against tools/_ab/libsf_g14.so, v7w parity,
# and the v7 / v7w crossover at r = 17..24
mkdir -p gpurun_out; O=gpurun_out/ab_g16.log; : > $O
B=tools/_ab/libsf_g14.so
CASES="cfg5 64 cfg5 48 cfg5 32 cfg5 25 cfg4 64"
for rep in 1 2; do
  echo "-- g14" >> $O; SF_LIB_OVERRIDE=$B timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
  echo "-- in-tree" >> $O; timeout 300 python tools/time_cfg.py $CASES >> $O 2>&1
done
echo "-- crossover: default (v7)" >> $O; timeout 300 python tools/time_cfg.py cfg5 18 cfg5 20 cfg5 22 cfg5 24 >> $O 2>&1
echo "-- crossover: v7w" >> $O; SF_VARIANT=v7w timeout 300 python tools/time_cfg.py cfg5 16 cfg5 18 cfg5 20 cfg5 22 cfg5 24 >> $O 2>&1
echo "-- v7w_check" >> $O; timeout 600 python tools/v7w_check.py >> $O 2>&1
cut -c1-160 $O
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q --timeout 600 -x -k "every_radius" 2>&1 | tail -4
