#!/bin/bash
# v6 walker width A/B at R = 16 + one ncu --set full capture of v6 (cfg5 r=16)
mkdir -p gpurun_out; O=gpurun_out/v6b.log; : > $O
for g in 16 20 24; do
  for v in v6 v6m; do
    echo "-- $v G=$g" >> $O
    SF_V6_G=$g SF_VARIANT=$v timeout 300 python tools/time_cfg.py cfg5 16 cfg4 16 >> $O 2>&1
  done
done
echo "-- v5 ref" >> $O
SF_VARIANT=v5 timeout 300 python tools/time_cfg.py cfg5 16 >> $O 2>&1
SF_VARIANT=v6 timeout 300 python tools/profile_case.py 8192 8192 16 0 15 118 2 > gpurun_out/prof_plain.log 2>&1 && \
SF_VARIANT=v6 ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v6 -s 1 -c 1 \
  -o gpurun_out/prof_v6_r16 python tools/profile_case.py 8192 8192 16 0 15 118 2 > gpurun_out/ncu_v6.log 2>&1
echo "ncu exit $?" >> $O
