#!/bin/bash
# default dispatch = v7m: tests, configs timing, one ncu capture
mkdir -p gpurun_out; O=gpurun_out/r2a.log; : > $O
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_precision.py -x -q >> $O 2>&1
echo "pytest exit $?" >> $O
echo "-- default" >> $O
timeout 300 python tools/time_cfg.py cfg1 5 cfg2 8 cfg3 10 cfg4 16 cfg5 4 cfg5 16 cfg5 64 cfg5 24 cfg5 32 >> $O 2>&1
echo "-- v4r" >> $O
SF_VARIANT=v4 timeout 300 python tools/time_cfg.py cfg2 8 cfg5 4 >> $O 2>&1
echo "-- v5m" >> $O
SF_VARIANT=v5m timeout 300 python tools/time_cfg.py cfg1 5 cfg2 8 >> $O 2>&1
timeout 300 python tools/profile_case.py 8192 8192 16 0 15 118 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v7 -s 1 -c 1 \
  -o gpurun_out/prof_v7m_r16 python tools/profile_case.py 8192 8192 16 0 15 118 2 > gpurun_out/ncu_v7.log 2>&1
echo "ncu exit $?" >> $O
