#!/bin/bash
mkdir -p gpurun_out
SF_V7_PS=1 timeout 300 python tools/cfg1_probe.py || exit 1
SF_V7_PS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:bilateral_box_v7 --launch-skip 2 --launch-count 2 -o gpurun_out/cfg1_full -f python tools/cfg1_probe.py > gpurun_out/cfg1b.log 2>&1
