#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/prof_cfg.py cfg5 64 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bilateral_box --launch-skip 1 --launch-count 1 -o gpurun_out/prof_v5_r64 -f python tools/prof_cfg.py cfg5 64 > gpurun_out/prof_r64.log 2>&1
