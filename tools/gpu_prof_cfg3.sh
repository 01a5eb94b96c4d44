#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/prof_cfg.py cfg3 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:v7q --launch-skip 1 --launch-count 1 -o gpurun_out/prof_v7q_cfg3 -f python tools/prof_cfg.py cfg3 > gpurun_out/prof_v7q.log 2>&1
