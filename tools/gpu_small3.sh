#!/bin/bash
mkdir -p gpurun_out
SF_VARIANT=vs ncu --set full --import-source on --clock-control none -k regex:bilateral_box_small -c 1 -o gpurun_out/prof_vs_cfg1 -f python tools/profile_case.py 256 256 5 0 30 30 2 > gpurun_out/prof_vs.log 2>&1
ncu -i gpurun_out/prof_vs_cfg1.ncu-rep --page details --csv > gpurun_out/prof_vs_details.csv 2>&1
ncu -i gpurun_out/prof_vs_cfg1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_vs_source.csv 2>&1
tail -3 gpurun_out/prof_vs.log
