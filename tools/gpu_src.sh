#!/bin/bash
# ncu --set full of the bench kernel (v7, cfg5 r = 16) with source-level
# stall attribution exported as CSV (SASS + CUDA source views)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v7 -s 3 -c 1 \
  -o gpurun_out/prof_v7_r16 -f python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_bench.log 2>&1
echo "ncu bench exit $?" >> gpurun_out/ncu_bench.log
ncu -i gpurun_out/prof_v7_r16.ncu-rep --page source --csv --print-source sass > gpurun_out/src_sass.csv 2> gpurun_out/src.err
ncu -i gpurun_out/prof_v7_r16.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_cuda.csv 2>> gpurun_out/src.err
ls -la gpurun_out
