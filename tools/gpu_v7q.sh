#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/v7q.log; : > $O
timeout 600 python tools/v7q_check.py >> $O 2>&1
echo "-- v1 (tile kernel)" >> $O
SF_VARIANT=v1 timeout 600 python tools/v7q_check.py 2>&1 | grep cfg3_size >> $O
