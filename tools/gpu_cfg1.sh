#!/bin/bash
mkdir -p gpurun_out
for ps in 1 2 4; do
  SF_V7_PS=$ps timeout 300 python tools/cfg1_probe.py || exit 1
  SF_V7_PS=$ps timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/cfg1_ps$ps.csv python tools/cfg1_probe.py > /dev/null 2>&1
done
