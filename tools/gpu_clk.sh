#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/clk.log; : > $O
timeout 300 python tools/time_cfg.py cfg5 16 cfg5 16 >> $O 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__cycles_elapsed.avg.per_second,sm__cycles_active.avg --clock-control none --csv -k regex:bilateral --log-file gpurun_out/clk_ncu.csv python tools/time_cfg.py cfg5 16 >> $O 2>&1
echo "exit $?" >> $O
