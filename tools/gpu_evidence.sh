#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/evidence.log; : > $O
timeout 900 python tools/drift_stress.py > gpurun_out/precision_stress.jsonl 2>> $O
echo "drift exit $?" >> $O
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_short.json 2>> $O && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "ncu exit $?" >> $O
