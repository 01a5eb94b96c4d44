#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/bench_r2.log; : > $O
timeout 600 python bench.py > gpurun_out/bench_line.json 2> gpurun_out/bench_err.log
echo "bench exit $?" >> $O
timeout 600 python bench.py --workload cfg4 --no-cpu --no-configs > gpurun_out/bench_cfg4.json 2>> gpurun_out/bench_err.log
echo "bench cfg4 exit $?" >> $O
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench_err.log
echo "ref exit $?" >> $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "ncu exit $?" >> $O
