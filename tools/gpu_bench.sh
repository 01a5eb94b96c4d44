#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/bench_r2.log; : > $O
timeout 600 python bench.py > gpurun_out/bench_line.json 2> gpurun_out/bench_err.log
echo "bench exit $?" >> $O
timeout 600 python bench.py --workload cfg4 --no-cpu --no-configs > gpurun_out/bench_cfg4.json 2>> gpurun_out/bench_err.log
echo "bench cfg4 exit $?" >> $O
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench_err.log
echo "ref exit $?" >> $O
