#!/bin/bash
# the whole GPU test suite + bench line + launch list (round-end evidence)
mkdir -p gpurun_out; O=gpurun_out/full.log; : > $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_full.log 2>&1
echo "pytest exit $?" >> $O
tail -3 gpurun_out/pytest_gpu_full.log >> $O
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full_err.log
echo "bench exit $?" >> $O
