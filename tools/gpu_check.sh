#!/bin/bash
# full GPU test suite + default-dispatch radius sweep + one bench line
mkdir -p gpurun_out; O=gpurun_out/check.log; : > $O
timeout 1500 python -m pytest tests -m gpu -x -q >> $O 2>&1
echo "pytest exit $?" >> $O
timeout 600 python tools/variants.py 8192 8192 ${RS:-1 3 4 5 6 8 10 12 16 20 24 32 33 40 48 56 64} > gpurun_out/radius_sweep.jsonl 2>&1
timeout 600 python bench.py >> $O 2>&1
echo "bench exit $?" >> $O
