#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/poly.log; : > $O
timeout 900 python -m pytest tests/test_gpu_poly.py -x -q >> $O 2>&1
echo "pytest exit $?" >> $O
timeout 600 python tools/poly_errors.py > gpurun_out/poly_errors.jsonl 2>> $O
echo "table exit $?" >> $O
