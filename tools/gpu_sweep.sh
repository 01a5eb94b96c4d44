#!/bin/bash
# radius sweep of v5 (rotation) vs v5m (MUFU outgoing rows) on cfg5, plus the every-radius parity test
mkdir -p gpurun_out; O=gpurun_out/sweep.log; : > $O
timeout 900 python -m pytest tests/test_gpu_variants.py -k "every_radius" -x -q >> $O 2>&1
echo "pytest exit $?" >> $O
RS="${RS:-1 2 3 4 5 6 7 8 9 10 11 12 14 16 18 20 24 28 32}"
SF_VARIANT=v5 timeout 600 python tools/variants.py 8192 8192 $RS >> $O 2>&1
SF_VARIANT=v5m timeout 600 python tools/variants.py 8192 8192 $RS >> $O 2>&1
timeout 600 python tools/variants.py 8192 8192 33 40 48 56 64 >> $O 2>&1
