#!/bin/bash
# v6 bring-up: variant parity, A/B timing against v5, speck-image precision
mkdir -p gpurun_out; O=gpurun_out/v6.log; : > $O
timeout 900 python -m pytest tests/test_gpu_variants.py -x -q -k "v6" >> $O 2>&1
echo "pytest exit $?" >> $O
for v in v5 v6 v6d v5m v6m; do
  echo "-- $v" >> $O
  SF_VARIANT=$v timeout 300 python tools/time_cfg.py cfg5 16 cfg5 4 cfg5 8 cfg5 32 cfg4 16 >> $O 2>&1
done
for v in v5 v6; do
  echo "-- drift $v" >> $O
  SF_VARIANT=$v timeout 600 python tools/drift_stress.py >> $O 2>&1
done
