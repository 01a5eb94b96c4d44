#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/v5c3.log; : > $O
timeout 120 python tools/v5c_quick.py >> $O 2>&1
timeout 300 python tools/variants.py 8192 8192 33 48 64 >> $O 2>&1
SF_DIAG=3 timeout 300 python tools/variants.py 8192 8192 33 48 64 >> $O 2>&1
SF_VARIANT=v5nc timeout 300 python tools/variants.py 8192 8192 33 48 64 >> $O 2>&1
echo "exit $?" >> $O
