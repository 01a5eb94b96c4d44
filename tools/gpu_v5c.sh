#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/v5c4.log; : > $O
SF_VARIANT=v5c timeout 120 python tools/v5c_quick.py >> $O 2>&1
echo "quick exit $?" >> $O
SF_VARIANT=v5c timeout 300 python tools/variants.py 8192 8192 33 48 64 >> $O 2>&1
timeout 300 python tools/variants.py 8192 8192 33 48 64 >> $O 2>&1
