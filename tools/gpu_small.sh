O=gpurun_out/small.log; : > $O
for v in default v1 v4b v5m; do echo "-- $v" >> $O
 if [ $v = default ]; then timeout 300 python tools/small_scan.py >> $O 2>&1; else SF_VARIANT=$v timeout 300 python tools/small_scan.py >> $O 2>&1; fi; done
SF_V7_PS=1 timeout 300 python tools/small_scan.py >> $O 2>&1
