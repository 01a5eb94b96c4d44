cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/diag.log gpurun_out/variants.log
for r in 16 10 64; do
  timeout 40 python tools/hangcheck.py 300 400 $r 30 30.0 >> gpurun_out/diag.log 2>&1
  rc=$?; echo "default r=$r exit $rc" >> gpurun_out/diag.log
  if [ $rc -ne 0 ]; then echo "ABORT" >> gpurun_out/diag.log; exit 3; fi
done
SF_VARIANT=v5 timeout 300 python tools/variants.py 8192 8192 4 10 16 >> gpurun_out/variants.log 2>&1
SF_VARIANT=v5m timeout 300 python tools/variants.py 8192 8192 4 10 16 >> gpurun_out/variants.log 2>&1
timeout 300 python tools/variants.py 8192 8192 64 >> gpurun_out/variants.log 2>&1
