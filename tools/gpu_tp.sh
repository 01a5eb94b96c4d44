cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -f gpurun_out/tp.log
for r in 16 4 10; do
  for N in 30 31; do
    SF_VARIANT=v5t timeout 60 python tools/hangcheck.py 300 400 $r $N 30.0 >> gpurun_out/tp.log 2>&1
    rc=$?; echo "v5t r=$r N=$N exit $rc" >> gpurun_out/tp.log
    if [ $rc -ne 0 ]; then exit 3; fi
  done
done
SF_VARIANT=v5t timeout 120 python tools/variants.py 8192 8192 4 5 8 10 16 >> gpurun_out/tp.log 2>&1
timeout 120 python tools/variants.py 8192 8192 16 >> gpurun_out/tp.log 2>&1
