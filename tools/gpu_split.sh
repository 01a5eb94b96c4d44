cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -f gpurun_out/split.log
for r in 16 4; do
  SF_VARIANT=v5s timeout 60 python tools/hangcheck.py 300 400 $r 30 30.0 >> gpurun_out/split.log 2>&1
  rc=$?; echo "v5s r=$r exit $rc" >> gpurun_out/split.log
  if [ $rc -ne 0 ]; then exit 3; fi
done
SF_VARIANT=v5s timeout 120 python tools/variants.py 8192 8192 4 10 16 >> gpurun_out/split.log 2>&1
SF_VARIANT=v5 timeout 120 python tools/variants.py 8192 8192 16 >> gpurun_out/split.log 2>&1
