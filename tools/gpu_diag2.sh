cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -f gpurun_out/diag2.log
for d in 0 1 2; do
  SF_DIAG=$d timeout 120 python tools/variants.py 8192 8192 16 >> gpurun_out/diag2.log 2>&1
done
