cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -f gpurun_out/flip.log
for f in 0 1; do
  SF_FLIP=$f timeout 60 python tools/hangcheck.py 300 400 16 30 30.0 >> gpurun_out/flip.log 2>&1
  SF_FLIP=$f timeout 120 python tools/variants.py 8192 8192 4 16 >> gpurun_out/flip.log 2>&1
done
