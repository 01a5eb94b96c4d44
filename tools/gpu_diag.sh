# hang/parity matrix: every variant x radius on a small image, 40 s each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda(); print('cuda ok')" > gpurun_out/diag.log 2>&1
for r in 0 1 3 17 32 33 64 4 5 8 10 16; do
  SF_VARIANT=v4 timeout 40 python tools/hangcheck.py 300 400 $r 30 30.0 >> gpurun_out/diag.log 2>&1
  echo "v4 r=$r exit $?" >> gpurun_out/diag.log
done
for v in v2 v3; do
  for r in 4 16; do
    SF_VARIANT=$v timeout 40 python tools/hangcheck.py 300 400 $r 30 30.0 >> gpurun_out/diag.log 2>&1
    echo "$v r=$r exit $?" >> gpurun_out/diag.log
  done
done
timeout 60 ./tools/ubench2 > gpurun_out/ubench2.log 2>&1
