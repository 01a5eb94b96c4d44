# v5m experiment: variant timings at all ring radii; ncu of v5m.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/diag.log gpurun_out/variants.log
for r in 16 4; do
  SF_VARIANT=v5m timeout 40 python tools/hangcheck.py 300 400 $r 30 30.0 >> gpurun_out/diag.log 2>&1
  rc=$?; echo "v5m r=$r exit $rc" >> gpurun_out/diag.log
  if [ $rc -ne 0 ]; then echo "ABORT" >> gpurun_out/diag.log; exit 3; fi
done
for v in v5m v5 v4; do
  SF_VARIANT=$v timeout 300 python tools/variants.py 8192 8192 4 5 8 10 16 >> gpurun_out/variants.log 2>&1
  echo "variants $v exit $?" >> gpurun_out/variants.log
done
SF_VARIANT=v5m timeout 300 ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v5 -s 1 -c 1 -o gpurun_out/prof_v5m_16 python tools/profile_case.py 2368 2048 16 0 15 118 2 > gpurun_out/ncu_v5m.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_v5m.log
