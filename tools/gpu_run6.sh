# v4r / v4b GPU session: hang check, variant timings, parity, bench, ncu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 16 4 5 8 10 64; do
  SF_VARIANT=v4 timeout 40 python tools/hangcheck.py 300 400 $r 30 30.0 >> gpurun_out/diag.log 2>&1
  rc=$?; echo "v4 r=$r exit $rc" >> gpurun_out/diag.log
  if [ $rc -ne 0 ]; then echo "ABORT: hang/failure at r=$r" >> gpurun_out/diag.log; exit 3; fi
done
for v in v4 v2; do
  SF_VARIANT=$v timeout 300 python tools/variants.py 8192 8192 4 16 64 >> gpurun_out/variants.log 2>&1
  echo "variants $v exit $?" >> gpurun_out/variants.log
done
SF_VARIANT=v1 timeout 300 python tools/variants.py 4096 4096 16 64 >> gpurun_out/variants.log 2>&1
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch exit $?" >> gpurun_out/ncu_launch.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v4r -s 1 -c 1 -o gpurun_out/prof_v4r16 python tools/profile_case.py 2048 2048 16 0 15 118 2 > gpurun_out/ncu_v4r.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_v4r.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v4b -s 1 -c 1 -o gpurun_out/prof_v4b64 python tools/profile_case.py 2048 2048 64 0 15 118 2 > gpurun_out/ncu_v4b.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_v4b.log
timeout 1000 python -m pytest tests -m gpu -q --timeout 600 -rf -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
