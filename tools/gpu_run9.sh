cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/diag.log gpurun_out/variants.log
timeout 40 python tools/hangcheck.py 300 400 64 30 30.0 >> gpurun_out/diag.log 2>&1
rc=$?; echo "default r=64 exit $rc" >> gpurun_out/diag.log
if [ $rc -ne 0 ]; then echo "ABORT" >> gpurun_out/diag.log; exit 3; fi
timeout 40 python tools/hangcheck.py 129 200 64 118 15.0 >> gpurun_out/diag.log 2>&1
echo "default r=64 small exit $?" >> gpurun_out/diag.log
timeout 300 python tools/variants.py 8192 8192 4 16 64 >> gpurun_out/variants.log 2>&1
echo "variants default exit $?" >> gpurun_out/variants.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -rf -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch exit $?" >> gpurun_out/ncu_launch.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v5 -s 3 -c 1 -o gpurun_out/prof_bench_r16 python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_bench.log 2>&1
echo "ncu bench exit $?" >> gpurun_out/ncu_bench.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v5 -s 1 -c 1 -o gpurun_out/prof_v5_64 python tools/profile_case.py 2368 2048 64 0 15 118 2 > gpurun_out/ncu_v5_64.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_v5_64.log
