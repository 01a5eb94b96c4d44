cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -rf -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
timeout 900 python tools/parity_report.py > gpurun_out/parity.log 2>&1
python tools/profile_case.py 2048 2048 16 0 15 118 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v3 -s 1 -c 1 -o gpurun_out/prof_v3 python tools/profile_case.py 2048 2048 16 0 15 118 2 > gpurun_out/ncu_v3.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_v3.log
