# full GPU validation + bench + ncu evidence of the current build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
timeout 300 python tools/configs_bench.py > gpurun_out/configs.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch exit $?" >> gpurun_out/ncu_launch.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v5 -s 3 -c 1 -o gpurun_out/prof_bench_r16 python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_bench.log 2>&1
echo "ncu bench exit $?" >> gpurun_out/ncu_bench.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bilateral_q2 -s 1 -c 1 -o gpurun_out/prof_q2_cfg3 python tools/profile_case.py 2048 2048 10 1 40 17 2 > gpurun_out/ncu_q2.log 2>&1
echo "ncu q2 exit $?" >> gpurun_out/ncu_q2.log
