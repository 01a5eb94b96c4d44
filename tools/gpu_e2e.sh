cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "host" --timeout 600 -rf > gpurun_out/pytest_host.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_host.log
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
