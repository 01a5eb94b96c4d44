cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "truncated" --timeout 600 -rf > gpurun_out/pytest_trunc.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_trunc.log
timeout 600 python tools/configs_bench.py > gpurun_out/configs.log 2>&1
echo "exit $?" >> gpurun_out/configs.log
