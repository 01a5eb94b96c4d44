cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 200 -k "cfg3 or edge or constant or qM or spatial" -rf > gpurun_out/pytest_q2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_q2.log
timeout 300 python tools/configs_bench.py > gpurun_out/configs.log 2>&1
SF_VARIANT=v1 timeout 300 python tools/configs_bench.py > gpurun_out/configs_v1.log 2>&1
