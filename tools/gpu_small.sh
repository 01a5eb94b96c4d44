cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -f gpurun_out/small.log
timeout 60 python tools/hangcheck.py 256 256 5 30 30.0 >> gpurun_out/small.log 2>&1
timeout 60 python tools/hangcheck.py 300 400 8 66 20.0 >> gpurun_out/small.log 2>&1
timeout 300 python tools/configs_bench.py >> gpurun_out/small.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -rf -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
