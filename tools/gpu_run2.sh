cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./tools/ubench > gpurun_out/ubench.log 2>&1
timeout 900 python tools/parity_report.py > gpurun_out/parity_v1.log 2>&1
