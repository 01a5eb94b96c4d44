cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SF_DIAG=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v5 -s 1 -c 1 -o gpurun_out/prof_v5_ponly python tools/profile_case.py 2368 2048 16 0 15 118 2 > gpurun_out/ncu_ponly.log 2>&1
SF_DIAG=2 timeout 300 ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v5 -s 1 -c 1 -o gpurun_out/prof_v5_conly python tools/profile_case.py 2368 2048 16 0 15 118 2 > gpurun_out/ncu_conly.log 2>&1
