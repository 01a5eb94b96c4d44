cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/profile_case.py 2048 2048 16 0 15 118 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v2 -s 1 -c 1 -o gpurun_out/prof_v2a python tools/profile_case.py 2048 2048 16 0 15 118 2 > gpurun_out/ncu_v2a.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_v2a.log
