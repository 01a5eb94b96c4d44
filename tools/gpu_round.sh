#!/bin/bash
# round evidence of the current build: bench line, launch list, ncu --set full
# of the bench kernel (v7, cfg5 r = 16), smoke, precision stress
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch exit $?" >> gpurun_out/ncu_launch.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bilateral_box_v7 -s 3 -c 1 \
  -o gpurun_out/prof_v7_r16 -f python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_bench.log 2>&1
echo "ncu bench exit $?" >> gpurun_out/ncu_bench.log
timeout 600 python tools/drift_stress.py > gpurun_out/precision_stress.jsonl 2> gpurun_out/precision_stress.err
tail -3 gpurun_out/smoke.log gpurun_out/bench.err gpurun_out/ncu_launch.log gpurun_out/ncu_bench.log
cat gpurun_out/bench.json
