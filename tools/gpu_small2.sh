#!/bin/bash
mkdir -p gpurun_out
(for v in vs v7m; do SF_VARIANT=$v python tools/small_probe.py; done) > gpurun_out/small_probe.jsonl 2>&1
SF_VARIANT=vs ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,smsp__cycles_active.avg --clock-control none --csv python tools/small_probe.py > gpurun_out/small_ncu.csv 2>&1
cat gpurun_out/small_probe.jsonl; grep -i "bilateral\|fill\|Kernel" gpurun_out/small_ncu.csv | head -40
