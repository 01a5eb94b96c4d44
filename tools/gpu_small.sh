#!/bin/bash
# small-image kernel: parity tests, then the crossover sweep against v7m
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_small.py -x -q 2>&1 | tail -15 > gpurun_out/small_tests.log
SHAPES="256 256 5 30 30  256 256 5 15 118  256 256 8 20 66  256 256 1 30 30  384 384 5 30 30  512 512 5 30 30  512 512 8 20 66  480 640 8 20 66"
for v in vs ${SWEEP_V7:+v7m}; do SF_VARIANT=$v timeout 300 python tools/small_sweep.py $SHAPES; done > gpurun_out/small_sweep.jsonl 2>&1
python tools/time_cfg.py cfg1 5 >> gpurun_out/small_sweep.jsonl 2>&1
SF_VARIANT=vs python tools/small_probe.py >> gpurun_out/small_sweep.jsonl 2>&1
cat gpurun_out/small_tests.log gpurun_out/small_sweep.jsonl
