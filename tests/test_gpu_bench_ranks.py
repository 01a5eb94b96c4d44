"""The bench's N > 1 GPU arm (row bands for cfg5, term split for cfg4) run as
two ranks on the one GPU this pool offers: SF_BENCH_SHARED_GPU=1 puts both
ranks on cuda:0 over gloo (NCCL refuses two ranks on one device).  This checks
the multi-rank code path end to end — launcher, band split, max/sum over
ranks, the JSON line — not its timing."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["cfg5", "cfg4"])
def test_bench_two_ranks_shared_gpu(workload):
    env = dict(os.environ, SF_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3",
           "--no-sweep", "--no-cpu", "--no-configs", "--workload", workload]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and "diagnostic" in line
    assert line["value"] > 0 and line["ms_per_step"] > 0
    assert line["gpu_launches"] >= 1
    assert line["config"]["parallelism"] == ("rowband2" if workload == "cfg5" else "termsplit2")
    assert line["e2e"]["value"] > 0
