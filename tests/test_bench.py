"""bench.py's launcher and reference arm on CPU (no GPU needed): `--gpus 2`
outside torchrun re-executes itself as two ranks under
torch.distributed.run on 127.0.0.1; under the reference arm rank 0 alone
runs the oracle sample and prints one JSON line whose n_gpus is 2, the other
rank exits 0 (the task's reference-arm contract)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None, timeout=600):
    env = dict(os.environ, SF_BENCH_ORACLE_S="0.2", OMP_NUM_THREADS="2")
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                          text=True, timeout=timeout, env=env, cwd=ROOT)


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_reference_arm_one_process():
    res = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert res.returncode == 0, res.stderr[-2000:]
    lines = _json_lines(res.stdout)
    assert len(lines) == 1
    ln = lines[0]
    assert ln["impl"] == "reference" and ln["n_gpus"] == 1 and ln["value"] > 0
    assert ln["e2e"]["value"] == ln["value"] and ln["cpu_baseline"]["kind"] == "oracle"
    rows = int(ln["cpu_baseline"]["sample"].split("[0,")[1].split(")")[0])
    assert rows >= 32 * ln["cpu_baseline"]["cores"]           # every host core gets oracle bands


def test_gpus_2_spawns_two_ranks():
    res = _run(["--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert res.returncode == 0, res.stderr[-2000:]
    lines = _json_lines(res.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2      # rank 0 only


def test_world_size_must_match_gpus():
    """Under an external launcher the world size must equal --gpus."""
    res = _run(["--gpus", "2", "--steps", "1", "--warmup", "0"], env_extra={"WORLD_SIZE": "1", "RANK": "0"})
    assert res.returncode == 2 and "world size 1 != --gpus 2" in res.stderr
