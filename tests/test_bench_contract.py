"""bench.py's JSON contract, checked on the CPU through the reference arm
(the oracle on host cores; the GPU arm is exercised on the B200)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config", ["c1", "c2", "c6", "c5"])
def test_reference_arm_line(config):
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", config, "--steps", "1",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["steps"] == 1 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["unit"] == line["unit"]
    assert "workload" in line["config"]


def _env_without_launcher():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    return env


def test_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` with no launcher spawns 2 ranks itself
    (torch.distributed.run, 127.0.0.1); they meet in a process group (gloo on
    the CPU here, NCCL on the GPU box) and rank 0 reports the world size."""
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--check-launch"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300, env=_env_without_launcher())
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["rank_sum"] == 1


def test_gpus_flag_must_match_launcher():
    """Under a launcher, WORLD_SIZE != --gpus fails loudly (it never times one
    GPU while claiming N)."""
    env = _env_without_launcher()
    env.update(WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--check-launch"], cwd=ROOT, capture_output=True,
                       text=True, timeout=120, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
