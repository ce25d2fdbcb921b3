"""bench.py's reference arm on CPU: `--impl reference` runs the oracle port
of the reference path (the reference itself cannot be built here) and prints
one JSON line with the contract's keys; under a multi-rank launch only rank 0
prints."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config",
                        "c0", "--steps", "1", "--warmup", "3", "--cpu-bins", "4"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr
    return [l for l in r.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_prints_contract_line(built):
    lines = _run({})
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "c0"


def test_reference_arm_other_ranks_exit_quietly(built):
    assert _run({"RANK": "1", "WORLD_SIZE": "2"}) == []
