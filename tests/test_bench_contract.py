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


def test_default_workload_is_c3_and_arms_share_config():
    """The headline config is BASELINE configs[3]; both arms print the same
    `config` dict (the driver compares them), strong scaling shards ONE
    mixture's bins."""
    import argparse
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", ROOT / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    from paper_2101_08563_b200 import synth
    src = (ROOT / "bench.py").read_text()
    assert 'os.environ.get("FFCA_BENCH_CONFIG", "c3")' in src
    c3 = synth.CONFIGS["c3"]
    for world in (1, 2, 8):
        wl, scaling = bench.workload(c3, world)
        assert scaling == "strong" and wl.batch == 1  # one mixture, bins split over ranks
        a = bench.config_dict(c3, wl.batch, world, scaling)
        assert a["workload"] == "c3" and (a["M"], a["N"], a["F"], a["T"], a["iters"]) == (8, 12, 2049, 8000, 30)
    wl, scaling = bench.workload(c3, 4, "weak")
    assert scaling == "weak" and wl.batch == 4
    assert bench.alg_bytes(8, 12) == 160 and bench.alg_flops(8, 12) == 3176
    assert src.count("config_dict(") >= 3  # defined once, used by both arms
