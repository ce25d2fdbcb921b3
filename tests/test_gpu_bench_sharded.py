"""bench.py's frequency-sharded (strong-scaling) harness, launched the way the
driver launches it (torch.distributed.run, one process per rank): ONE
mixture's bins are split over the ranks (the reference's parallel_for over
bins, parallel.cpp:16-45), the per-bin NLL slots are all-gathered and the
trace is summed in bin order -- so the 2-rank line must carry the same trace,
bit for bit, as the single-rank line.  Only one GPU exists here, so the two
ranks share it and the all-gather runs over gloo (--dist-backend gloo); the
ranks' fits are independent kernels (no rank waits on another).  On a
multi-GPU node the same command runs over NCCL, one GPU per rank."""
import json
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

COMMON = ["--config", "c0", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"]


def _line(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_two_rank_strong_scaling_line_matches_single_rank(gpu):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    one = _line([sys.executable, str(ROOT / "bench.py"), "--gpus", "1", *COMMON])
    two = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                 "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
                 "--gpus", "2", "--dist-backend", "gloo", *COMMON])
    assert two["n_gpus"] == 2 and two["scaling"] == "strong" and one["scaling"] == "strong"
    for k in ("workload", "M", "N", "F", "T", "iters", "batch"):
        assert two["config"][k] == one["config"][k], k  # the same total work
    assert two["config"]["batch"] == 1  # one mixture, its 513 bins split over the ranks
    assert two["trace"]["failed_bins"] == 0 and two["trace"]["monotone"]
    assert two["trace"]["nll_first"] == one["trace"]["nll_first"]  # bitwise
    assert two["trace"]["nll_last"] == one["trace"]["nll_last"]
    assert two["value"] > 0 and two["gpu_launches"] == 3
