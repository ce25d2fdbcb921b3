"""Frequency sharding host logic on CPU: world_size-2 gloo processes split the
(mixture, bin) problems, all-gather the per-bin NLL slots and assemble the
same bin-order trace a single process computes.  The per-bin
"fit" here is the fp64 oracle, so the check is end to end on real traces."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2101_08563_b200 import synth
from paper_2101_08563_b200.shard import bin_order_trace, gather_slots, shard

CFG = synth.small(2, 2, 7, 80, seed=3)
ITERS = 4
BATCH = 2


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem_slots(lo: int, hi: int) -> np.ndarray:
    """Per-bin NLL slots [(iters+1), hi-lo] of problems [lo, hi) via the oracle."""
    import oracle
    cfg = CFG
    out = []
    for p in range(lo, hi):
        b, f = divmod(p, cfg.F)
        x = synth.mixture(cfg, b)[f:f + 1].astype(np.complex128)
        W, L, H = synth.init_params(cfg, b)
        _, _, _, _, sl, _ = oracle.fit(x, W[f:f + 1], L[f:f + 1], H[f:f + 1], ITERS, slots=True)
        out.append(sl[:, 0])
    return np.stack(out, axis=1) if out else np.zeros((ITERS + 1, 0))


def _worker(rank, world, port, q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = BATCH * CFG.F
    lo, hi = shard(P, world, rank)
    local = torch.from_numpy(_problem_slots(lo, hi))
    full = gather_slots(local, P, world, rank, dist)
    if rank == 0:
        q.put(bin_order_trace(full, BATCH, CFG.F))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_partition():
    for P in (1, 7, 513, 513 * 256 + 5):
        for world in (1, 2, 3, 8):
            spans = [shard(P, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == P
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - lo for lo, h in spans]
            assert max(sizes) - min(sizes) <= 1


def test_gloo_two_ranks_match_single_process(built):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    trace2 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    single = bin_order_trace(_problem_slots(0, BATCH * CFG.F), BATCH, CFG.F)
    np.testing.assert_array_equal(trace2, single)  # bitwise: same slots, same order


@pytest.mark.parametrize("world", [1, 2, 4])
def test_trace_is_independent_of_shard_count(built, world):
    P = BATCH * CFG.F
    slots = _problem_slots(0, P)
    parts = [slots[:, slice(*shard(P, world, r))] for r in range(world)]
    assembled = np.concatenate(parts, axis=1)
    np.testing.assert_array_equal(bin_order_trace(assembled, BATCH, CFG.F),
                                  bin_order_trace(slots, BATCH, CFG.F))
