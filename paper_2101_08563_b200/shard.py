"""Frequency sharding across GPUs.

Frequencies (and, for batches, mixtures x frequencies) are independent, so
the flattened problem index p = b*F + f is split into contiguous balanced
ranges, one per rank; no data moves during the fit.  The only collective is
the final all-gather of the per-bin NLL slots, from which every mixture's
trace is assembled in bin order exactly like the reference's
`nll[t] = sum_i nll_slots(t, i)` (fastfca.cpp:186-189) -- so the trace does
not depend on the number of GPUs.
"""
from __future__ import annotations

import numpy as np


def shard(P: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced range [lo, hi) of P problems for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard: bad world/rank")
    base, rem = divmod(P, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def gather_slots(local, P: int, world: int, rank: int, dist=None):
    """All-gather per-bin slots [(iters+1), P_local] (torch tensor) into the
    full [(iters+1), P] array (numpy), in global problem order."""
    if dist is None or world == 1:
        return local.detach().cpu().numpy()
    import torch
    sizes = [shard(P, world, r)[1] - shard(P, world, r)[0] for r in range(world)]
    width = max(sizes)
    pad = torch.zeros((local.shape[0], width), dtype=local.dtype, device=local.device)
    pad[:, : local.shape[1]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[:, :n] for p, n in zip(parts, sizes)], dim=1).cpu().numpy()


def bin_order_trace(all_slots: np.ndarray, batch: int, F: int) -> np.ndarray:
    """Per-mixture traces [(iters+1), batch] summed over bins in bin order."""
    T1 = all_slots.shape[0]
    out = np.zeros((T1, batch))
    s = all_slots.reshape(T1, batch, F)
    for i in range(F):  # sequential, bin order (fastfca.cpp:188)
        out += s[:, :, i]
    return out
