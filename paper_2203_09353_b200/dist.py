"""Replica sharding across processes (one process per GPU) and the single end-of-run
collective.

Replicas are independent: replica p runs on rank p mod world (the
reference's binding rule p mod devices, bench.cpp:171, 349-351), with no data-path
collective. The only exchange is at the end: an all-gather of the per-replica final
entropies (8 B each) so every rank can form the procedure-order average
(spinmc.cpp:253-269) and the best replica (max final entropy) — over NCCL on a GPU
box, over gloo in the CPU tests. torch.distributed is plumbing only.
"""
from __future__ import annotations

import numpy as np


def shard_procedures(procedures: int, rank: int, world: int) -> np.ndarray:
    """Procedures owned by `rank`: p = rank, rank + world, ... (< procedures)."""
    return np.arange(rank, procedures, world, dtype=np.int64)


def gather_finals(final_local: np.ndarray, procedures: int, rank: int, world: int, device=None):
    """All-gather per-rank final entropies into procedure order.

    Returns (finals[procedures], average_entropy, best_procedure, best_entropy). The average
    is summed sequentially in procedure order, as the reference does (spinmc.cpp:259-268).
    """
    import torch
    import torch.distributed as dist

    per_rank = (procedures + world - 1) // world
    buf = torch.full((per_rank,), float("nan"), dtype=torch.float64, device=device)
    n = len(final_local)
    if n:
        buf[:n] = torch.as_tensor(np.asarray(final_local, dtype=np.float64), device=device)
    if world > 1:
        out = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(out, buf)
        gathered = torch.stack(out).cpu().numpy()  # [world, per_rank]
    else:
        gathered = buf.cpu().numpy()[None]
    finals = np.empty(procedures, dtype=np.float64)
    for r in range(world):
        ps = shard_procedures(procedures, r, world)
        finals[ps] = gathered[r, : len(ps)]
    total = 0.0
    for x in finals:
        total += float(x)
    best = int(np.argmax(finals))
    return finals, total / procedures, best, float(finals[best])
