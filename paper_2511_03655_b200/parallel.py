"""Host-side multi-GPU plumbing (one process per GPU, torch.distributed).

Two ways the path shards:

* Ensembles (configs 2-4): independent trajectories -> contiguous batch slices
  per rank, no data-path collective.  `batch_slice` / `gather_batch`.
* One large N-body system (config 5): body shards; the library's
  irk_set_comm + in-kernel-loop ncclAllGather of stage positions per
  fixed-point iteration does the exchange.  Here: the NCCL unique-id bootstrap
  over the process group (`nccl_bootstrap`), and the row bookkeeping between the
  global state [q (3N) | v (3N)] and a rank's local rows [q_loc | v_loc]
  (`shard_rows` / `assemble_rows`).

Nothing here does any of the method's arithmetic.
"""
from __future__ import annotations

import numpy as np


def batch_slice(batch: int, rank: int, world: int) -> slice:
    """Contiguous, balanced slice of trajectories for `rank` (first ranks get the extra)."""
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return slice(start, start + base + (1 if rank < extra else 0))


def gather_batch(local: np.ndarray, group=None) -> np.ndarray:
    """All-gather per-rank (rows, local_batch) arrays into (rows, batch), rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, np.ascontiguousarray(local), group=group)
    return np.concatenate(parts, axis=-1)


def body_range(nbody: int, rank: int, world: int) -> tuple[int, int]:
    if nbody % world:
        raise ValueError("N must be divisible by the number of ranks")
    n = nbody // world
    return rank * n, (rank + 1) * n


def shard_rows(y: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Global N-body state y = [q (3N) | v (3N)] (rows, ...) -> this rank's rows
    [q_loc (3N/P) | v_loc (3N/P)] (the layout irk_set_comm expects)."""
    N = y.shape[0] // 6
    b0, b1 = body_range(N, rank, world)
    return np.concatenate([y[3 * b0:3 * b1], y[3 * N + 3 * b0:3 * N + 3 * b1]])


def assemble_rows(parts: list[np.ndarray]) -> np.ndarray:
    """Inverse of shard_rows over all ranks (parts in rank order)."""
    world = len(parts)
    nl = parts[0].shape[0] // 2
    q = [p[:nl] for p in parts]
    v = [p[nl:] for p in parts]
    assert all(p.shape[0] == 2 * nl for p in parts)
    del world
    return np.concatenate(q + v)


def nccl_bootstrap(rank: int, group=None) -> bytes:
    """Rank 0 creates a 128-byte ncclUniqueId (through the library), every rank
    receives it over the process group (gloo or nccl)."""
    import torch.distributed as dist
    obj = [None]
    if rank == 0:
        from . import irk
        obj[0] = irk.nccl_unique_id()
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def max_over_ranks(value: float, group=None, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
