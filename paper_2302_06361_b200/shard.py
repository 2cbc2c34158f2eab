"""Inference sharding across ranks.

Garbled inferences are independent (one seed, one garbled circuit each), so a
global batch is split into contiguous per-rank shards with no data-path
exchange; the only collective is one all-gather of the decoded outputs
(int64, n_out per inference) so that rank 0 holds the whole batch.  On B200
the process group is NCCL over NVLink; the CPU tests use gloo.
"""
from __future__ import annotations

from typing import List

import numpy as np


def shard_range(global_batch: int, world: int, rank: int):
    """Contiguous [start, stop) slice of the global batch owned by `rank`."""
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def step_seeds(step: int, global_batch: int, first: int = 0x5EED0000) -> List[bytes]:
    """Fresh 16-byte seeds (seed_from_string(hex(v)) form) for every inference of a step."""
    return [int(first + step * global_batch + i).to_bytes(16, "big") for i in range(global_batch)]


def gather_outputs(local: np.ndarray, global_batch: int, n_out: int, group=None, device=None) -> np.ndarray:
    """All-gathers per-rank decoded outputs into the [global_batch, n_out] array."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    counts = [shard_range(global_batch, world, r) for r in range(world)]
    width = max(b - a for a, b in counts)
    buf = torch.zeros((width, n_out), dtype=torch.int64, device=device)
    buf[: local.shape[0]] = torch.as_tensor(local, dtype=torch.int64, device=device)
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return np.concatenate([p[: b - a].cpu().numpy() for p, (a, b) in zip(parts, counts)], axis=0)
