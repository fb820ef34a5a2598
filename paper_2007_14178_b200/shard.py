"""Batch sharding across the GPUs of one node (BASELINE config 5).

Every (image, filter) pair is independent, so the batch is
cut into contiguous per-rank slices, each rank packs its own replica of the
weights from the same host tensor, and there is NO collective on the hot path.
The only collectives are outside it: a max-reduce of per-rank device times
(timing protocol) and an optional gather of the outputs to rank 0.

Works with any torch.distributed backend: NCCL over NVLink on the GPU box,
gloo for the CPU tests (tests/test_shard.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(global_batch: int, world_size: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) slice of the batch for `rank`; the first
    global_batch % world_size ranks take one extra image."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError(f"bad rank {rank} for world size {world_size}")
    if global_batch < 0:
        raise ValueError("global_batch must be >= 0")
    base, extra = divmod(global_batch, world_size)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Max of a per-rank scalar (e.g. device milliseconds) over all ranks."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_to_rank0(local: torch.Tensor, global_batch: int, group=None):
    """Concatenate every rank's batch slice on rank 0 (None elsewhere).

    Uneven shards are padded to the largest shard for the collective and
    trimmed afterwards.  Off the timed hot path by design."""
    if not (dist.is_available() and dist.is_initialized()):
        return local
    ws = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if ws == 1:
        return local
    sizes = [shard_bounds(global_batch, ws, r) for r in range(ws)]
    biggest = max(b - a for a, b in sizes)
    pad_shape = (biggest,) + tuple(local.shape[1:])
    buf = torch.zeros(pad_shape, dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    if rank == 0:
        parts = [torch.empty_like(buf) for _ in range(ws)]
        dist.gather(buf, parts, dst=0, group=group)
        return torch.cat([p[: b - a] for p, (a, b) in zip(parts, sizes)])
    dist.gather(buf, None, dst=0, group=group)
    return None
