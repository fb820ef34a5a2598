"""Multi-rank host logic of the batch-sharded path, world_size 2 on gloo (CPU)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_14178_b200.shard import gather_to_rank0, max_over_ranks, shard_bounds


@pytest.mark.parametrize("gb", [0, 1, 7, 256, 2048, 2049])
@pytest.mark.parametrize("ws", [1, 2, 4, 8])
def test_shard_bounds_partition_exactly(gb, ws):
    covered = []
    for r in range(ws):
        a, b = shard_bounds(gb, ws, r)
        covered.extend(range(a, b))
        assert b - a in (gb // ws, gb // ws + 1)
    assert covered == list(range(gb))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, gb, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    a, b = shard_bounds(gb, ws, rank)
    # stand-in for the per-rank layer output: a function of the global image index
    local = torch.arange(a, b, dtype=torch.float32).view(-1, 1, 1, 1).expand(-1, 3, 2, 2).contiguous()
    full = gather_to_rank0(local, gb)
    t = max_over_ranks(10.0 + rank)
    if rank == 0:
        q.put((full.shape[0], bool(torch.equal(full[:, 0, 0, 0], torch.arange(gb, dtype=torch.float32))), t))
    dist.destroy_process_group()


@pytest.mark.parametrize("gb", [8, 7])
def test_gloo_two_ranks_gather_and_max(gb):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, gb, q)) for r in range(2)]
    for p in procs:
        p.start()
    n, ordered, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert n == gb and ordered and t == 11.0
