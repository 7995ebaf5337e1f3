"""World-size-2 gloo test of the multi-GPU bench aggregation (CPU, 127.0.0.1 rendezvous)."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_2211_13939_b200.harness import merge_rank_stats, nearest_rank


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    local = {"fcl": [10.0 * (rank + 1) + i for i in range(5)], "fcl_c": [1.0], "lcl": [2.0], "rtf": [0.1],
             "window": 1.5 + rank, "missing": rank, "launch": 100, "h2d": 8, "d2h": 16}
    merged = merge_rank_stats(local, dist)
    if rank == 0:
        out.put(merged)
    else:
        assert merged is None
    dist.barrier()
    dist.destroy_process_group()


def test_merge_over_two_gloo_ranks():
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in procs]
    merged = q.get(timeout=120)
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    assert sorted(merged["fcl"]) == sorted([10.0 + i for i in range(5)] + [20.0 + i for i in range(5)])
    assert merged["window"] == 2.5                 # max over ranks
    assert merged["missing"] == 1 and merged["launch"] == 200
    assert nearest_rank(merged["fcl"], 99) == 24.0


def test_single_rank_passthrough():
    local = {"fcl": [1.0], "fcl_c": [], "lcl": [], "rtf": [], "window": 3.0}
    assert merge_rank_stats(local, None) == local
