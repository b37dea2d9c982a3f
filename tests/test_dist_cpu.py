"""Multi-process (world_size 2, gloo, CPU) coverage of the batch-sharding
logic bench.py uses on N GPUs: disjoint shards, no data-path collective, and
the max-over-ranks timing reduction.  Each rank runs the CPU oracle on its
own shard exactly as a GPU rank runs the device pipeline on its own."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import oracle as O

    B = 2
    seeds = bench.shard_seeds(rank, B)
    clouds = bench.clouds_for(rank, B, n_points=600)
    idx = [O.mdps(c, 150, exponent=0.45, rng_seed=rank * B + b).indices for b, c in enumerate(clouds)]
    t = bench.max_over_ranks(10.0 + rank)  # per-rank "time"
    all_seeds = [None] * world
    dist.all_gather_object(all_seeds, seeds)  # test-only check of disjointness
    q.put((rank, seeds, t, [i.tolist() for i in idx], all_seeds))
    dist.barrier()
    dist.destroy_process_group()


def test_batch_shards_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    seeds0, seeds1 = res[0][1], res[1][1]
    assert not set(seeds0) & set(seeds1), "shards must be disjoint"
    assert res[0][2] == res[1][2] == 11.0, "time is the max over ranks"
    # every rank's samples are distinct indices of its own shard
    for r in res:
        for idx in r[3]:
            assert len(idx) == 150 and len(set(idx)) == 150
