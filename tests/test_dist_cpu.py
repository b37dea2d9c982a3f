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


# ---- point-split FPS (C5) host logic ------------------------------------------------

def _split_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2507_23480_b200 import pointsplit

    # shard partition used by the kernel, and the chunk-merge rule it relies on:
    # each rank reduces its own shard, the G records merge to the reference FPS
    N, n = 700, 120
    c = np.random.default_rng(3).random((N, 3), dtype=np.float32)
    c[350:360] = c[0]  # duplicates across the shard boundary
    lo, hi = pointsplit.shard_range(N, world, rank)
    x, y, z = O.columns_f64(c)
    md = np.full(N, np.inf)
    taken = np.zeros(N, np.uint8)
    out = [0]
    taken[0] = 1
    for _ in range(1, n):
        p = out[-1]
        best, bj = O.CKernels.fps_update_chunk(x, y, z, x[p], y[p], z[p], md, lo, hi)
        recs = [None] * world
        dist.all_gather_object(recs, (float(best), int(bj), bool(bj >= 0 and taken[bj])))
        mb, mj, mt = max((r for r in recs if r[1] >= 0), key=lambda r: (r[0], -r[1]))
        if mb <= 0.0 or mt:
            fu = [None] * world
            local = [j for j in range(lo, hi) if not taken[j]]
            dist.all_gather_object(fu, local[0] if local else -1)
            cand = [j for j in fu if j >= 0]
            if cand:
                mj = min(cand)
        # every rank refolds its own shard only; md outside [lo, hi) is never read
        taken[mj] = 1
        out.append(mj)
    q.put((rank, (lo, hi), out))


def test_point_split_host_protocol_gloo_world2():
    """World-2 (gloo, CPU) restatement of the point-split exchange: shards
    [g*ceil(N/G), ...) merged by (max md, lowest index) with the cross-rank
    lowest-untaken fallback reproduce the single-process reference FPS."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import oracle as O

    N, n = 700, 120
    c = np.random.default_rng(3).random((N, 3), dtype=np.float32)
    c[350:360] = c[0]
    ref = O.fps(c, n, 0)[0]
    (r0, s0, o0), (r1, s1, o1) = res
    assert s0 == (0, 350) and s1 == (350, 700)
    assert o0 == o1 == ref.tolist()
