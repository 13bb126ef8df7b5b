"""Multi-rank path on CPU (gloo, world_size 2): element sharding, generation by global index and
the post-timing reductions (max step time, checksum sum).  The device STP is replaced by the CPU
oracle here, so this checks the host-side plumbing the B200 ranks run, not the kernel."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2003_12787_b200.shard import (Shard, chunks, max_over_ranks, strong_shard, sum_over_ranks,
                                         weak_shard)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_strong_shard_partitions_exactly():
    for total in (0, 1, 7, 1048576, 1048577):
        for world in (1, 2, 3, 4, 8):
            shards = [strong_shard(total, world, r) for r in range(world)]
            assert shards[0].start == 0
            for a, b in zip(shards, shards[1:]):
                assert a.start + a.count == b.start
            assert sum(s.count for s in shards) == total
            assert max(s.count for s in shards) - min(s.count for s in shards) <= 1
    # BASELINE C5: 1,048,576 elements over 8 GPUs -> 131,072 per GPU
    assert strong_shard(1048576, 8, 5) == Shard(5, 8, 5 * 131072, 131072)


def test_weak_shard_and_chunks():
    s = weak_shard(131072, 4, 3)
    assert (s.start, s.count) == (3 * 131072, 131072)
    got = list(chunks(strong_shard(1000, 3, 1), 97))
    assert sum(c for _, c in got) == 333 and got[0][0] == 334 and got[-1][1] == 333 - 3 * 97
    with pytest.raises(ValueError):
        strong_shard(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, total, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = O.Oracle()
        sh = strong_shard(total, world, rank)
        q, rcc = orc.generate(0, 2024, n, sh.start, sh.count)
        cp_max = max_over_ranks(float(rcc[:, 1].max()) if sh.count else 0.0)
        dt = O.cfl_dt(n, cp_max)
        out = orc.stp(n, 9, q, dt, par=orc.material_lmr(rcc), threads=1)
        checksum = sum_over_ranks(float(out.qavg.sum() + out.face_f.sum()))
        slowest = max_over_ranks(float(rank + 1))
        if rank == 0:
            out_q.put((dt, checksum, slowest))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process():
    import oracle as O
    n, total, world = 4, 13, 2
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, total, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    dt, checksum, slowest = out_q.get(timeout=10)
    orc = O.Oracle()
    q, rcc = orc.generate(0, 2024, n, 0, total)
    assert dt == O.cfl_dt(n, float(rcc[:, 1].max()))
    out = orc.stp(n, 9, q, dt, par=orc.material_lmr(rcc), threads=1)
    want = float(out.qavg.sum() + out.face_f.sum())
    assert abs(checksum - want) <= 1e-12 * max(1.0, abs(want))
    assert slowest == 2.0


def _slab_worker(rank, world, port, out):
    import torch.distributed as dist
    from paper_2003_12787_b200.shard import make_rank_sync, slab_neighbours, slab_partition
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        sync = make_rank_sync()
        # the stability flag is the max over ranks: rank 1 reports non-finite in round 2
        flags = [sync(0), sync(3 if rank == 1 else 0), sync(0)]
        out.put((rank, slab_partition(7, world, rank), slab_neighbours(rank, world), flags))
    finally:
        dist.destroy_process_group()


def test_slab_partition_and_rank_sync_gloo():
    """The multi-GPU time loop's host logic (paper_2003_12787_b200/timeloop.py): z-slabs cover
    the mesh exactly once, periodic neighbours, and the per-step rank sync is a max over ranks."""
    import multiprocessing as mp
    from paper_2003_12787_b200.shard import slab_partition
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, out)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(out.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res[0][1] == (0, 4) and res[1][1] == (4, 3)
    assert res[0][2] == (1, 1) and res[1][2] == (0, 0)
    assert res[0][3] == [0, 3, 0] and res[1][3] == [0, 3, 0]
    layers = [slab_partition(10, 4, r) for r in range(4)]
    assert [z for z0, nz in layers for z in range(z0, z0 + nz)] == list(range(10))
