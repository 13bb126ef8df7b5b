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
