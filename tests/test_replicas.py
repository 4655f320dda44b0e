"""Multi-GPU host logic (query replicas) on CPU: two gloo ranks
take disjoint query batches at every step and reduce their timings (max) and
query counts (sum) into the whole-job throughput bench.py reports."""

import os
import socket

import pytest

torch = pytest.importorskip("torch")

from paper_1912_08756_b200.replicas import aggregate, rank_batch  # noqa: E402


def test_rank_batch_single_process():
    assert [rank_batch(0, 1, i, 4) for i in range(6)] == [0, 1, 2, 3, 0, 1]
    nq, (t,) = aggregate(None, "cpu", 512, [0.25])
    assert nq == 512 and t == 0.25
    with pytest.raises(ValueError):
        rank_batch(2, 2, 0, 4)


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nb = 5
        mine = [rank_batch(rank, world, i, nb) for i in range(7)]
        got = [None] * world
        dist.all_gather_object(got, mine)
        # per-rank figures: rank r ran 100 + r queries in 1 + r seconds (two timings)
        nq_all, times = aggregate(dist, "cpu", 100 + rank, [1.0 + rank, 0.5 - 0.1 * rank])
        out.put((rank, got, nq_all, times))
    finally:
        dist.destroy_process_group()


def test_two_gloo_ranks_partition_and_reduce():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    res = [out.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, nq_all, times in res:
        # every step: the two ranks run different, consecutive batches
        for a, b in zip(got[0], got[1]):
            assert a != b and b == (a + 1) % 5
        # over the steps every batch is covered
        assert set(got[0]) | set(got[1]) == set(range(5))
        # whole-job figures: queries summed, times maxed over the ranks
        assert nq_all == 201
        assert times == [2.0, 0.5]
