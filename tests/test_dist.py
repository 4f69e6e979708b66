"""The N > 1 path on CPU: two gloo ranks, round-robin workunit shards, int64
all-reduce of the counts (the oracle stands in for the GPU search here)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1709_02599_b200.dist import shard_workunits


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import oracle
    import paper_1709_02599_b200 as D
    from paper_1709_02599_b200.dist import allreduce_count, allreduce_max, shard_workunits

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 6
    d = D.default_split_depth(n)
    recs = D.dls_split(n, d)
    mine = shard_workunits(recs, rank, world)
    order = oracle.plan(n)[d:]
    import synth
    local = sum(oracle.count(n, False, synth.to_int_grid(r), order)[0] for r in mine)
    total = allreduce_count(local)
    slowest = allreduce_max(float(rank + 1))
    q.put((rank, len(mine), local, total, slowest))
    dist.destroy_process_group()


def test_shards_partition_the_workunits():
    recs = np.arange(10 * 4, dtype=np.uint8).reshape(10, 2, 2)
    parts = [shard_workunits(recs, r, 3) for r in range(3)]
    got = np.concatenate(parts)
    assert sorted(map(bytes, got)) == sorted(map(bytes, recs))
    assert [len(p) for p in parts] == [4, 3, 3]
    with pytest.raises(ValueError):
        shard_workunits(recs, 3, 3)


def test_two_rank_gloo_count():
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = oracle.count_all(6)
    assert all(r[3] == want for r in res)                 # every rank sees the sum
    assert sum(r[2] for r in res) == want                 # shards add up
    assert all(r[4] == 2.0 for r in res)                  # max over ranks


def test_bench_split_depth_grows_with_ranks():
    """bench.py: every rank gets >= ~3.5 workunits per lane (148 SMs x 1024 lanes)."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    import paper_1709_02599_b200 as D
    lib = D.load()
    prev = 0
    for world in (1, 2, 4, 8):
        d = bench.pick_depth(world)
        assert d >= prev
        prev = d
        assert lib.dls_split(8, 0, 1, d, None, 0) >= 3.5 * 148 * 1024 * world
    assert bench.pick_depth(1) == D.default_split_depth(8)      # config 3: diagonals
