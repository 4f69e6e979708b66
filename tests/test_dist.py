"""The N > 1 path on CPU: two gloo ranks, round-robin workunit shards, int64
all-reduce of the counts (the oracle stands in for the GPU search here)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1709_02599_b200.dist import shard_ranges, shard_workunits


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


def _oracle_sb_range(n, b, e, vs):
    """Stand-in for dls_count_sb_range on CPU (oracle only): Alg. 6 over the
    diagonal workunits [b, e) -- every hourglass below them (row N-1 completed),
    canonic ones weighted by their class size (Corollary 1)."""
    import oracle
    plan = oracle.plan(n, vs)
    diag = {i * n + j for i in range(1, n) for j in (i, n - 1 - i)}
    dd = next(k for k in range(len(plan) + 1) if diag <= {c for c in plan[:k]} | {(c // n) * n + n - 1 - c % n for c in plan[:k] if vs})
    units = oracle.prefixes(n, vs, oracle.first_row_grid(n), plan, dd)[b:e]
    last = [(n - 1) * n + j for j in range(n) if (not vs or 2 * j <= n - 1)]
    total = hg = cls = 0
    for u in units:
        cells = [c for c in last if u.reshape(-1)[c] == -1]
        for h in oracle.prefixes(n, vs, u, cells, len(cells)):
            hg += 1
            m = oracle.canonize(n, vs, h)
            if m:
                cls += 1
                total += m * oracle.count(n, vs, h)[0]
    return {"count": total, "hourglasses": hg, "classes": cls, "nodes": 0}


def _sb_worker(rank, world, port, q):
    import torch.distributed as dist
    import oracle
    from paper_1709_02599_b200.dist import count_sb_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 6
    plan = oracle.plan(n)
    n_units = oracle.count_prefixes(n, False, oracle.first_row_grid(n), plan, 8)
    r = count_sb_sharded(n, False, rank, world, 1, n_units, count_range=_oracle_sb_range)
    q.put((rank, r))
    dist.destroy_process_group()


def test_shard_ranges_partition():
    from paper_1709_02599_b200.dist import shard_ranges
    for n_units, world, chunk in ((10, 3, 2), (7, 2, 5), (0, 2, 3), (100, 4, 7)):
        got = sorted(x for r in range(world) for b, e in shard_ranges(n_units, r, world, chunk) for x in range(b, e))
        assert got == list(range(n_units))
    with pytest.raises(ValueError):
        shard_ranges(5, 2, 2, 1)


def test_two_rank_gloo_symmetry_broken_count():
    """Alg. 6 sharded over two gloo ranks by diagonal-workunit ranges: the rank
    totals add up to the full first-row-fixed count, the all-reduced total equals
    it on both ranks (the oracle stands in for dls_count_sb_range)."""
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sb_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = oracle.count_all(6)
    assert all(res[r]["count"] == want for r in res)
    assert sum(res[r]["local_count"] for r in res) == want
    assert all(res[r]["local_count"] > 0 for r in res)
