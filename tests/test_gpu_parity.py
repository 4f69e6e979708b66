"""GPU parity: the sm_100a kernel (through the C ABI) against the CPU oracle.

Bar: counts are integers, so every comparison is bit-exact.
Node counts are compared too wherever the oracle enumerates the same tree (same
Section 2.3 order below the same prefixes).  The five BASELINE.json configs:

  1  N=6, no first-row fixing: every prefix and the total
  2  N=7, first row fixed: every prefix, total and the N! scaled total
  3  N=8, first row fixed: full count = 7 447 587 840, sampled prefixes
  4  VS N=8 full (every prefix) and VS N=10 on 4096 seeded prefixes
  5  N=9 on 1024 seeded prefixes
"""
import math

import numpy as np
import pytest

import oracle
import synth
import paper_1709_02599_b200 as D
from paper_1709_02599_b200 import _binding as B
from conftest import golden, paper_counts

pytestmark = pytest.mark.gpu


def _oracle_per_prefix(n, vs, recs, depth, fixed=True):
    """Oracle counts of every record, and the oracle's node total of the search
    the GPU runs: the plan cells below the records down to the level
    dls_search_levels reports (the two-row closure level, R15)."""
    pre = np.zeros((n, n), np.int32)
    if fixed:
        pre[0, :] = 1
    order = oracle.plan(n, vs, pre)[depth:]
    levels = D.dls_search_levels(n, depth, vs, fixed) if len(order) else 0
    out = [oracle.count_levels(n, vs, synth.to_int_grid(r), order) for r in recs]
    return np.array([c for c, _ in out], dtype=np.uint64), sum(sum(lv[:levels]) for _, lv in out)


class closure_off:
    """DLS_CLOSE=0 for the calls inside: the plain search over every level (its
    node count is the oracle's full-tree count)."""
    def __enter__(self):
        import os
        self.old = os.environ.get("DLS_CLOSE")
        os.environ["DLS_CLOSE"] = "0"

    def __exit__(self, *a):
        import os
        if self.old is None:
            os.environ.pop("DLS_CLOSE", None)
        else:
            os.environ["DLS_CLOSE"] = self.old


def _gpu(n, vs, recs, depth, fixed=True):
    counts, total, nodes = D.count_prefixes(n, recs, vs, fixed, depth)
    assert int(counts.sum()) == total
    return counts, total, nodes


# ------------------------------------------------------------------ config 1

def test_config1_dls6_no_symmetry_breaking():
    n, vs, fixed = 6, False, False
    d = D.default_split_depth(n, vs, fixed)
    recs = D.dls_split(n, d, vs, fixed)
    counts, total, nodes = _gpu(n, vs, recs, d, fixed)
    want, want_nodes = _oracle_per_prefix(n, vs, recs, d, fixed)
    assert (counts == want).all()
    assert nodes == want_nodes
    assert total == oracle.count_all(n, fixed_first_row=False)
    assert total == math.factorial(n) * oracle.count_all(n, fixed_first_row=True)


# ------------------------------------------------------------------ config 2

@pytest.mark.parametrize("extra", [0, 3])
def test_config2_dls7_first_row(extra):
    n = 7
    d = D.default_split_depth(n) + extra
    recs = D.dls_split(n, d)
    counts, total, nodes = _gpu(n, False, recs, d)
    want, want_nodes = _oracle_per_prefix(n, False, recs, d)
    assert (counts == want).all()
    assert nodes == want_nodes
    assert total == oracle.count_all(n)
    r = D.count_squares(n)
    assert r["count"] == total and r["total_all_first_rows"] == math.factorial(7) * total


# ------------------------------------------------------------------ config 3

def test_config3_dls8_full_count_matches_paper():
    r = D.count_squares(8)
    assert r["n_prefix"] == 547896
    assert r["count"] == paper_counts()["dls8_first_row_fixed"]
    assert r["total_all_first_rows"] == math.factorial(8) * 7447587840


def test_config3_dls8_sampled_prefixes():
    n, d = 8, D.default_split_depth(8)
    recs = D.dls_split(n, d)
    counts, total, _ = _gpu(n, False, recs, d)
    assert total == paper_counts()["dls8_first_row_fixed"]
    rng = np.random.default_rng(8)
    idx = np.concatenate([rng.choice(len(recs), 150, replace=False), [0, len(recs) - 1]])
    want, _ = _oracle_per_prefix(n, False, recs[idx], d)
    assert (counts[idx] == want).all()


# ------------------------------------------------------------------ config 4

def test_config4_vs8_full():
    n, vs = 8, True
    d = D.default_split_depth(n, vs)
    recs = D.dls_split(n, d, vs)
    counts, total, nodes = _gpu(n, vs, recs, d)
    want, want_nodes = _oracle_per_prefix(n, vs, recs, d)
    assert (counts == want).all()
    assert nodes == want_nodes
    assert total == oracle.count_all(n, vs=True)


def _read_golden(name):
    """index -> (count, nodes) from the round-1 file and the stratified round-2
    sample next to it (scripts/make_golden.py, make_golden_r2.py: oracle only)."""
    rows = {}
    for fn in (name, name.replace(".txt", "_r2.txt")):
        for line in open(golden(fn)):
            if line.startswith("#") or not line.strip():
                continue
            i, c, nd = line.split()[:3]
            rows[int(i)] = (int(c), int(nd))
    return rows


def test_config4_vs10_seeded_prefixes():
    n, vs = 10, True
    recs = synth.diagonal_prefixes(synth.SEED_VS10, n, synth.N_VS10, vs=True)
    d = D.default_split_depth(n, vs)
    counts, total, _ = _gpu(n, vs, recs, d)
    gold = _read_golden("vs10_prefix_counts.txt")
    for i, (c, _) in gold.items():
        assert int(counts[i]) == c, i
    # the golden prefixes alone: same counts, and the plain search (closure off)
    # visits exactly the oracle's full-tree nodes (full-size workunits, refined
    # to ~1.2M records on the host)
    idx = sorted(gold)
    c2, t2, _ = _gpu(n, vs, recs[idx], d)
    assert [int(x) for x in c2] == [gold[i][0] for i in idx]
    with closure_off():
        c3, t3, nodes = _gpu(n, vs, recs[idx], d)
    assert [int(x) for x in c3] == [gold[i][0] for i in idx]
    assert nodes == sum(gold[i][1] for i in idx)


def test_config4_vs10_children_vs_oracle():
    """Deepen two seeded VS10 prefixes by two rows with the oracle's own prefix
    enumeration; GPU counts of sampled children must equal the oracle's."""
    n, vs = 10, True
    recs = synth.diagonal_prefixes(synth.SEED_VS10, n, 3, vs=True)
    d = D.default_split_depth(n, vs)
    order = oracle.plan(n, vs)
    extra = 8
    rng = np.random.default_rng(10)
    for r in recs[:2]:
        kids = oracle.prefixes(n, vs, synth.to_int_grid(r), order[d:], extra)
        pick = rng.choice(len(kids), min(12, len(kids)), replace=False)
        kid_recs = np.where(kids[pick] < 0, 255, kids[pick]).astype(np.uint8)
        counts, _, nodes = _gpu(n, vs, kid_recs, d + extra)
        want, want_nodes = _oracle_per_prefix(n, vs, kid_recs, d + extra)
        assert (counts == want).all()
        assert nodes == want_nodes


# ------------------------------------------------------------------ config 5

def test_config5_dls9_seeded_prefixes():
    n = 9
    recs = synth.diagonal_prefixes(synth.SEED_DLS9, n, synth.N_DLS9)
    d = D.default_split_depth(n)
    counts, total, _ = _gpu(n, False, recs, d)
    gold = _read_golden("dls9_prefix_counts.txt")
    for i, (c, _) in gold.items():
        assert int(counts[i]) == c, i
    idx = sorted(gold)
    c2, t2, _ = _gpu(n, False, recs[idx], d)
    assert [int(x) for x in c2] == [gold[i][0] for i in idx]
    with closure_off():
        c3, t3, nodes = _gpu(n, False, recs[idx], d)
    assert [int(x) for x in c3] == [gold[i][0] for i in idx]
    assert nodes == sum(gold[i][1] for i in idx)


def test_config5_dls9_children_vs_oracle():
    n = 9
    recs = synth.diagonal_prefixes(synth.SEED_DLS9, n, 2)
    d = D.default_split_depth(n)
    order = oracle.plan(n)
    extra = 9
    rng = np.random.default_rng(9)
    for r in recs:
        kids = oracle.prefixes(n, False, synth.to_int_grid(r), order[d:], extra)
        pick = rng.choice(len(kids), min(10, len(kids)), replace=False)
        kid_recs = np.where(kids[pick] < 0, 255, kids[pick]).astype(np.uint8)
        counts, _, nodes = _gpu(n, False, kid_recs, d + extra)
        want, want_nodes = _oracle_per_prefix(n, False, kid_recs, d + extra)
        assert (counts == want).all()
        assert nodes == want_nodes


class env_set:
    """Environment knobs of the library (read at every call) for the calls inside."""
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        import os
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update(self.kv)

    def __exit__(self, *a):
        import os
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("rng_la,close", [("51-60", "1"), ("51-60", "0"), ("30-60", "1"), ("20-72", "0")])
def test_lookahead_dls9_never_changes_counts(rng_la, close):
    """Section 2.4.2: the lookahead only cuts branches that cannot be
    completed, so every per-prefix count stays the oracle's; the kernel with it
    visits no more nodes than without."""
    n = 9
    r = synth.diagonal_prefixes(synth.SEED_DLS9, n, 1)[0]
    d = D.default_split_depth(n)
    order = oracle.plan(n)
    extra = 10
    kids = oracle.prefixes(n, False, synth.to_int_grid(r), order[d:], extra)
    pick = np.random.default_rng(5).choice(len(kids), min(12, len(kids)), replace=False)
    kid_recs = np.where(kids[pick] < 0, 255, kids[pick]).astype(np.uint8)
    want, _ = _oracle_per_prefix(n, False, kid_recs, d + extra)
    with env_set(DLS_CLOSE=close):
        c0, _, nodes0 = _gpu(n, False, kid_recs, d + extra)
        with env_set(DLS_LOOKAHEAD=rng_la):
            c1, _, nodes1 = _gpu(n, False, kid_recs, d + extra)
    assert (c0 == want).all() and (c1 == want).all()
    assert nodes1 <= nodes0


# ------------------------------------------------------------------ edge cases

@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_small_orders(n):
    r = D.count_squares(n)
    assert r["count"] == oracle.count_all(n)
    r = D.count_squares(n, fixed_first_row=False)
    assert r["count"] == oracle.count_all(n, fixed_first_row=False)


def test_empty_input():
    recs = np.zeros((0, 8, 8), np.uint8)
    counts, total, nodes = D.count_prefixes(8, recs)
    assert total == 0 and nodes == 0 and counts.shape == (0,)


@pytest.mark.parametrize("back", [0, 1, 2, 5])
def test_deep_prefixes_ragged_tail(back):
    # L = levels left for the kernel: 0 (records are complete squares), 1, 2, 5
    n = 6
    steps = len(D.dls_plan(n)[0])
    d = steps - back
    recs = D.dls_split(n, d)
    counts, total, nodes = _gpu(n, False, recs, d)
    want, want_nodes = _oracle_per_prefix(n, False, recs, d)
    assert (counts == want).all() and nodes == want_nodes
    assert total == oracle.count_all(n)


def test_ragged_prefix_counts_not_multiple_of_warp():
    n = 7
    d = D.default_split_depth(n)
    recs = D.dls_split(n, d)[:1001]
    counts, total, _ = _gpu(n, False, recs, d)
    want, _ = _oracle_per_prefix(n, False, recs, d)
    assert (counts == want).all()


def test_inconsistent_prefix_is_reported():
    n = 7
    d = D.default_split_depth(n)
    recs = D.dls_split(n, d)[:64].copy()
    recs[5, 1, 1] = recs[5, 0, 1]     # value repeated in column 1
    with pytest.raises(D.DlsError) as e:
        D.count_prefixes(n, recs, depth=d)
    assert e.value.code == B.DLS_E_PREFIX


def test_depth_below_diagonals_rejected():
    n = 8
    recs = D.dls_split(n, 5)
    with pytest.raises(D.DlsError) as e:
        D.dls_count(n, 5, recs)
    assert e.value.code == B.DLS_E_ARG


def test_device_buffers_and_async_stats():
    import torch
    n = 7
    d = D.default_split_depth(n)
    recs = D.dls_split(n, d)
    dev = torch.from_numpy(recs).cuda()
    out = torch.zeros(len(recs), dtype=torch.int64, device="cuda")
    stats = torch.zeros(B.DLS_STATS_WORDS, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    D.dls_count_async(n, d, dev, out, stats, stream=s.cuda_stream)
    torch.cuda.synchronize()
    want = oracle.count_all(n)
    assert int(stats[0]) == want and int(out.sum()) == want and int(stats[2]) == 0
    total, _ = D.dls_count(n, d, dev, out_counts=out, stream=s.cuda_stream)
    assert total == want and int(out.sum()) == want


def test_concurrent_streams_and_threads():
    """Calls on different streams / from different host threads at once: the
    search kernel is a cooperative launch (every warp of the grid must be resident
    for its exit protocol), so concurrent launches run one after the other instead
    of dead-locking, and every call returns the oracle's count."""
    import threading
    import torch
    want7, want6 = oracle.count_all(7), oracle.count_all(6, vs=True)
    d7, d6 = D.default_split_depth(7), D.default_split_depth(6, True)
    dev7 = torch.from_numpy(D.dls_split(7, d7)).cuda()
    dev6 = torch.from_numpy(D.dls_split(6, d6, True)).cuda()
    streams = [torch.cuda.Stream() for _ in range(4)]
    stats = [torch.zeros(B.DLS_STATS_WORDS, dtype=torch.int64, device="cuda") for _ in range(4)]
    torch.cuda.synchronize()
    for rep in range(3):
        for k, s in enumerate(streams):
            if k % 2 == 0:
                D.dls_count_async(7, d7, dev7, None, stats[k], stream=s.cuda_stream)
            else:
                D.dls_count_async(6, d6, dev6, None, stats[k], True, stream=s.cuda_stream)
        torch.cuda.synchronize()
        for k in range(4):
            assert int(stats[k][0]) == (want7 if k % 2 == 0 else want6) and int(stats[k][2]) == 0
    got = {}

    def work(k):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        if k % 2 == 0:
            got[k] = D.dls_count(7, d7, dev7, stream=s.cuda_stream)[0]
        else:
            got[k] = D.dls_count(6, d6, dev6, True, stream=s.cuda_stream)[0]

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert got == {0: want7, 1: want6, 2: want7, 3: want6}


def test_repeatable():
    n = 8
    d = D.default_split_depth(n)
    recs = D.dls_split(n, d)[:20000]
    a = _gpu(n, False, recs, d)
    b = _gpu(n, False, recs, d)
    assert (a[0] == b[0]).all() and a[1:] == b[1:]


@pytest.mark.parametrize("n,vs,k,reps", [(8, False, 1, 12), (8, False, 4, 8), (8, True, 6, 8)])
def test_pool_stress_repeated_launches(n, vs, k, reps):
    """The device-wide pool under contention: the k largest of 40 seeded
    workunits (no host refinement) spread over all 148 x 1024 lanes, launched
    `reps` times on one stream.  Every launch must give the oracle's
    per-workunit counts and node total; a torn or lost donated subtree would
    show as a count or node difference."""
    import torch
    d = D.default_split_depth(n, vs)
    recs = D.dls_split(n, d, vs)
    rng = np.random.default_rng(100 + n + vs)
    pool = np.ascontiguousarray(recs[rng.choice(len(recs), 40, replace=False)])
    sizes = [_oracle_per_prefix(n, vs, pool[i:i + 1], d)[1] for i in range(len(pool))]
    recs = np.ascontiguousarray(pool[np.argsort(sizes)[::-1][:k]])
    want, want_nodes = _oracle_per_prefix(n, vs, recs, d)
    dev = torch.from_numpy(recs).cuda()
    s = torch.cuda.current_stream().cuda_stream
    outs = [torch.zeros(k, dtype=torch.int64, device="cuda") for _ in range(reps)]
    stats = [torch.zeros(B.DLS_STATS_WORDS, dtype=torch.int64, device="cuda") for _ in range(reps)]
    for o, st in zip(outs, stats):
        D.dls_count_async(n, d, dev, o, st, vs, stream=s)
    torch.cuda.synchronize()
    donated = 0
    for o, st in zip(outs, stats):
        st = st.cpu().tolist()
        assert (o.cpu().numpy().astype(np.uint64) == want).all()
        assert st[2] == 0 and st[0] == int(want.sum()) and st[1] == want_nodes
        donated += st[4]
    assert donated > 0                       # the pool / donation path really ran


@pytest.mark.parametrize("n,vs,k", [(7, False, 3), (8, False, 2), (8, True, 5), (10, True, 1), (9, False, 2)])
def test_few_workunits_spread_by_device_pool(n, vs, k):
    """dls_count_async does no host refinement: k workunits start on k lanes and
    reach the rest of the GPU only through warp donation and the device-wide pool."""
    import torch
    d = D.default_split_depth(n, vs)
    if n >= 9:
        recs = synth.diagonal_prefixes(synth.SEED_VS10 if vs else synth.SEED_DLS9, n, 3, vs=vs)
        recs = recs[:k]
        # deepen (VS10: one row; DLS9: two rows) so the oracle finishes in seconds
        extra = 6 if vs else 14
        order = oracle.plan(n, vs)
        kids = oracle.prefixes(n, vs, synth.to_int_grid(recs[0]), order[d:], extra)
        recs = np.where(kids[:k] < 0, 255, kids[:k]).astype(np.uint8)
        d += extra
    else:
        recs = D.dls_split(n, d, vs)
        rng = np.random.default_rng(n)
        recs = recs[rng.choice(len(recs), k, replace=False)]
    dev = torch.from_numpy(np.ascontiguousarray(recs)).cuda()
    out = torch.zeros(k, dtype=torch.int64, device="cuda")
    stats = torch.zeros(B.DLS_STATS_WORDS, dtype=torch.int64, device="cuda")
    D.dls_count_async(n, d, dev, out, stats, vs, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    want, want_nodes = _oracle_per_prefix(n, vs, recs, d)
    assert (out.cpu().numpy().astype(np.uint64) == want).all()
    st = stats.cpu().tolist()
    assert st[2] == 0 and st[0] == int(want.sum()) and st[1] == want_nodes


@pytest.mark.parametrize("n,vs,fixed", [(4, False, True), (5, False, True), (6, False, True), (5, False, False),
                                        (4, True, True), (6, True, True), (6, True, False)])
def test_emit_squares_equal_oracle(n, vs, fixed):
    """The compact emit of squares (north_star (4)): the very same squares as the oracle."""
    import torch
    d = D.default_split_depth(n, vs, fixed)
    recs = torch.from_numpy(D.dls_split(n, d, vs, fixed)).cuda()
    want = oracle.squares(n, vs, oracle.first_row_grid(n) if fixed else oracle.empty_grid(n))
    total = D.dls_emit(n, d, recs, None, vs, fixed)                      # count only
    assert total == len(want)
    out = torch.zeros((total + 5, n, n), dtype=torch.uint8, device="cuda")
    assert D.dls_emit(n, d, recs, out, vs, fixed) == total
    got = out[:total].cpu().numpy().astype(np.int64)
    key = lambda a: sorted(tuple(x.reshape(-1).tolist()) for x in a)
    assert key(got) == key(want)
    for sq in got:
        assert oracle.is_diagonal(sq) and (not vs or oracle.is_vertically_symmetric(sq))
    small = torch.zeros((3, n, n), dtype=torch.uint8, device="cuda")
    assert D.dls_emit(n, d, recs, small, vs, fixed) == total               # capacity < total


@pytest.mark.parametrize("n,vs,k", [(7, False, 21), (8, False, 26), (8, True, 24), (6, False, 20), (9, False, 22), (10, False, 20)])
def test_count_cells_row_major_vs_oracle(n, vs, k):
    """N_n^k: consistent assignments of the first k row-major cells, row 0 fixed."""
    g = oracle.first_row_grid(n)
    cells = [c for c in range(n, k) if not vs or 2 * (c % n) <= n - 1]
    want = oracle.count_prefixes(n, vs, g, cells, len(cells))
    got, _ = D.dls_count_cells(n, np.where(g < 0, 255, g).astype(np.uint8), cells, vs)
    assert got == want


@pytest.mark.parametrize("k,key", [(30, "dls10_k30_prefixes"), (32, "dls10_k32_prefixes")])
def test_count_cells_dls10_paper(k, key):
    """N_10^30 = 284 086 571 712 and N_10^32 = 12 611 543 636 160."""
    n = 10
    g = oracle.first_row_grid(n)
    got, _ = D.dls_count_cells(n, np.where(g < 0, 255, g).astype(np.uint8), list(range(n, k)))
    assert got == paper_counts()[key]


def test_monte_carlo_estimate_small_order():
    """Section 5.3 on the GPU for N = 7, k = 14: the Knuth estimate of the number of
    DLS with row 0 fixed is within 4 standard errors of the exact count."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("mc", __import__("conftest").ROOT + "/scripts/mc_estimate.py")
    mc = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mc)
    r = mc.estimate(7, 14, 600, 3)
    exact = oracle.count_all(7)
    assert abs(r["knuth"] - exact) < 4 * r["knuth_se"]
    assert r["N_k"] == oracle.count_prefixes(7, False, oracle.first_row_grid(7), list(range(7, 14)), 7)


# ------------------------------------------------------------------ two-row closure

@pytest.mark.parametrize("n,vs,fixed", [(5, False, True), (6, False, False), (7, False, True), (4, True, True),
                                        (6, True, True), (8, True, True), (6, True, False)])
def test_closure_equals_plain_search(n, vs, fixed):
    """The closure kernel and the plain search (DLS_CLOSE=0) give the same
    per-prefix counts; each one's nodes are the oracle's nodes of the levels it
    searches (truncated tree / full tree)."""
    d = D.default_split_depth(n, vs, fixed)
    recs = D.dls_split(n, d, vs, fixed)
    want, want_nodes = _oracle_per_prefix(n, vs, recs, d, fixed)
    c1, t1, nd1 = _gpu(n, vs, recs, d, fixed)
    with closure_off():
        c0, t0, nd0 = _gpu(n, vs, recs, d, fixed)
        levels_full = D.dls_search_levels(n, d, vs, fixed)
    assert (c1 == want).all() and (c0 == want).all()
    assert nd1 == want_nodes
    pre = np.zeros((n, n), np.int32)
    if fixed:
        pre[0, :] = 1
    order = oracle.plan(n, vs, pre)[d:]
    assert levels_full == len(order)
    full = sum(oracle.count(n, vs, synth.to_int_grid(r), order)[1] for r in recs)
    assert nd0 == full and nd1 <= full


def test_closure_dls8_sample_and_nodes():
    """DLS8 workunits: closure counts = oracle counts; nodes = the oracle's nodes
    of levels 1..30 (the plan's rows 3/4 tail, 12 cells, is closed in form)."""
    n, d = 8, D.default_split_depth(8)
    assert D.dls_search_levels(n, d) == 30 and len(D.dls_plan(n)[0]) - d == 42
    recs = D.dls_split(n, d)
    rng = np.random.default_rng(30)
    recs = recs[rng.choice(len(recs), 40, replace=False)]
    counts, _, nodes = _gpu(n, False, recs, d)
    want, want_nodes = _oracle_per_prefix(n, False, recs, d)
    assert (counts == want).all() and nodes == want_nodes


def test_closure_event_count_in_stats():
    """stats[8] = two-row states counted in closed form = the oracle's number of
    consistent partial squares at the closure level (every one is an event)."""
    import torch
    n, vs = 7, False
    d = D.default_split_depth(n, vs)
    recs = D.dls_split(n, d, vs)
    levels = D.dls_search_levels(n, d, vs)
    order = oracle.plan(n, vs)[d:]
    assert levels < len(order)
    want = sum(oracle.count_levels(n, vs, synth.to_int_grid(r), order)[1][levels - 1] for r in recs)
    dev = torch.from_numpy(recs).cuda()
    stats = torch.zeros(B.DLS_STATS_WORDS, dtype=torch.int64, device="cuda")
    D.dls_count_async(n, d, dev, None, stats, vs, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    st = stats.cpu().tolist()
    assert st[8] == want and st[0] == oracle.count_all(n)


def _children(tag, n):
    idx, recs, cnt, nodes, nodes2 = [], [], [], [], []
    extra = None
    for line in open(golden("children_%s.txt" % tag)):
        if line.startswith("#"):
            if "random descent of" in line:
                extra = int(line.split("random descent of")[1].split()[0])
            continue
        i, r, c, nd, nd2 = line.split()
        idx.append(int(i))
        recs.append([255 if ch == "." else int(ch) for ch in r])
        cnt.append(int(c))
        nodes.append(int(nd))
        nodes2.append(int(nd2))
    return idx, np.array(recs, np.uint8).reshape(-1, n, n), np.array(cnt, np.uint64), sum(nodes), sum(nodes2), extra


@pytest.mark.parametrize("tag,n,vs,seed,count", [("vs10", 10, True, synth.SEED_VS10, synth.N_VS10),
                                                 ("dls9", 9, False, synth.SEED_DLS9, synth.N_DLS9)])
def test_every_seeded_prefix_has_an_oracle_checked_child(tag, n, vs, seed, count):
    """Configs 4/5: for EVERY one of the seeded prefixes, one seeded-random child
    (scripts/make_golden_children.py, oracle only) -- the GPU count of each child
    equals the oracle's; nodes equal the oracle's two-row-level nodes (closure on)
    and its full-tree nodes (closure off); each child extends its seeded prefix."""
    idx, kids, want, nodes_full, nodes_two, extra = _children(tag, n)
    assert idx == list(range(count))
    pre = synth.diagonal_prefixes(seed, n, count, vs=vs)
    given = pre != 255
    assert (kids[given] == pre[given]).all()
    d = D.default_split_depth(n, vs) + extra
    counts, total, nodes = _gpu(n, vs, kids, d)
    assert (counts == want).all()
    assert nodes == nodes_two
    with closure_off():
        counts0, _, nodes0 = _gpu(n, vs, kids, d)
    assert (counts0 == want).all() and nodes0 == nodes_full
