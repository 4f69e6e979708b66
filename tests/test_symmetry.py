"""Symmetry breaking with hourglass designs (Section 4).

CPU: pins of the oracle's M-transformations and canonisation (Alg. 5): the
class count 116 857 of P:436, classes partition the hourglasses, class sizes are
orbit sizes (divide the group order), Proposition 1 (equal completion counts
inside a class), Corollary 1 / Alg. 6 (weighted sum = plain count).
GPU: dls_canonize and dls_count_sb against the oracle and the paper's counts.
"""
import math

import numpy as np
import pytest

import oracle
import synth
import paper_1709_02599_b200 as D
from conftest import paper_counts


@pytest.mark.parametrize("n", [4, 5, 6, 7])
def test_classes_partition_hourglasses(n):
    reps, mult, nh = oracle.hourglass_classes(n)
    assert nh == len(oracle.hourglasses(n))
    assert int(mult.sum()) == nh                      # every design in exactly one class
    g = oracle.group_size(n)
    assert all(g % int(m) == 0 for m in mult)         # orbit sizes divide |G|


def test_group_orders_from_paper():
    # Alg. 5 loops: 2 x 2^h x (h-1)!  -> 192 for N = 8, 9 ("at most 192")
    assert oracle.group_size(8) == 192 and oracle.group_size(9) == 192
    assert oracle.group_size(10, vs=True) == 768      # P:524 "2^5 x 4! = 768"
    # full classes of DLS have at most 4 * 2^h * h! members
    assert 4 * 2 ** 4 * math.factorial(4) == 1536     # N = 9
    assert 4 * 2 ** 5 * math.factorial(5) == 15360    # N = 10


def test_fig2_vertical_mirror():
    """Fig. 2: the right design is the vertical mirror of the left one
    (before renaming row 0), i.e. our transform with mirror only, up
    to the renaming of P:312."""
    left = np.array([[0, 1, 2, 3, 4, 5, 6, 7, 8, 9],
                     [-1, 4, -1, -1, -1, -1, -1, -1, 6, -1],
                     [-1, -1, 1, -1, -1, -1, -1, 3, -1, -1],
                     [-1, -1, -1, 6, -1, -1, 7, -1, -1, -1],
                     [-1, -1, -1, -1, 7, 1, -1, -1, -1, -1],
                     [-1, -1, -1, -1, 2, 8, -1, -1, -1, -1],
                     [-1, -1, -1, 8, -1, -1, 2, -1, -1, -1],
                     [-1, -1, 0, -1, -1, -1, -1, 9, -1, -1],
                     [-1, 5, -1, -1, -1, -1, -1, -1, 3, -1],
                     [4, 2, 3, 1, 8, 6, 9, 0, 7, 5]])
    right = np.array([[9, 8, 7, 6, 5, 4, 3, 2, 1, 0],
                      [-1, 6, -1, -1, -1, -1, -1, -1, 4, -1],
                      [-1, -1, 3, -1, -1, -1, -1, 1, -1, -1],
                      [-1, -1, -1, 7, -1, -1, 6, -1, -1, -1],
                      [-1, -1, -1, -1, 1, 7, -1, -1, -1, -1],
                      [-1, -1, -1, -1, 8, 2, -1, -1, -1, -1],
                      [-1, -1, -1, 2, -1, -1, 8, -1, -1, -1],
                      [-1, -1, 9, -1, -1, -1, -1, 0, -1, -1],
                      [-1, 3, -1, -1, -1, -1, -1, -1, 5, -1],
                      [5, 7, 0, 9, 6, 8, 1, 3, 2, 4]])
    n = 10
    img = oracle.transform(n, left, list(range(n // 2)), 0, True)
    # renaming right's row 0 to 0..9 gives the same design
    ren = {int(v): j for j, v in enumerate(right[0])}
    right_norm = np.where(right < 0, -1, np.vectorize(lambda v: ren.get(int(v), -1))(right))
    assert (img == right_norm).all()


@pytest.mark.parametrize("n", [5, 6, 7])
def test_proposition1_equal_counts_in_a_class(n):
    """designs related by an M-transformation have equally many completions."""
    rng = np.random.default_rng(n)
    reps, mult, _ = oracle.hourglass_classes(n)
    h = n // 2
    for r in reps[rng.choice(len(reps), min(6, len(reps)), replace=False)]:
        c0 = oracle.count(n, False, r)[0]
        for _ in range(4):
            pi = [0] + list(1 + rng.permutation(h - 1))
            img = oracle.transform(n, r, pi, int(rng.integers(1 << h)), bool(rng.integers(2)))
            assert oracle.count(n, False, img)[0] == c0


@pytest.mark.parametrize("n,vs", [(5, False), (6, False), (7, False), (4, True), (6, True)])
def test_corollary1_weighted_sum(n, vs):
    """Alg. 6: sum over canonic designs of count x class size = plain count."""
    reps, mult, _ = oracle.hourglass_classes(n, vs)
    total = sum(oracle.count(n, vs, r)[0] * int(m) for r, m in zip(reps, mult))
    assert total == oracle.count_all(n, vs)


def test_hourglass_classes_order8_paper():
    """"we still need to store about 100 000 (116 857) classes representatives"."""
    k, _, nh = oracle.hourglass_classes(8, keep=False)
    assert nh == paper_counts()["hourglass8"]
    assert k == paper_counts()["hourglass8_classes"]


# ------------------------------------------------------------------ GPU

def _rec(a):
    return np.where(np.asarray(a) < 0, 255, a).astype(np.uint8)


@pytest.mark.gpu
@pytest.mark.parametrize("n,vs", [(4, False), (5, False), (6, False), (7, False), (4, True), (6, True), (8, True)])
def test_gpu_canonize_all_hourglasses(n, vs):
    H = oracle.hourglasses(n, vs)
    got = D.dls_canonize(n, _rec(H), vs)
    want = np.array([oracle.canonize(n, vs, h) for h in H])
    assert (got.astype(np.int64) == want).all()


@pytest.mark.gpu
@pytest.mark.parametrize("n,vs,k", [(8, False, 3000), (9, False, 1500), (10, True, 1500)])
def test_gpu_canonize_sampled(n, vs, k):
    # hourglasses below seeded diagonal workunits: canonic and non-canonic mixed
    rng = np.random.default_rng(n)
    order = oracle.hourglass_cells(n)
    if vs:
        order = [c for c in order if 2 * (c % n) <= n - 1]
    recs = synth.diagonal_prefixes(7, n, 40, vs=vs)
    H = []
    for r in recs:
        g = synth.to_int_grid(r)
        last = [c for c in order if c // n == n - 1 and g.reshape(-1)[c] < 0]
        H.extend(oracle.prefixes(n, vs, g, last, len(last)))
    H = np.array(H)[rng.permutation(len(H))[:k]]
    got = D.dls_canonize(n, _rec(H), vs)
    want = np.array([oracle.canonize(n, vs, h) for h in H])
    assert (got.astype(np.int64) == want).all()
    # include the canonic forms of some classes
    reps = []
    for h in H[:50]:
        pi = list(range(n // 2))
        best = h
        for m in (False, True) if not vs else (False,):
            for s in range(1 << (n // 2)):
                img = oracle.transform(n, h, pi, s, m)
                if tuple(img.reshape(-1)) < tuple(best.reshape(-1)):
                    best = img
        reps.append(best)
    got = D.dls_canonize(n, _rec(np.array(reps)), vs)
    want = np.array([oracle.canonize(n, vs, h) for h in reps])
    assert (got.astype(np.int64) == want).all()


@pytest.mark.gpu
@pytest.mark.parametrize("n,vs", [(4, False), (5, False), (6, False), (7, False), (4, True), (6, True), (8, True)])
def test_gpu_count_sb_matches_oracle(n, vs):
    r = D.dls_count_sb(n, vs)
    assert r["count"] == oracle.count_all(n, vs)
    reps, mult, nh = oracle.hourglass_classes(n, vs)
    assert r["hourglasses"] == nh and r["classes"] == len(reps)


@pytest.mark.gpu
def test_gpu_count_sb_order8_paper():
    r = D.dls_count_sb(8)
    assert r["count"] == paper_counts()["dls8_first_row_fixed"]
    assert r["hourglasses"] == paper_counts()["hourglass8"]
    assert r["classes"] == paper_counts()["hourglass8_classes"]


@pytest.mark.gpu
def test_gpu_count_sb_vs10_paper():
    """82 731 715 264 512 vertically symmetric DLS of order 10 (row 0 fixed)."""
    r = D.dls_count_sb(10, True)
    assert r["count"] == paper_counts()["vsdls10_first_row_fixed"]


@pytest.mark.gpu
def test_gpu_count_sb_ranges_add_up():
    n = 7
    full = D.dls_count_sb(n)
    total = D.load().dls_split(n, 0, 1, D.default_split_depth(n), None, 0)
    cuts = [0, 5, total // 3, total - 1, total]
    parts = [D.dls_count_sb_range(n, a, b) for a, b in zip(cuts[:-1], cuts[1:])]
    for key in ("count", "hourglasses", "classes"):
        assert sum(p[key] for p in parts) == full[key]


@pytest.mark.gpu
@pytest.mark.parametrize("n,vs,world,chunk", [(7, False, 3, 5), (8, False, 2, 20000), (8, True, 4, 3)])
def test_gpu_count_sb_round_robin_shards(n, vs, world, chunk):
    """The multi-GPU split of Alg. 6 (paper_1709_02599_b200.dist.shard_ranges):
    diagonal-workunit ranges dealt round-robin to `world` ranks; the ranks'
    dls_count_sb_range totals add up to dls_count_sb (run here one rank after
    the other on one GPU; the all-reduce is covered by the gloo test)."""
    from paper_1709_02599_b200.dist import shard_ranges
    full = D.dls_count_sb(n, vs)
    d = D.default_split_depth(n, vs)
    n_units = len(D.dls_split(n, d, vs))
    tot = {"count": 0, "hourglasses": 0, "classes": 0}
    for r in range(world):
        for b, e in shard_ranges(n_units, r, world, chunk):
            part = D.dls_count_sb_range(n, b, e, vs)
            for k in tot:
                tot[k] += part[k]
    assert tot == {k: full[k] for k in tot}
