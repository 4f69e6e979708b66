"""The two-row closure (reading R15), CPU only.

1. Where it applies: dls_search_levels (host C++ in libdls_b200.so) must report
   the first level after which exactly two rows have empty cells, in the same
   columns and on neither diagonal -- recomputed here from the oracle's plan.
2. What it computes: at such a state the completions are the solutions of
   XOR_{j in J} x_j e_j = t over GF(2) (e_j: the two values column j misses;
   t: the values row r1 misses XOR the lower value of every e_j; vertical
   symmetry: the same over value pairs).  The count written out here by brute
   force over all 2^|J| choices must equal the oracle's count of completions
   (oracle.count, a plain recursion over the remaining cells), on every record
   below randomly chosen ancestors, zero counts included.
"""
import functools

import numpy as np
import pytest

import oracle
import paper_1709_02599_b200 as D


def _pre(n, fixed):
    pre = np.zeros((n, n), np.int32)
    if fixed:
        pre[0, :] = 1
    return pre


def _word(n, i, r1=None, r2=None):
    """Mask word of row i in the kernel's layouts 3 (n = 9) / 4 (n = 10).  With a
    closure, row r1 trades places with the first row of word 2 other than r2
    (unless r1 is in word 2 already), so that the event store always takes word 2."""
    first = 6 if n == 9 else 7
    if r1 is not None and r1 < first:
        b = first + 1 if first == r2 else first
        i = b if i == r1 else (r1 if i == b else i)
    return i // 3 if n == 9 else (3 if i == 0 else (i - 1) // 3)


def closure_level(n, vs, order, depth, fixed=True, walk=False):
    """(l, r1, forced): l >= 1 is the first level after which only two rows r1 < r2
    have empty cells, with equal empty columns and no empty diagonal cell, moved
    back over up to two forced cells (DLS only) -- cells outside rows r1, r2 whose
    row or column has every other cell assigned before them (n = 9, 10: in row
    r1's mask word) -- which the closure assigns itself; None if there is none
    (or the condition already holds at l = 0)."""
    pre = _pre(n, fixed)
    empty = np.ones((n, n), bool)
    empty[pre == 1] = False

    def take(e, c):
        i, j = divmod(c, n)
        e[i, j] = False
        if vs:
            e[i, n - 1 - j] = False

    for c in order[:depth]:
        take(empty, c)
    for l in range(0, len(order) - depth + 1):
        if l:
            take(empty, order[depth + l - 1])
        rows = [i for i in range(n) if empty[i].any()]
        if len(rows) != 2:
            continue
        r1, r2 = rows
        if (empty[r1] != empty[r2]).any():
            continue
        if any(empty[r, j] and (r == j or r + j == n - 1) for r in rows for j in range(n)):
            continue
        if l == 0:
            return None
        forced = []
        while walk and len(forced) < 2 and l - 1 >= 1 and not vs:
            i, j = divmod(order[depth + l - 1], n)
            if i in (r1, r2) or (n >= 9 and _word(n, i, r1, r2) != _word(n, r1, r1, r2)):
                break
            before = np.ones((n, n), bool)          # still empty before level l
            before[pre == 1] = False
            for c in order[:depth + l - 1]:
                take(before, c)
            row_full = sum(not before[i, k] for k in range(n) if k != j) == n - 1
            col_full = sum(not before[k, j] for k in range(n) if k != i) == n - 1
            if not (row_full or col_full):
                break
            forced.insert(0, order[depth + l - 1])
            l -= 1
        return l, r1, forced
    return None


@pytest.mark.parametrize("n", range(3, 11))
@pytest.mark.parametrize("vs", [False, True])
@pytest.mark.parametrize("fixed", [True, False])
@pytest.mark.parametrize("walk", [False, True])
def test_search_levels_is_first_two_row_level(n, vs, fixed, walk, monkeypatch):
    if walk:
        monkeypatch.setenv("DLS_CLOSE_FORCED", "1")
    if vs and n % 2:
        return
    order = oracle.plan(n, vs, _pre(n, fixed))
    dd = D.default_split_depth(n, vs, fixed)
    for depth in sorted({dd, dd + 1, dd + 3, len(order) - 6, len(order) - 2}):
        if depth < dd or depth > len(order):
            continue
        got = D.dls_search_levels(n, depth, vs, fixed)
        want = closure_level(n, vs, order, depth, fixed, walk)
        # the closure is used when the open columns fit the kernel's column list
        # (<= n-2 DLS / n/2-1 VS: always true here) and is not the whole row
        assert got == (want[0] if want else len(order) - depth), (depth, got, want)
    if n == 8 and not vs and fixed:
        # rows 3/4 closed after level 30; with the walk-back (7,6) is forced too
        assert D.dls_search_levels(n, dd, vs, fixed) == (29 if walk else 30)


def gf2_count(n, vs, g, r1, forced=()):
    """Completions of a two-row state by the GF(2) formula, brute force over x,
    after assigning the forced cells (their one candidate; none -> 0)."""
    g = np.array(g)
    for c in forced:
        i, j = divmod(c, n)
        cand = [v for v in range(n) if v not in set(g[i].tolist()) | set(g[:, j].tolist())]
        if not cand:
            return 0
        assert len(cand) == 1
        g[i, j] = cand[0]
    cols = [j for j in range(n) if g[r1, j] == -1 and (not vs or 2 * j < n - 1)]
    pair = (lambda v: 1 << min(v, n - 1 - v)) if vs else (lambda v: 1 << v)
    x, es = 0, []
    for j in cols:
        miss = [v for v in range(n) if v not in set(g[:, j].tolist())]
        assert len(miss) == 2
        es.append(pair(miss[0]) ^ pair(miss[1]) if vs else pair(miss[0]) | pair(miss[1]))
        x ^= pair(min(miss))
    m1 = 0
    for v in range(n):
        if v not in set(g[r1].tolist()):
            m1 |= pair(v)
    t = m1 ^ x
    sums = [functools.reduce(lambda a, k: a ^ (es[k] if m >> k & 1 else 0), range(len(es)), 0)
            for m in range(1 << len(es))]
    return sum(1 for s in sums if s == t)


@pytest.mark.parametrize("walk", [False, True])
@pytest.mark.parametrize("n,vs,k,back", [(5, False, 30, 6), (6, False, 30, 8), (7, False, 25, 10), (8, False, 12, 10),
                                         (4, True, 10, 3), (6, True, 20, 6), (8, True, 15, 8), (10, True, 6, 8),
                                         (9, False, 12, 9)])
def test_gf2_closure_equals_oracle_count(n, vs, k, back, walk):
    g0 = oracle.first_row_grid(n)
    order = oracle.plan(n, vs)
    lc, r1, forced = closure_level(n, vs, order, 0, walk=walk)
    rng = np.random.default_rng(n * 10 + vs)
    d0 = max(lc - back, 0)
    base = oracle.prefixes(n, vs, g0, order, min(d0, 12), cap=20000)
    checked = zeros = 0
    for _ in range(k):
        for _try in range(200):          # random descent to depth d0 (restart on dead ends)
            g = base[rng.integers(len(base))]
            for l in range(min(d0, 12), d0):
                kids = oracle.prefixes(n, vs, g, order[l:], 1, cap=64)
                if len(kids) == 0:
                    break
                g = kids[rng.integers(len(kids))]
            else:
                break
        for rec in oracle.prefixes(n, vs, g, order[d0:], lc - d0, cap=2000):
            want = oracle.count(n, vs, rec, order[lc:])[0]
            assert gf2_count(n, vs, rec, r1, forced) == want
            checked += 1
            zeros += want == 0
    assert checked >= 1
    if not vs and n == 7:
        assert zeros > 0          # the "no completion" outcome (t outside the span) is exercised
