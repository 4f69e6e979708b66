"""Pins for the CPU oracle (oracle/), CPU only.

Each oracle function is checked against something other than itself:
brute force over permutation-row stackings for N <= 5, the N!
first-row invariant, the vertical-symmetry definition
checked square by square, Fig. 1 and the hourglass count of P:436.
"""
import math

import numpy as np
import pytest

import oracle
from conftest import golden, paper_counts


def fig1():
    rows = []
    with open(golden("fig1_dls9_order.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append([int(x) for x in line.split()])
    return np.array(rows)


# ------------------------------------------------------------------ definitions

def test_definitions_on_hand_examples():
    # a DLS of order 4 with row 0 = 0123, checked by hand
    sq = np.array([[0, 1, 2, 3], [2, 3, 0, 1], [3, 2, 1, 0], [1, 0, 3, 2]])
    assert oracle.is_latin(sq) and oracle.is_diagonal(sq)
    # rows are vertically symmetric: 0+3 = 1+2 = 3 etc.
    assert oracle.is_vertically_symmetric(sq)
    bad = sq.copy()
    bad[1], bad[2] = sq[2].copy(), sq[1].copy()      # still Latin, breaks main diagonal
    assert oracle.is_latin(bad) and not oracle.is_diagonal(bad)
    cyc = np.array([[(i + j) % 4 for j in range(4)] for i in range(4)])
    assert oracle.is_latin(cyc) and not oracle.is_diagonal(cyc)


def test_brute_force_latin_counts():
    # the brute force itself: Latin squares (no diagonal filter) of orders 1..5
    # are 1, 2, 12, 576, 161280 in total; with row 0 fixed divide by N!.
    for n, total in ((1, 1), (2, 2), (3, 12), (4, 576)):
        assert oracle.brute_force_count(n, diagonal=False, fixed_first_row=False) == total
    assert oracle.brute_force_count(5, diagonal=False, fixed_first_row=True) == 161280 // 120


# ------------------------------------------------------------------ plan (Section 2.3)

def test_plan_reproduces_fig1():
    n = 9
    order = oracle.plan(n)
    got = np.zeros((n, n), dtype=int)
    for step, cell in enumerate(order):
        got[cell // n, cell % n] = step + 1
    assert (got[1:] == fig1()).all()


@pytest.mark.parametrize("n", range(1, 11))
@pytest.mark.parametrize("fixed", [True, False])
def test_plan_is_permutation_of_free_cells(n, fixed):
    pre = np.zeros((n, n), dtype=np.int32)
    if fixed:
        pre[0, :] = 1
    order = oracle.plan(n, False, pre)
    assert sorted(order) == [c for c in range(n * n) if not pre.reshape(-1)[c]]


@pytest.mark.parametrize("n", [4, 6, 8, 10])
def test_vs_plan_covers_left_half(n):
    order = oracle.plan(n, True)
    assert sorted(order) == [i * n + j for i in range(1, n) for j in range(n // 2)]


@pytest.mark.parametrize("n", range(5, 11))
def test_plan_puts_diagonals_first(n):
    # P:174 "we start with diagonal elements, and then fill the rest"
    order = oracle.plan(n)
    diag = {i * n + j for i in range(1, n) for j in range(n) if i == j or i + j == n - 1}
    assert set(order[:len(diag)]) == diag


def _units_of(n, i, j):
    """The uniqueness units through cell (i, j): row, column, and the
    main diagonal / antidiagonal when the cell lies on them."""
    out = [[(i, k) for k in range(n)], [(k, j) for k in range(n)]]
    if i == j:
        out.append([(k, k) for k in range(n)])
    if i + j == n - 1:
        out.append([(k, n - 1 - k) for k in range(n)])
    return out


def _all_units(n):
    """Rows 0..N-1, columns 0..N-1, main diagonal, antidiagonal (R5 scan order)."""
    return ([[(i, k) for k in range(n)] for i in range(n)] + [[(k, j) for k in range(n)] for j in range(n)]
            + [[(k, k) for k in range(n)], [(k, n - 1 - k) for k in range(n)]])


@pytest.mark.parametrize("n", [4, 6, 8, 10])
@pytest.mark.parametrize("fixed", [True, False])
def test_vs_plan_replay_against_section_2_3(n, fixed):
    """Pin of the vertically symmetric plan (reading R4) by replaying it on a
    board, checked against the text of Section 2.3 rather than the planner:
      * every step takes a left-half cell ("fill only the left half") that
        is still empty together with its mirror, and marks both;
      * forced rule: when some unit has exactly N-1 assigned cells, the
        step takes that unit's remaining cell (or its mirror), the first such
        unit in the R5 scan order;
      * otherwise the step takes a left-half cell of the largest
        V = r_i + c_j + md(i,j) + ad(i,j), the first in lexicographic order;
      * with the first row fixed and N >= 6 the left-half diagonal cells come
        first (for N = 4 the V rule itself interleaves row cells), and
        the plan ends with every cell assigned."""
    order = oracle.plan(n, True, _pre_rows(n, fixed))
    a = np.zeros((n, n), dtype=int)
    if fixed:
        a[0, :] = 1
    ndiag = sum(1 for i in range(n) for j in range(n // 2) if (i == j or i + j == n - 1) and not a[i, j])
    for step, cell in enumerate(order):
        i, j = divmod(cell, n)
        m = n - 1 - j
        assert 2 * j < n and not a[i, j] and not a[i, m], (step, i, j)
        forced = None
        for u in _all_units(n):
            if sum(a[p] for p in u) == n - 1:
                forced = next(p for p in u if not a[p])
                break
        if forced is not None:
            assert forced in ((i, j), (i, m)), (step, forced, (i, j))
        else:
            def v(ii, jj):
                return sum(sum(a[p] for p in u) for u in _units_of(n, ii, jj))
            free = [(ii, jj) for ii in range(n) for jj in range(n) if 2 * jj < n and not a[ii, jj]]
            best = max(v(*c) for c in free)
            assert v(i, j) == best and (i, j) == min(c for c in free if v(*c) == best), (step, (i, j))
        if fixed and n >= 6 and step < ndiag:
            assert i == j or i + j == n - 1, (step, i, j)
        a[i, j] = a[i, m] = 1
    assert a.all()


def _pre_rows(n, fixed):
    pre = np.zeros((n, n), dtype=np.int32)
    if fixed:
        pre[0, :] = 1
    return pre


@pytest.mark.parametrize("n", range(4, 11))
def test_dls_plan_replay_forced_rule(n):
    """The non-symmetric plan replayed the same way: every step where some unit
    has N-1 assigned cells takes the remaining cell of the first such unit
    (R5 scan order), every other step a cell of maximal V."""
    order = oracle.plan(n)
    a = np.zeros((n, n), dtype=int)
    a[0, :] = 1
    nforced = 0
    for cell in order:
        i, j = divmod(cell, n)
        assert not a[i, j]
        forced = next((next(p for p in u if not a[p]) for u in _all_units(n) if sum(a[p] for p in u) == n - 1), None)
        if forced is not None:
            assert forced == (i, j)
            nforced += 1
        else:
            def v(ii, jj):
                return sum(sum(a[p] for p in u) for u in _units_of(n, ii, jj))
            free = [(ii, jj) for ii in range(n) for jj in range(n) if not a[ii, jj]]
            best = max(v(*c) for c in free)
            assert v(i, j) == best and (i, j) == min(c for c in free if v(*c) == best)
        a[i, j] = 1
    # the last cell of rows 1..N-1 and of both diagonals at least (Fig. 1)
    assert nforced >= n + 1


def test_plan_forced_cells_are_forced():
    # a cell taken because its unit reached N-1 assigned cells really is
    # the last free cell of that unit at that step (replay check).
    n = 9
    order = oracle.plan(n)
    a = np.zeros((n, n), dtype=int)
    a[0, :] = 1
    forced_steps = 0
    for cell in order:
        i, j = divmod(cell, n)
        units = [a[i, :].sum(), a[:, j].sum()]
        if i == j:
            units.append(sum(a[k, k] for k in range(n)))
        if i + j == n - 1:
            units.append(sum(a[k, n - 1 - k] for k in range(n)))
        if max(units) == n - 1:
            forced_steps += 1
        a[i, j] = 1
    # Fig. 1: the last cell of each of rows 1..8 and both diagonals is forced at least
    assert forced_steps >= 10


# ------------------------------------------------------------------ counts vs brute force

@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_count_matches_brute_force_first_row_fixed(n):
    assert oracle.count_all(n, fixed_first_row=True) == oracle.brute_force_count(n, True, False, True)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_count_matches_brute_force_free(n):
    assert oracle.count_all(n, fixed_first_row=False) == oracle.brute_force_count(n, True, False, False)


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("fixed", [True, False])
def test_vs_count_matches_brute_force(n, fixed):
    assert oracle.count_all(n, vs=True, fixed_first_row=fixed) == \
        oracle.brute_force_count(n, True, True, fixed)


@pytest.mark.parametrize("n", [4, 5])
def test_squares_equal_brute_force_set(n):
    # not only the number: the very same squares
    got = oracle.squares(n, False, oracle.first_row_grid(n))
    want = oracle.brute_force_squares(n, True, False, True)
    key = lambda s: tuple(np.asarray(s).reshape(-1).tolist())
    assert sorted(map(key, got)) == sorted(map(key, want))
    assert all(oracle.is_diagonal(s) for s in got)


# ------------------------------------------------------------------ invariants

@pytest.mark.parametrize("n", [4, 5, 6])
def test_first_row_factor_is_n_factorial(n):
    # renaming symbols maps DLS to DLS bijectively, so total = N! * (row 0 fixed)
    assert oracle.count_all(n, fixed_first_row=False) == \
        math.factorial(n) * oracle.count_all(n, fixed_first_row=True)


@pytest.mark.parametrize("n", [4, 6])
def test_vs_first_row_factor(n):
    # reading R3: only renamings commuting with x -> N-1-x keep vertical symmetry
    assert oracle.count_all(n, vs=True, fixed_first_row=False) == \
        oracle.vs_first_row_multiplier(n) * oracle.count_all(n, vs=True, fixed_first_row=True)


@pytest.mark.parametrize("n", [4, 6])
def test_vs_squares_by_definition(n):
    """VS enumeration == DLS enumeration filtered by LS[i][j]+LS[i][N-1-j]=N-1."""
    g = oracle.first_row_grid(n)
    vs_sq = oracle.squares(n, True, g)
    assert len(vs_sq) == oracle.count_all(n, vs=True)
    for s in vs_sq:
        assert oracle.is_diagonal(s) and oracle.is_vertically_symmetric(s)
    all_sq = oracle.squares(n, False, g)
    filt = [s for s in all_sq if oracle.is_vertically_symmetric(s)]
    key = lambda s: tuple(np.asarray(s).reshape(-1).tolist())
    assert sorted(map(key, filt)) == sorted(map(key, vs_sq))


def test_odd_order_has_no_vs_squares():
    for n in (3, 5, 7):
        assert oracle.count_all(n, vs=True) == 0


@pytest.mark.parametrize("n,depth", [(6, 8), (7, 12), (7, 14)])
def test_prefix_additivity(n, depth):
    """Workunits partition the search: sum over all depth-k prefixes of
    their completions equals the count, and nodes add up level by level."""
    g = oracle.first_row_grid(n)
    order = oracle.plan(n)
    total, nodes = oracle.count(n, False, g, order)
    pre = oracle.prefixes(n, False, g, order, depth)
    parts = [oracle.count(n, False, p, order[depth:]) for p in pre]
    assert sum(c for c, _ in parts) == total
    upper = sum(oracle.count_prefixes(n, False, g, order, d) for d in range(1, depth + 1))
    assert upper + sum(nd for _, nd in parts) == nodes


def test_count_is_order_independent():
    # the count is a property of the partial square, not of the cell order
    n = 6
    g = oracle.first_row_grid(n)
    a = oracle.count(n, False, g)[0]
    b = oracle.count(n, False, g, [c for c in range(n, n * n)])[0]          # row-major
    c = oracle.count(n, False, g, list(reversed(range(n, n * n))))[0]
    assert a == b == c > 0


def test_inconsistent_grid_counts_zero():
    g = oracle.first_row_grid(5)
    g[1, 1] = 1          # column 1 already holds 1
    assert oracle.count(5, False, g)[0] == 0


def test_hourglass_count_order8():
    """'for diagonal Latin squares of order N=8 it is equal to 22 192 248'
    hourglass designs (row 0, row N-1 and both diagonals assigned)."""
    n = 8
    g = oracle.first_row_grid(n)
    diag = [i * n + j for i in range(1, n) for j in range(n) if i == j or i + j == n - 1]
    last = [(n - 1) * n + j for j in range(n) if (n - 1) * n + j not in diag]
    assert oracle.count_prefixes(n, False, g, diag + last, len(diag) + len(last)) == \
        paper_counts()["hourglass8"]


@pytest.mark.parametrize("n,vs,fixed", [(4, False, True), (5, False, False), (6, False, True), (6, True, True),
                                        (7, False, True)])
def test_count_levels_pins(n, vs, fixed):
    """oracle.count_levels: entry k = consistent assignments of the first k+1
    cells (= count_prefixes, an independent enumeration), the entries add up to
    count()'s nodes, and the last one is the number of completions."""
    g = oracle.first_row_grid(n) if fixed else oracle.empty_grid(n)
    order = oracle.plan_for_grid(n, vs, g)
    c, lv = oracle.count_levels(n, vs, g, order)
    cc, nodes = oracle.count(n, vs, g, order)
    assert c == cc and sum(lv) == nodes and lv[-1] == c
    for k in range(0, len(order), max(1, len(order) // 9)):
        assert lv[k] == oracle.count_prefixes(n, vs, g, order, k + 1)
