"""Host-side product logic (CPU only): the C ABI loads and exports what the header
declares; the Section 2.3 planner and the prefix splitter (both host C++ in
libdls_b200.so) agree with the oracle; the GPU entry points refuse to run
without a device (no CPU fallback)."""
import re

import numpy as np
import pytest

import oracle
import synth
import paper_1709_02599_b200 as D
from paper_1709_02599_b200 import _binding as B
from conftest import ROOT, golden
from test_oracle import fig1


def header_functions():
    src = open(ROOT + "/include/dls_b200.h").read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\s*\*?\s*(dls_[a-z_]+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    lib = D.load()
    names = header_functions()
    assert set(names) >= {"dls_plan", "dls_split", "dls_count", "dls_count_async"}
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(B.EXPORTS)
    assert "sm_100a" in D.dls_version()


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", D.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


@pytest.mark.parametrize("n", range(1, 11))
@pytest.mark.parametrize("vs", [False, True])
@pytest.mark.parametrize("fixed", [True, False])
def test_plan_matches_oracle(n, vs, fixed):
    if vs and n % 2:
        with pytest.raises(D.DlsError):
            D.dls_plan(n, vs, fixed)
        return
    cells, forced, dd = D.dls_plan(n, vs, fixed)
    pre = np.zeros((n, n), np.int32)
    if fixed:
        pre[0, :] = 1
    assert cells.tolist() == oracle.plan(n, vs, pre)
    # diag depth: the first prefix covering both diagonals
    diag = {i * n + j for i in range(n) for j in range(n) if (i == j or i + j == n - 1) and not pre[i, j]}
    covered = set()
    for c in cells[:dd]:
        i, j = divmod(int(c), n)
        covered |= {i * n + j, i * n + (n - 1 - j)} if vs else {i * n + j}
    assert diag <= covered
    if dd:
        i, j = divmod(int(cells[dd - 1]), n)
        last = {i * n + j, i * n + (n - 1 - j)} if vs else {i * n + j}
        assert last & diag


def test_plan_fig1_and_forced_flags():
    cells, forced, dd = D.dls_plan(9)
    got = np.zeros((9, 9), int)
    for s, c in enumerate(cells):
        got[c // 9, c % 9] = s + 1
    assert (got[1:] == fig1()).all()
    assert dd == 15
    # Fig. 1 step 13 (cell (8,0)) and step 15 (cell (8,8)) complete the antidiagonal
    # and the main diagonal
    assert forced[12] == 1 and forced[14] == 1 and forced[0] == 0


@pytest.mark.parametrize("n,vs,fixed,depth", [
    (4, False, True, 3), (5, False, True, 6), (6, False, True, 8), (6, False, False, 14),
    (7, False, True, 12), (8, False, True, 9), (4, True, True, 3), (6, True, True, 5),
    (8, True, True, 9), (10, True, True, 6), (9, False, True, 10)])
def test_split_equals_oracle_prefixes(n, vs, fixed, depth):
    got = D.dls_split(n, depth, vs, fixed)
    g = oracle.first_row_grid(n) if fixed else oracle.empty_grid(n)
    pre = np.zeros((n, n), np.int32)
    if fixed:
        pre[0, :] = 1
    want = oracle.prefixes(n, vs, g, oracle.plan(n, vs, pre), depth)
    # same records in the same (depth-first, increasing value) order
    assert got.shape[0] == want.shape[0]
    assert (synth.to_int_grid(got) == want).all()


def test_split_sizes_and_edges():
    assert D.dls_split(8, 14).shape == (547896, 8, 8)   # N=8 diagonal workunits
    assert D.dls_split(2, 2).shape[0] == 0               # no DLS of order 2
    assert D.dls_split(1, 0).shape == (1, 1, 1)
    assert D.dls_split(5, 0).shape == (1, 5, 5)
    with pytest.raises(D.DlsError):
        D.dls_split(8, 99)
    with pytest.raises(D.DlsError):
        D.dls_split(11, 1)
    with pytest.raises(D.DlsError):
        D.dls_split(7, 1, symmetric=True)


def test_dls9_decomposition_workunits():
    """P:481 decomposes N=9 by the first 10 Fig. 1 cells.  The paper prints
    1 225 884; the oracle (scripts/make_golden.py) finds 1 255 884 (reading R8)."""
    want = int(open(golden("dls9_k10_workunits.txt")).read().split("\n")[-2])
    lib = D.load()
    assert lib.dls_split(9, 0, 1, 10, None, 0) == want


def test_count_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    pre = D.dls_split(6, 8)
    with pytest.raises(D.DlsError) as e:
        D.dls_count(6, 8, pre)
    assert e.value.code == B.DLS_E_NODEVICE


@pytest.mark.parametrize("n,vs,extra", [(6, False, 3), (7, False, 4), (8, True, 3), (10, True, 2)])
def test_refine_equals_oracle_children(n, vs, extra):
    """dls_refine (P:481 below given records) == the oracle's enumeration of the
    next `extra` plan cells below each record, in record order."""
    d = D.default_split_depth(n, vs)
    if n == 10:
        recs = synth.diagonal_prefixes(3, n, 3, vs=True)
    else:
        recs = D.dls_split(n, d, vs)[:5]
    kids, parent = D.dls_refine(n, d, recs, d + extra, vs)
    order = oracle.plan(n, vs)
    want, want_par = [], []
    for p, r in enumerate(recs):
        k = oracle.prefixes(n, vs, synth.to_int_grid(r), order[d:], extra)
        want.extend(k)
        want_par.extend([p] * len(k))
    assert len(kids) == len(want)
    assert (synth.to_int_grid(kids) == np.array(want)).all()
    assert parent.tolist() == want_par


def test_refine_rejects_bad_records():
    n = 7
    d = D.default_split_depth(n)
    recs = D.dls_split(n, d)[:3].copy()
    recs[1, 2, 2] = recs[1, 1, 1]          # repeated value on the main diagonal
    with pytest.raises(D.DlsError) as e:
        D.dls_refine(n, d, recs, d + 2)
    assert e.value.code == B.DLS_E_PREFIX
    with pytest.raises(D.DlsError):
        D.dls_refine(n, d, recs[:1], d - 1)


def test_reference_arm_json():
    import json
    import os
    import subprocess
    import sys
    env = dict(os.environ, DLS_REF_STEP_SECONDS="0.5")
    out = subprocess.run([sys.executable, ROOT + "/bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "cpu_baseline", "e2e", "config"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"


def test_knuth_descent_unbiased_prefix_count():
    """Section 5.3 estimator, host half: E[weight] of the random descent over the
    first k row-major cells = N_n^k, checked against the oracle's exact
    count within 4 standard errors; deterministic per seed."""
    n, k = 6, 18
    g = oracle.first_row_grid(n)
    rec = np.where(g < 0, 255, g).astype(np.uint8)
    cells = list(range(n, k))
    ws = np.array([D.dls_random_prefix(n, rec, cells, s)[1] for s in range(6000)])
    exact = oracle.count_prefixes(n, False, g, cells, len(cells))
    assert abs(ws.mean() - exact) < 4 * ws.std() / np.sqrt(len(ws))
    a, wa = D.dls_random_prefix(n, rec, cells, 77)
    b, wb = D.dls_random_prefix(n, rec, cells, 77)
    assert (a == b).all() and wa == wb
    if wa > 0:
        full = synth.to_int_grid(a)
        assert oracle.count(n, False, full)[0] >= 0     # a consistent partial square


def test_cli_host_commands():
    import subprocess
    import sys
    out = subprocess.run([sys.executable, "-m", "paper_1709_02599_b200", "plan", "--n", "9"], capture_output=True,
                         text=True, cwd=ROOT)
    assert out.returncode == 0
    rows = [list(map(int, l.split())) for l in out.stdout.splitlines()[1:9]]
    assert (np.array(rows) == fig1()).all()
    out = subprocess.run([sys.executable, "-m", "paper_1709_02599_b200", "split", "--n", "8", "--depth", "14"],
                         capture_output=True, text=True, cwd=ROOT)
    assert out.stdout.strip() == "547896"


def test_binding_validates_buffers():
    """Marshalling guards (no GPU needed: they run before the C call): records must
    be uint8 (k, n, n); counts 8-byte integers with room for every record."""
    recs = np.zeros((4, 7, 7), np.uint8)
    with pytest.raises(ValueError):
        B.dls_count(7, 11, recs.astype(np.int32))
    with pytest.raises(ValueError):
        B.dls_count(7, 11, np.zeros((4, 6, 6), np.uint8))
    with pytest.raises(ValueError):
        B.dls_count(7, 11, recs, out_counts=np.zeros(4, np.int32))
    with pytest.raises(ValueError):
        B.dls_count(7, 11, recs, out_counts=np.zeros(3, np.uint64))
    with pytest.raises(ValueError):
        B.dls_emit(7, 11, recs, np.zeros((5, 49), np.int8))


@pytest.mark.parametrize("n", range(1, 11))
def test_scale_total_multipliers(n):
    """dls_scale_total: N! for DLS, (N/2)! 2^(N/2) for vertical symmetry (R3,
    pinned against the oracle's brute force in tests/test_oracle.py), 128-bit product."""
    import math
    tot, m = B.dls_scale_total(n, 12345678901234567, False)
    assert m == math.factorial(n) and tot == 12345678901234567 * math.factorial(n)
    tot, m = B.dls_scale_total(n, 987654321987, True)
    want = math.factorial(n // 2) * 2 ** (n // 2) if n % 2 == 0 else 0
    assert m == want == oracle.vs_first_row_multiplier(n) and tot == 987654321987 * want


def test_scale_total_reproduces_paper_totals():
    """5 056 994 653 507 584 x 9! = 1 835 082 219 864 832 081 920 (needs 128 bits)."""
    tot, m = B.dls_scale_total(9, 5056994653507584, False)
    assert m == 362880 and tot == 5056994653507584 * 362880 and tot > 2 ** 64
    tot8, _ = B.dls_scale_total(8, 7447587840, False)
    assert tot8 == 7447587840 * 40320


def test_mc_estimate_arithmetic():
    """dls_mc_estimate against the same sums written with numpy (Section 5.3)."""
    rng = np.random.default_rng(7)
    w = rng.integers(1, 50, 40).astype(np.float64) * 1e3
    c = rng.integers(0, 10 ** 9, 40).astype(np.uint64)
    r = B.dls_mc_estimate(w, c, 1.5e6)
    wc = w * c.astype(np.float64)
    assert r["knuth"] == pytest.approx(wc.mean(), rel=1e-12)
    assert r["knuth_se"] == pytest.approx(wc.std(ddof=1) / np.sqrt(len(wc)), rel=1e-12)
    assert r["ratio"] == pytest.approx(1.5e6 * wc.sum() / w.sum(), rel=1e-12)
    assert r["mean_completions_weighted"] == pytest.approx(wc.sum() / w.sum(), rel=1e-12)
    assert np.isnan(B.dls_mc_estimate(w[:1], c[:1], 1.0)["knuth_se"])
