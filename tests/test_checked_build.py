"""The kernels' internal invariants (DLS_CHECK / SB_CHECK in csrc/): stack and
table indices inside levels -1..L+1, pool slots never overwritten before they
are read, donated subtrees in range, every lane idle at exit, class sizes
dividing |G|.  They are compiled only into libdls_b200_checked.so
(-DDLS_CHECKS); a violation fails the call with DLS_E_CUDA.

compute-sanitizer is not available on the GPU pool, so these checks stand in
for it.  The test reruns a cross-section of the GPU parity tests (every
kernel, the pool and donation paths, emit, symmetry breaking) with DLS_LIB
pointing at the checked build, so the oracle comparisons stay the same.
"""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

SELECT = ("config1 or config2 or config3_dls8_full or config4_vs8 or small_orders or empty or ragged "
          "or inconsistent or device_buffers or few_workunits or pool_stress or emit or count_cells_row_major "
          "or gpu_canonize_all or gpu_count_sb")


def _checked_lib():
    from paper_1709_02599_b200 import build as _build
    return _build.build_checked()


def test_checked_build_compiles_the_checks_in():
    """Host-only: the checked library loads, exports the ABI and says it is checked."""
    lib = _checked_lib()
    code = ("import paper_1709_02599_b200 as D; L = D.load(); "
            "assert L._name == %r, L._name; print(D.dls_version())" % lib)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT,
                         env=dict(os.environ, DLS_LIB=lib), timeout=300)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip().endswith("sm_100a checked")


@pytest.mark.gpu
def test_parity_cross_section_under_checked_build():
    lib = _checked_lib()
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu", "-k", SELECT,
           "tests/test_gpu_parity.py", "tests/test_symmetry.py"]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, env=dict(os.environ, DLS_LIB=lib),
                         timeout=1500)
    tail = (out.stdout + out.stderr)[-3000:]
    assert out.returncode == 0, tail
    assert " passed" in out.stdout and "failed" not in out.stdout, tail
