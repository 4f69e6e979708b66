"""The driver's smoke() entry point, run as a GPU test so that a change that
breaks it (e.g. a new node-count convention) fails the GPU suite too."""
import pytest

pytestmark = pytest.mark.gpu


def test_graft_entry_smoke():
    import __graft_entry__
    __graft_entry__.smoke()
