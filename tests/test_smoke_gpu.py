"""The driver's round-end smoke() must pass on the GPU box: run it as a GPU test."""
import pytest


@pytest.mark.gpu
def test_graft_smoke():
    import __graft_entry__ as g
    g.smoke()
