import pytest


@pytest.mark.gpu
def test_smoke_entry():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.smoke()
