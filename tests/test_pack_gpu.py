"""The fused allreduce-payload kernel (spb_pack_grads) against the torch packing path."""
import pytest
import torch

from paper_2501_11407_b200.parallel import GradPacker


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("n,k,kp,m,B", [(37, 13, 16, 3, 5), (1024, 700, 768, 20, 256)])
def test_pack_grads_matches_torch(dtype, n, k, kp, m, B):
    g = torch.Generator().manual_seed(n + k)
    acc = torch.randn(n, kp, dtype=torch.float64, generator=g)
    gwo = torch.randn(m, n, dtype=torch.float64, generator=g)
    loss = torch.rand(B, dtype=torch.float64, generator=g)
    correct = torch.randint(0, 2, (B,), dtype=torch.int32, generator=g)
    cpu = GradPacker(n, k, m, "cpu", dtype=dtype)
    want = cpu.pack(acc, gwo, loss, correct).clone()
    dev = GradPacker(n, k, m, "cuda", dtype=dtype)
    got = dev.pack(acc.cuda(), gwo.cuda(), loss.cuda(), correct.cuda())
    torch.cuda.synchronize()
    got = got.cpu()
    # element copies are exact; the loss sum is in sample order (torch's may differ by ulps)
    assert torch.equal(got[:-2], want[:-2])
    assert got[-1].item() == want[-1].item()
    tol = 1e-6 if dtype == torch.float32 else 1e-12
    assert abs(got[-2].item() - want[-2].item()) <= tol * abs(want[-2].item())
