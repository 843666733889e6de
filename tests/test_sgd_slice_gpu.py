"""spb_sgd_slice_update (SGD on W fused with the INT8 re-slicing) against the two
launches it replaces (spb_sgd_update then spb_slice_weights): bitwise W, digits and
exponents, for fp32 and fp64 weights and both gradient sources."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.parametrize("w_f64", [False, True])
@pytest.mark.parametrize("g_f64", [False, True])
@pytest.mark.parametrize("n,k", [(1024, 700), (37, 5), (100, 129)])
def test_sgd_slice_matches_two_launches(w_f64, g_f64, n, k):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_11407_b200 import _lib
    from paper_2501_11407_b200.engine import EpropEngine
    eng_a = EpropEngine(n, k, 3, 2, alif=False, w_f64=w_f64, chunk=63)
    eng_b = EpropEngine(n, k, 3, 2, alif=False, w_f64=w_f64, chunk=63)
    rng = np.random.default_rng(n + k)
    w = rng.standard_normal((n, k)) * np.exp(rng.uniform(-12, 0, (n, k)))
    w[rng.random((n, k)) < 0.05] = 0.0
    wo = rng.standard_normal((3, n))
    for e in (eng_a, eng_b):
        e.set_weights(torch.from_numpy(w), torch.from_numpy(wo))
    ld = k + 3
    g = torch.from_numpy(rng.standard_normal((n, ld))).to(
        torch.float64 if g_f64 else torch.float32).cuda()
    scale, lr = 1.0 / 7.0, 0.013
    eng_a.sgd_slice(g, g_f64, ld, scale, lr)
    v = ctypes.c_void_p
    st = v(torch.cuda.current_stream().cuda_stream)
    _lib.call("spb_sgd_update", v(eng_b.w.data_ptr()), int(w_f64), n, k, v(g.data_ptr()),
              int(g_f64), ld, scale, lr, None, st)
    eng_b.slice_weights()
    torch.cuda.synchronize()
    assert torch.equal(eng_a.w, eng_b.w)
    assert torch.equal(eng_a.sexp, eng_b.sexp)
    assert torch.equal(eng_a.wq, eng_b.wq)
    # and the digits reconstruct the updated weights (digits.cuh format)
    P = eng_a.P
    # rows are stored in slot order within groups of 16 neurons (digits.cuh wq_slot)
    i = np.arange(n)
    j = i & 15
    slot = (i & ~15) | (((j & 3) >> 1) * 8 + (j >> 2) * 2 + (j & 1))
    wq = eng_a.wq.cpu().numpy().astype(np.float64)[:, slot, :k]
    s = eng_a.sexp.cpu().numpy()[:n].astype(np.float64)
    if P == 6:
        rec = sum(wq[p] * 2.0 ** (8 * (5 - p)) for p in range(6)) * (2.0 ** (s - 46))[:, None]
    else:
        rec = sum(wq[p] * 2.0 ** (-6 - 7 * p) for p in range(P)) * (2.0 ** s)[:, None]
    wn = eng_a.w.cpu().numpy().astype(np.float64)
    tol = (2.0 ** (s - (46 if P == 6 else 6 + 7 * (P - 1))))[:, None]
    assert np.all(np.abs(rec - wn) <= tol)
