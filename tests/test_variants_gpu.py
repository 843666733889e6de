"""Engine variants that must reproduce the default path: the segmented chunk scan and
filter, the raw-spike operand over several chunks, the pack writing K5's operand,
parked psi, and CUDA-graph replay of a whole update (bitwise where the arithmetic is
the same, to fp32 rounding where only the summation order differs)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _run(net, x, y, *, smooth=False):
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    B, T, _ = x.shape
    chunk = next(c for c in (63, 127, 255, 511) if T <= c)
    eng = EpropEngine(net.n, net.k, net.m, B, alif=net.is_alif,
                      w_f64=net.neuron.w.dtype == np.float64, chunk=chunk)
    eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
    r = torch.zeros((B, T, (net.n + 31) // 32), dtype=torch.int32, device="cuda")
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    eng.run(xd, yd, raster=r, smooth=smooth, **_neuron_kwargs(net))
    torch.cuda.synchronize()
    return dict(raster=r.cpu().numpy().copy(), loss=eng.loss.cpu().numpy().copy(),
                gw=eng.grad_w_acc.cpu().numpy().copy(), gwo=eng.grad_wout.cpu().numpy().copy())


@pytest.mark.parametrize("kind,n,B,T", [("lif", 256, 6, 100), ("alif", 192, 5, 120),
                                         ("alif", 70, 3, 300)])
def test_segmented_scan_matches_one_sweep(kind, n, B, T, monkeypatch):
    """K1s on 4 time segments (chunk_scan_seg_kernel) vs the one-sweep scan."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=50, n_classes=4,
                                       precision="f32", seed=3))
    x, y = poisson_batch(B, 50, T, 4, seed=5)
    monkeypatch.setenv("SPB_SCAN_SEG", "1")
    a = _run(net, x, y)
    monkeypatch.setenv("SPB_SCAN_SEG", "0")
    b = _run(net, x, y)
    assert np.array_equal(a["raster"], b["raster"])
    assert _rel(a["gw"], b["gw"]) < 1e-5


@pytest.mark.parametrize("kind,n,k,B,T,chunk", [("alif", 128, 700, 4, 250, 255),
                                                 ("lif", 96, 37, 3, 300, 127),
                                                 ("alif", 64, 130, 2, 700, 511)])
def test_segmented_xbar_matches_sequential(kind, n, k, B, T, chunk, monkeypatch):
    """K4 on 64-row time segments (xbar_seg_kernel) vs the sequential 4-channel filter,
    one and several chunks (the carried fp64 filter state crosses chunk boundaries)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=4,
                                       precision="f32", seed=9))
    x, y = poisson_batch(B, k, T, 4, seed=2)
    out = {}
    monkeypatch.setenv("SPB_PACK_XH", "0")   # keep K4 in the one-chunk case (it is tested here)
    for flag in ("1", "0"):
        monkeypatch.setenv("SPB_XBAR_SEG", flag)
        eng = EpropEngine(n, k, 4, B, alif=net.is_alif, chunk=chunk)
        eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
        eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), **_neuron_kwargs(net))
        torch.cuda.synchronize()
        out[flag] = (eng.grad_w_acc.cpu().numpy().copy(), eng.xbar_state.cpu().numpy().copy(),
                     eng.xh.float().cpu().numpy().copy())
    a, b = out["1"], out["0"]
    np.testing.assert_allclose(a[1], b[1], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(a[2], b[2], rtol=2 ** -7, atol=0)
    assert _rel(a[0], b[0]) < 1e-6


@pytest.mark.parametrize("kind,n,k,B,T,chunk", [("alif", 256, 130, 5, 300, 63),
                                                 ("lif", 200, 64, 9, 400, 127),
                                                 ("alif", 1024, 96, 40, 600, 255)])
def test_raw_operand_multichunk_matches_xbar(kind, n, k, B, T, chunk, monkeypatch):
    """Several chunks on the raw-spike operand (filter folded into C / W, the carried
    filter state through the K = B row-0 GEMM and the K6 epilogue) vs the filtered-input
    operand: the same sums in another order (gradient to fp32 rounding)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=5,
                                       precision="f32", seed=21))
    x, y = poisson_batch(B, k, T, 5, seed=22)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("SPB_FILT", flag)
        eng = EpropEngine(n, k, 5, B, alif=net.is_alif, chunk=chunk)
        assert eng.filt == (flag == "1")
        eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
        eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), **_neuron_kwargs(net))
        torch.cuda.synchronize()
        out[flag] = (eng.grad_w_acc.cpu().numpy().copy(), eng.loss.cpu().numpy().copy())
    assert np.array_equal(out["1"][1], out["0"][1])
    assert _rel(out["1"][0], out["0"][0]) < 1e-5


@pytest.mark.parametrize("bits", [False, True])
def test_pack_writes_raw_operand_bitwise(bits, monkeypatch):
    """One chunk: the pack writing K5's raw-spike operand (spb_pack_spikes_xh) instead of
    K4 -- the same bf16 rows, so the whole update is bitwise equal."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    n, k, B, T = 256, 700, 6, 200
    net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=n, n_inputs=k, n_classes=5,
                                       precision="f32", seed=31))
    x, y = poisson_batch(B, k, T, 5, seed=32)
    xin = np.packbits(x, axis=-1, bitorder="little") if bits else x
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("SPB_PACK_XH", flag)
        eng = EpropEngine(n, k, 5, B, alif=True, chunk=255)
        eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
        eng.run(torch.from_numpy(xin).cuda(), torch.from_numpy(y).cuda(), bits=bits,
                **_neuron_kwargs(net))
        torch.cuda.synchronize()
        out[flag] = (eng.grad_w_acc.cpu().numpy().copy(), eng.xh.float().cpu().numpy().copy())
    assert np.array_equal(out["1"][1], out["0"][1])
    assert np.array_equal(out["1"][0], out["0"][0])


@pytest.mark.parametrize("kind,T,chunk", [("alif", 300, 63), ("lif", 400, 127)])
def test_parked_psi_is_bitwise_the_recompute(kind, T, chunk):
    """Opt-in psi parking (park_budget): pass B reads the psi pass A parked instead of
    re-running the projection and the dynamics -- the same psi, so bitwise the same update."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    n, k, B = 200, 96, 6
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=4,
                                       precision="f32", seed=41))
    x, y = poisson_batch(B, k, T, 4, seed=42)
    out = {}
    for budget in (0, 1 << 30):
        eng = EpropEngine(n, k, 4, B, alif=net.is_alif, chunk=chunk)
        eng.park_budget = budget
        eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
        eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), **_neuron_kwargs(net))
        torch.cuda.synchronize()
        assert (eng.psi_park is not None) == (budget > 0)
        out[budget] = (eng.grad_w_acc.cpu().numpy().copy(), eng.loss.cpu().numpy().copy(),
                       eng.grad_wout.cpu().numpy().copy())
    for a, b in zip(out[0], out[1 << 30]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("T", [150, 60])   # three chunks / one chunk (side-stream K4)
def test_graphed_update_equals_eager(T):
    """EpropEngine.graphed: the captured CUDA graph replays the same update bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=200, n_inputs=90, n_classes=5,
                                       precision="f32", seed=4))
    kw = _neuron_kwargs(net)
    eng = EpropEngine(200, 90, 5, 12, alif=True, chunk=63)
    eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
    outs = []
    for seed in (1, 2):
        x, y = poisson_batch(12, 90, T, 5, seed=seed)
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        eng.run(xd, yd, **kw)
        torch.cuda.synchronize()
        outs.append((eng.grad_w_acc.cpu().numpy().copy(), eng.loss.cpu().numpy().copy()))
    step = eng.graphed(xd, yd, **kw)
    for seed, (gw, ls) in zip((1, 2), outs):
        x, y = poisson_batch(12, 90, T, 5, seed=seed)
        step(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
        torch.cuda.synchronize()
        assert np.array_equal(eng.grad_w_acc.cpu().numpy(), gw)
        assert np.array_equal(eng.loss.cpu().numpy(), ls)


@pytest.mark.parametrize("kind,n,k,B,T,chunk,reset,filt", [
    ("alif", 256, 130, 5, 300, 63, False, "1"),     # kp = 256: one pair column tile
    ("alif", 384, 700, 7, 600, 127, False, "1"),    # n_pad % 256 = 128: the idle half-pair
    ("alif", 200, 90, 9, 400, 127, False, "0"),     # filtered operand (3 MMAs), kp = 128
    ("lif", 130, 64, 4, 300, 63, True, "1"),        # LIF reset: the G_u trace
    ("alif", 1024, 700, 40, 700, 255, False, "1"),  # C3-like, several sample splits
])
def test_carry_pairs_vs_oracle(kind, n, k, B, T, chunk, reset, filt, monkeypatch):
    """K6 on CTA pairs (cta_group::2, streamed eps boxes) over several chunks, at the
    geometries the pair tiling makes special (one pair column tile, a half pair past
    n_pad, the filtered 3-MMA operand, LIF reset, several sample splits) against the f64
    oracle: rasters bit-exact, gradient within the north-star tolerance."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    from oracle import eprop_ref as O
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=5,
                                       precision="f32", reset=reset, seed=31))
    x, y = poisson_batch(B, k, T, 5, seed=32)
    monkeypatch.setenv("SPB_FILT", filt)
    eng = EpropEngine(n, k, 5, B, alif=kind == "alif", chunk=chunk, reset=reset)
    assert -(-T // chunk) >= 3 and eng.ntr == 1
    eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
    eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), **_neuron_kwargs(net))
    torch.cuda.synchronize()
    p = O.Params(alif=kind == "alif", reset=reset)
    if reset:   # the per-sample forward-mode e-prop (gradients.py:132-185), summed
        rs = [O.eprop_forward_mode(net.neuron.w, net.readout.w_out, p,
                                   x[b].astype(np.float64), int(y[b])) for b in range(B)]
        ref_gw = np.sum([r.grad_w for r in rs], axis=0)
        ref_loss = np.array([r.loss for r in rs])
    else:       # feed-forward, no reset: BPTT == e-prop (test_gradients.py:157-168)
        ref = O.bptt_batch(net.neuron.w, net.readout.w_out, p, x, y)
        ref_gw, ref_loss = ref.grad_w, ref.loss
    gw = eng.grad_w(torch.float64).cpu().numpy()
    assert _rel(gw, ref_gw) < 1e-4
    cos = float(gw.ravel() @ ref_gw.ravel() / (np.linalg.norm(gw) * np.linalg.norm(ref_gw)))
    assert cos >= 0.9999
    assert np.allclose(eng.loss.cpu().numpy(), ref_loss, rtol=1e-9, atol=1e-12)
