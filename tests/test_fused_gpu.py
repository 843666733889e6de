"""K21 (fused projection + dynamics, csrc/fused.cu) against the reference goldens and
against the two-kernel path K2 + K1 it replaces: the same arithmetic, so rasters,
losses and the whole gradient accumulator must be bitwise identical."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from conftest import load_golden  # noqa: E402
from oracle import eprop_ref as O  # noqa: E402


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _engine_run(net, x, y, *, fused, chunk, smooth=False, bits=False):
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    B, T, _ = x.shape
    eng = EpropEngine(net.n, net.k, net.m, B, alif=net.is_alif,
                      w_f64=net.neuron.w.dtype == np.float64, chunk=chunk, fused=fused,
                      reset=net.neuron.reset)
    assert eng.fused == fused
    eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
    r = torch.zeros((B, T, (net.n + 31) // 32), dtype=torch.int32, device="cuda")
    xin = np.packbits(x, axis=-1, bitorder="little") if bits else x
    eng.run(torch.from_numpy(xin).cuda(), torch.from_numpy(y).cuda(), raster=r, smooth=smooth,
            bits=bits, **_neuron_kwargs(net))
    torch.cuda.synchronize()
    rr = r.cpu().numpy().view(np.uint32)
    ras = ((rr[..., None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool)
    return (ras.reshape(B, T, -1)[..., :net.n], eng.loss.cpu().numpy().copy(),
            eng.grad_w_acc.cpu().numpy().copy(), eng.grad_wout.cpu().numpy().copy(),
            eng.zsum.cpu().numpy().copy())


@pytest.mark.parametrize("name", ["c1_lif_f64", "c1_alif_f64", "c1_lif_f32", "c1_alif_f32",
                                  "mid_alif_f64", "c1_lif_reset_f64", "c1_alif_reset_f64"])
@pytest.mark.parametrize("chunk", [63, 127])
def test_fused_vs_reference_and_unfused(name, chunk):
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    g = load_golden(name)
    net = P.init_network(P.NetworkSpec(kind=str(g["kind"]), n_hidden=int(g["n"]),
                                       n_inputs=int(g["k"]), n_classes=int(g["m"]),
                                       precision=str(g["precision"]), reset=bool(g["reset"]),
                                       seed=int(g["seed_net"])))
    x, y = poisson_batch(int(g["B"]), int(g["k"]), int(g["T"]), int(g["m"]),
                         seed=int(g["seed_data"]))
    fu = _engine_run(net, x, y, fused=True, chunk=chunk)
    un = _engine_run(net, x, y, fused=False, chunk=chunk)
    for a, b in zip(fu, un):
        assert np.array_equal(a, b)
    if str(g["precision"]) == "f64":
        want = np.unpackbits(g["raster_packed"], axis=-1)[..., :int(g["n"])].astype(bool)
        assert np.array_equal(fu[0], want)
        assert np.allclose(fu[1], g["loss"], rtol=1e-9, atol=1e-12)
    gw = fu[2][:, :int(g["k"])]
    assert _rel(gw, g["eprop_w"].sum(0)) <= 1e-4


@pytest.mark.parametrize("kind,reset,smooth,wdt,bits", [
    ("alif", False, False, "f32", True), ("lif", False, False, "f64", False),
    ("alif", True, False, "f64", False), ("alif", False, True, "f32", False),
    ("lif", True, False, "f32", True)])
def test_fused_ragged_many_chunks(kind, reset, smooth, wdt, bits):
    """3 sample blocks (last partial), ragged neuron tile, 4 chunks, bits / counts input."""
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    B, n, k, m, T = 300, 70, 130, 5, 200
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m,
                                       precision=wdt, reset=reset, seed=9))
    x, y = poisson_batch(B, k, T, m, seed=9)
    fu = _engine_run(net, x, y, fused=True, chunk=63, smooth=smooth, bits=bits)
    un = _engine_run(net, x, y, fused=False, chunk=63, smooth=smooth, bits=bits)
    for a, b in zip(fu, un):
        assert np.array_equal(a, b)
    # and the oracle on a few samples (f64 forward of the same weights)
    p = O.Params(alif=kind == "alif", reset=reset)
    w64 = net.neuron.w.astype(np.float64)
    wo64 = net.readout.w_out.astype(np.float64)
    for b in (0, 127, 128, 299):
        _, _, ras = O.network_loss(w64, wo64, p, x[b].astype(np.float64), int(y[b]),
                                   smooth=smooth)
        assert np.array_equal(fu[0][b], ras)


@pytest.mark.parametrize("T", [150, 60])   # three chunks / one chunk (side-stream K4)
def test_graphed_update_equals_eager(T):
    """EpropEngine.graphed: the captured CUDA graph replays the same update bit for bit."""
    _need_gpu()
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


@pytest.mark.parametrize("parts", [2, 3])
def test_microbatch_engine_matches_single(parts):
    """MicroBatchEngine (half batches on concurrent streams): losses/readouts bitwise, the
    gradient up to the summation order of the per-part fp32 GEMM partials."""
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    from paper_2501_11407_b200.engine import EpropEngine, MicroBatchEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=150, n_inputs=80, n_classes=4,
                                       precision="f32", seed=8))
    kw = _neuron_kwargs(net)
    x, y = poisson_batch(11, 80, 300, 4, seed=8)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    w, wo = torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out)
    one = EpropEngine(150, 80, 4, 11, alif=True, chunk=127)
    one.set_weights(w, wo)
    one.run(xd, yd, **kw)
    mb = MicroBatchEngine(150, 80, 4, 11, parts=parts, alif=True, chunk=127)
    mb.set_weights(w, wo)
    mb.run(xd, yd, **kw)
    torch.cuda.synchronize()
    assert torch.equal(one.loss, mb.loss) and torch.equal(one.s, mb.s)
    assert torch.equal(one.correct, mb.correct)
    assert _rel(mb.grad_w(torch.float64).cpu().numpy(),
                one.grad_w(torch.float64).cpu().numpy()) <= 1e-6
    assert _rel(mb.grad_wout.cpu().numpy(), one.grad_wout.cpu().numpy()) <= 1e-12
