"""GPU parity of the reset=True path: the soft reset u -= theta z
makes the LIF trace G_u per-synapse and couples it to the ALIF trace G_a
(neurons.py:266-271), so the chunk algebra carries one (LIF) or two (ALIF) per-synapse
traces (forward.cu K1r, elig.cu / elig_reset.cu).  Checked against the reference's own
outputs (c1_*_reset_f64 goldens) and, for many chunks and ragged tiles, against the
oracle's per-step forward-mode restatement of gradients.py:132-185."""

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


def _cos(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(a @ b / max(np.linalg.norm(a) * np.linalg.norm(b), 1e-300))


def _run(net, x, y, chunk):
    from paper_2501_11407_b200.gradients import _neuron_kwargs, get_engine
    B, T, _ = x.shape
    eng = get_engine(net, B, chunk=chunk, T=T)
    eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
    r = torch.zeros((B, T, (net.n + 31) // 32), dtype=torch.int32, device="cuda")
    eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), raster=r,
            **_neuron_kwargs(net))
    torch.cuda.synchronize()
    rr = r.cpu().numpy().view(np.uint32)
    bits = ((rr[..., None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool)
    return eng, bits.reshape(B, T, -1)[..., :net.n]


@pytest.mark.parametrize("name", ["c1_lif_reset_f64", "c1_alif_reset_f64"])
@pytest.mark.parametrize("chunk", [63, 127])
def test_reset_vs_reference(name, chunk):
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    g = load_golden(name)
    net = P.init_network(P.NetworkSpec(kind=str(g["kind"]), n_hidden=int(g["n"]),
                                       n_inputs=int(g["k"]), n_classes=int(g["m"]),
                                       precision="f64", reset=True, seed=int(g["seed_net"])))
    x, y = poisson_batch(int(g["B"]), int(g["k"]), int(g["T"]), int(g["m"]),
                         seed=int(g["seed_data"]))
    eng, raster = _run(net, x, y, chunk)
    want = np.unpackbits(g["raster_packed"], axis=-1)[..., :int(g["n"])].astype(bool)
    assert np.array_equal(raster, want)
    assert np.allclose(eng.loss.cpu().numpy(), g["loss"], rtol=1e-9, atol=1e-12)
    gw = eng.grad_w(torch.float64).cpu().numpy()
    for ref in (g["eprop_w"].sum(0), g["bptt_w"].sum(0)):
        assert _rel(gw, ref) <= 1e-4, _rel(gw, ref)
        assert _cos(gw, ref) >= 0.9999
    assert _rel(eng.grad_wout.cpu().numpy(), g["eprop_w_out"].sum(0)) <= 1e-9


@pytest.mark.parametrize("kind", ["lif", "alif"])
@pytest.mark.parametrize("n,k,T,chunk", [(160, 200, 200, 63), (40, 30, 300, 127)])
def test_reset_many_chunks_vs_oracle(kind, n, k, T, chunk):
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    B, m = 5, 4
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m,
                                       precision="f64", reset=True, seed=4))
    x, y = poisson_batch(B, k, T, m, seed=4)
    eng, raster = _run(net, x, y, chunk)
    p = O.Params(alif=kind == "alif", reset=True)
    gw_ref = np.zeros((n, k))
    loss_ref = []
    for b in range(B):
        r = O.eprop_forward_mode(net.neuron.w, net.readout.w_out, p, x[b].astype(np.float64),
                                 int(y[b]))
        gw_ref += r.grad_w
        loss_ref.append(r.loss)
        assert np.array_equal(raster[b], O.network_loss(net.neuron.w, net.readout.w_out, p,
                                                        x[b].astype(np.float64), int(y[b]))[2])
    assert np.allclose(eng.loss.cpu().numpy(), loss_ref, rtol=1e-9, atol=1e-12)
    gw = eng.grad_w(torch.float64).cpu().numpy()
    assert _rel(gw, gw_ref) <= 1e-4, _rel(gw, gw_ref)
    assert _cos(gw, gw_ref) >= 0.9999


def test_reset_drop_in_api():
    """eprop_sparse_gradient on a reset network (per sample, like the reference call)."""
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    g = load_golden("c1_alif_reset_f64")
    net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=32, n_inputs=16, n_classes=2,
                                       precision="f64", reset=True, seed=int(g["seed_net"])))
    x, y = poisson_batch(8, 16, 100, 2, seed=int(g["seed_data"]))
    for b in range(3):
        res = P.eprop_sparse_gradient(net, x[b].astype(np.float64), int(y[b]))
        assert res.loss == pytest.approx(float(g["loss"][b]), rel=1e-9, abs=1e-12)
        if np.linalg.norm(g["eprop_w"][b]) > 1e-8:
            assert _rel(res.grads["w"], g["eprop_w"][b]) <= 1e-4
