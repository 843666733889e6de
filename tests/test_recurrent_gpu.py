"""Recurrent extension on the B200 -- PARITY UNPINNED: the reference has
no recurrent weights, so the checks are (1) W_rec = 0 reproduces the feed-forward path
(the reference path) and (2) agreement with the oracle's restatement
(oracle/eprop_ref.py: eprop_forward_mode_rec), which builds the e-prop traces exactly as
the reference does with the presynaptic input [x_t, z_{t-1}]."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

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


def _run(net, x, y, chunk, recurrent=True):
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    B, T, _ = x.shape
    eng = EpropEngine(net.n, net.k, net.m, B, alif=net.is_alif,
                      w_f64=net.neuron.w.dtype == np.float64, chunk=chunk,
                      reset=net.neuron.reset, recurrent=recurrent)
    # the recurrent path keeps the filtered-input (xbar) GEMM operand; compare it with the
    # feed-forward engine on that same operand (the raw-spike fold sums in another order)
    eng.filt = False
    eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out),
                    w_rec=torch.from_numpy(net.neuron.w_rec) if recurrent else None)
    r = torch.zeros((B, T, (net.n + 31) // 32), dtype=torch.int32, device="cuda")
    eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), raster=r,
            **_neuron_kwargs(net))
    torch.cuda.synchronize()
    rr = r.cpu().numpy().view(np.uint32)
    ras = ((rr[..., None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool)
    return eng, ras.reshape(B, T, -1)[..., :net.n]


@pytest.mark.parametrize("kind", ["lif", "alif"])
@pytest.mark.parametrize("chunk", [63, 255])
def test_zero_recurrent_weights_reproduce_feed_forward(kind, chunk):
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=96, n_inputs=50, n_classes=4,
                                       precision="f64", seed=2, recurrent=True))
    net.neuron.w_rec = np.zeros_like(net.neuron.w_rec)
    x, y = poisson_batch(7, 50, 150, 4, seed=2)
    e_rec, r_rec = _run(net, x, y, chunk, recurrent=True)
    gw_rec = e_rec.grad_w(torch.float64).cpu().numpy()
    gwr = e_rec.grad_w_rec(torch.float64).cpu().numpy()
    loss_rec = e_rec.loss.cpu().numpy().copy()
    e_ff, r_ff = _run(net, x, y, chunk, recurrent=False)
    assert np.array_equal(r_rec, r_ff)
    assert np.array_equal(loss_rec, e_ff.loss.cpu().numpy())
    assert _rel(gw_rec, e_ff.grad_w(torch.float64).cpu().numpy()) <= 1e-6
    # the W_rec gradient itself (traces of z_{t-1}) vs the oracle
    p = O.Params(alif=kind == "alif")
    ref = np.zeros((96, 96))
    for b in range(7):
        r, _ = O.eprop_forward_mode_rec(net.neuron.w, net.neuron.w_rec, net.readout.w_out, p,
                                        x[b].astype(np.float64), int(y[b]))
        ref += r.grad_w[:, 50:]
    assert _rel(gwr, ref) <= 1e-4


@pytest.mark.parametrize("kind,reset,chunk,T,prec", [
    ("lif", False, 255, 120, "f64"), ("alif", False, 63, 200, "f64"),
    ("alif", True, 63, 150, "f64"), ("lif", True, 127, 300, "f32"),
    ("alif", False, 127, 140, "f32")])
def test_recurrent_vs_oracle(kind, reset, chunk, T, prec):
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    n, k, m, B = 130, 70, 5, 6
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m,
                                       precision=prec, reset=reset, seed=5, recurrent=True))
    net.neuron.w_rec = (net.neuron.w_rec * 3).astype(net.neuron.w.dtype)  # visible recurrence
    x, y = poisson_batch(B, k, T, m, seed=5)
    eng, ras = _run(net, x, y, chunk)
    p = O.Params(alif=kind == "alif", reset=reset)
    w64, wr64, wo64 = (a.astype(np.float64) for a in (net.neuron.w, net.neuron.w_rec,
                                                       net.readout.w_out))
    gref = np.zeros((n, k + n))
    losses = []
    for b in range(B):
        r, rr = O.eprop_forward_mode_rec(w64, wr64, wo64, p, x[b].astype(np.float64), int(y[b]))
        assert np.array_equal(ras[b], rr)
        gref += r.grad_w
        losses.append(r.loss)
    assert np.allclose(eng.loss.cpu().numpy(), losses, rtol=1e-9, atol=1e-12)
    got = np.concatenate([eng.grad_w(torch.float64).cpu().numpy(),
                          eng.grad_w_rec(torch.float64).cpu().numpy()], axis=1)
    assert _rel(got, gref) <= 1e-4, _rel(got, gref)
    assert _cos(got, gref) >= 0.9999
    assert np.any(ras)  # the network spikes


def test_recurrent_drop_in_and_training():
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import generate_poisson_dataset
    from paper_2501_11407_b200.training import train
    spec = P.NetworkSpec(kind="alif", n_hidden=40, n_inputs=20, n_classes=3, precision="f64",
                         seed=1, recurrent=True)
    net = P.init_network(spec)
    ds = generate_poisson_dataset(6, 20, 60, 3, seed=1)
    r = P.eprop_batch_gradient(net, ds.counts(), ds.label_array())
    assert set(r.grads) == {"w", "w_out", "w_rec"} and r.grads["w_rec"].shape == (40, 40)
    net2, rows = train(spec, ds, optimizer="adam", lr=1e-3, batch_size=3)
    assert len(rows) == 2 and all(np.isfinite(rw.loss) for rw in rows)
    assert not np.array_equal(net2.neuron.w_rec, net.neuron.w_rec)
