"""GPU tests of the rows next to the gradient path: the on-device
optimizers and training loop against the reference's own ``train`` (goldens produced by
the unmodified reference) and the CPU oracle, and the smooth-spike mode against the
reference's ``eprop_sparse_gradient(..., smooth=True)``."""

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


def _dataset_and_spec(g):
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import generate_poisson_dataset
    spec = P.NetworkSpec(kind=str(g["kind"]), n_hidden=int(g["n"]), n_inputs=int(g["k"]),
                         n_classes=int(g["m"]), precision=str(g["precision"]),
                         seed=int(g["seed"]))
    ds = generate_poisson_dataset(int(g["N"]), int(g["k"]), int(g["T"]), int(g["m"]),
                                  seed=int(g["seed"]))
    return spec, ds


@pytest.mark.parametrize("name", ["train_lif_sgd_f64", "train_alif_adam_f64",
                                  "train_lif_adam_f32", "train_alif_sgd_f32"])
def test_online_training_matches_reference_train(name, tmp_path):
    """batch_size=1 is the reference's per-sample online loop (training.py:116-166)."""
    _need_gpu()
    from paper_2501_11407_b200.training import init_network, train
    g = load_golden(name)
    spec, ds = _dataset_and_spec(g)
    mu = int(g["max_updates"])
    path = tmp_path / "m.csv"
    net, rows = train(spec, ds, optimizer=str(g["optimizer"]), lr=float(g["lr"]),
                      epochs=int(g["epochs"]), max_updates=None if mu < 0 else mu,
                      metrics_path=path)
    f64 = str(g["precision"]) == "f64"
    assert [r.epoch for r in rows] == list(g["epoch"])
    assert [r.step for r in rows] == list(range(1, len(rows) + 1))
    assert np.array_equal([r.accuracy for r in rows], g["accuracy"])
    # fp64 forward + readout: losses track the reference; the fp32 eligibility path
    # perturbs the weights by ~1e-6 of each update, which the losses see at that level
    assert np.allclose([r.loss for r in rows], g["loss"], rtol=1e-5 if f64 else 1e-3,
                       atol=1e-6 if f64 else 1e-3)
    w0 = init_network(spec)
    dw_ref = g["w"].astype(np.float64) - w0.neuron.w
    dw = net.neuron.w.astype(np.float64) - w0.neuron.w
    assert net.neuron.w.dtype == w0.neuron.w.dtype
    assert _rel(dw, dw_ref) <= (1e-4 if f64 else 1e-3)
    assert _rel(net.readout.w_out, g["w_out"]) <= (1e-6 if f64 else 1e-5)
    lines = path.read_text().strip().splitlines()
    assert lines[0] == "epoch,step,loss,accuracy" and len(lines) == len(rows) + 1


@pytest.mark.parametrize("kind,opt", [("lif", "sgd"), ("alif", "adam")])
def test_batched_training_matches_oracle(kind, opt):
    """batch_size=B applies the batch-mean gradient; checked against the
    oracle's loop with the same batching."""
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import generate_poisson_dataset
    from paper_2501_11407_b200.training import train
    spec = P.NetworkSpec(kind=kind, n_hidden=40, n_inputs=30, n_classes=4, precision="f64",
                         seed=7)
    ds = generate_poisson_dataset(10, 30, 70, 4, seed=7)
    lr = 1e-4 if opt == "sgd" else 1e-3
    net, rows = train(spec, ds, optimizer=opt, lr=lr, epochs=2, batch_size=4)
    w, wo = O.init_network_arrays(40, 30, 4, seed=7)
    x, y = O.poisson_batch(10, 30, 70, 4, seed=7)
    w2, wo2, orows = O.train_online(w, wo, O.Params(alif=kind == "alif"), x, y, opt, lr, 2,
                                    None, batch_size=4)
    assert len(rows) == len(orows) == 6       # 4 + 4 + 2 samples per epoch
    assert np.allclose([r.loss for r in rows], [r[1] for r in orows], rtol=1e-5, atol=1e-6)
    assert np.array_equal([r.accuracy for r in rows], [r[2] for r in orows])
    assert _rel(net.neuron.w - w, w2 - w) <= 1e-4


def test_evaluate_matches_oracle():
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import generate_poisson_dataset
    from paper_2501_11407_b200.training import evaluate
    net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=48, n_inputs=25, n_classes=3,
                                       precision="f64", seed=2))
    ds = generate_poisson_dataset(11, 25, 90, 3, seed=2)
    loss, acc = evaluate(net, ds, batch_size=4)
    x, y = O.poisson_batch(11, 25, 90, 3, seed=2)
    p = O.Params(alif=True)
    ls, corr = [], 0
    for b in range(11):
        lb, s, _ = O.network_loss(net.neuron.w, net.readout.w_out, p, x[b].astype(np.float64),
                                  int(y[b]))
        ls.append(lb)
        corr += int(np.argmax(s) == y[b])
    assert loss == pytest.approx(float(np.mean(ls)), rel=1e-10)
    assert acc == corr / 11


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_optimizer_kernels_bit_exact(dtype):
    """spb_sgd_update / spb_adam_update restate training.py:58-91 operation by operation."""
    _need_gpu()
    import ctypes

    from paper_2501_11407_b200 import _lib
    from paper_2501_11407_b200.training import AdamState, adam_update, sgd_update
    rng = np.random.default_rng(0)
    rows, cols, ld = 37, 53, 64
    p0 = rng.standard_normal((rows, cols)).astype(dtype)
    v = ctypes.c_void_p
    f64 = int(dtype == np.float64)
    # SGD (gradient from an fp64 accumulator with padded rows, rounded to dtype first)
    acc = rng.standard_normal((rows, ld))
    pd = torch.from_numpy(p0.copy()).cuda()
    ad = torch.from_numpy(acc).cuda()
    mirror = torch.empty((rows, cols), dtype=torch.float64, device="cuda")
    _lib.call("spb_sgd_update", v(pd.data_ptr()), f64, rows, cols, v(ad.data_ptr()), 1, ld, 1.0,
              0.03, v(mirror.data_ptr()), None)
    want = sgd_update({"w": p0}, {"w": acc[:, :cols].astype(dtype)}, 0.03)["w"]
    assert np.array_equal(pd.cpu().numpy(), want)
    assert np.array_equal(mirror.cpu().numpy(), want.astype(np.float64))
    # Adam, three steps, fp32 gradient source with a 1/4 batch-mean scale
    pd = torch.from_numpy(p0.copy()).cuda()
    md, vd = torch.zeros_like(pd), torch.zeros_like(pd)
    st = AdamState()
    p = {"w": p0.copy()}
    for t in range(1, 4):
        g32 = rng.standard_normal((rows, cols)).astype(np.float32)
        gd = torch.from_numpy(g32).cuda()
        _lib.call("spb_adam_update", v(pd.data_ptr()), v(md.data_ptr()), v(vd.data_ptr()), f64,
                  rows, cols, v(gd.data_ptr()), 0, cols, 0.25, 1e-3, 0.9, 0.999, 1e-8, t, None,
                  None)
        gscaled = (g32.astype(np.float64) * 0.25).astype(dtype)
        p = adam_update(p, {"w": gscaled}, 1e-3, st)
    torch.cuda.synchronize()
    assert np.array_equal(pd.cpu().numpy(), p["w"])
    assert np.array_equal(md.cpu().numpy(), st.m["w"])
    assert np.array_equal(vd.cpu().numpy(), st.v["w"])


@pytest.mark.parametrize("name", ["smooth_lif_f64", "smooth_alif_f64", "smooth_alif_f32"])
@pytest.mark.parametrize("chunk", [63, 127])
def test_smooth_mode_vs_reference(name, chunk):
    """eprop with surrogate_smooth spikes (the reference's FD mode, smooth=True)."""
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    from paper_2501_11407_b200.gradients import _neuron_kwargs, get_engine
    g = load_golden(name)
    net = P.init_network(P.NetworkSpec(kind=str(g["kind"]), n_hidden=int(g["n"]),
                                       n_inputs=int(g["k"]), n_classes=int(g["m"]),
                                       precision=str(g["precision"]), seed=0))
    B, T, n = int(g["B"]), int(g["T"]), int(g["n"])
    x, y = poisson_batch(B, int(g["k"]), T, int(g["m"]), seed=0)
    eng = get_engine(net, B, chunk=chunk, T=T)
    eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
    r = torch.zeros((B, T, (n + 31) // 32), dtype=torch.int32, device="cuda")
    eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), raster=r, smooth=True,
            **_neuron_kwargs(net))
    torch.cuda.synchronize()
    f64 = str(g["precision"]) == "f64"
    rr = r.cpu().numpy().view(np.uint32)
    bits = ((rr[..., None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool)
    got = bits.reshape(B, T, -1)[..., :n]
    want = np.unpackbits(g["raster_packed"], axis=-1)[..., :n].astype(bool)
    if f64:
        assert np.array_equal(got, want)
    assert np.allclose(eng.loss.cpu().numpy(), g["loss"], rtol=1e-9 if f64 else 1e-4,
                       atol=1e-12 if f64 else 1e-6)
    gw = eng.grad_w(torch.float64).cpu().numpy()
    ref = g["eprop_w"].sum(0)
    assert _rel(gw, ref) <= 1e-4
    assert float(gw.ravel() @ ref.ravel()) / (np.linalg.norm(gw) * np.linalg.norm(ref)) >= 0.9999
    assert _rel(eng.grad_wout.cpu().numpy(), g["eprop_w_out"].sum(0)) <= (1e-9 if f64 else 1e-5)
    # the drop-in accepts smooth=True as the reference does
    res = P.eprop_batch_gradient(net, x, y, smooth=True)
    assert _rel(res.grads["w"], ref) <= 1e-4


def test_device_poisson_generator():
    """spb_poisson_bits: per-class/channel firing rates match sample_events' distribution,
    deterministic per seed, no stray bits past k, and the engine trains on it directly."""
    _need_gpu()
    from paper_2501_11407_b200.datasets import DevicePoisson
    k, m, B, T = 37, 3, 64, 400
    gen = DevicePoisson(m, k, seed=3)
    bits, labels = gen.batch(B, T)
    x = np.unpackbits(bits.cpu().numpy(), axis=-1, bitorder="little")
    assert np.all(x[..., k:] == 0)
    x = x[..., :k].astype(np.float64)
    lab = labels.cpu().numpy()
    for c in range(m):
        sel = x[lab == c]
        if len(sel) < 4:
            continue
        emp = sel.mean(axis=(0, 1))
        p = gen.rates_np[c]
        sd = np.sqrt(p * (1 - p) / (sel.shape[0] * T))
        assert np.all(np.abs(emp - p) <= 5 * sd + 1e-9)
    again = DevicePoisson(m, k, seed=3).batch(B, T)[0]
    assert torch.equal(again, bits)
    other = DevicePoisson(m, k, seed=4).batch(B, T)[0]
    assert not torch.equal(other, bits)
