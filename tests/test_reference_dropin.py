"""The drop-in against the UNMODIFIED reference package (``sparseprop`` 0.1.0).

The reference is imported from ``baseline/_ref`` (installed with pip from
/root/reference/pkg; git-ignored, shipped to the GPU box with the repo snapshot) and the
tests skip when it is absent.  They show what INTEGRATION.md promises:

* the reference's own ``Network`` / ``LIFParams`` / ``ALIFParams`` objects go straight
  into ``eprop_sparse_gradient`` / ``eprop_batch_gradient`` / ``network_loss``;
* ``ENGINES["eprop-b200"]`` registered with the INTEGRATION.md stub drives the
  reference's own ``train()`` (training.py:116-166) and ``cli gradcheck``
  (cli.py:95-113) on the B200 kernels;
* the public single-step trace helpers (``initial_trace``, ``eprop_trace_update``,
  ``learning_signal``, ``accumulate_param_grad``; gradients.py:78-111) reproduce the
  reference's on the reference's own compressed tensors (CPU).
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_REF = os.path.join(ROOT, "baseline", "_ref")


def _sparseprop():
    if os.path.isdir(os.path.join(_REF, "sparseprop")) and _REF not in sys.path:
        sys.path.insert(0, _REF)
    try:
        import sparseprop  # noqa: F401
    except ImportError:
        pytest.skip("reference package not installed in baseline/_ref")
    import sparseprop
    return sparseprop


def _ref_network(sp, kind="lif", n=8, k=6, m=3, seed=0, dtype=np.float64, **kw):
    # the reference's own test constructor (test_gradients.py:40-45)
    from sparseprop.neurons import ALIFParams, LIFParams, Network, ReadoutParams
    rng = np.random.default_rng(seed)
    w = (rng.uniform(-1, 1, (n, k)) / np.sqrt(k)).astype(dtype)
    w_out = (rng.uniform(-1, 1, (m, n)) / np.sqrt(n)).astype(dtype)
    neuron = ALIFParams(w, **kw) if kind == "alif" else LIFParams(w, **kw)
    return Network(kind, neuron, ReadoutParams(w_out))


def _sample(net, T, seed=1):
    # test_gradients.py:48-51
    rng = np.random.default_rng(seed)
    x = (rng.random((T, net.k)) < 0.3).astype(net.neuron.w.dtype)
    return x, int(rng.integers(net.m))


def eprop_b200_gradient(net, x_seq, label, smooth=False):
    """The INTEGRATION.md stub a maintainer adds to sparseprop (sparseprop/b200.py)."""
    import paper_2501_11407_b200.gradients as b200
    from sparseprop.gradients import GradResult
    r = b200.eprop_sparse_gradient(net, x_seq, label, smooth=smooth)
    return GradResult(r.loss, r.grads, np.asarray(r.readout_sum), None)


# ----------------------------------------------------------------------------------
# CPU: the single-step trace helpers on the reference's own tensors
# ----------------------------------------------------------------------------------

@pytest.mark.parametrize("kind", ["lif", "alif"])
@pytest.mark.parametrize("reset", [False, True])
def test_trace_helpers_match_reference(kind, reset):
    sp = _sparseprop()
    from sparseprop import gradients as RG
    from sparseprop.neurons import NeuronState, step_jacobians

    from paper_2501_11407_b200 import gradients as G
    net = _ref_network(sp, kind, n=7, k=5, seed=3, reset=reset)
    x, label = _sample(net, 12, seed=4)
    rng = np.random.default_rng(0)
    g_ref = RG.initial_trace(net.neuron)
    g_ours = G.initial_trace(net.neuron)
    assert g_ours.G.values.shape == g_ref.G.values.shape
    acc_ref = np.zeros((net.n, net.k))
    acc_ours = np.zeros((net.n, net.k))
    u = rng.standard_normal(net.n)
    a = np.abs(rng.standard_normal(net.n))
    for t in range(x.shape[0]):
        h_i, f = step_jacobians(net.neuron, NeuronState(u, np.zeros(net.n), a), x[t])
        g_ref = RG.eprop_trace_update(g_ref, h_i, f)
        g_ours = G.eprop_trace_update(g_ours, h_i, f)           # reference SparseTensors
        np.testing.assert_allclose(g_ours.G.values, g_ref.G.values, rtol=1e-14, atol=1e-15)
        # plain compressed arrays work too
        g2 = G.eprop_trace_update(G.TraceState(g_ref.G.values), h_i.values, f.values)
        np.testing.assert_allclose(g2.values, RG.eprop_trace_update(g_ref, h_i, f).G.values,
                                   rtol=1e-14, atol=1e-15)
        dl_dv = rng.standard_normal(net.m)
        sg = rng.random(net.n)
        c_ref = RG.learning_signal(dl_dv, net.readout, sg)
        c_ours = G.learning_signal(dl_dv, net.readout, sg)
        np.testing.assert_allclose(c_ours, c_ref, rtol=1e-15, atol=0)
        RG.accumulate_param_grad(acc_ref, c_ref, g_ref)
        G.accumulate_param_grad(acc_ours, c_ours, g_ref)
        np.testing.assert_allclose(acc_ours, acc_ref, rtol=1e-13, atol=1e-15)
        u = rng.standard_normal(net.n)
    with pytest.raises(G.ShapeMismatch):
        G.learning_signal(np.zeros(net.m + 1), net.readout, np.ones(net.n))
    with pytest.raises(G.ShapeMismatch):
        G.accumulate_param_grad(np.zeros((net.n + 1, net.k)), np.zeros(net.n + 1), g_ref)


def test_trace_update_rejects_dense_operand():
    """A densified H_I raises StructureFallback, like the reference (gradients.py:91-92)."""
    _sparseprop()
    from sparseprop.gradients import initial_trace
    from sparseprop.neurons import LIFParams, NeuronState, step_jacobians
    from sparseprop.tensor import dense_tensor

    from paper_2501_11407_b200 import gradients as G
    p = LIFParams(np.zeros((2, 3)))
    _, f = step_jacobians(p, NeuronState(np.zeros(2), np.zeros(2)), np.ones(3))
    with pytest.raises(G.StructureFallback):
        G.eprop_trace_update(initial_trace(p), dense_tensor(np.eye(2), 1), f)


# ----------------------------------------------------------------------------------
# GPU: the reference's objects and loops on the B200 path
# ----------------------------------------------------------------------------------

def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["lif", "alif"])
@pytest.mark.parametrize("n,T", [(8, 10), (8, 100), (32, 10), (32, 100)])
def test_reference_network_objects_vs_reference_engines(kind, n, T):
    """TestEngineAgreement (test_gradients.py:157-168) with the B200 engine in place of
    the reference's e-prop: the reference's Network objects, its BPTT as the oracle."""
    _need_gpu()
    sp = _sparseprop()
    from sparseprop.gradients import bptt_gradient, network_loss

    from paper_2501_11407_b200 import gradients as G
    for seed in range(3):
        net = _ref_network(sp, kind, n=n, seed=seed)
        x, label = _sample(net, T, seed=seed + 100)
        a = G.eprop_sparse_gradient(net, x, label)
        b = bptt_gradient(net, x, label)
        for key in ("w", "w_out"):
            assert a.grads[key].dtype == net.neuron.w.dtype
            scale = max(np.max(np.abs(b.grads[key])), 1e-300)
            assert np.max(np.abs(a.grads[key] - b.grads[key])) <= 1e-5 * scale + 1e-12
        assert a.loss == pytest.approx(b.loss, rel=1e-10, abs=1e-12)
        # forward-only loss and raster on the B200 = the reference's network_loss
        l_ours, s_ours, r_ours = G.network_loss(net, x, label)
        l_ref, s_ref, r_ref = network_loss(net, x, label)
        assert np.array_equal(r_ours, r_ref)
        assert l_ours == pytest.approx(l_ref, rel=1e-12, abs=1e-12)
        np.testing.assert_allclose(s_ours, s_ref, rtol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["lif", "alif"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_real_valued_inputs_vs_reference(kind, dtype):
    """Inputs that are not spike counts (any float x_seq, as the reference accepts,
    gradients.py:132): the B200 path projects them in fp64 and feeds the gradient GEMM
    bf16 hi/lo pairs -- the reference's own e-prop and BPTT on its own Network objects
    are matched to the fp32 gradient tolerance, the forward raster and loss exactly."""
    _need_gpu()
    sp = _sparseprop()
    from sparseprop.gradients import bptt_gradient, eprop_sparse_gradient, network_loss

    from paper_2501_11407_b200 import gradients as G
    for seed in range(3):
        net = _ref_network(sp, kind, n=32, k=12, seed=seed, dtype=dtype)
        rng = np.random.default_rng(seed + 7)
        x = (rng.random((90, 12)) * 1.3 * (rng.random((90, 12)) < 0.4)).astype(dtype)
        label = int(rng.integers(net.m))
        a = G.eprop_sparse_gradient(net, x, label)
        for ref in (eprop_sparse_gradient(net, x, label), bptt_gradient(net, x, label)):
            for key in ("w", "w_out"):
                assert a.grads[key].dtype == net.neuron.w.dtype
                g, r = a.grads[key].astype(np.float64), ref.grads[key].astype(np.float64)
                rel = np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300)
                assert rel <= (1e-4 if dtype == np.float64 else 2e-4), (key, rel)
        l_ours, s_ours, r_ours = G.network_loss(net, x, label)
        l_ref, s_ref, r_ref = network_loss(net, x, label)
        assert np.array_equal(r_ours, r_ref)
        # (the reference runs an f32 net in f32 arithmetic, the B200 path in fp64)
        assert l_ours == pytest.approx(l_ref, rel=1e-4 if dtype == np.float32 else 1e-10)
    # the batched entry point with a float batch (B = 5, T = 90)
    xb = (np.random.default_rng(3).random((5, 90, 12)) * 0.9).astype(dtype)
    yb = np.arange(5) % net.m
    rb = G.eprop_batch_gradient(net, xb, yb)
    gs = sum(eprop_sparse_gradient(net, xb[i], int(yb[i])).grads["w"].astype(np.float64)
             for i in range(5))
    rel = np.linalg.norm(rb.grads["w"] - gs) / np.linalg.norm(gs)
    assert rel <= 2e-4, rel


@pytest.mark.gpu
@pytest.mark.parametrize("kind,precision,optimizer", [("lif", "f64", "sgd"),
                                                     ("alif", "f64", "adam"),
                                                     ("alif", "f32", "sgd")])
def test_reference_train_through_engines_registry(kind, precision, optimizer, tmp_path):
    """The reference's own train() with ENGINES["eprop-b200"] (INTEGRATION.md stub)
    against the same train() with its CPU engine: identical accuracy rows, losses and
    final weights within the fp32 gradient tolerance."""
    _need_gpu()
    sp = _sparseprop()
    from sparseprop.datasets import generate_poisson_dataset
    from sparseprop.gradients import ENGINES
    from sparseprop.training import NetworkSpec, train
    ENGINES["eprop-b200"] = eprop_b200_gradient
    try:
        spec = NetworkSpec(kind=kind, n_hidden=24, n_inputs=16, n_classes=3,
                           precision=precision, seed=2)
        ds = generate_poisson_dataset(12, 16, 60, 3, seed=5)
        net_c, rows_c = train(spec, ds, method="eprop-sparse", optimizer=optimizer, lr=0.01,
                              epochs=2, metrics_path=tmp_path / "cpu.csv")
        net_g, rows_g = train(spec, ds, method="eprop-b200", optimizer=optimizer, lr=0.01,
                              epochs=2, metrics_path=tmp_path / "gpu.csv")
    finally:
        ENGINES.pop("eprop-b200", None)
    assert len(rows_c) == len(rows_g) == 24
    assert [r.accuracy for r in rows_c] == [r.accuracy for r in rows_g]
    tol = 1e-5 if precision == "f64" else 1e-3
    np.testing.assert_allclose([r.loss for r in rows_g], [r.loss for r in rows_c],
                               rtol=tol, atol=tol)
    # weights after 24 online updates: the fp32 eligibility path perturbs each update's
    # gradient at ~1e-6 relative, accumulated over the run
    wtol = 1e-4 if precision == "f64" else 1e-3
    for a, b in ((net_g.neuron.w, net_c.neuron.w), (net_g.readout.w_out, net_c.readout.w_out)):
        assert a.dtype == b.dtype
        assert np.linalg.norm(a - b) <= wtol * np.linalg.norm(b)


@pytest.mark.gpu
@pytest.mark.parametrize("neuron", ["lif", "alif"])
def test_reference_cli_gradcheck_on_b200(neuron, capsys, monkeypatch):
    """`sparseprop gradcheck` (cli.py:95-113) with its e-prop call routed to the B200
    (what a maintainer's --method switch would do): the CSV row of e-prop vs BPTT
    deviations stays at the fp32 level the paper reports (median ~1e-6)."""
    _need_gpu()
    sp = _sparseprop()
    import sparseprop.cli as cli
    monkeypatch.setattr(cli, "eprop_sparse_gradient", eprop_b200_gradient)
    rc = cli.main(["gradcheck", "--neuron", neuron, "--hidden", "32", "--steps", "100",
                   "--seed", "0", "--precision", "f64"])
    out = capsys.readouterr().out.strip().splitlines()
    assert rc == 0
    assert out[0] == ",".join(cli.GRADCHECK_HEADER)
    fields = out[1].split(",")
    assert fields[:5] == [neuron, "f64", "32", "100", "0"]
    median, q_hi = float(fields[5]), float(fields[7])
    assert median <= 1e-6 and q_hi <= 1e-4


@pytest.mark.gpu
def test_weights_cached_between_calls_but_inplace_edits_seen():
    """The drop-in re-uploads W only when it changed; an in-place edit (the reference's
    finite differences perturb weights in place, gradients.py:403-408) is seen."""
    _need_gpu()
    sp = _sparseprop()
    from sparseprop.gradients import eprop_sparse_gradient as ref_eprop

    from paper_2501_11407_b200 import gradients as G
    net = _ref_network(sp, "alif", n=16, k=10, seed=1)
    x, label = _sample(net, 40, seed=2)
    a = G.eprop_sparse_gradient(net, x, label)
    net.neuron.w[3, 4] += 0.5                      # in place, same array object
    b = G.eprop_sparse_gradient(net, x, label)
    r = ref_eprop(net, x, label)
    assert not np.array_equal(a.grads["w"], b.grads["w"])
    assert b.loss == pytest.approx(r.loss, rel=1e-10)
    assert np.max(np.abs(b.grads["w"] - r.grads["w"])) <= 1e-5 * np.max(np.abs(r.grads["w"]))
