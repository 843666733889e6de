"""Parity at the configurations the bench reports, and over long horizons.

* C3 exactly as ``bench.py`` times it: ALIF 700->1024->20, f32 weights from
  ``init_network(seed=0)``, B=256, T=250, inputs ``poisson_batch(seed=1000)`` (rank 0),
  0/1 spikes promised (``binary=True``), both as bytes and bit-packed (the e2e format).
* C4 as benched per GPU: ALIF 700->2048->35, f32, B=128, T=500.
* ALIF over T = 6000 steps: 12 chunks of 511 and 96 chunks of 63, so the per-synapse
  trace is carried through bf16 hi/lo operands many times (drift bound).

Oracle: ``oracle.eprop_ref.bptt_batch`` in f64 -- the reference's BPTT engine
(gradients.py:188-231) batched in GEMM form, equal to the reference's e-prop for this
feed-forward layer (test_gradients.py:157-194) and pinned against the reference's own
outputs in tests/test_oracle.py.  Tolerances (north_star): rasters bit-exact over the
whole horizon; batch-summed grad W relative L2 <= 1e-4 and cosine >= 0.9999; grad W_out
relative <= 1e-6 (fp64 readout path); losses relative <= 1e-9.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import eprop_ref as O  # noqa: E402

REL_TOL = 1e-4
COS_TOL = 0.9999


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _cos(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(a @ b / max(np.linalg.norm(a) * np.linalg.norm(b), 1e-300))


def _unpack_raster(r, n):
    r = r.cpu().numpy().view(np.uint32)
    B, T, nw = r.shape
    bits = ((r[..., None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool)
    return bits.reshape(B, T, nw * 32)[..., :n]


def _run(kind, n, k, m, x, y, w, w_out, chunk, bits=False):
    from paper_2501_11407_b200.engine import EpropEngine, default_chunk
    B, T, _ = x.shape
    chunk = chunk or default_chunk(T, B, n, k, kind == "alif")
    eng = EpropEngine(n, k, m, B, alif=kind == "alif", w_f64=w.dtype == np.float64,
                      chunk=chunk, device="cuda")
    eng.set_weights(torch.from_numpy(w), torch.from_numpy(w_out))
    xin = np.packbits(x, axis=-1, bitorder="little") if bits else x
    xd = torch.from_numpy(np.ascontiguousarray(xin)).cuda()
    yd = torch.from_numpy(y).cuda()
    raster = torch.zeros((B, T, (n + 31) // 32), dtype=torch.int32, device="cuda")
    eng.run(xd, yd, raster=raster, bits=bits, binary=True, alpha=0.95, theta=1.0,
            slope=10.0, beta=0.8, rho=0.96, kappa=0.95)
    torch.cuda.synchronize()
    return eng, _unpack_raster(raster, n)


def _check(eng, raster, ref, n):
    assert np.array_equal(raster, ref.raster), \
        f"{int((raster != ref.raster).sum())} spike flips"
    gw = eng.grad_w(torch.float64).cpu().numpy()
    gwo = eng.grad_wout.cpu().numpy()
    rel, cos = _rel(gw, ref.grad_w), _cos(gw, ref.grad_w)
    assert rel <= REL_TOL and cos >= COS_TOL, (rel, cos)
    assert _rel(gwo, ref.grad_w_out) <= 1e-6
    assert np.allclose(eng.loss.cpu().numpy(), ref.loss, rtol=1e-9, atol=1e-12)
    return rel, cos


@pytest.mark.parametrize("bits", [False, True])
def test_c3_as_benched(bits):
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    kind, n, k, m, T, B = "alif", 1024, 700, 20, 250, 256
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m,
                                       precision="f32", seed=0))
    x, y = poisson_batch(B, k, T, m, seed=1000)
    eng, raster = _run(kind, n, k, m, x, y, net.neuron.w, net.readout.w_out, 0, bits=bits)
    ref = O.bptt_batch(net.neuron.w, net.readout.w_out, O.Params(alif=True), x, y)
    _check(eng, raster, ref, n)


def test_c4_as_benched():
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    kind, n, k, m, T, B = "alif", 2048, 700, 35, 500, 128
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m,
                                       precision="f32", seed=0))
    x, y = poisson_batch(B, k, T, m, seed=1000)
    eng, raster = _run(kind, n, k, m, x, y, net.neuron.w, net.readout.w_out, 0)
    ref = O.bptt_batch(net.neuron.w, net.readout.w_out, O.Params(alif=True), x, y)
    _check(eng, raster, ref, n)


def test_c2_lif_as_benched():
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    kind, n, k, m, T, B = "lif", 256, 700, 20, 250, 128
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m,
                                       precision="f32", seed=0))
    x, y = poisson_batch(B, k, T, m, seed=1000)
    eng, raster = _run(kind, n, k, m, x, y, net.neuron.w, net.readout.w_out, 0)
    ref = O.bptt_batch(net.neuron.w, net.readout.w_out, O.Params(alif=False), x, y)
    _check(eng, raster, ref, n)


@pytest.mark.parametrize("chunk", [511, 63])
@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_alif_long_horizon(chunk, precision):
    """T = 6000: 12 (Tc=511) or 96 (Tc=63) chunk boundaries, each one a bf16 hi/lo
    round of the carried per-synapse trace; the error must stay inside the fp32 gate."""
    _need_gpu()
    n, k, m, T, B = 64, 40, 4, 6000, 8
    dt = np.float64 if precision == "f64" else np.float32
    w, w_out = O.init_network_arrays(n, k, m, seed=3, dtype=dt)
    w_out = (w_out * 2e-3).astype(dt)   # keep the T-summed logits off saturation
    x, y = O.poisson_batch(B, k, T, m, seed=7)
    eng, raster = _run("alif", n, k, m, x, y, w, w_out, chunk)
    ref = O.bptt_batch(w, w_out, O.Params(alif=True), x, y)
    assert ref.raster.mean() > 0.005
    rel, cos = _check(eng, raster, ref, n)
    print(f"T={T} chunk={chunk} {precision}: rel {rel:.2e} cos {cos:.10f}")


@pytest.mark.parametrize("chunk,T", [(1023, 900), (1023, 2500), (2047, 2000), (2047, 4500)])
@pytest.mark.parametrize("kind", ["alif", "lif"])
def test_long_chunks(chunk, T, kind):
    """Tc = 1023 / 2047: one chunk (the trace never materialised, pass B reuses pass A)
    and several chunks (the carry path with K = 1024 / 2048 per-sample GEMMs)."""
    _need_gpu()
    n, k, m, B = 72, 40, 4, 5
    w, w_out = O.init_network_arrays(n, k, m, seed=5, dtype=np.float32)
    w_out = (w_out * 2e-3).astype(np.float32)
    x, y = O.poisson_batch(B, k, T, m, seed=9)
    eng, raster = _run(kind, n, k, m, x, y, w, w_out, chunk)
    ref = O.bptt_batch(w, w_out, O.Params(alif=kind == "alif"), x, y)
    _check(eng, raster, ref, n)


@pytest.mark.parametrize("chunk", [1023, 2047])
@pytest.mark.parametrize("kind", ["alif", "lif"])
def test_long_chunks_reset(chunk, kind):
    """reset=True (the per-synapse G_u, K1r + K6 / K6r) with the long chunks."""
    _need_gpu()
    from paper_2501_11407_b200.engine import EpropEngine
    n, k, m, B, T = 48, 30, 3, 4, 2500
    w, w_out = O.init_network_arrays(n, k, m, seed=6, dtype=np.float64)
    w_out = w_out * 2e-3
    x, y = O.poisson_batch(B, k, T, m, seed=10)
    eng = EpropEngine(n, k, m, B, alif=kind == "alif", w_f64=True, chunk=chunk,
                      device="cuda", reset=True)
    eng.set_weights(torch.from_numpy(w), torch.from_numpy(w_out))
    raster = torch.zeros((B, T, (n + 31) // 32), dtype=torch.int32, device="cuda")
    eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), raster=raster,
            reset=True, binary=True)
    torch.cuda.synchronize()
    ref = O.bptt_batch(w, w_out, O.Params(alif=kind == "alif", reset=True), x, y)
    _check(eng, _unpack_raster(raster, n), ref, n)
