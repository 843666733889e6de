"""Pin the CPU oracle (oracle/eprop_ref.py) against the reference's own outputs.

The fixtures in tests/golden/ were produced by running the unmodified reference
(tests/golden/make_golden.py).  These tests run on CPU only.
"""

import hashlib

import numpy as np
import pytest

from conftest import load_golden
from oracle import eprop_ref as O

SMALL = ["c1_lif_f64", "c1_alif_f64", "c1_lif_f32", "c1_alif_f32",
         "c1_lif_reset_f64", "c1_alif_reset_f64", "mid_alif_f64"]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def _setup(g):
    dtype = np.float64 if str(g["precision"]) == "f64" else np.float32
    B, T, k, m, n = (int(g[x]) for x in ("B", "T", "k", "m", "n"))
    x, labels = O.poisson_batch(B, k, T, m, seed=int(g["seed_data"]))
    w, w_out = O.init_network_arrays(n, k, m, seed=int(g["seed_net"]), dtype=dtype)
    assert _sha(x) == str(g["x_checksum"])
    assert _sha(w) == str(g["w_checksum"])
    assert np.array_equal(labels, g["labels"])
    p = O.Params(alif=str(g["kind"]) == "alif", reset=bool(g["reset"]))
    return p, w, w_out, x.astype(dtype), labels


@pytest.mark.parametrize("name", SMALL)
def test_forward_mode_port_matches_reference(name):
    g = load_golden(name)
    p, w, w_out, x, labels = _setup(g)
    f64 = w.dtype == np.float64
    for b in range(int(g["B"])):
        r = O.eprop_forward_mode(w, w_out, p, x[b], int(labels[b]))
        gw, gwo = g["eprop_w"][b], g["eprop_w_out"][b]
        if f64:
            # same algorithm, different summation order inside BLAS / einsum
            scale = max(np.max(np.abs(gw)), 1e-300)
            assert np.max(np.abs(r.grad_w - gw)) <= 1e-12 * scale + 1e-300
            assert np.max(np.abs(r.grad_w_out - gwo)) <= 1e-12 * max(np.max(np.abs(gwo)), 1e-300)
            assert r.loss == pytest.approx(float(g["loss"][b]), rel=1e-12, abs=1e-12)
        else:
            # the f32 reference mixes f64 traces with f32 filters (SURVEY App. C cmd C1)
            num = np.linalg.norm(r.grad_w - gw)
            assert num <= 1e-4 * np.linalg.norm(gw) + 1e-30
        assert np.allclose(r.readout_sum, g["readout_sum"][b], rtol=1e-5 if not f64 else 1e-12)


@pytest.mark.parametrize("name", SMALL)
def test_raster_bit_exact(name):
    g = load_golden(name)
    p, w, w_out, x, labels = _setup(g)
    for b in range(int(g["B"])):
        _, _, raster = O.network_loss(w, w_out, p, x[b], int(labels[b]))
        assert np.array_equal(np.packbits(raster, axis=-1), g["raster_packed"][b])


@pytest.mark.parametrize("name", [n for n in SMALL if "f64" in n])
def test_bptt_port_matches_reference(name):
    g = load_golden(name)
    p, w, w_out, x, labels = _setup(g)
    for b in range(int(g["B"])):
        r = O.bptt(w, w_out, p, x[b], int(labels[b]))
        scale = max(np.max(np.abs(g["bptt_w"][b])), 1e-300)
        assert np.max(np.abs(r.grad_w - g["bptt_w"][b])) <= 1e-12 * scale + 1e-300
        # e-prop == BPTT on feed-forward nets (test_gradients.py:157-168)
        assert np.max(np.abs(g["eprop_w"][b] - g["bptt_w"][b])) <= 1e-10


@pytest.mark.parametrize("name", ["c1_lif_f64", "c1_alif_f64", "mid_alif_f64"])
def test_two_pass_batch_matches_reference(name):
    g = load_golden(name)
    p, w, w_out, x, labels = _setup(g)
    r = O.eprop_two_pass_batch(w, w_out, p, x, labels)
    ref = g["eprop_w_batch_sum"]
    assert np.linalg.norm(r.grad_w - ref) <= 1e-12 * np.linalg.norm(ref)
    assert np.linalg.norm(r.grad_w_out - g["eprop_w_out_batch_sum"]) <= \
        1e-12 * np.linalg.norm(g["eprop_w_out_batch_sum"])
    assert np.allclose(r.loss, g["loss"], rtol=1e-12, atol=1e-12)
    packed = np.packbits(r.raster, axis=-1)
    assert np.array_equal(packed, g["raster_packed"])


@pytest.mark.parametrize("name", ["c2_lif_f64", "c3_alif_f64", "c4_alif_f64"])
def test_two_pass_batch_large_shapes(name):
    """SHD-shaped cases: rasters bit-exact, sampled gradient entries and norms."""
    g = load_golden(name)
    p, w, w_out, x, labels = _setup(g)
    r = O.eprop_two_pass_batch(w, w_out, p, x, labels)
    assert np.array_equal(np.packbits(r.raster, axis=-1), g["raster_packed"])
    idx = g["grad_idx"]
    ref = g["eprop_w_batch_sum"]
    got = r.grad_w.ravel()[idx]
    assert np.linalg.norm(got - ref) <= 1e-11 * np.linalg.norm(ref)
    assert abs(np.linalg.norm(r.grad_w) - float(g["eprop_w_batch_norm"])) <= \
        1e-11 * float(g["eprop_w_batch_norm"])
    assert np.allclose(r.loss, g["loss"], rtol=1e-12)


@pytest.mark.parametrize("name", [n for n in SMALL if "f64" in n])
def test_bptt_batch_matches_reference(name):
    """The batched GEMM-form BPTT (checker of the benched configs) against the
    reference's per-sample e-prop and BPTT, summed over the batch (reset on and off)."""
    g = load_golden(name)
    p, w, w_out, x, labels = _setup(g)
    r = O.bptt_batch(w, w_out, p, x, labels)
    for key in ("eprop_w", "bptt_w"):
        ref = g[key].sum(0)
        assert np.linalg.norm(r.grad_w - ref) <= 1e-11 * np.linalg.norm(ref)
    ref_o = g["eprop_w_out"].sum(0)
    assert np.linalg.norm(r.grad_w_out - ref_o) <= 1e-11 * np.linalg.norm(ref_o)
    assert np.allclose(r.loss, g["loss"], rtol=1e-12, atol=1e-12)
    assert np.array_equal(np.packbits(r.raster, axis=-1), g["raster_packed"])


@pytest.mark.parametrize("name", ["c2_lif_f64", "c3_alif_f64", "c4_alif_f64"])
def test_bptt_batch_large_shapes(name):
    """SHD/SSC shapes: bit-exact rasters and the reference's gradient samples."""
    g = load_golden(name)
    p, w, w_out, x, labels = _setup(g)
    r = O.bptt_batch(w, w_out, p, x, labels)
    assert np.array_equal(np.packbits(r.raster, axis=-1), g["raster_packed"])
    ref = g["eprop_w_batch_sum"]
    got = r.grad_w.ravel()[g["grad_idx"]]
    assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)
    assert np.allclose(r.loss, g["loss"], rtol=1e-12)


def test_bptt_batch_equals_two_pass_long_horizon():
    """Long horizon (T = 3000, ALIF, the regime of the >= 10-chunk GPU tests): the
    GEMM-form BPTT and the per-synapse two-pass e-prop restatement agree in f64."""
    p = O.Params(alif=True)
    x, labels = O.poisson_batch(3, 24, 3000, 3, seed=5)
    w, w_out = O.init_network_arrays(16, 24, 3, seed=2)
    w = w * 4.0   # enough drive that neurons spike and adapt over the whole horizon
    a = O.bptt_batch(w, w_out, p, x, labels)
    b = O.eprop_two_pass_batch(w, w_out, p, x, labels)
    assert a.raster.any() and np.array_equal(a.raster, b.raster)
    assert np.linalg.norm(a.grad_w - b.grad_w) <= 1e-10 * np.linalg.norm(b.grad_w)


def test_poisson_generator_statistics():
    x, labels = O.poisson_batch(4, 700, 50, 20, seed=0)
    assert x.dtype == np.uint8 and set(np.unique(x)) <= {0, 1}
    assert 0.08 < x.mean() < 0.13
    assert labels.min() >= 0 and labels.max() < 20


def test_readout_coeffs():
    c = O.readout_coeffs(5, 0.5)
    assert np.allclose(c, [1 + .5 + .25 + .125 + .0625, 1 + .5 + .25 + .125, 1.75, 1.5, 1.0])


def test_hand_values():
    # graph.py:40-52 known answers (test_graph.py:23-36)
    assert O.surrogate_grad(np.array([0.0]))[0] == 1.0
    assert O.surrogate_grad(np.array([0.5]))[0] == pytest.approx(1 / 36)
    assert O.heaviside(np.array([0.0]))[0] == 1.0
    # LIF hand example u=0.5, I=0.6 -> 1.075, spike (test_neurons.py:27-32)
    p = O.Params(alif=False)
    u, a, z, _ = O.step_state(np.array([[0.6]]), p, np.array([0.5]), np.array([0.0]), np.array([1.0]))
    assert u[0] == pytest.approx(1.075) and z[0] == 1.0
