"""Training-loop host logic: the reference's optimizer tests (pkg/tests/test_training.py)
against the drop-in's numpy optimizers, and the CPU oracle's training loop pinned to the
reference's own ``train`` (tests/golden/train_*.npz).  CPU only."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import eprop_ref as O
from paper_2501_11407_b200.errors import ShapeMismatch
from paper_2501_11407_b200.training import (AdamState, NetworkSpec, adam_update, init_network,
                                            sgd_update)

TRAIN = ["train_lif_sgd_f64", "train_alif_adam_f64", "train_lif_adam_f32", "train_alif_sgd_f32"]


class TestOptimizers:
    def test_sgd_zero_grad_is_noop(self):
        p = {"w": np.ones((2, 2))}
        out = sgd_update(p, {"w": np.zeros((2, 2))}, 0.1)
        assert np.array_equal(out["w"], p["w"])

    def test_sgd_exact_step(self):
        out = sgd_update({"w": np.array([1.0, 2.0])}, {"w": np.array([0.5, -0.5])}, 0.1)
        assert np.allclose(out["w"], [0.95, 2.05])

    def test_sgd_shape_mismatch(self):
        with pytest.raises(ShapeMismatch):
            sgd_update({"w": np.ones(2)}, {"w": np.ones(3)}, 0.1)

    def test_adam_first_step_magnitude(self):
        for scale in (1e-4, 1.0, 1e4):
            out = adam_update({"w": np.zeros(3)}, {"w": np.full(3, scale)}, 0.01, AdamState())
            assert np.allclose(np.abs(out["w"]), 0.01, rtol=1e-4)

    def test_adam_state_advances(self):
        st = AdamState()
        p, g = {"w": np.zeros(2)}, {"w": np.ones(2)}
        adam_update(p, g, 0.01, st)
        adam_update(p, g, 0.01, st)
        assert st.t == 2

    def test_init_network(self):
        spec = NetworkSpec(seed=3)
        a, b = init_network(spec), init_network(spec)
        assert np.array_equal(a.neuron.w, b.neuron.w)
        assert init_network(NetworkSpec(precision="f32")).neuron.w.dtype == np.float32
        assert init_network(NetworkSpec(kind="alif")).neuron.beta == 0.8
        with pytest.raises(ValueError):
            init_network(NetworkSpec(kind="izhikevich"))


def _golden_setup(g):
    dt = np.float64 if str(g["precision"]) == "f64" else np.float32
    w, wo = O.init_network_arrays(int(g["n"]), int(g["k"]), int(g["m"]), seed=int(g["seed"]),
                                  dtype=dt)
    x, y = O.poisson_batch(int(g["N"]), int(g["k"]), int(g["T"]), int(g["m"]), seed=int(g["seed"]))
    mu = int(g["max_updates"])
    return w, wo, x, y, (None if mu < 0 else mu)


@pytest.mark.parametrize("name", TRAIN)
def test_oracle_training_loop_matches_reference(name):
    g = load_golden(name)
    w, wo, x, y, mu = _golden_setup(g)
    w2, wo2, rows = O.train_online(w, wo, O.Params(alif=str(g["kind"]) == "alif"), x, y,
                                   str(g["optimizer"]), float(g["lr"]), int(g["epochs"]), mu)
    assert [r[0] for r in rows] == list(g["epoch"])
    assert np.allclose([r[1] for r in rows], g["loss"], rtol=1e-12, atol=1e-12)
    assert np.array_equal([r[2] for r in rows], g["accuracy"])
    tol = 0 if w.dtype == np.float64 else 1e-6
    assert np.max(np.abs(w2 - g["w"])) <= tol * np.max(np.abs(g["w"]))
    assert np.max(np.abs(wo2 - g["w_out"])) <= tol * np.max(np.abs(g["w_out"]))


def test_device_optimizer_kernels_are_exported():
    from paper_2501_11407_b200 import _lib
    lib = _lib.load()
    for name in ("spb_sgd_update", "spb_adam_update"):
        assert hasattr(lib, name)


def test_recurrent_spec_keeps_the_reference_weights():
    """recurrent=True draws W_rec AFTER the reference's two blocks (zero diagonal), so the
    input and readout weights are the reference's; positional constructors unchanged."""
    a = init_network(NetworkSpec(kind="alif", n_hidden=12, n_inputs=7, seed=3))
    b = init_network(NetworkSpec(kind="alif", n_hidden=12, n_inputs=7, seed=3, recurrent=True))
    assert np.array_equal(a.neuron.w, b.neuron.w)
    assert np.array_equal(a.readout.w_out, b.readout.w_out)
    assert a.neuron.w_rec is None and not a.is_recurrent and b.is_recurrent
    assert b.neuron.w_rec.shape == (12, 12) and np.all(np.diag(b.neuron.w_rec) == 0)
    from paper_2501_11407_b200.neurons import ALIFParams
    p = ALIFParams(np.zeros((2, 3)), 0.9, 1.0, 10.0, False, 0.5, 0.9)
    assert p.beta == 0.5 and p.rho == 0.9 and p.w_rec is None
    with pytest.raises(ValueError):
        ALIFParams(np.zeros((2, 3)), w_rec=np.zeros((3, 3)))


def test_oracle_recurrent_with_zero_w_rec_is_the_feed_forward_oracle():
    w, wo = O.init_network_arrays(20, 12, 3, seed=1)
    x, y = O.poisson_batch(2, 12, 60, 3, seed=1)
    for alif in (False, True):
        for rst in (False, True):
            p = O.Params(alif=alif, reset=rst)
            r0 = O.eprop_forward_mode(w, wo, p, x[0].astype(float), int(y[0]))
            r1, ras = O.eprop_forward_mode_rec(w, np.zeros((20, 20)), wo, p,
                                               x[0].astype(float), int(y[0]))
            assert np.array_equal(r0.grad_w, r1.grad_w[:, :12]) and r0.loss == r1.loss
            assert np.array_equal(ras, O.network_loss(w, wo, p, x[0].astype(float),
                                                      int(y[0]))[2])
