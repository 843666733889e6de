"""Network construction for the drop-in: ``NetworkSpec`` / ``init_network``.

Same seeded initialisation as the reference (training.py:18-50): weights drawn
U(+-1/sqrt(fan_in)) from ``numpy.random.default_rng(seed)`` in f64, input block first,
then cast to the requested precision, so parity runs start from identical weights.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .neurons import ALIFParams, LIFParams, Network, ReadoutParams

_DTYPES = {"f32": np.float32, "f64": np.float64}


@dataclass
class NetworkSpec:
    kind: str = "lif"
    n_hidden: int = 64
    n_inputs: int = 140
    n_classes: int = 3
    alpha: float = 0.95
    theta: float = 1.0
    slope: float = 10.0
    beta: float = 0.8
    rho: float = 0.96
    kappa: float = 0.95
    reset: bool = False
    precision: str = "f64"
    seed: int = 0


def init_network(spec: NetworkSpec) -> Network:
    """Seeded uniform +-1/sqrt(fan_in) initialisation (training.py:35-50)."""
    if spec.precision not in _DTYPES:
        raise ValueError(f"precision must be one of {sorted(_DTYPES)}")
    dtype = _DTYPES[spec.precision]
    gen = np.random.default_rng(spec.seed)
    lim_in = 1.0 / np.sqrt(spec.n_inputs)
    lim_out = 1.0 / np.sqrt(spec.n_hidden)
    w = gen.uniform(-lim_in, lim_in, size=(spec.n_hidden, spec.n_inputs)).astype(dtype)
    w_out = gen.uniform(-lim_out, lim_out, size=(spec.n_classes, spec.n_hidden)).astype(dtype)
    if spec.kind == "lif":
        neuron = LIFParams(w, spec.alpha, spec.theta, spec.slope, spec.reset)
    elif spec.kind == "alif":
        neuron = ALIFParams(w, spec.alpha, spec.theta, spec.slope, spec.reset, spec.beta, spec.rho)
    else:
        raise ValueError(f"unknown neuron kind {spec.kind!r}")
    return Network(spec.kind, neuron, ReadoutParams(w_out, spec.kappa))
