"""Neuron-model parameter types of the drop-in (same names/fields as the reference).

The reference defines these in /root/reference/pkg/src/sparseprop/neurons.py:30-101;
callers construct them the same way here.  Only the parameter containers live on the
host: the per-step dynamics (neurons.py:109-137) and the step Jacobians
(neurons.py:246-279) are evaluated in closed form inside the CUDA kernels
(csrc/forward.cu, csrc/elig.cu).
"""

from __future__ import annotations

from dataclasses import KW_ONLY, dataclass

import numpy as np

DEFAULT_SLOPE = 10.0  # graph.py:37


@dataclass
class LIFParams:
    """Leaky integrate-and-fire layer: ``w`` is [n, k] (neurons.py:30-50)."""

    w: np.ndarray
    alpha: float = 0.95
    theta: float = 1.0
    slope: float = DEFAULT_SLOPE
    reset: bool = False
    _: KW_ONLY
    # recurrent extension (not in the reference, parity unpinned):
    # W_rec [n, n] feeding z_{t-1} back into the current; None = the reference's
    # feed-forward layer.  Keyword-only so the reference's positional constructors
    # (LIFParams(w, alpha, theta, slope, reset), ALIFParams(..., beta, rho)) are unchanged.
    w_rec: np.ndarray | None = None

    def __post_init__(self):
        if not (0.0 < self.alpha < 1.0):
            raise ValueError("alpha must be in (0, 1)")
        if not self.theta > 0.0:
            raise ValueError("theta must be positive")
        if self.w_rec is not None and np.shape(self.w_rec) != (self.n, self.n):
            raise ValueError("w_rec must be [n, n]")

    @property
    def n(self) -> int:
        return int(self.w.shape[0])

    @property
    def k(self) -> int:
        return int(self.w.shape[1])


@dataclass
class ALIFParams(LIFParams):
    """Adaptive-threshold LIF: threshold theta + beta*a, a <- rho*a + z (neurons.py:53-63)."""

    beta: float = 0.8
    rho: float = 0.96

    def __post_init__(self):
        super().__post_init__()
        if self.beta < 0.0:
            raise ValueError("beta must be non-negative")
        if not (0.0 < self.rho < 1.0):
            raise ValueError("rho must be in (0, 1)")


@dataclass
class ReadoutParams:
    """Leaky non-spiking readout v <- kappa*v + W_out z, ``w_out`` [m, n] (neurons.py:73-80)."""

    w_out: np.ndarray
    kappa: float = 0.95

    def __post_init__(self):
        if not (0.0 < self.kappa < 1.0):
            raise ValueError("kappa must be in (0, 1)")


@dataclass
class Network:
    """One hidden spiking layer plus the leaky readout (neurons.py:83-101)."""

    kind: str  # "lif" | "alif"
    neuron: LIFParams
    readout: ReadoutParams

    @property
    def n(self) -> int:
        return self.neuron.n

    @property
    def k(self) -> int:
        return self.neuron.k

    @property
    def m(self) -> int:
        return int(self.readout.w_out.shape[0])

    @property
    def is_alif(self) -> bool:
        return isinstance(self.neuron, ALIFParams)

    @property
    def is_recurrent(self) -> bool:
        return self.neuron.w_rec is not None
