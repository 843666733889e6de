"""Gradient entry points of the drop-in (same names and signatures as the reference).

Reference: /root/reference/pkg/src/sparseprop/gradients.py
  GradResult                 :54-63
  softmax_cross_entropy      :66-75
  eprop_sparse_gradient      :132-185   <- the hot path, here on B200 kernels
  gradient_deviation_stats   :418-433
  ENGINES                    :436-441

``eprop_sparse_gradient(net, x_seq, label)`` keeps the reference's single-sample
contract (numpy in, numpy out, dtype of ``net.neuron.w``).  ``eprop_batch_gradient``
is the batched form the kernels are built for: per-sample losses/readouts and the
batch-SUMMED gradients.  Every number is computed by the CUDA
kernels in libsparseprop_b200.so; there is no CPU path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .engine import EpropEngine, default_chunk
from .errors import LabelOutOfRange, ShapeMismatch
from .neurons import ALIFParams, Network


@dataclass
class DeviationStats:
    median: float
    q_low: float
    q_high: float


@dataclass
class GradResult:
    """Result of one gradient evaluation (gradients.py:54-63)."""

    loss: float
    grads: dict
    readout_sum: np.ndarray
    live_bytes_per_step: list | None = None

    @property
    def prediction(self) -> int:
        return int(np.argmax(self.readout_sum))


@dataclass
class BatchGradResult:
    """Batched e-prop result: per-sample loss/readout, batch-summed gradients."""

    loss: np.ndarray          # [B]
    grads: dict               # {"w": [n, k], "w_out": [m, n]}, summed over the batch
    readout_sum: np.ndarray   # [B, m]
    correct: np.ndarray       # [B] bool, argmax(readout_sum) == label

    @property
    def prediction(self) -> np.ndarray:
        return np.argmax(self.readout_sum, axis=1)


def softmax_cross_entropy(v: np.ndarray, label: int):
    """Loss and dL/dv = softmax(v) - onehot(label) (gradients.py:66-75); host helper."""
    if not 0 <= label < v.shape[0]:
        raise LabelOutOfRange(f"label {label} out of range for {v.shape[0]} classes")
    z = v - np.max(v)
    lse = np.log(np.sum(np.exp(z)))
    p = np.exp(z - lse)
    p[label] -= 1.0
    return float(lse - z[label]), p


_ENGINES: dict = {}


def get_engine(net: Network, B: int, *, chunk: int | None = None, T: int | None = None,
               device=None) -> EpropEngine:
    """Engine cache keyed by shape, neuron kind, weight precision, chunk and device."""
    dev = torch.device(device if device is not None else "cuda")
    if chunk is None:
        chunk = default_chunk(T or 127, B, net.n, net.k, net.is_alif)
    w_f64 = net.neuron.w.dtype == np.float64
    reset = bool(net.neuron.reset)
    rec = net.is_recurrent
    key = (net.n, net.k, net.m, B, net.is_alif, w_f64, chunk, str(dev), reset, rec)
    eng = _ENGINES.get(key)
    if eng is None:
        eng = EpropEngine(net.n, net.k, net.m, B, alif=net.is_alif, w_f64=w_f64, chunk=chunk,
                          device=dev, reset=reset, recurrent=rec)
        _ENGINES[key] = eng
    return eng


def _as_counts(x: np.ndarray) -> np.ndarray:
    """Spike inputs as uint8 event counts (binary spikes or pooled counts <= 255)."""
    if x.dtype == np.uint8:
        return x
    if x.dtype == np.bool_:
        return x.astype(np.uint8)
    xi = np.rint(x)
    if not np.array_equal(xi, x) or (x.size and (x.min() < 0 or x.max() > 255)):
        raise ValueError("inputs must be non-negative integer spike counts <= 255 "
                         "(binary spikes or pooled counts, datasets.py:46-52/138-159)")
    return xi.astype(np.uint8)


def _neuron_kwargs(net: Network) -> dict:
    p = net.neuron
    kw = dict(alpha=p.alpha, theta=p.theta, slope=p.slope, reset=p.reset, kappa=net.readout.kappa)
    if isinstance(p, ALIFParams):
        kw.update(beta=p.beta, rho=p.rho)
    return kw


def eprop_batch_gradient(net: Network, x, labels, *, chunk: int | None = None,
                         device=None, smooth: bool = False) -> BatchGradResult:
    """Batched online e-prop on the B200: x [B, T, k] spike counts, labels [B].

    Returns per-sample losses and readout sums and the gradients SUMMED over the batch
    (= sum of the reference's per-sample ``eprop_sparse_gradient`` grads).  ``smooth``
    replaces the hard threshold by surrogate_smooth in the forward (graph.py:45-47), the
    reference's finite-difference mode (gradients.py:114-115).
    """
    x = np.asarray(x)
    if x.ndim != 3 or x.shape[2] != net.k:
        raise ShapeMismatch(f"x must be [B, T, k={net.k}], got {x.shape}")
    labels = np.asarray(labels, dtype=np.int64).reshape(-1)
    B, T = x.shape[0], x.shape[1]
    if labels.shape[0] != B:
        raise ShapeMismatch("one label per sample required")
    if B and (labels.min() < 0 or labels.max() >= net.m):
        bad = labels[(labels < 0) | (labels >= net.m)][0]
        raise LabelOutOfRange(f"label {int(bad)} out of range for {net.m} classes")
    xc = np.ascontiguousarray(_as_counts(x))
    eng = get_engine(net, B, chunk=chunk, T=T, device=device)
    dev = eng.device
    xd = torch.from_numpy(xc).to(dev)
    ld = torch.from_numpy(labels).to(dev)
    eng.set_weights(torch.from_numpy(np.ascontiguousarray(net.neuron.w)),
                    torch.from_numpy(np.ascontiguousarray(net.readout.w_out)),
                    w_rec=(torch.from_numpy(np.ascontiguousarray(net.neuron.w_rec))
                           if net.is_recurrent else None))
    eng.run(xd, ld, smooth=smooth, **_neuron_kwargs(net))
    wdt = torch.float64 if net.neuron.w.dtype == np.float64 else torch.float32
    gw = eng.grad_w(wdt)
    gwo = eng.grad_wout.to(wdt)
    out_dtype = net.neuron.w.dtype
    grads = {"w": gw.cpu().numpy().astype(out_dtype, copy=False),
             "w_out": gwo.cpu().numpy().astype(out_dtype, copy=False)}
    if net.is_recurrent:
        grads["w_rec"] = eng.grad_w_rec(wdt).cpu().numpy().astype(out_dtype, copy=False)
    return BatchGradResult(
        loss=eng.loss.cpu().numpy().copy(),
        grads=grads,
        readout_sum=eng.s.cpu().numpy().astype(out_dtype),
        correct=eng.correct.cpu().numpy().astype(bool),
    )


def eprop_sparse_gradient(net: Network, x_seq: np.ndarray, label: int,
                          smooth: bool = False) -> GradResult:
    """Online sparse e-prop for one sample -- the reference entry point (gradients.py:132).

    Same contract: ``x_seq`` [T, k], integer ``label``; returns the loss, the gradients
    {"w": [n, k], "w_out": [m, n]} in the dtype of ``net.neuron.w`` and the time-summed
    readout.  Inputs must be spike counts (binary or pooled integers).
    """
    x_seq = np.asarray(x_seq)
    if x_seq.ndim != 2 or x_seq.shape[1] != net.k:
        raise ShapeMismatch(f"x_seq must be [T, k={net.k}], got {x_seq.shape}")
    if not 0 <= int(label) < net.m:
        raise LabelOutOfRange(f"label {label} out of range for {net.m} classes")
    r = eprop_batch_gradient(net, x_seq[None], np.array([int(label)]), smooth=smooth)
    return GradResult(float(r.loss[0]), r.grads, r.readout_sum[0], None)


def gradient_deviation_stats(g1, g2) -> DeviationStats:
    """Median and 2.5/97.5 % quantiles of |g1 - g2| over all parameters (gradients.py:418-433)."""

    def flat(g):
        if isinstance(g, (GradResult, BatchGradResult)):
            g = g.grads
        if isinstance(g, dict):
            return np.concatenate([np.asarray(g[key]).ravel() for key in sorted(g)])
        return np.asarray(g).ravel()

    a, b = flat(g1), flat(g2)
    if a.shape != b.shape:
        raise ShapeMismatch("gradient shapes disagree")
    d = np.abs(a.astype(np.float64) - b.astype(np.float64))
    lo, med, hi = np.quantile(d, [0.025, 0.5, 0.975], method="linear")
    return DeviationStats(float(med), float(lo), float(hi))


ENGINES = {
    "eprop-sparse": eprop_sparse_gradient,
}
