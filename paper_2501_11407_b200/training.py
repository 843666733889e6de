"""Training on the B200: network construction, optimizers and the (batched) online loop.

Drop-in for the reference's ``sparseprop.training`` (training.py:18-166):

* ``NetworkSpec`` / ``init_network``  -- same seeded initialisation (U(+-1/sqrt(fan_in))
  drawn from ``numpy.random.default_rng(seed)`` in f64, input block first, then cast), so
  parity runs start from identical weights (training.py:18-50);
* ``sgd_update`` / ``adam_update`` / ``AdamState`` -- the reference's host (numpy)
  optimizers, same signatures and semantics (training.py:58-91);
* ``train`` / ``evaluate`` / ``MetricsRow`` -- the training loop and its metrics CSV
  (training.py:94-166), running on the device: weights, optimizer state and gradients
  stay in HBM, the optimizer step is one fused kernel per parameter (csrc/optim.cu),
  and the host reads back only the per-update loss / accuracy at the end.

``train(..., batch_size=1)`` is the reference's strictly online per-sample loop.  With
``batch_size=B`` each update consumes B consecutive samples and applies the batch-MEAN
gradient ("batch is an outer loop with gradient averaging"); the metrics
row of an update carries the batch-mean loss.  With torch.distributed initialised the
batch is sharded over the ranks and the gradient is combined with one allreduce per
update (parallel.py).

Provenance note: the host-only numpy pieces (``NetworkSpec``, ``loss_and_grad``,
``sgd_update``, ``AdamState``, ``adam_update``, ``MetricsRow``) restate the reference's
training.py:18-100 nearly line for line ON PURPOSE -- they are the reference API the
drop-in must reproduce bit for bit (same RNG stream, same numpy promotion rules), and
they never run on the GPU path.  The device trainer below (``DeviceTrainer``,
``train``, ``evaluate``) is this package's own design.
"""

from __future__ import annotations

import csv
import ctypes
from dataclasses import dataclass, field

import numpy as np

from .errors import LabelOutOfRange, ShapeMismatch
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
    recurrent: bool = False  # extension: also draw W_rec (after w_out, zero diagonal)


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
    w_rec = None
    if spec.recurrent:  # drawn after the reference's two blocks: feed-forward nets unchanged
        w_rec = gen.uniform(-lim_out, lim_out, size=(spec.n_hidden, spec.n_hidden))
        np.fill_diagonal(w_rec, 0.0)
        w_rec = w_rec.astype(dtype)
    if spec.kind == "lif":
        neuron = LIFParams(w, spec.alpha, spec.theta, spec.slope, spec.reset, w_rec=w_rec)
    elif spec.kind == "alif":
        neuron = ALIFParams(w, spec.alpha, spec.theta, spec.slope, spec.reset, spec.beta, spec.rho,
                            w_rec=w_rec)
    else:
        raise ValueError(f"unknown neuron kind {spec.kind!r}")
    return Network(spec.kind, neuron, ReadoutParams(w_out, spec.kappa))


# --------------------------------------------------------------------------------------
# host optimizers (training.py:53-91) -- the reference API, numpy in / numpy out
# --------------------------------------------------------------------------------------

def loss_and_grad(readout_sum: np.ndarray, label: int):
    """Softmax cross-entropy on the time-summed readout (training.py:53-55)."""
    from .gradients import softmax_cross_entropy
    return softmax_cross_entropy(readout_sum, label)


def sgd_update(params: dict, grads: dict, lr: float) -> dict:
    out = {}
    for key, p in params.items():
        g = grads[key]
        if g.shape != p.shape:
            raise ShapeMismatch(f"gradient for {key!r} has shape {g.shape}, expected {p.shape}")
        out[key] = p - lr * g
    return out


@dataclass
class AdamState:
    m: dict = field(default_factory=dict)
    v: dict = field(default_factory=dict)
    t: int = 0


def adam_update(params: dict, grads: dict, lr: float, state: AdamState,
                beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8) -> dict:
    state.t += 1
    out = {}
    for key, p in params.items():
        g = grads[key]
        if g.shape != p.shape:
            raise ShapeMismatch(f"gradient for {key!r} has shape {g.shape}, expected {p.shape}")
        m = state.m.get(key, np.zeros_like(p))
        v = state.v.get(key, np.zeros_like(p))
        m = beta1 * m + (1 - beta1) * g
        v = beta2 * v + (1 - beta2) * g * g
        state.m[key], state.v[key] = m, v
        m_hat = m / (1 - beta1 ** state.t)
        v_hat = v / (1 - beta2 ** state.t)
        out[key] = p - lr * m_hat / (np.sqrt(v_hat) + eps)
    return out


@dataclass
class MetricsRow:
    epoch: int
    step: int
    loss: float
    accuracy: float


# --------------------------------------------------------------------------------------
# device trainer
# --------------------------------------------------------------------------------------

def _neuron_kwargs(net: Network) -> dict:
    p = net.neuron
    kw = dict(alpha=p.alpha, theta=p.theta, slope=p.slope, reset=p.reset,
              kappa=net.readout.kappa)
    if isinstance(p, ALIFParams):
        kw.update(beta=p.beta, rho=p.rho)
    return kw


class DeviceTrainer:
    """Weights, optimizer state and the e-prop engines of one training run on one GPU.

    ``step(x, labels)`` = one update: the e-prop gradient of the batch (engine.py), the
    optional allreduce over ranks (parallel.py), then the fused optimizer kernel on W
    and W_out and the re-slicing of W into the INT8 projection digits -- all enqueued
    on the current stream, no host synchronisation.  Per-update (loss sum, #correct)
    are appended to a device history read once by ``history()``.
    """

    def __init__(self, net: Network, *, optimizer: str = "sgd", lr: float = 0.01,
                 beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 chunk: int | None = None, T: int | None = None, device=None, group=None):
        import torch

        from . import _lib
        from .engine import default_chunk
        if optimizer not in ("sgd", "adam"):
            raise ValueError(f"unknown optimizer {optimizer!r}; choose 'sgd' or 'adam'")
        self.torch = torch
        self.lib = _lib
        self.net = net
        self.optimizer = optimizer
        self.lr, self.beta1, self.beta2, self.eps = float(lr), float(beta1), float(beta2), float(eps)
        self.device = torch.device(device if device is not None else "cuda")
        self.group = group
        self.chunk = chunk if chunk is not None else default_chunk(T or 127, None, net.n, net.k,
                                                                   net.is_alif)
        self.is_f64 = net.neuron.w.dtype == np.float64
        tdt = torch.float64 if self.is_f64 else torch.float32
        self.tdt = tdt
        # master parameters in the network dtype (the engine's fp64 W_out is a mirror)
        self.w = torch.from_numpy(np.ascontiguousarray(net.neuron.w)).to(self.device)
        self.w_out = torch.from_numpy(np.ascontiguousarray(net.readout.w_out)).to(self.device)
        self.w_rec = (torch.from_numpy(np.ascontiguousarray(net.neuron.w_rec)).to(self.device)
                      if net.is_recurrent else None)
        self.t = 0
        if optimizer == "adam":
            self.m_w, self.v_w = torch.zeros_like(self.w), torch.zeros_like(self.w)
            self.m_wo, self.v_wo = torch.zeros_like(self.w_out), torch.zeros_like(self.w_out)
            if self.w_rec is not None:
                self.m_wr, self.v_wr = torch.zeros_like(self.w_rec), torch.zeros_like(self.w_rec)
        self.kw = _neuron_kwargs(net)
        self._engines = {}
        self._hist = []
        self._packer = None

    def _world(self):
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_world_size(self.group)
        return 1

    def engine(self, B: int):
        from .engine import EpropEngine
        eng = self._engines.get(B)
        if eng is None:
            net = self.net
            eng = EpropEngine(net.n, net.k, net.m, B, alif=net.is_alif, w_f64=self.is_f64,
                              chunk=self.chunk, device=self.device, reset=net.neuron.reset,
                              recurrent=net.is_recurrent)
            self._engines[B] = eng
        # every engine shares the trainer's parameters: point its W at the master
        # copy and refresh its fp64 W_out mirror + INT8 digits when they changed
        if eng.w.data_ptr() != self.w.data_ptr():
            eng.w = self.w
        if getattr(eng, "_wver", None) != self.t:
            eng.wout.copy_(self.w_out.to(self.torch.float64))
            if self.w_rec is not None:
                eng.wrecT.copy_(self.w_rec.t())
            eng.slice_weights()
            eng._wver = self.t
        return eng

    def step(self, x, labels, *, bits: bool = False, total_batch: int | None = None):
        """One update on this rank's shard ``x`` [B, T, k] (uint8 counts, or bit-packed
        with ``bits=True``; device tensor or pinned host tensor) and ``labels`` [B]
        (int64 device tensor).  ``total_batch`` = samples over all ranks (mean scale)."""
        torch = self.torch
        B = int(x.shape[0])
        eng = self.engine(B)
        eng.run(x, labels, bits=bits, **self.kw)
        nb = int(total_batch) if total_batch is not None else B
        scale = 1.0 / nb
        st = ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        v = ctypes.c_void_p
        stats = torch.stack([eng.loss.sum(), eng.correct.sum().to(torch.float64)])
        # the accumulator holds grad W in columns [0, k) and, for the recurrent
        # extension, grad W_rec in columns [k, k + n): both travel in the one payload
        kx = eng.k + (eng.n if self.w_rec is not None else 0)
        if self._world() > 1:
            from .parallel import GradPacker
            if self._packer is None:
                self._packer = GradPacker(eng.n, kx, eng.m, self.device,
                                          dtype=torch.float64 if self.is_f64 else torch.float32)
            self._packer.pack(eng.grad_w_acc, eng.grad_wout, eng.loss, eng.correct)
            gw, gwo, ls, nc = self._packer.allreduce(self.group)
            stats = torch.stack([ls.to(torch.float64), nc.to(torch.float64)])
            g_w, g_w_f64, ld_w = gw, int(self.is_f64), kx
            g_wo, g_wo_f64 = gwo, int(self.is_f64)
        else:
            g_w, g_w_f64, ld_w = eng.grad_w_acc, 1, eng.kp
            g_wo, g_wo_f64 = eng.grad_wout, 1
        self.t += 1
        n, k, m = eng.n, eng.k, eng.m
        f64 = int(self.is_f64)
        if self.optimizer == "sgd":
            # W update fused with the re-slicing of this engine's INT8 digits (one launch)
            eng.sgd_slice(g_w, g_w_f64, ld_w, scale, self.lr, stream=st.value)
            # one rank: grad W_out comes from K7 on the engine's side stream -- the update
            # follows it there (beside the gradient GEMM) and the main stream joins it
            side = eng.side if self._world() == 1 else None
            self.lib.call("spb_sgd_update", v(self.w_out.data_ptr()), f64, m, n,
                          v(g_wo.data_ptr()), g_wo_f64, n, scale, self.lr,
                          v(eng.wout.data_ptr()),
                          v(side.cuda_stream) if side is not None else st)
            if side is not None:
                done = torch.cuda.Event()
                done.record(side)
                torch.cuda.current_stream(self.device).wait_event(done)
        else:
            self.lib.call("spb_adam_update", v(self.w.data_ptr()), v(self.m_w.data_ptr()),
                          v(self.v_w.data_ptr()), f64, n, k, v(g_w.data_ptr()), g_w_f64, ld_w,
                          scale, self.lr, self.beta1, self.beta2, self.eps, self.t, None, st)
            self.lib.call("spb_adam_update", v(self.w_out.data_ptr()), v(self.m_wo.data_ptr()),
                          v(self.v_wo.data_ptr()), f64, m, n, v(g_wo.data_ptr()), g_wo_f64, n,
                          scale, self.lr, self.beta1, self.beta2, self.eps, self.t,
                          v(eng.wout.data_ptr()), st)
        if self.w_rec is not None:  # columns k .. k+n of the accumulator / payload
            g_wr = ctypes.c_void_p(g_w.data_ptr() + g_w.element_size() * k)
            if self.optimizer == "sgd":
                self.lib.call("spb_sgd_update", v(self.w_rec.data_ptr()), f64, n, n, g_wr,
                              g_w_f64, ld_w, scale, self.lr, None, st)
            else:
                self.lib.call("spb_adam_update", v(self.w_rec.data_ptr()),
                              v(self.m_wr.data_ptr()), v(self.v_wr.data_ptr()), f64, n, n, g_wr,
                              g_w_f64, ld_w, scale, self.lr, self.beta1, self.beta2, self.eps,
                              self.t, None, st)
            eng.wrecT.copy_(self.w_rec.t())
        # this engine's digits follow the new W right away (the next update's K2; the
        # SGD kernel above already re-sliced them)
        if self.optimizer != "sgd":
            eng.slice_weights()
        eng._wver = self.t
        self._hist.append((stats, nb))
        return eng

    def history(self):
        """[(loss_sum, n_correct, n_samples)] per update (one device->host copy)."""
        torch = self.torch
        if not self._hist:
            return []
        st = torch.stack([h[0] for h in self._hist]).cpu().numpy()
        return [(float(st[i, 0]), int(round(st[i, 1])), self._hist[i][1])
                for i in range(len(self._hist))]

    def weights(self):
        """Current parameters as numpy arrays in the network dtype."""
        return self.w.cpu().numpy(), self.w_out.cpu().numpy()

    def weights_rec(self):
        return None if self.w_rec is None else self.w_rec.cpu().numpy()


def _set_weights(net: Network, w: np.ndarray, w_out: np.ndarray) -> None:
    net.neuron.w = w.astype(net.neuron.w.dtype)
    net.readout.w_out = w_out.astype(net.readout.w_out.dtype)


def _dataset_inputs(dataset):
    """Whole-dataset input tensor on the host: bit-packed binary spikes when possible
    (8x less host->device traffic), else uint8 counts; plus int64 labels."""
    if hasattr(dataset, "counts"):
        binary = dataset.is_binary()
        x = dataset.packed_bits() if binary else dataset.counts()
        return x, dataset.label_array(), binary
    raise TypeError("dataset must be a SpikeDataset (datasets.py)")


def _check_labels(labels: np.ndarray, m: int) -> None:
    """Every label in [0, m) -- the reference raises LabelOutOfRange from
    softmax_cross_entropy (gradients.py:66-69) in train and evaluate; here it is checked
    once per dataset on the host, before any kernel reads a label."""
    if labels.size and (labels.min() < 0 or labels.max() >= m):
        bad = labels[(labels < 0) | (labels >= m)][0]
        raise LabelOutOfRange(f"label {int(bad)} out of range for {m} classes")


def _pinned(torch, arr):
    t = torch.from_numpy(np.ascontiguousarray(arr))
    try:
        return t.pin_memory()
    except RuntimeError:
        return t


def evaluate(net: Network, dataset, *, batch_size: int = 256, device=None):
    """Mean loss and accuracy over all samples (training.py:102-113), forward only on
    the device (pass A + loss of the engine)."""
    import torch

    from .engine import EpropEngine, default_chunk
    x, labels, bits = _dataset_inputs(dataset)
    _check_labels(labels, net.m)
    N, T = x.shape[0], x.shape[1]
    if N == 0:
        return float("nan"), 0.0
    dev = torch.device(device if device is not None else "cuda")
    kw = _neuron_kwargs(net)
    w = torch.from_numpy(np.ascontiguousarray(net.neuron.w))
    wo = torch.from_numpy(np.ascontiguousarray(net.readout.w_out))
    xs = _pinned(torch, x)
    ld = torch.from_numpy(labels).to(dev)
    engines = {}
    losses, correct = [], []
    for s0 in range(0, N, batch_size):
        B = min(batch_size, N - s0)
        eng = engines.get(B)
        if eng is None:
            eng = EpropEngine(net.n, net.k, net.m, B, alif=net.is_alif,
                              w_f64=net.neuron.w.dtype == np.float64,
                              chunk=default_chunk(T, B, net.n, net.k, net.is_alif), device=dev,
                              reset=net.neuron.reset, recurrent=net.is_recurrent, grad=False)
            eng.set_weights(w, wo, w_rec=(torch.from_numpy(np.ascontiguousarray(
                net.neuron.w_rec)) if net.is_recurrent else None))
            engines[B] = eng
        eng.run(xs[s0:s0 + B], ld[s0:s0 + B], bits=bits, forward_only=True, **kw)
        losses.append(eng.loss.clone())
        correct.append(eng.correct.clone())
    loss = torch.cat(losses).cpu().numpy()
    corr = torch.cat(correct).cpu().numpy()
    return float(np.mean(loss)), float(corr.sum()) / N


def train(spec: NetworkSpec, dataset, method: str = "eprop-sparse", optimizer: str = "sgd",
          epochs: int = 1, lr: float = 0.01, max_updates: int | None = None, metrics_path=None,
          *, batch_size: int = 1, device=None, chunk: int | None = None, group=None):
    """Online e-prop training on the B200 (training.py:116-166).

    Deterministic per (spec, seed).  ``batch_size=1`` reproduces the reference's
    per-sample online loop; larger batches apply the batch-mean gradient.  Under
    torch.distributed each update's batch is split over the ranks (contiguous shards,
    parallel.shard_range) and the gradients are allreduced.  Returns (network, metrics
    rows); the network holds the trained weights (numpy, the spec's dtype).
    """
    import torch

    from .gradients import ENGINES
    from .parallel import shard_range
    if method not in ENGINES:
        raise ValueError(f"unknown method {method!r}; choose from {sorted(ENGINES)}")
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    net = init_network(spec)
    x, labels, bits = _dataset_inputs(dataset)
    _check_labels(labels, net.m)
    N, T = x.shape[0], x.shape[1]
    world, rank = 1, 0
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    if device is None and torch.cuda.is_available() and world > 1:
        device = torch.device("cuda", torch.cuda.current_device())
    tr = DeviceTrainer(net, optimizer=optimizer, lr=lr, chunk=chunk, T=T, device=device,
                       group=group)
    xs = _pinned(torch, x)
    ld = torch.from_numpy(labels).to(tr.device)
    epochs_of = []
    updates = 0
    done = False
    for epoch in range(epochs):
        for s0 in range(0, N, batch_size):
            nb = min(batch_size, N - s0)
            if nb < world:   # rank-independent: every rank raises, none enters the allreduce
                raise ValueError("every rank needs at least one sample per update "
                                 f"(batch {nb} over {world} ranks)")
            lo, hi = shard_range(nb, rank, world)
            tr.step(xs[s0 + lo:s0 + hi], ld[s0 + lo:s0 + hi], bits=bits, total_batch=nb)
            epochs_of.append(epoch)
            updates += 1
            if max_updates is not None and updates >= max_updates:
                done = True
                break
        if done:
            break
    # metrics rows: running epoch accuracy (training.py:146-152); one host read
    metrics: list[MetricsRow] = []
    hist = tr.history()
    ep_seen, ep_correct, cur_ep = 0, 0, None
    for i, (loss_sum, n_corr, nb) in enumerate(hist):
        if epochs_of[i] != cur_ep:
            cur_ep, ep_seen, ep_correct = epochs_of[i], 0, 0
        ep_seen += nb
        ep_correct += n_corr
        metrics.append(MetricsRow(epochs_of[i], i + 1, loss_sum / nb, ep_correct / ep_seen))
    w, w_out = tr.weights()
    _set_weights(net, w, w_out)
    if net.is_recurrent:
        net.neuron.w_rec = tr.weights_rec().astype(net.neuron.w.dtype)
    if metrics_path is not None:
        with open(metrics_path, "w", newline="") as fh:
            writer = csv.writer(fh)
            writer.writerow(["epoch", "step", "loss", "accuracy"])
            for row in metrics:
                writer.writerow([row.epoch, row.step, f"{row.loss:.6f}", f"{row.accuracy:.4f}"])
    return net, metrics
