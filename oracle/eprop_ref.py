"""CPU oracle for the e-prop training step -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``sparseprop`` 0.1.0
(arXiv 2501.11407 artifact, ``/root/reference/pkg/src/sparseprop``) for the one hot
path this repository rebuilds on B200: ``eprop_sparse_gradient``
(``gradients.py:132-185``).  It exists so that ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs have a checker and a
CPU timing arm.  The product package ``paper_2501_11407_b200`` never imports it:
there is no CPU fallback on the product path.

Parity of this restatement is PINNED: ``tests/golden/make_golden.py`` ran the
reference itself (imported from ``/root/reference/pkg/src`` in the build
container) and stored its outputs in ``tests/golden/*.npz``;
``tests/test_oracle.py`` checks every function here against those fixtures
(bit-identical rasters, gradients to <=1e-12 relative in f64).

Contents
--------
* ``surrogate_grad``, ``surrogate_smooth``, ``heaviside``  -- ``graph.py:40-52``
* ``step_state``                       -- ``gradients.py:118-129`` (``_step_state``)
* ``softmax_cross_entropy``            -- ``gradients.py:66-75``
* ``eprop_forward_mode``               -- ``gradients.py:132-185`` restated with the
  closed-form step Jacobians of ``neurons.py:246-279`` (pinned by
  ``test_neurons.py:127-155``): per-sample, per-step, per-synapse traces exactly
  as the reference carries them.  This is the CPU baseline ("port").
* ``bptt``                             -- ``gradients.py:188-231``
* ``network_loss``                     -- ``gradients.py:349-365`` (spike raster)
* ``eprop_two_pass_batch``             -- the batched two-pass form the GPU kernels
  implement, vectorised over the batch; the fast checker for
  large batches.
* ``init_network_arrays``              -- ``training.py:35-50``
* ``poisson_batch``                    -- vectorised ``generate_poisson_dataset``
  (``datasets.py:60-83``), same RNG call sequence, bit-identical output.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


# --------------------------------------------------------------------------------------
# elementwise pieces (graph.py:40-52)
# --------------------------------------------------------------------------------------

def surrogate_grad(x, slope=10.0):
    """sigma'(x) = 1 / (1 + slope*|x|)^2  -- graph.py:40-42."""
    return 1.0 / (1.0 + slope * np.abs(x)) ** 2


def surrogate_smooth(x, slope=10.0):
    """Smooth spike 0.5 + x/(1+slope|x|) -- graph.py:45-47."""
    return 0.5 + x / (1.0 + slope * np.abs(x))


def heaviside(x):
    """Theta(x) = [x >= 0] in x.dtype (tie spikes) -- graph.py:50-52."""
    return (x >= 0.0).astype(x.dtype)


def _spike(x, slope, smooth):
    # gradients.py:114-115
    return surrogate_smooth(x, slope) if smooth else heaviside(x)


@dataclass
class Params:
    """Hyper-parameters of one network (neurons.py:30-80); beta=rho=0 means LIF."""

    alif: bool
    alpha: float = 0.95
    theta: float = 1.0
    slope: float = 10.0
    reset: bool = False
    beta: float = 0.8
    rho: float = 0.96
    kappa: float = 0.95

    @property
    def beta_eff(self):
        return self.beta if self.alif else 0.0

    @property
    def rho_eff(self):
        return self.rho if self.alif else 0.0


def step_state(w, p: Params, u, a, x_t, smooth=False):
    """One forward step; returns (u', a', z', psi') -- gradients.py:118-129."""
    beta, rho = p.beta_eff, p.rho_eff
    z = _spike(u - p.theta - beta * a, p.slope, smooth)
    a_next = rho * a + z
    u_next = p.alpha * u + w @ x_t
    if p.reset:
        u_next = u_next - p.theta * z
    drive = u_next - p.theta - beta * a_next
    return u_next, a_next, _spike(drive, p.slope, smooth), surrogate_grad(drive, p.slope)


def softmax_cross_entropy(v, label):
    """(loss, softmax(v) - onehot(label)) -- gradients.py:66-75."""
    if not 0 <= label < v.shape[0]:
        raise ValueError(f"label {label} out of range for {v.shape[0]} classes")
    shifted = v - np.max(v)
    logz = np.log(np.sum(np.exp(shifted)))
    loss = float(logz - shifted[label])
    grad = np.exp(shifted - logz)
    grad[label] -= 1.0
    return loss, grad


# --------------------------------------------------------------------------------------
# per-sample engines
# --------------------------------------------------------------------------------------

@dataclass
class Result:
    loss: float
    grad_w: np.ndarray
    grad_w_out: np.ndarray
    readout_sum: np.ndarray


def eprop_forward_mode(w, w_out, p: Params, x_seq, label, smooth=False) -> Result:
    """Online sparse e-prop for one sample, restating gradients.py:132-185.

    The per-step Jacobians the reference derives by vertex elimination
    (neurons.py:246-279) are used in their closed form (test_neurons.py:127-155):
      LIF   H_I = diag(alpha - rst*theta*psi^-)
      ALIF  H_I = [[alpha - rst*theta*psi^-, rst*theta*beta*psi^-],
                   [psi^-,                  rho - beta*psi^-     ]]   per neuron
      F     rows = x_t on the u component, 0 on the a component.
    The trace G = (G_u, G_a) is carried per synapse ([n, k] each) exactly as the
    reference's compressed tensors store it (gradients.py:78-94).
    """
    dtype = w.dtype
    n, k = w.shape
    m = w_out.shape[0]
    T = x_seq.shape[0]
    beta, rho = p.beta_eff, p.rho_eff
    rst = 1.0 if p.reset else 0.0
    u = np.zeros(n, dtype=dtype)
    a = np.zeros(n, dtype=dtype)
    g_u = np.zeros((n, k), dtype=dtype)          # gradients.py:148 (initial_trace)
    g_a = np.zeros((n, k), dtype=dtype) if p.alif else None
    xbar = np.zeros((n, k), dtype=dtype)         # gradients.py:149
    xsum = np.zeros((n, k), dtype=dtype)         # gradients.py:150
    zbar = np.zeros(n, dtype=dtype)
    zsum = np.zeros(n, dtype=dtype)
    v = np.zeros(m, dtype=dtype)
    s = np.zeros(m, dtype=dtype)
    for t in range(T):                           # gradients.py:157
        x_t = x_seq[t]
        psi_prev = surrogate_grad(u - p.theta - beta * a, p.slope)
        # eprop_trace_update: G <- H_I G + F  (gradients.py:89-94)
        h_uu = p.alpha - rst * p.theta * psi_prev
        if p.alif:
            h_ua = rst * p.theta * beta * psi_prev
            h_au = psi_prev
            h_aa = rho - beta * psi_prev
            g_u_new = h_uu[:, None] * g_u + h_ua[:, None] * g_a + x_t[None, :]
            g_a = h_au[:, None] * g_u + h_aa[:, None] * g_a
            g_u = g_u_new
        else:
            g_u = h_uu[:, None] * g_u + x_t[None, :]
        u, a, z, sg = step_state(w, p, u, a, x_t, smooth)      # gradients.py:162
        v = p.kappa * v + w_out @ z                             # gradients.py:163
        s = s + v                                               # gradients.py:164
        if p.alif:                                              # gradients.py:165-169
            x_step = sg[:, None] * (g_u - beta * g_a)
        else:
            x_step = sg[:, None] * g_u
        xbar *= p.kappa                                         # gradients.py:170-172
        xbar += x_step
        xsum += xbar
        zbar = p.kappa * zbar + z                               # gradients.py:173-174
        zsum = zsum + zbar
    loss, g = softmax_cross_entropy(s, label)                   # gradients.py:177
    w_sig = w_out.T @ g                                         # gradients.py:178
    return Result(loss, (w_sig[:, None] * xsum).astype(dtype),
                  np.outer(g, zsum).astype(dtype), s)


def bptt(w, w_out, p: Params, x_seq, label, smooth=False) -> Result:
    """Reverse sweep over stored states -- gradients.py:188-231."""
    dtype = w.dtype
    n = w.shape[0]
    m = w_out.shape[0]
    T = x_seq.shape[0]
    u = np.zeros(n, dtype=dtype)
    a = np.zeros(n, dtype=dtype)
    zs = np.zeros((T, n), dtype=dtype)
    sgs = np.zeros((T, n), dtype=dtype)
    v = np.zeros(m, dtype=dtype)
    s = np.zeros(m, dtype=dtype)
    for t in range(T):
        u, a, z, sg = step_state(w, p, u, a, x_seq[t], smooth)
        zs[t], sgs[t] = z, sg
        v = p.kappa * v + w_out @ z
        s = s + v
    loss, g = softmax_cross_entropy(s, label)
    grad_w = np.zeros_like(w)
    grad_w_out = np.zeros_like(w_out)
    lam_u = np.zeros(n, dtype=dtype)
    lam_a = np.zeros(n, dtype=dtype)
    c_t = 0.0
    for t in range(T - 1, -1, -1):
        c_t = 1.0 + p.kappa * c_t
        lam_v = c_t * g
        mu = w_out.T @ lam_v
        grad_w_out += np.outer(lam_v, zs[t])
        xi = mu
        if p.alif:
            xi = xi + lam_a
        if p.reset:
            xi = xi - p.theta * lam_u
        new_lam_u = p.alpha * lam_u + xi * sgs[t]
        if p.alif:
            lam_a = p.rho * lam_a - p.beta * xi * sgs[t]
        lam_u = new_lam_u
        grad_w += np.outer(lam_u, x_seq[t])
    return Result(loss, grad_w, grad_w_out, s)


def network_loss(w, w_out, p: Params, x_seq, label, smooth=False):
    """Forward-only loss, readout sum and bool spike raster -- gradients.py:349-365."""
    dtype = w.dtype
    n = w.shape[0]
    m = w_out.shape[0]
    u = np.zeros(n, dtype=dtype)
    a = np.zeros(n, dtype=dtype)
    v = np.zeros(m, dtype=dtype)
    s = np.zeros(m, dtype=dtype)
    raster = np.zeros((x_seq.shape[0], n), dtype=bool)
    for t in range(x_seq.shape[0]):
        u, a, z, _ = step_state(w, p, u, a, x_seq[t], smooth)
        raster[t] = z > 0.5
        v = p.kappa * v + w_out @ z
        s = s + v
    loss, _ = softmax_cross_entropy(s, label)
    return loss, s, raster


# --------------------------------------------------------------------------------------
# batched two-pass form (what the kernels compute)
# --------------------------------------------------------------------------------------

@dataclass
class BatchResult:
    loss: np.ndarray          # [B]
    readout_sum: np.ndarray   # [B, m]
    grad_w: np.ndarray        # [n, k]   summed over the batch
    grad_w_out: np.ndarray    # [m, n]   summed over the batch
    raster: np.ndarray        # [B, T, n] bool
    zsum: np.ndarray          # [B, n]


def readout_coeffs(T, kappa):
    """c_t = sum_{tau=t}^{T-1} kappa^(tau-t), the readout filter gain seen by step t."""
    c = np.empty(T)
    acc = 0.0
    for t in range(T - 1, -1, -1):
        acc = 1.0 + kappa * acc
        c[t] = acc
    return c


def eprop_two_pass_batch(w, w_out, p: Params, x, labels, dtype=np.float64) -> BatchResult:
    """Batched e-prop in the two-pass closed form, rst=0 (the default, neurons.py:36).

    Pass A: forward, time-summed readout s (gradients.py:163-164), loss and
    g = softmax - onehot, w_sig = W_out^T g, L_t = c_t * w_sig.
    Pass B: the same forward again with the traces
      xbar_t = alpha*xbar_{t-1} + x_t                       (LIF G_u, factorised)
      eps_t  = (rho - beta psi_{t-1}) eps_{t-1} + psi_{t-1} (x) xbar_{t-1}   (ALIF G_a)
    and grad_W = sum_{b,t} (L_t psi_t)[b,i] * (xbar_t[b,j] - beta*eps_t[b,i,j]).
    """
    if p.reset:
        raise NotImplementedError("two-pass batch oracle covers reset=False")
    w = w.astype(dtype)
    w_out = w_out.astype(dtype)
    x = x.astype(dtype)
    B, T, k = x.shape
    n, m = w.shape[0], w_out.shape[0]
    beta, rho = p.beta_eff, p.rho_eff

    def forward():
        u = np.zeros((B, n), dtype)
        a = np.zeros((B, n), dtype)
        for t in range(T):
            z_prev = heaviside(u - p.theta - beta * a)
            a = rho * a + z_prev
            u = p.alpha * u + x[:, t, :] @ w.T
            d = u - p.theta - beta * a
            yield t, heaviside(d), surrogate_grad(d, p.slope)

    raster = np.zeros((B, T, n), dtype=bool)
    zbar = np.zeros((B, n), dtype)
    zsum = np.zeros((B, n), dtype)
    v = np.zeros((B, m), dtype)
    s = np.zeros((B, m), dtype)
    for t, z, _ in forward():
        raster[:, t] = z > 0.5
        v = p.kappa * v + z @ w_out.T
        s = s + v
        zbar = p.kappa * zbar + z
        zsum = zsum + zbar
    loss = np.zeros(B)
    g = np.zeros((B, m), dtype)
    for b in range(B):
        loss[b], g[b] = softmax_cross_entropy(s[b], int(labels[b]))
    w_sig = g @ w_out                                   # [B, n]
    c = readout_coeffs(T, p.kappa).astype(dtype)

    grad_w = np.zeros((n, k), dtype)
    xbar = np.zeros((B, k), dtype)
    eps = np.zeros((B, n, k), dtype) if p.alif else None
    psi_prev = None
    for t, z, psi in forward():
        if p.alif and t > 0:
            eps = (rho - beta * psi_prev)[:, :, None] * eps + psi_prev[:, :, None] * xbar[:, None, :]
        xbar = p.alpha * xbar + x[:, t, :]
        lpsi = c[t] * w_sig * psi                        # [B, n]
        grad_w += lpsi.T @ xbar
        if p.alif:
            grad_w -= beta * np.einsum("bi,bij->ij", lpsi, eps)
        psi_prev = psi
    grad_w_out = g.T @ zsum
    return BatchResult(loss, s, grad_w, grad_w_out, raster, zsum)


def bptt_batch(w, w_out, p: Params, x, labels, dtype=np.float64, smooth=False) -> BatchResult:
    """Batched ``bptt_gradient`` (gradients.py:188-231) in GEMM form: the checker for the
    benched configurations (C3 at B=256, C4 at B=128), where the per-synapse e-prop
    restatement would take hours in numpy.

    For the reference's feed-forward layer e-prop is the exact gradient (the reference
    pins sparse e-prop == BPTT to <=1e-10 in f64, test_gradients.py:157-194, reset on and
    off), so this is an oracle for ``eprop_sparse_gradient`` summed over the batch.
    Forward: one [B*T, k] x [k, n] GEMM for every step's current (x is integer counts,
    so the f64 sums differ from the reference's matvec only in the last ulp), then the
    per-step state update of gradients.py:118-129 over [B, n].  Reverse sweep exactly as
    gradients.py:216-230, storing lambda_u per step; grad_W = one [n, B*T] x [B*T, k] GEMM.
    """
    w = np.asarray(w).astype(dtype)
    w_out = np.asarray(w_out).astype(dtype)
    B, T, k = x.shape
    n, m = w.shape[0], w_out.shape[0]
    beta, rho = p.beta_eff, p.rho_eff
    xf = x.reshape(B * T, k).astype(dtype)
    cur = (xf @ w.T).reshape(B, T, n)                  # every step's W x_t
    sgs = np.empty((B, T, n), dtype)
    raster = np.zeros((B, T, n), dtype=bool)
    u = np.zeros((B, n), dtype)
    a = np.zeros((B, n), dtype)
    v = np.zeros((B, m), dtype)
    s = np.zeros((B, m), dtype)
    zbar = np.zeros((B, n), dtype)
    zsum = np.zeros((B, n), dtype)
    for t in range(T):                                  # gradients.py:118-129
        z_prev = _spike(u - p.theta - beta * a, p.slope, smooth)
        a = rho * a + z_prev
        u = p.alpha * u + cur[:, t]
        if p.reset:
            u = u - p.theta * z_prev
        d = u - p.theta - beta * a
        z = _spike(d, p.slope, smooth)
        sgs[:, t] = surrogate_grad(d, p.slope)
        raster[:, t] = z > 0.5
        cur[:, t] = z                                   # z_t kept for the readout grad
        v = p.kappa * v + z @ w_out.T
        s = s + v
        zbar = p.kappa * zbar + z
        zsum = zsum + zbar
    loss = np.zeros(B)
    g = np.zeros((B, m), dtype)
    for b in range(B):
        loss[b], g[b] = softmax_cross_entropy(s[b], int(labels[b]))
    lam_u = np.zeros((B, n), dtype)
    lam_a = np.zeros((B, n), dtype)
    c_t = 0.0
    mu0 = g @ w_out                                      # W_out^T g per sample
    for t in range(T - 1, -1, -1):                      # gradients.py:216-230
        c_t = 1.0 + p.kappa * c_t
        xi = c_t * mu0
        if p.alif:
            xi = xi + lam_a
        if p.reset:
            xi = xi - p.theta * lam_u
        new_lam_u = p.alpha * lam_u + xi * sgs[:, t]
        if p.alif:
            lam_a = rho * lam_a - beta * xi * sgs[:, t]
        lam_u = new_lam_u
        sgs[:, t] = lam_u                               # lambda_u,t overwrites psi_t
    grad_w = sgs.reshape(B * T, n).T @ xf               # sum_{b,t} lambda_u (x) x_t
    grad_w_out = g.T @ zsum                             # sum_t c_t g (x) z_t = g (x) zsum
    return BatchResult(loss, s, grad_w, grad_w_out, raster, zsum)


# --------------------------------------------------------------------------------------
# parity inputs (training.py:35-50, datasets.py:60-83)
# --------------------------------------------------------------------------------------

def init_network_arrays(n_hidden, n_inputs, n_classes, seed=0, dtype=np.float64):
    """Seeded U(+-1/sqrt(fan_in)) weights, drawn in f64 then cast -- training.py:35-50."""
    rng = np.random.default_rng(seed)
    bound_w = 1.0 / np.sqrt(n_inputs)
    bound_out = 1.0 / np.sqrt(n_hidden)
    w = rng.uniform(-bound_w, bound_w, size=(n_hidden, n_inputs)).astype(dtype)
    w_out = rng.uniform(-bound_out, bound_out, size=(n_classes, n_hidden)).astype(dtype)
    return w, w_out


def poisson_batch(n_samples, n_channels, n_steps, n_classes, seed=0):
    """Dense uint8 [B, T, k] inputs + labels, bit-identical to
    generate_poisson_dataset(...).input_array(s) (datasets.py:60-83): the same RNG
    calls in the same order (rates, then per sample: label, Bernoulli grid)."""
    rng = np.random.default_rng(seed)
    rates = rng.uniform(0.01, 0.2, size=(n_classes, n_channels))    # datasets.py:60-62
    x = np.empty((n_samples, n_steps, n_channels), dtype=np.uint8)
    labels = np.empty(n_samples, dtype=np.int64)
    for s in range(n_samples):
        label = int(rng.integers(n_classes))                          # datasets.py:77
        labels[s] = label
        x[s] = rng.random((n_steps, n_channels)) < rates[label]        # datasets.py:65-67
    return x, labels


# --------------------------------------------------------------------------------------
# training loop (training.py:58-166) -- checker for the device trainer
# --------------------------------------------------------------------------------------

def sgd_update(params, grads, lr):
    """p - lr*g per parameter, numpy weak-scalar promotion -- training.py:58-65."""
    return {key: p - lr * grads[key] for key, p in params.items()}


def adam_update(params, grads, lr, state, beta1=0.9, beta2=0.999, eps=1e-8):
    """training.py:75-91; ``state`` is a dict {"m": {}, "v": {}, "t": int}."""
    state["t"] += 1
    out = {}
    for key, p in params.items():
        g = grads[key]
        m = state["m"].get(key, np.zeros_like(p))
        v = state["v"].get(key, np.zeros_like(p))
        m = beta1 * m + (1 - beta1) * g
        v = beta2 * v + (1 - beta2) * g * g
        state["m"][key], state["v"][key] = m, v
        m_hat = m / (1 - beta1 ** state["t"])
        v_hat = v / (1 - beta2 ** state["t"])
        out[key] = p - lr * m_hat / (np.sqrt(v_hat) + eps)
    return out


def train_online(w, w_out, p: Params, x, labels, optimizer="sgd", lr=0.01, epochs=1,
                 max_updates=None, batch_size=1):
    """Online e-prop training -- training.py:116-166 with eprop_forward_mode as the
    engine.  ``batch_size > 1`` applies the batch-MEAN gradient, the
    device trainer's batched mode.  Returns (w, w_out, [(epoch, loss, accuracy)])."""
    dtype = w.dtype
    w, w_out = w.copy(), w_out.copy()
    state = {"m": {}, "v": {}, "t": 0}
    rows, updates = [], 0
    N = x.shape[0]
    for epoch in range(epochs):
        seen, correct = 0, 0
        for s0 in range(0, N, batch_size):
            nb = min(batch_size, N - s0)
            gw = np.zeros_like(w, dtype=np.float64)
            gwo = np.zeros_like(w_out, dtype=np.float64)
            losses = []
            for s in range(s0, s0 + nb):
                r = eprop_forward_mode(w, w_out, p, x[s].astype(dtype), int(labels[s]))
                gw += r.grad_w
                gwo += r.grad_w_out
                losses.append(r.loss)
                correct += int(np.argmax(r.readout_sum) == labels[s])
            grads = {"w": (gw / nb).astype(dtype), "w_out": (gwo / nb).astype(dtype)}
            params = {"w": w, "w_out": w_out}
            if optimizer == "adam":
                params = adam_update(params, grads, lr, state)
            else:
                params = sgd_update(params, grads, lr)
            w, w_out = params["w"].astype(dtype), params["w_out"].astype(dtype)
            seen += nb
            updates += 1
            rows.append((epoch, float(np.mean(losses)), correct / seen))
            if max_updates is not None and updates >= max_updates:
                return w, w_out, rows
    return w, w_out, rows


# --------------------------------------------------------------------------------------
# recurrent extension -- PARITY UNPINNED: the reference has no
# recurrent weights (neurons.py:165-172), so this restatement is the
# spec of the GPU kernels, not a copy of reference behaviour.  It is pinned only by
# (1) w_rec = 0 reproducing the feed-forward functions above bit for bit and (2) the
# e-prop trace construction being the reference's own with the presynaptic input
# x_t replaced by [x_t, z_{t-1}] (the standard e-prop treatment of recurrent weights,
# H_E dropped).
# --------------------------------------------------------------------------------------

def step_state_rec(w, w_rec, p: Params, u, a, x_t, smooth=False):
    """One forward step with recurrent input: I_t = W x_t + W_rec z_{t-1}, added to the
    leak as ONE current (u' = alpha*u + I_t), z_{t-1} = spike(d_{t-1})."""
    beta, rho = p.beta_eff, p.rho_eff
    z = _spike(u - p.theta - beta * a, p.slope, smooth)
    a_next = rho * a + z
    current = w @ x_t + (w_rec @ z if w_rec is not None else 0.0)
    u_next = p.alpha * u + current
    if p.reset:
        u_next = u_next - p.theta * z
    drive = u_next - p.theta - beta * a_next
    return u_next, a_next, _spike(drive, p.slope, smooth), surrogate_grad(drive, p.slope), z


def eprop_forward_mode_rec(w, w_rec, w_out, p: Params, x_seq, label, smooth=False):
    """Per-sample online e-prop of a recurrent layer: eprop_forward_mode with the trace
    input x~_t = [x_t, z_{t-1}] and the forward of step_state_rec.  Returns
    (Result with grad_w = [n, k + n] over [W | W_rec], raster [T, n])."""
    dtype = w.dtype
    n, k = w.shape
    m = w_out.shape[0]
    T = x_seq.shape[0]
    beta, rho = p.beta_eff, p.rho_eff
    rst = 1.0 if p.reset else 0.0
    kk = k + n
    u = np.zeros(n, dtype=dtype)
    a = np.zeros(n, dtype=dtype)
    g_u = np.zeros((n, kk), dtype=dtype)
    g_a = np.zeros((n, kk), dtype=dtype) if p.alif else None
    xbar = np.zeros((n, kk), dtype=dtype)
    xsum = np.zeros((n, kk), dtype=dtype)
    zbar = np.zeros(n, dtype=dtype)
    zsum = np.zeros(n, dtype=dtype)
    v = np.zeros(m, dtype=dtype)
    s = np.zeros(m, dtype=dtype)
    raster = np.zeros((T, n), dtype=bool)
    for t in range(T):
        psi_prev = surrogate_grad(u - p.theta - beta * a, p.slope)
        u, a_new, z, sg, z_prev = step_state_rec(w, w_rec, p, u, a, x_seq[t], smooth)
        xt = np.concatenate([x_seq[t].astype(dtype), z_prev.astype(dtype)])
        h_uu = p.alpha - rst * p.theta * psi_prev
        if p.alif:
            h_ua = rst * p.theta * beta * psi_prev
            g_u_new = h_uu[:, None] * g_u + h_ua[:, None] * g_a + xt[None, :]
            g_a = psi_prev[:, None] * g_u + (rho - beta * psi_prev)[:, None] * g_a
            g_u = g_u_new
            x_step = sg[:, None] * (g_u - beta * g_a)
        else:
            g_u = h_uu[:, None] * g_u + xt[None, :]
            x_step = sg[:, None] * g_u
        a = a_new
        raster[t] = z > 0.5
        v = p.kappa * v + w_out @ z
        s = s + v
        xbar *= p.kappa
        xbar += x_step
        xsum += xbar
        zbar = p.kappa * zbar + z
        zsum = zsum + zbar
    loss, g = softmax_cross_entropy(s, label)
    w_sig = w_out.T @ g
    return Result(loss, (w_sig[:, None] * xsum).astype(dtype), np.outer(g, zsum).astype(dtype),
                  s), raster
