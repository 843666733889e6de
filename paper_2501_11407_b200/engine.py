"""Device-side e-prop engine: buffers and the chunked two-pass update.

One ``EpropEngine`` owns every device buffer for a fixed problem shape (batch B,
hidden n, inputs k, classes m, chunk length Tc) and replays the update

    weights   K2s  slice W into exact INT8 digits (once per update)
    pass A    per chunk: pack x -> K2 INT8 tcgen05 current I = W x_t -> K1 dynamics(A)
    readout   K3 loss / g / w_sig ; K7 grad W_out
    pass B    per chunk: pack -> K2 -> K1 dynamics(B) + backward chunk scan -> K4 operand
                         -> K5 tcgen05 chunk-gradient GEMM   (all intra-chunk terms)
                         -> K6 tcgen05 ALIF trace carry      (inter-chunk terms, ALIF)
                         -> fixed-order reduction of the split partials

which is the reference's per-sample online loop (gradients.py:157-176) restated for a
batch: the learning signal L_t = c_t W_out^T (softmax - onehot) is only known after the
whole sequence (gradients.py:177-182), so pass B recomputes the (deterministic) forward
with L_t known (two-pass form), and the per-synapse ALIF trace is
carried chunk to chunk (forward.cu / elig.cu headers give the algebra).  With reset=False
the presynaptic filter is folded into the scan's coefficients, so K5 / K6 run on the raw
spikes (2 MMAs); a one-chunk sequence reuses pass A's current and parked psi (pass B =
scan + K5), and its pack also writes K5's operand.  Memory is independent of T: state is
per (sample, neuron[, input]) and chunk buffers are sized by Tc (opt-in `park_budget`
trades that for skipping pass B's recompute).

All work is enqueued on torch's current CUDA stream through the C-ABI (``_lib``); the
engine never synchronises.  PyTorch provides allocation and streams only.
"""

from __future__ import annotations

import ctypes
import os
import math

import numpy as np
import torch

from . import _lib
from .errors import LabelOutOfRange, ShapeMismatch

SM_COUNT_DEFAULT = 148
# Tc with Tc + 1 a multiple of the 64-wide K block.  Longer chunks are strictly less work
# (one per-synapse trace round trip per chunk; a sequence that fits one chunk never
# materialises the trace and skips pass B's recompute); the chunk buffers grow with Tc,
# never with T.
CHUNKS = (63, 127, 255, 511, 1023, 2047)


def ctypes_void(p):
    return ctypes.c_void_p(p)


def _round_up(a, b):
    return (a + b - 1) // b * b


def readout_gains(T: int, kappa: float) -> np.ndarray:
    """c_t = sum_{tau=t}^{T-1} kappa^(tau-t): the gain with which the time-summed leaky
    readout (gradients.py:163-164) sees a spike at step t; the recurrence matches
    bptt_gradient's c_t = 1 + kappa*c_{t+1} (gradients.py:218)."""
    c = np.empty(T, dtype=np.float64)
    acc = 0.0
    for t in range(T - 1, -1, -1):
        acc = 1.0 + kappa * acc
        c[t] = acc
    return c


def _wave_split(tiles: int, B: int, sms: int) -> int:
    """Number of sample ranges for K6 (one CTA per SM): the smallest split whose grid
    fills whole waves to >= 90 %, else the best of splits <= 8 waves."""
    best, best_eff = 1, 0.0
    for s in range(1, B + 1):
        ctas = tiles * s
        waves = math.ceil(ctas / sms)
        if waves > 8:
            break
        eff = ctas / (waves * sms)
        if eff >= 0.9:
            return s
        if eff > best_eff + 1e-9:
            best, best_eff = s, eff
    return best


def chunk_bytes(Tc: int, B: int, n: int, k: int, alif: bool = True) -> int:
    """Device bytes of the Tc-sized chunk buffers of an engine (current, packed spikes,
    psi scratch, C/W operands, xbar operands): the part of the footprint that grows with
    the chunk length (none of it grows with T)."""
    KR = Tc + 1
    kp = _round_up(k, 128)
    ldc = _round_up(n, 8)
    ops = 2 * (2 if alif else 1) * 2 * B * KR * ldc
    return (8 * B * KR * n + B * KR * kp + 4 * B * (KR + 1) * n + ops + 4 * B * KR * kp)


def default_chunk(T: int, B: int | None = None, n: int | None = None, k: int | None = None,
                  alif: bool = True, budget: int = 32 << 30) -> int:
    """Chunk length Tc for a sequence of T steps: the smallest Tc covering the whole
    sequence, else the longest one whose chunk buffers fit ``budget`` bytes.  Longer
    chunks are strictly less work (the per-synapse ALIF trace makes one HBM round trip per
    chunk, K6) and memory stays independent of T."""
    for c in CHUNKS:
        if T <= c and (B is None or chunk_bytes(c, B, n, k, alif) <= budget):
            return c
    best = CHUNKS[0]
    for c in CHUNKS:
        if B is None or chunk_bytes(c, B, n, k, alif) <= budget:
            best = c
    return best


class EpropEngine:
    """Buffers + launch sequence for one problem shape on one device."""

    def __init__(self, n: int, k: int, m: int, B: int, *, alif: bool, w_f64: bool = False,
                 chunk: int = 127, device=None, sm_count: int | None = None,
                 reset: bool = False, recurrent: bool = False, grad: bool = True):
        if chunk not in CHUNKS:
            raise ValueError(f"chunk must be one of {CHUNKS} (Tc + 1 a multiple of 64)")
        self.lib = _lib.load()
        self.n, self.k, self.m, self.B = int(n), int(k), int(m), int(B)
        if min(self.n, self.k, self.m, self.B) <= 0:
            raise ShapeMismatch("n, k, m and B must be positive")
        self.alif = bool(alif)
        # carried per-synapse traces: ALIF G_a (reset=False); LIF G_u (reset=True, the soft
        # reset makes G_u non-factorisable); ALIF (G_u, G_a) pair (reset=True)
        self.reset = bool(reset)
        self.ntr = (2 if self.reset else 1) if self.alif else (1 if self.reset else 0)
        self.w_f64 = bool(w_f64)
        self.Tc = int(chunk)
        self.KR = self.Tc + 1
        dev = torch.device(device if device is not None else "cuda")
        if dev.type == "cuda" and dev.index is None and torch.cuda.is_available():
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        # grad=False: forward-only engine (evaluate(), network_loss): none of the pass-B
        # buffers (psi scratch, GEMM operands, the per-synapse trace, partials) exist
        self.grad = bool(grad)
        self.n_pad = _round_up(self.n, 128)
        # recurrent layer: the eligibility kernels see the extended
        # input x~_t = [x_t, z_{t-1}] of width kx = k + n (forward_rec.cu)
        self.recurrent = bool(recurrent)
        if self.recurrent and self.n > 2048:
            raise ValueError("the recurrent path supports n <= 2048 hidden neurons")
        self.kx = self.k + (self.n if self.recurrent else 0)
        self.kp = _round_up(self.kx, 128)
        self.ke = _round_up(self.kx, 4)
        sms = sm_count or (torch.cuda.get_device_properties(self.device).multi_processor_count
                           if self.device.type == "cuda" else SM_COUNT_DEFAULT)
        self.sm_count = sms
        dev = self.device
        f32, f64, bf16 = torch.float32, torch.float64, torch.bfloat16
        B, n, k, m = self.B, self.n, self.k, self.m
        Bn = (B, n)
        K = B * self.KR
        self.K = K
        # K2 exact INT8 tensor-core projection: x chunk operand, sliced weights, current
        self.Kpad = _round_up(k, 128)
        self.n_pad32 = _round_up(n, 32)
        self.P = 8 if self.w_f64 else 6   # digit format, csrc/digits.cuh
        # sample-aligned rows b*KR + s (KR = Tc + 1, a multiple of 64; rows s >= len zero)
        self.xq = torch.zeros((B * self.KR, self.Kpad), dtype=torch.uint8, device=dev)
        self.cur = torch.empty((B * self.KR, n), dtype=f64, device=dev)
        self.wq = torch.zeros((self.P, self.n_pad32, self.Kpad), dtype=torch.int8, device=dev)
        self.sexp = torch.zeros(n, dtype=torch.int32, device=dev)
        # neuron state (fp64) and readout filters
        self.u = torch.empty(Bn, dtype=f64, device=dev)
        self.a = torch.empty(Bn, dtype=f64, device=dev)
        self.zbar = torch.empty(Bn, dtype=f64, device=dev)
        self.zsum = torch.empty(Bn, dtype=f64, device=dev)
        # readout / loss
        self.wsig = torch.empty(Bn, dtype=f32, device=dev)
        self.s = torch.empty((B, m), dtype=f64, device=dev)
        self.loss = torch.empty(B, dtype=f64, device=dev)
        self.g = torch.empty((B, m), dtype=f64, device=dev)
        self.correct = torch.empty(B, dtype=torch.int32, device=dev)
        self.ldc = _round_up(n, 8)   # C/W are MN-major [K][ldc] (neurons contiguous)
        self.xbar_state = torch.empty((B, self.kx), dtype=f64, device=dev)
        if self.recurrent:
            self.wrecT = torch.zeros((n, n), dtype=f64 if self.w_f64 else f32, device=dev)
            self.nw = (n + 31) // 32
            self.Kx2 = _round_up(self.kx, 4)
        # weights
        self.w = torch.empty((n, k), dtype=f64 if self.w_f64 else f32, device=dev)
        self.wout = torch.empty((m, n), dtype=f64, device=dev)
        # fold the input filter into the one-chunk coefficients (SPB_FILT=0: xbar operand)
        self.filt = os.environ.get("SPB_FILT", "1") != "0"
        self.pack_xh = os.environ.get("SPB_PACK_XH", "1") != "0"
        # SPB_COMPACT_ROWS=0: the one-chunk projection over all KR rows per sample (A/B)
        self.compact_rows = os.environ.get("SPB_COMPACT_ROWS", "1") != "0"
        # opt-in memory-for-time trade (off by default: memory then grows with T): park the
        # psi of every chunk in pass A when all of it fits `park_budget` bytes, so pass B
        # skips the projection and the dynamics recompute.  SPB_PARK_GB sets it too.
        self.park_budget = int(float(os.environ.get("SPB_PARK_GB", "0")) * (1 << 30))
        self.psi_park = None
        self._ctab_T = None
        self.ctab = None
        self.launches = 0
        # where K4 of a one-chunk sequence runs when the pack does not write K5's operand
        # itself (SPB_PACK_XH=0, unaligned byte rows, recurrent engines): "fa"
        # (default, measured best: C4 1.66 -> 1.59 ms) = side stream after K2, overlapping
        # K1; "proj" = side stream from the start of pass A, overlapping K2; "main" =
        # serially before K5
        self.xbar_sched = os.environ.get("SPB_XBAR_SCHED", "fa")
        # side stream for work off the critical path (K4 xbar of a one-chunk sequence, K7)
        if self.device.type == "cuda":
            self.side = torch.cuda.Stream(device=dev)
            self._ev = {nm: torch.cuda.Event() for nm in ("start", "xbar", "ro", "rg")}
        else:
            self.side = None
            self._ev = None
        self.splits5 = self.splits6 = 0
        self.psi = self.c_hi = self.c_lo = self.xh = self.xl = self.xs_hi = self.xs_lo = None
        self.w_hi = self.w_lo = self.wa_hi = self.wa_lo = self.mdt = self.eps = self.eps2 = None
        self.partial = self.grad_w_acc = self.grad_wout = self.zchunk = self.xq2 = None
        if self.grad:
            self._alloc_grad_buffers()

    def device_bytes(self) -> int:
        """Device memory held by the engine's buffers (each tensor counted once)."""
        seen, total = set(), 0
        for v in vars(self).values():
            if isinstance(v, torch.Tensor) and v.device.type == "cuda":
                key = v.untyped_storage().data_ptr()
                if key not in seen:
                    seen.add(key)
                    total += v.untyped_storage().nbytes()
        return total

    def _alloc_grad_buffers(self):
        """Pass-B buffers: psi scratch, the chunk GEMM / carry operands (bf16 hi/lo,
        K-major over (sample, rho)), the per-synapse trace, split partials, accumulators."""
        dev, sms = self.device, self.sm_count
        f32, f64, bf16 = torch.float32, torch.float64, torch.bfloat16
        B, n, m, K = self.B, self.n, self.m, self.K
        self.psi = torch.zeros((B, self.KR + 1, n), dtype=f32, device=dev)   # K1 scan scratch
        self.c_hi = torch.zeros((K, self.ldc), dtype=bf16, device=dev)
        self.c_lo = torch.zeros((K, self.ldc), dtype=bf16, device=dev)
        if self.recurrent:
            self.zchunk = torch.zeros((B, self.KR, self.nw), dtype=torch.int32, device=dev)
            self.xq2 = torch.zeros((B * self.Tc, self.Kx2), dtype=torch.uint8, device=dev)
        self.xh = torch.zeros((K, self.kp), dtype=bf16, device=dev)   # MN-major [K][kp]
        self.xl = torch.zeros((K, self.kp), dtype=bf16, device=dev)
        # entry filter state xbar_{t0-1} of a later chunk (raw-spike operand), bf16 hi/lo
        self.xs_hi = torch.zeros((B, self.kp), dtype=bf16, device=dev)
        self.xs_lo = torch.zeros((B, self.kp), dtype=bf16, device=dev)
        # split-K (K5) and sample-split (K6) partial slices, reduced in fixed order
        tiles5 = 2 * math.ceil(self.kp / 256) * math.ceil(n / 256)   # K5: CTA pairs, 256 x 256
        # split-K so the grid fills whole waves of SMs (C4: 96 tiles x 3 = 1.95 waves)
        self.splits5 = _wave_split(tiles5, max(1, K // 64), sms)
        self.wa_hi = self.wa_lo = self.eps2 = None
        if self.ntr:
            self.w_hi = torch.zeros((K, self.ldc), dtype=bf16, device=dev)
            self.w_lo = torch.zeros((K, self.ldc), dtype=bf16, device=dev)
            # chunk coefficients: (M, Dt) per (sample, neuron); the reset pair needs
            # (M_u, M_a, Dt 2x2) padded to 8 floats
            self.mdt = torch.empty((B, n, 2 if self.ntr == 1 else 8), dtype=f32, device=dev)
            self.eps = torch.zeros((B, self.n_pad, self.ke), dtype=f32, device=dev)
            if self.ntr == 2:
                self.wa_hi = torch.zeros((K, self.ldc), dtype=bf16, device=dev)
                self.wa_lo = torch.zeros((K, self.ldc), dtype=bf16, device=dev)
                self.eps2 = torch.zeros((B, self.n_pad, self.ke), dtype=f32, device=dev)
            if self.ntr == 1:   # K6: CTA pairs over 256 x 256 synapse tiles
                tiles6 = 2 * math.ceil(self.kp / 256) * math.ceil(self.n_pad / 256)
            else:               # K6r: 128 x 64 tiles
                tiles6 = (self.kp // 64) * (self.n_pad // 128)
            self.splits6 = _wave_split(tiles6, B, sms)
        else:
            self.w_hi = self.w_lo = self.mdt = self.eps = None
            self.splits6 = 0
        # partial slices: [K5 splits | K6 splits | 1 for the carried-filter row-0 GEMM]
        self.partial = torch.zeros((self.splits5 + self.splits6 + 1, self.n_pad, self.kp),
                                   dtype=f32, device=dev)
        self.grad_w_acc = torch.empty((n, self.kp), dtype=f64, device=dev)
        self.grad_wout = torch.empty((m, n), dtype=f64, device=dev)

    # ----------------------------------------------------------------------------------
    def set_weights(self, w, w_out, stream=None, w_rec=None):
        """Upload input weights and readout weights (fp64) and slice W into the INT8
        digits of the exact tensor-core projection (K2); recurrent engines also take
        ``w_rec`` [n, n] (stored transposed for the coalesced spike gather)."""
        w = torch.as_tensor(w)
        w_out = torch.as_tensor(w_out)
        if self.recurrent:
            if w_rec is None:
                raise ShapeMismatch("a recurrent engine needs w_rec")
            w_rec = torch.as_tensor(w_rec)
            if tuple(w_rec.shape) != (self.n, self.n):
                raise ShapeMismatch(f"w_rec must be [{self.n}, {self.n}]")
            self.wrecT.copy_(w_rec.to(self.wrecT.dtype).t().contiguous(), non_blocking=True)
        elif w_rec is not None:
            raise ShapeMismatch("w_rec given to a feed-forward engine")
        if tuple(w.shape) != (self.n, self.k) or tuple(w_out.shape) != (self.m, self.n):
            raise ShapeMismatch(f"weights {tuple(w.shape)}/{tuple(w_out.shape)} do not match "
                                f"engine (n={self.n}, k={self.k}, m={self.m})")
        self.w.copy_(w.to(self.w.dtype), non_blocking=True)
        self.wout.copy_(w_out.to(torch.float64), non_blocking=True)
        self.slice_weights(stream)

    def slice_weights(self, stream=None):
        """Re-derive the INT8 weight digits from ``self.w`` (after an in-place update)."""
        st = ctypes_void(stream if stream is not None else self._stream())
        _lib.call("spb_slice_weights", ctypes_void(self.w.data_ptr()), int(self.w_f64), self.n,
                  self.k, self.Kpad, self.n_pad32, self.P, ctypes_void(self.wq.data_ptr()),
                  ctypes_void(self.sexp.data_ptr()), st)

    def sgd_slice(self, g, g_is_f64: bool, ld_g: int, g_scale: float, lr: float, stream=None):
        """``self.w <- self.w - lr * g_scale * g`` (the fused SGD kernel's arithmetic) and
        the INT8 digits re-derived from the new W, in one launch (spb_sgd_slice_update)."""
        st = ctypes_void(stream if stream is not None else self._stream())
        _lib.call("spb_sgd_slice_update", ctypes_void(self.w.data_ptr()), int(self.w_f64),
                  self.n, self.k, ctypes_void(g.data_ptr()), int(g_is_f64), int(ld_g),
                  float(g_scale), float(lr), self.Kpad, self.n_pad32, self.P,
                  ctypes_void(self.wq.data_ptr()), ctypes_void(self.sexp.data_ptr()), st)

    def _stream(self):
        if self.device.type != "cuda":
            return 0
        return torch.cuda.current_stream(self.device).cuda_stream

    def _gains(self, T, kappa):
        if self._ctab_T != (T, kappa):
            self.ctab = torch.as_tensor(readout_gains(T, kappa).astype(np.float32),
                                        device=self.device)
            self._ctab_T = (T, kappa)
        return self.ctab

    def _pack(self, xp, strideb, bits, ln, st, xh=False, compact=False):
        """Chunk spikes (bytes or bits) -> zero-padded projection operand xq [B*KR][Kpad]
        (rows b*KR + s, rows s >= len zero; also K4's row source).  xh: also
        write the one-chunk raw-spike GEMM operand (K4 folded into the pack).  compact
        (with xh): only the live steps, xq rows b*len + s (spb_input_proj_rows)."""
        if xh:
            _lib.call("spb_pack_spikes_xh", ctypes_void(xp), strideb, self.B, self.k, int(bits),
                      ln, ln if compact else self.KR, self.Kpad, self.KR,
                      ctypes_void(self.xq.data_ptr()), ctypes_void(self.xh.data_ptr()), st)
            return
        _lib.call("spb_pack_spikes", ctypes_void(xp), strideb, self.B, self.k, int(bits), ln,
                  self.KR, self.Kpad, 0, ctypes_void(self.xq.data_ptr()), st)

    def _project(self, ln, st, timed=None, binary=False, compact=False):
        """K2: cur = W x_t exactly on INT8 tensor cores from the packed chunk (binary:
        0/1 spikes, single-int64 digit recombination).  compact: xq holds only the chunk's
        live steps (rows b*len + s), written to cur rows b*KR + s."""
        v = ctypes_void
        if compact:
            args = ("spb_input_proj_rows", v(self.xq.data_ptr()), v(self.wq.data_ptr()),
                    v(self.sexp.data_ptr()), self.B, ln, self.KR, self.n, self.n_pad32, self.k,
                    self.Kpad, self.P, v(self.cur.data_ptr()), self.sm_count, int(bool(binary)),
                    st)
        else:
            args = ("spb_input_proj", v(self.xq.data_ptr()),
                    v(self.wq.data_ptr()), v(self.sexp.data_ptr()), self.B * self.KR, self.n,
                    self.n_pad32, self.k, self.Kpad, self.P, v(self.cur.data_ptr()),
                    self.sm_count, int(bool(binary)), st)
        if timed is not None:
            timed("proj", ln, *args)
        else:
            _lib.call(*args)

    # ----------------------------------------------------------------------------------
    def run(self, x: torch.Tensor, labels: torch.Tensor, *, alpha=0.95, theta=1.0, slope=10.0,
            beta=0.8, rho=0.96, kappa=0.95, reset=False, raster: torch.Tensor | None = None,
            stream=None, timers: dict | None = None, bits: bool = False, smooth: bool = False,
            forward_only: bool = False, binary: bool | None = None):
        """One full e-prop update.

        x       uint8 [B, T, k] spike counts, or with ``bits=True`` uint8 [B, T, ceil(k/8)]
                bit-packed binary spikes (numpy.packbits(..., axis=-1, bitorder="little")).
                A CUDA tensor is used in place; a CPU (ideally pinned) tensor is STREAMED:
                each time chunk is copied into a double-buffered device chunk on a copy
                stream, overlapped with the previous chunk's kernels, so device memory is
                independent of T.
        labels  int64 [B] (CUDA)
        raster  optional int32 [B, T, ceil(n/32)] bit-packed spike output (pass A)
        timers  optional dict; CUDA event pairs are appended per launch of the main
                kernels under "proj", "forward_a", "forward", "gemm", "carry".
        smooth  spikes are surrogate_smooth(d) instead of Theta(d) (the reference's
                smooth=True mode, gradients.py:114-115); the trace algebra is unchanged.
        forward_only  pass A + loss only (network_loss, gradients.py:349-365): no
                gradients are computed (evaluate()).
        binary  promise that every input count is 0 or 1 (default: True for bit-packed
                input); K2 then recombines its digit sums in one int64 (same bits).
        Results stay on device: ``grad_w_acc`` (fp64 [n, kp]), ``grad_wout``, ``loss``,
        ``s`` (readout sums), ``correct``.
        """
        if binary is None:
            binary = bits
        if bool(reset) != self.reset:
            raise ValueError(f"engine built for reset={self.reset}, called with reset={reset}")
        kb = (self.k + 7) // 8 if bits else self.k
        # real-valued inputs (fp32/fp64, not spike counts): fp64 projection, hi/lo operand
        real = x.dtype in (torch.float32, torch.float64) and not bits
        if ((x.dtype != torch.uint8 and not real) or x.dim() != 3 or x.shape[0] != self.B
                or x.shape[2] != kb):
            raise ShapeMismatch(f"x must be uint8 [B={self.B}, T, {kb}] "
                                f"({'bit-packed' if bits else 'counts'}) or fp32/fp64 "
                                f"[B, T, k], got {tuple(x.shape)} {x.dtype}")
        if not x.is_contiguous():
            raise ShapeMismatch("x must be contiguous")
        if (labels.dtype != torch.int64 or tuple(labels.shape) != (self.B,)
                or labels.device != self.device):
            raise ShapeMismatch(f"labels must be int64 [{self.B}] on {self.device}, got "
                                f"{labels.dtype} {tuple(labels.shape)} on {labels.device}")
        if not self.grad and not forward_only:
            raise ValueError("engine built with grad=False runs forward_only updates only")
        streaming = x.device.type == "cpu" and self.device.type == "cuda"
        T = int(x.shape[1])
        if T <= 0:
            raise ShapeMismatch("T must be positive")
        if real and (streaming or T > self.Tc or self.recurrent or self.reset
                     or stream is not None or x.device != self.device
                     or self.device.type != "cuda"):
            raise ValueError("real-valued (non-count) inputs are supported for one-chunk "
                             f"sequences (T <= {self.Tc}) on the engine's device, reset=False, "
                             "without the recurrent extension; spike-count inputs have no "
                             "such limits")
        call = _lib.call
        st = ctypes_void(stream if stream is not None else self._stream())
        beta_e, rho_e = (float(beta), float(rho)) if self.alif else (0.0, 0.0)
        B, n, k, m, Tc, KR, K = self.B, self.n, self.k, self.m, self.Tc, self.KR, self.K
        ctab = self._gains(T, float(kappa))
        nchunks = (T + Tc - 1) // Tc
        one = nchunks == 1
        slab = B * (self.KR + 1) * n
        park = (not one and not forward_only and not self.recurrent
                and self.park_budget > 0 and 4 * slab * nchunks <= self.park_budget
                and self.device.type == "cuda")
        if park and (self.psi_park is None or self.psi_park.shape[0] < nchunks):
            self.psi_park = torch.empty((nchunks, B, self.KR + 1, n), dtype=torch.float32,
                                        device=self.device)

        def psi_ptr(c):
            return v(self.psi_park[c].data_ptr()) if park else v(self.psi.data_ptr())
        strideb = T * kb
        self.launches = 0
        v = ctypes_void
        common = (float(alpha), float(theta), float(slope), beta_e, rho_e, float(kappa),
                  int(self.reset), int(self.alif), int(bool(smooth)))
        # K4 reads the packed operand (sample-major rows)
        xq_sb, xq_st = KR * self.Kpad, self.Kpad
        # K5/K6 operand: the filtered input xbar (reset=False: G_u = 1 (x) xbar), or with
        # reset=True the raw input (G_u is carried per synapse; K4 with alpha = 0 = copy)
        x_alpha = 0.0 if self.reset else float(alpha)
        # one fresh chunk, reset=False: the input filter is folded into the coefficients
        # (scan pass 3), so K5 too runs on the raw spikes (forward.cu FILT).  Raw-spike
        # operands are exact in bf16: no lo part (K4 writes hi only, K5 does 2 MMAs).
        # Several chunks: the same on every chunk (scan pass 4 / 3), with the entry state
        # xbar_{t0-1} of each later chunk handled apart -- K4 writes it to xs_hi/lo, a
        # K = B GEMM adds Ct_0 (x) xbar_{t0-1} and K6 adds Wt_0 xbar_{t0-1} in its epilogue.
        # (the recurrent extension: one chunk only -- its x~ operand is built in pass B)
        filt = (not self.reset and (one or not self.recurrent) and not forward_only
                and self.filt)
        if filt and one:
            x_alpha = 0.0   # K4 = byte -> bf16 copy (the filter state is never needed)
        raw_x = (filt or self.reset) and (filt or not self.recurrent)
        xl_ptr = None if (raw_x or self.xl is None) else v(self.xl.data_ptr())
        if real and self.xl is not None:
            xl_ptr = v(self.xl.data_ptr())   # real inputs are not exact in bf16: hi + lo
        # one chunk: the pack writes the raw-spike GEMM operand itself (no K4 at all)
        pack_xh = (filt and one and not self.recurrent and self.pack_xh
                   and (bits or (self.k % 4 == 0 and x.data_ptr() % 4 == 0)))
        if real:
            pack_xh = True   # spb_pack_real writes the operand (hi and lo)
        # one chunk with the operand folded into the pack: xq holds only the live steps
        # (K2 over B*len rows instead of B*KR; C3: 500 instead of 512 row tiles)
        compact = pack_xh and not real and self.compact_rows

        def timed(name, meta, fn, *args):
            if timers is None:
                return call(fn, *args)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = call(fn, *args)
            e1.record()
            timers.setdefault(name, []).append((e0, e1, meta))
            return rc

        use_side = self.side is not None and stream is None
        sst = ctypes_void(self.side.cuda_stream) if use_side else st
        main = torch.cuda.current_stream(self.device) if self.device.type == "cuda" else None
        if use_side:
            # the side stream must not run ahead of the previous update's consumers
            self._ev["start"].record(main)
            self.side.wait_event(self._ev["start"])

        # ---- input access: resident (device tensor) or streamed chunk by chunk ----
        if streaming:
            if stream is not None:
                raise ValueError("streamed inputs use the engine's own streams")
            xs = self._stream_buffers(kb)
            uses = list(range(nchunks)) * (1 if (one or forward_only) else 2)
            xhost = x.data_ptr()
            for e in self._sev_free:
                e.record(main)

            def _copy(u):
                cc = uses[u]
                t0c = cc * Tc
                lnc = min(Tc, T - t0c)
                bb = u % 2
                self._cs.wait_event(self._sev_free[bb])
                call("spb_copy_chunk_h2d", v(xs[bb].data_ptr()), Tc * kb, v(xhost + t0c * kb),
                     T * kb, lnc * kb, B, ctypes_void(self._cs.cuda_stream))
                self._sev_ready[bb].record(self._cs)

            state = {"u": 0}

            def pack_chunk(c, ln):
                u = state["u"]
                if u == 0:
                    _copy(0)
                if u + 1 < len(uses):
                    _copy(u + 1)
                main.wait_event(self._sev_ready[u % 2])
                self._pack(xs[u % 2].data_ptr(), Tc * kb, bits, ln, st, xh=pack_xh,
                           compact=compact)
                self._sev_free[u % 2].record(main)
                state["u"] += 1
        elif real:
            def pack_chunk(c, ln):
                # operand: bf16 hi/lo rows; projection I = x W^T in fp64 (cuBLAS DGEMM via
                # torch, on this stream): the exact INT8 path needs integer counts
                if self.xh is not None:   # (forward-only engines have no GEMM operand)
                    call("spb_pack_real", v(x.data_ptr()), int(x.dtype == torch.float64),
                         T * k, B, k, ln, KR, self.kp, v(self.xh.data_ptr()),
                         v(self.xl.data_ptr()), st)
                cur3 = self.cur.view(B, KR, n)
                cur3[:, :ln].copy_(torch.matmul(x[:, :ln].to(torch.float64),
                                                self.w.to(torch.float64).t()))
        else:
            def pack_chunk(c, ln):
                self._pack(x.data_ptr() + c * Tc * kb, strideb, bits, ln, st, xh=pack_xh,
                           compact=compact)

        # ---------------- pass A ----------------
        for c in range(nchunks):  # chunk 0 starts from fresh state inside the kernels
            t0 = c * Tc
            ln = min(Tc, T - t0)
            pack_chunk(c, ln)
            side_x = one and use_side and not forward_only and not self.recurrent
            if pack_xh:  # the pack wrote K5's raw operand: no K4 (pass B's wait is a no-op)
                if use_side:
                    self._ev["xbar"].record(main)
                side_x = False
            if side_x and self.xbar_sched == "fa":
                self._project(ln, st, timed, binary)
            if side_x and self.xbar_sched != "main":
                # K4 needs only x: overlap it with pass A
                self._ev["xbar"].record(main)
                self.side.wait_event(self._ev["xbar"])
                call("spb_xbar_chunk", v(self.xq.data_ptr()), xq_sb, xq_st, B, k, self.kp, KR,
                     ln, 1, x_alpha, v(self.xbar_state.data_ptr()), v(self.xh.data_ptr()),
                     xl_ptr, sst)
                self._ev["xbar"].record(self.side)
                self.launches += 1
            if not (side_x and self.xbar_sched == "fa") and not real:
                self._project(ln, st, timed, binary, compact=compact)
            if self.recurrent:
                self._forward_rec(0, ln, t0, T, common, raster,
                                  one and not forward_only, st, timed, (ln, 0, one))
                self.launches += 3
                continue
            timed("forward_a", (ln, 0, one), "spb_forward_chunk", 0,
                  v(self.cur.data_ptr()), B, n, Tc, KR, ln, t0, T,
                  *common, v(self.u.data_ptr()), v(self.a.data_ptr()),
                  v(self.zbar.data_ptr()), v(self.zsum.data_ptr()),
                  v(raster.data_ptr()) if raster is not None else None,
                  None, None, None, None, None, None, None, None, 0, None,
                  psi_ptr(c) if (park or (one and not forward_only)) else None, st)
            self.launches += 3
        # ---------------- readout / loss ----------------
        call("spb_readout_loss", v(self.wout.data_ptr()), v(self.zsum.data_ptr()),
             v(labels.data_ptr()), B, n, m, v(self.s.data_ptr()), v(self.loss.data_ptr()),
             v(self.g.data_ptr()), v(self.wsig.data_ptr()), v(self.correct.data_ptr()), st)
        self.launches += 1
        if forward_only:
            return self
        if use_side:  # K7 is off the critical path
            self._ev["ro"].record(main)
            self.side.wait_event(self._ev["ro"])
        call("spb_readout_grad", v(self.g.data_ptr()), v(self.zsum.data_ptr()), B, n, m,
             v(self.grad_wout.data_ptr()), sst)
        if use_side:
            self._ev["rg"].record(self.side)
        self.launches += 1
        # ---------------- pass B ----------------
        slice_stride = self.n_pad * self.kp
        part6 = self.partial.data_ptr() + self.splits5 * slice_stride * 4
        for c in range(nchunks):
            t0 = c * Tc
            ln = min(Tc, T - t0)
            last = c == nchunks - 1
            carry_out = bool(self.ntr) and not last   # only a later chunk needs the trace
            if park:     # psi of this chunk was parked in pass A: spikes (for K4) only
                pack_chunk(c, ln)
                self.launches += 1
            elif not one:  # one chunk: xq and cur of pass A are still valid (same W, same x)
                pack_chunk(c, ln)
                self._project(ln, st, timed, binary)
                if self.recurrent:
                    self._forward_rec(1, ln, t0, T, common, None, True, st, timed,
                                      (ln, 1, carry_out))
                    self.launches += 1
                self.launches += 2
            # one chunk (pass A parked psi) or K1rec (parks psi itself): scan only
            pid = 2 if (one or park or self.recurrent) else 1
            if filt:
                pid = 3 if pid == 2 else 4
            timed("forward", (ln, pid, carry_out), "spb_forward_chunk", pid,
                  v(self.cur.data_ptr()), B, n, Tc, KR,
                  ln, t0, T, *common, v(self.u.data_ptr()), v(self.a.data_ptr()), None, None,
                  None, v(self.wsig.data_ptr()), v(ctab.data_ptr()),
                  v(self.c_hi.data_ptr()), v(self.c_lo.data_ptr()),
                  v(self.w_hi.data_ptr()) if carry_out else None,
                  v(self.w_lo.data_ptr()) if carry_out else None,
                  v(self.wa_hi.data_ptr()) if carry_out and self.ntr == 2 else None,
                  v(self.wa_lo.data_ptr()) if carry_out and self.ntr == 2 else None, self.ldc,
                  v(self.mdt.data_ptr()) if self.ntr else None, psi_ptr(c), st)
            self.launches += 1 if pid >= 2 else 2
            if self.recurrent:
                # x~ = [x_t, z_{t-1}] bytes, then the usual filter over kx columns
                call("spb_pack_rec", v(self.xq.data_ptr()), xq_sb, xq_st,
                     v(self.zchunk.data_ptr()), B, k, n, Tc, KR, ln, self.Kx2,
                     v(self.xq2.data_ptr()), st)
                call("spb_xbar_chunk_seg", v(self.xq2.data_ptr()), Tc * self.Kx2, self.Kx2, B,
                     self.kx, self.kp, KR, ln, int(c == 0 or self.reset), x_alpha,
                     v(self.xbar_state.data_ptr()), v(self.xh.data_ptr()), xl_ptr, st)
                self.launches += 2
            elif pack_xh:
                pass   # the pass-A pack wrote the raw-spike operand
            elif one and use_side and self.xbar_sched != "main":
                main.wait_event(self._ev["xbar"])
            elif filt and not one:
                call("spb_xbar_chunk_raw", v(self.xq.data_ptr()), xq_sb, xq_st, B, k, self.kp,
                     KR, ln, int(c == 0), float(alpha), v(self.xbar_state.data_ptr()),
                     v(self.xh.data_ptr()), v(self.xs_hi.data_ptr()), v(self.xs_lo.data_ptr()),
                     st)
                self.launches += 1
            else:
                call("spb_xbar_chunk_seg", v(self.xq.data_ptr()), xq_sb, xq_st, B, k, self.kp, KR,
                     ln, int(c == 0 or self.reset), x_alpha, v(self.xbar_state.data_ptr()),
                     v(self.xh.data_ptr()), xl_ptr, st)
                self.launches += 1
            timed("gemm", (ln, raw_x), "spb_grad_gemm_partials", v(self.c_hi.data_ptr()),
                  v(self.c_lo.data_ptr()), self.ldc, v(self.xh.data_ptr()), xl_ptr,
                  self.kp, n, self.kp, K, self.splits5, v(self.partial.data_ptr()), self.kp,
                  slice_stride, st)
            self.launches += 1
            entry = filt and not one and c > 0   # row-0 terms of the carried filter state
            if entry:  # sum_b Ct_0[b,i] xbar_{t0-1}[b,j]: rows b*KR of C, K = B
                call("spb_grad_gemm_partials", v(self.c_hi.data_ptr()), v(self.c_lo.data_ptr()),
                     KR * self.ldc, v(self.xs_hi.data_ptr()), v(self.xs_lo.data_ptr()),
                     self.kp, n, self.kp, B, 1,
                     v(self.partial.data_ptr() + (self.splits5 + self.splits6) * slice_stride * 4),
                     self.kp, slice_stride, st)
                self.launches += 1
            slices = self.splits5
            if self.ntr and (c > 0 or not last):
                # first chunk: E0 = 0 (nothing to add, only carry); last chunk: no carry
                if self.ntr == 1:
                    timed("carry", (ln, c > 0, not last, raw_x), "spb_alif_carry_chunk",
                          v(self.w_hi.data_ptr()), v(self.w_lo.data_ptr()), self.ldc,
                          v(self.xh.data_ptr()), xl_ptr, v(self.mdt.data_ptr()),
                          v(self.eps.data_ptr()), v(part6), B, n, self.n_pad, self.kx, self.ke,
                          self.kp, KR, self.splits6, int(not last), int(c > 0), int(not last),
                          v(self.xs_hi.data_ptr()) if entry else None,
                          v(self.xs_lo.data_ptr()) if entry else None, st)
                else:
                    timed("carry", (ln, c > 0, not last, True), "spb_reset_carry_chunk",
                          v(self.w_hi.data_ptr()), v(self.w_lo.data_ptr()),
                          v(self.wa_hi.data_ptr()), v(self.wa_lo.data_ptr()), self.ldc,
                          v(self.xh.data_ptr()), v(self.mdt.data_ptr()), v(self.eps.data_ptr()),
                          v(self.eps2.data_ptr()), v(part6), B, n, self.n_pad, self.kx,
                          self.ke,
                          self.kp, KR, self.splits6, int(not last), int(c > 0), int(not last),
                          st)
                self.launches += 1
                if c > 0:
                    slices += self.splits6
            if entry:  # the row-0 slice sits after K6's (layout [K5 | K6 | row 0])
                slices = self.splits5 + self.splits6 + 1
            call("spb_reduce_partials", v(self.partial.data_ptr()), slices, n, self.n_pad,
                 self.kp, int(c > 0), v(self.grad_w_acc.data_ptr()), st)
            self.launches += 1
        if use_side:
            main.wait_event(self._ev["rg"])
        return self

    def graphed(self, x_like: torch.Tensor, labels_like: torch.Tensor, *,
                static_inputs: bool = False, **run_kwargs):
        """Capture one update on static device buffers shaped like ``x_like`` /
        ``labels_like`` into a CUDA graph; returns ``step(x, labels)`` that copies the batch
        into the static buffers and replays the graph (no per-kernel host launches).  With
        ``static_inputs=True`` the given device tensors ARE the static buffers (the caller
        refills them, e.g. by an async host-to-device copy; ``step()`` just replays).  The
        results land in the engine's buffers as with ``run``."""
        if self.device.type != "cuda":
            raise ValueError("CUDA graphs need a CUDA engine")
        if static_inputs:
            xs, ls = x_like, labels_like
        else:
            xs = torch.empty_like(x_like, device=self.device)
            ls = torch.empty_like(labels_like, device=self.device)
            xs.copy_(x_like)
            ls.copy_(labels_like)
        cs = torch.cuda.Stream(device=self.device)
        cs.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(cs):
            self.run(xs, ls, **run_kwargs)       # first launches (attributes, descriptors)
        torch.cuda.current_stream(self.device).wait_stream(cs)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cs):
            self.run(xs, ls, **run_kwargs)

        def step(x=None, labels=None):
            if x is not None:
                xs.copy_(x, non_blocking=True)
            if labels is not None:
                ls.copy_(labels, non_blocking=True)
            graph.replay()
            return self

        step.graph = graph
        return step

    def _stream_buffers(self, kb):
        """Double-buffered device chunk of the input + copy stream (streaming mode)."""
        if getattr(self, "_xs", None) is None or self._xs.shape[-1] != kb:
            self._xs = torch.empty((2, self.B, self.Tc, kb), dtype=torch.uint8,
                                   device=self.device)
            self._cs = torch.cuda.Stream(device=self.device)
            self._sev_free = [torch.cuda.Event() for _ in range(2)]
            self._sev_ready = [torch.cuda.Event() for _ in range(2)]
        return self._xs

    def check_labels(self, labels_np):
        labels_np = np.asarray(labels_np)
        if labels_np.shape != (self.B,):
            raise ShapeMismatch(f"labels must have shape ({self.B},)")
        if labels_np.size and (labels_np.min() < 0 or labels_np.max() >= self.m):
            bad = labels_np[(labels_np < 0) | (labels_np >= self.m)][0]
            raise LabelOutOfRange(f"label {int(bad)} out of range for {self.m} classes")

    def _forward_rec(self, pass_id, ln, t0, T, common, raster, park, st, timed, meta):
        """K1rec: recurrent dynamics of a chunk from K2's input current (pass 0: raster,
        zsum; parks psi and the chunk spikes for pass B when ``park``)."""
        v = ctypes_void
        alpha, theta, slope, beta, rho, kappa, reset, alif, smooth = common
        timed("forward_a" if pass_id == 0 else "forward_rec_b", meta, "spb_forward_rec_chunk",
              pass_id, v(self.cur.data_ptr()), v(self.wrecT.data_ptr()), int(self.w_f64),
              self.B, self.n, self.Tc, self.KR, ln, t0, T, alpha, theta, slope, beta, rho,
              kappa, reset, alif, smooth, v(self.u.data_ptr()), v(self.a.data_ptr()),
              v(self.zbar.data_ptr()) if pass_id == 0 else None,
              v(self.zsum.data_ptr()) if pass_id == 0 else None,
              v(raster.data_ptr()) if raster is not None else None,
              v(self.psi.data_ptr()) if park else None,
              v(self.zchunk.data_ptr()) if park else None, st)

    def grad_w_rec(self, dtype=torch.float32):
        """Finalised recurrent-weight gradient [n, n] (columns k .. k+n of the
        accumulator over the extended input)."""
        if not self.recurrent:
            raise ValueError("not a recurrent engine")
        out = torch.empty((self.n, self.n), dtype=dtype, device=self.device)
        _lib.call("spb_finalize_grad", ctypes_void(self.grad_w_acc.data_ptr() + 8 * self.k),
                  self.n, self.n, self.kp, ctypes_void(out.data_ptr()),
                  int(dtype == torch.float64), ctypes_void(self._stream()))
        return out

    def grad_w(self, dtype=torch.float32):
        """Finalised input-weight gradient [n, k] in ``dtype`` (device tensor)."""
        out = torch.empty((self.n, self.k), dtype=dtype, device=self.device)
        _lib.call("spb_finalize_grad", ctypes_void(self.grad_w_acc.data_ptr()), self.n, self.k,
                  self.kp, ctypes_void(out.data_ptr()), int(dtype == torch.float64),
                  ctypes_void(self._stream()))
        return out
