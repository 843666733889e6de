"""Spike-event datasets for the e-prop path: synthesis, SPIKES v1 I/O, channel pooling,
and the dense / bit-packed batch tensors the B200 engine consumes.

Drop-in for the reference's ``sparseprop.datasets`` (datasets.py:1-159): same names,
fields, file format, RNG call sequence and error types, so a caller of the reference
finds the same behaviour.  What changes is the representation: events live in one
int64 ``[E, 3]`` array (sample, t, channel) instead of a Python list of tuples, every
operation is vectorised (no O(events) Python loops -- SURVEY.md 8(f)-2), and a dataset
converts directly into the uint8 count tensor or the bit-packed spike tensor that the
engine streams to the GPU chunk by chunk (engine.py, ``bits=True``).

SPIKES v1 (datasets.py:1-11)::

    SPIKES v1 <n_samples> <n_channels> <n_steps>
    <sample> <t> <channel>        # one line per event
    LABELS
    <sample> <class>              # one line per sample
"""

from __future__ import annotations

from collections.abc import Sequence

import numpy as np

from .errors import NotDivisible, ParseError, RangeError


class EventList(Sequence):
    """Read-only sequence of ``(sample, t, channel)`` tuples backed by an int64 [E, 3]
    array; compares equal to a list of tuples with the same content (the reference's
    ``events`` field is such a list, datasets.py:28)."""

    __slots__ = ("array",)

    def __init__(self, array):
        a = np.asarray(array, dtype=np.int64)
        if a.size == 0:
            a = np.zeros((0, 3), dtype=np.int64)
        if a.ndim != 2 or a.shape[1] != 3:
            raise ValueError("events must be (sample, t, channel) triples")
        self.array = a

    def __len__(self):
        return self.array.shape[0]

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [tuple(int(v) for v in r) for r in self.array[i]]
        r = self.array[i]
        return (int(r[0]), int(r[1]), int(r[2]))

    def __iter__(self):
        return (tuple(r) for r in self.array.tolist())

    def __eq__(self, other):
        if isinstance(other, EventList):
            return np.array_equal(self.array, other.array)
        if isinstance(other, (list, tuple)):
            if len(other) != len(self):
                return False
            return len(other) == 0 or np.array_equal(self.array, np.asarray(other, np.int64))
        return NotImplemented

    def __repr__(self):
        return f"EventList({len(self)} events)"


def _as_events(events) -> np.ndarray:
    if isinstance(events, EventList):
        return events.array
    a = np.asarray(list(events) if not isinstance(events, np.ndarray) else events, dtype=np.int64)
    if a.size == 0:
        return np.zeros((0, 3), dtype=np.int64)
    if a.ndim != 2 or a.shape[1] != 3:
        raise ValueError("events must be (sample, t, channel) triples")
    return a


class SpikeDataset:
    """Event-list dataset (datasets.py:23-57).

    ``events``  (sample, t, channel) triples (list of tuples or int array [E, 3])
    ``labels``  (sample, class) pairs, one per sample
    ``weights`` per-event multiplicities after pooling (None = unit events)
    """

    def __init__(self, n_samples: int, n_channels: int, n_steps: int, events, labels,
                 weights=None):
        self.n_samples = int(n_samples)
        self.n_channels = int(n_channels)
        self.n_steps = int(n_steps)
        self.events = EventList(_as_events(events))
        self.labels = [(int(s), int(c)) for s, c in labels]
        self.weights = None if weights is None else np.asarray(weights, dtype=np.float64)
        self._validate()
        self._label_arr = None

    # datasets.py:32-43: the first offending event (in list order) raises, checking
    # time, then channel, then sample
    def _validate(self):
        ev = self.events.array
        if len(ev):
            s, t, c = ev[:, 0], ev[:, 1], ev[:, 2]
            bad_t = (t < 0) | (t >= self.n_steps)
            bad_c = (c < 0) | (c >= self.n_channels)
            bad_s = (s < 0) | (s >= self.n_samples)
            bad = bad_t | bad_c | bad_s
            if bad.any():
                e = int(np.argmax(bad))
                if bad_t[e]:
                    raise RangeError(f"event time {int(t[e])} out of range [0, {self.n_steps})")
                if bad_c[e]:
                    raise RangeError(f"event channel {int(c[e])} out of range "
                                     f"[0, {self.n_channels})")
                raise RangeError(f"event sample {int(s[e])} out of range [0, {self.n_samples})")
        if len(self.labels) != self.n_samples:
            raise RangeError("every sample needs exactly one label")
        if self.weights is not None and self.weights.shape != (len(ev),):
            raise RangeError("one weight per event required")

    def __eq__(self, other):
        if not isinstance(other, SpikeDataset):
            return NotImplemented
        same_w = (self.weights is None and other.weights is None) or (
            self.weights is not None and other.weights is not None
            and np.array_equal(self.weights, other.weights))
        return (self.n_samples, self.n_channels, self.n_steps) == (
            other.n_samples, other.n_channels, other.n_steps) and self.events == other.events \
            and self.labels == other.labels and same_w

    # ---- reference accessors ----
    def label_array(self) -> np.ndarray:
        """Labels as int64 [n_samples] indexed by sample (last pair wins, like dict())."""
        if self._label_arr is None:
            arr = np.zeros(self.n_samples, dtype=np.int64)
            for s, c in self.labels:
                if 0 <= s < self.n_samples:
                    arr[s] = c
            self._label_arr = arr
        return self._label_arr

    def label_of(self, sample: int) -> int:
        """datasets.py:45-46 (KeyError for a sample without a label pair)."""
        return dict(self.labels)[sample]

    def _sel(self, sample):
        return self.events.array[:, 0] == sample

    def input_array(self, sample: int, dtype=np.float64) -> np.ndarray:
        """Dense (n_steps, n_channels) input currents for one sample (datasets.py:48-54)."""
        out = np.zeros((self.n_steps, self.n_channels), dtype=dtype)
        m = self._sel(sample)
        ev = self.events.array[m]
        w = self.weights[m] if self.weights is not None else np.ones(len(ev))
        # per-sample event multiplicities add up in float64, then cast (the reference
        # accumulates in dtype; pooled counts are small integers, exact either way)
        acc = np.zeros((self.n_steps, self.n_channels), dtype=np.float64)
        np.add.at(acc, (ev[:, 1], ev[:, 2]), w)
        out[...] = acc
        return out

    def total_spikes(self, sample: int) -> float:
        m = self._sel(sample)
        if self.weights is None:
            return float(np.count_nonzero(m))
        return float(np.sum(self.weights[m]))

    # ---- device-side batch tensors ----
    def counts(self, samples=None) -> np.ndarray:
        """uint8 event counts [S, n_steps, n_channels] for ``samples`` (default: all), the
        engine's count input.  Pooled multiplicities must be integers <= 255."""
        samples = np.arange(self.n_samples) if samples is None else np.asarray(samples)
        pos = np.full(self.n_samples, -1, dtype=np.int64)
        pos[samples] = np.arange(len(samples))
        ev = self.events.array
        keep = pos[ev[:, 0]] >= 0 if len(ev) else np.zeros(0, bool)
        ev = ev[keep]
        w = self.weights[keep] if self.weights is not None else None
        acc = np.zeros((len(samples), self.n_steps, self.n_channels), dtype=np.int64)
        if w is None:
            np.add.at(acc, (pos[ev[:, 0]], ev[:, 1], ev[:, 2]), 1)
        else:
            wi = np.rint(w)
            if not np.array_equal(wi, w) or (len(w) and w.min() < 0):
                raise ValueError("pooled event weights must be non-negative integers")
            np.add.at(acc, (pos[ev[:, 0]], ev[:, 1], ev[:, 2]), wi.astype(np.int64))
        if acc.size and acc.max() > 255:
            raise ValueError("event counts above 255 do not fit the uint8 input operand")
        return acc.astype(np.uint8)

    def packed_bits(self, samples=None) -> np.ndarray:
        """Bit-packed binary spikes [S, n_steps, ceil(n_channels/8)] (numpy.packbits,
        little bit order): 8x less host->device traffic than counts.  Requires every
        count to be 0 or 1 (unpooled data)."""
        c = self.counts(samples)
        if c.size and c.max() > 1:
            raise ValueError("bit-packing needs binary spikes; use counts() for pooled data")
        return np.packbits(c, axis=-1, bitorder="little")

    def is_binary(self) -> bool:
        if self.weights is not None and len(self.weights) and np.any(self.weights != 1.0):
            return False
        ev = self.events.array
        if len(ev) == 0:
            return True
        key = (ev[:, 0] * self.n_steps + ev[:, 1]) * self.n_channels + ev[:, 2]
        return np.unique(key).size == key.size


# --------------------------------------------------------------------------------------
# synthesis (datasets.py:60-83)
# --------------------------------------------------------------------------------------

def sample_rate_patterns(n_classes: int, n_channels: int, rng) -> np.ndarray:
    """Per-class firing-rate patterns in [0.01, 0.2] spikes/step (datasets.py:60-62)."""
    return rng.uniform(0.01, 0.2, size=(n_classes, n_channels))


def sample_events(rates: np.ndarray, n_steps: int, rng) -> np.ndarray:
    """Independent per-step binary events at the given per-channel rates (datasets.py:65-67)."""
    return rng.random((n_steps, rates.shape[0])) < rates


def generate_poisson_dataset(n_samples: int, n_channels: int, n_steps: int, n_classes: int,
                             seed: int) -> SpikeDataset:
    """Synthetic classification task, deterministic per seed (datasets.py:70-83): the same
    RNG calls in the same order as the reference, events in (sample, t, channel) order."""
    rng = np.random.default_rng(seed)
    rates = sample_rate_patterns(n_classes, n_channels, rng)
    chunks, labels = [], []
    for s in range(n_samples):
        label = int(rng.integers(n_classes))
        labels.append((s, label))
        grid = sample_events(rates[label], n_steps, rng)
        t, c = np.nonzero(grid)
        if len(t):
            chunks.append(np.stack([np.full(len(t), s, np.int64), t, c], axis=1))
    ev = np.concatenate(chunks) if chunks else np.zeros((0, 3), np.int64)
    return SpikeDataset(n_samples, n_channels, n_steps, ev, labels)


def poisson_batch(n_samples: int, n_channels: int, n_steps: int, n_classes: int, seed: int = 0):
    """Dense uint8 [B, T, k] equivalent of ``generate_poisson_dataset`` followed by
    ``input_array`` for every sample, plus the labels: the same generator and RNG calls,
    so the bits are identical (checked against the reference in tests/test_oracle.py)."""
    rng = np.random.default_rng(seed)
    rates = rng.uniform(0.01, 0.2, size=(n_classes, n_channels))
    x = np.empty((n_samples, n_steps, n_channels), dtype=np.uint8)
    labels = np.empty(n_samples, dtype=np.int64)
    for s in range(n_samples):
        y = int(rng.integers(n_classes))
        labels[s] = y
        np.less(rng.random((n_steps, n_channels)), rates[y], out=x[s], casting="unsafe")
    return x, labels


class DevicePoisson:
    """Synthetic Poisson spike batches generated ON the device.

    Per-class rates come from ``sample_rate_patterns`` with ``numpy.random.default_rng(
    seed)`` exactly as the reference draws them (datasets.py:60-62, 75); labels per batch
    from a numpy generator; the Bernoulli grid itself is drawn by the kernel
    ``spb_poisson_bits`` (Philox4x32-10, counter = (channel byte, step, sample)), so a
    batch never crosses PCIe.  Same distribution as ``sample_events``, not numpy's bits --
    parity runs use ``poisson_batch``.  ``batch(B, T)`` returns (bits uint8 [B, T,
    ceil(k/8)] on the device, labels int64 [B] on the device) for ``engine.run(...,
    bits=True)``.
    """

    def __init__(self, n_classes: int, n_channels: int, seed: int = 0, device=None):
        import torch
        self.torch = torch
        self.k, self.m = int(n_channels), int(n_classes)
        rng = np.random.default_rng(seed)
        self.rates_np = sample_rate_patterns(n_classes, n_channels, rng)
        self.device = torch.device(device if device is not None else "cuda")
        self.rates = torch.from_numpy(self.rates_np.astype(np.float32)).to(self.device)
        self.seed = int(seed)
        self._label_rng = rng
        self._calls = 0

    def batch(self, B: int, T: int, out=None, labels=None):
        from . import _lib
        torch = self.torch
        if labels is None:
            lab = self._label_rng.integers(self.m, size=B).astype(np.int64)
            labels = torch.from_numpy(lab).to(self.device)
        kb = (self.k + 7) // 8
        if out is None:
            out = torch.empty((B, T, kb), dtype=torch.uint8, device=self.device)
        key = (self.seed * 0x9E3779B97F4A7C15 + self._calls) & 0xFFFFFFFFFFFFFFFF
        self._calls += 1
        import ctypes
        _lib.call("spb_poisson_bits", ctypes.c_void_p(self.rates.data_ptr()),
                  ctypes.c_void_p(labels.data_ptr()), B, T, self.k, 0, key,
                  ctypes.c_void_p(out.data_ptr()), T * kb,
                  ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))
        return out, labels


# --------------------------------------------------------------------------------------
# SPIKES v1 I/O (datasets.py:86-135)
# --------------------------------------------------------------------------------------

def _canonical(ev: np.ndarray) -> np.ndarray:
    if len(ev) == 0:
        return ev
    return ev[np.lexsort((ev[:, 2], ev[:, 1], ev[:, 0]))]


def save_spike_dataset(ds: SpikeDataset, path) -> None:
    """Write SPIKES v1 in canonical (sorted) order; byte-identical round trips."""
    if ds.weights is not None:
        raise ParseError("SPIKES v1 stores unit events only; save before pooling")
    ev = _canonical(ds.events.array)
    parts = [f"SPIKES v1 {ds.n_samples} {ds.n_channels} {ds.n_steps}"]
    if len(ev):
        parts.append("\n".join(" ".join(map(str, r)) for r in ev.tolist()))
    parts.append("LABELS")
    lab = sorted(ds.labels)
    if lab:
        parts.append("\n".join(f"{s} {c}" for s, c in lab))
    with open(path, "w") as fh:
        fh.write("\n".join(parts) + "\n")


_HEADER_MSG = "line 1: expected 'SPIKES v1 <n_samples> <n_channels> <n_steps>'"


def _parse_section_fast(lines, width):
    """Vectorised parse of whitespace-separated integer lines; None if any line is
    malformed (the slow path then finds it and reports its line number)."""
    if not lines:
        return np.zeros((0, width), dtype=np.int64)
    toks = " ".join(lines).split()
    if len(toks) != width * len(lines):
        return None
    try:
        arr = np.array(toks, dtype=np.int64)
    except (ValueError, OverflowError):
        return None
    arr = arr.reshape(len(lines), width)
    # a line with the right total token count but a wrong per-line count would shift
    # fields; check per line
    counts = np.fromiter((len(ln.split()) for ln in lines), dtype=np.int64, count=len(lines))
    if np.any(counts != width):
        return None
    return arr


def _parse_slow(lines, linenos, width, what, fmt):
    rows = []
    for ln, no in zip(lines, linenos):
        parts = ln.split()
        if len(parts) != width:
            raise ParseError(f"line {no}: expected '{fmt}'")
        try:
            rows.append(tuple(int(x) for x in parts))
        except ValueError:
            raise ParseError(f"line {no}: non-integer {what} field") from None
    return np.asarray(rows, dtype=np.int64).reshape(-1, width)


def load_spike_dataset(path) -> SpikeDataset:
    """Parse SPIKES v1 (datasets.py:101-135): same error messages with line numbers."""
    with open(path) as fh:
        raw = fh.read().splitlines()
    if not raw:
        raise ParseError("line 1: empty file")
    header = raw[0].split()
    if len(header) != 5 or header[0] != "SPIKES" or header[1] != "v1":
        raise ParseError(_HEADER_MSG)
    try:
        n_samples, n_channels, n_steps = (int(x) for x in header[2:])
    except ValueError:
        raise ParseError("line 1: header counts must be integers") from None
    ev_lines, ev_nos, lab_lines, lab_nos = [], [], [], []
    section = ev_lines, ev_nos
    for lineno, line in enumerate(raw[1:], start=2):
        st = line.strip()
        if not st:
            continue
        if st == "LABELS":
            section = lab_lines, lab_nos
            continue
        section[0].append(line)
        section[1].append(lineno)
    ev = _parse_section_fast(ev_lines, 3)
    if ev is None:
        ev = _parse_slow(ev_lines, ev_nos, 3, "event", "<sample> <t> <channel>")
    lab = _parse_section_fast(lab_lines, 2)
    if lab is None:
        lab = _parse_slow(lab_lines, lab_nos, 2, "label", "<sample> <class>")
    return SpikeDataset(n_samples, n_channels, n_steps, ev,
                        [(int(s), int(c)) for s, c in lab.tolist()])


# --------------------------------------------------------------------------------------
# channel pooling (datasets.py:138-159)
# --------------------------------------------------------------------------------------

def pool_channels(ds: SpikeDataset, factor: int) -> SpikeDataset:
    """Sum groups of ``factor`` adjacent channels into one input channel; pooled inputs
    are integer-valued counts, not re-binarised spikes (datasets.py:138-159)."""
    if ds.n_channels % factor != 0:
        raise NotDivisible(f"{ds.n_channels} channels not divisible by factor {factor}")
    ev = ds.events.array
    nc = ds.n_channels // factor
    w = ds.weights if ds.weights is not None else np.ones(len(ev))
    if len(ev) == 0:
        return SpikeDataset(ds.n_samples, nc, ds.n_steps, ev, list(ds.labels),
                            weights=np.zeros(0))
    key = (ev[:, 0] * ds.n_steps + ev[:, 1]) * nc + ev[:, 2] // factor
    uk, inv = np.unique(key, return_inverse=True)      # sorted = (s, t, c') order
    tot = np.zeros(len(uk), dtype=np.float64)
    # the reference sums each key's weights in event order (dict accumulation)
    np.add.at(tot, inv, w)
    c2 = uk % nc
    st = uk // nc
    out = np.stack([st // ds.n_steps, st % ds.n_steps, c2], axis=1)
    return SpikeDataset(ds.n_samples, nc, ds.n_steps, out, list(ds.labels), weights=tot)
