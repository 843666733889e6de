"""Synthetic spike inputs for parity and throughput runs.

``poisson_batch`` returns the dense uint8 [B, T, k] equivalent of the reference's
``generate_poisson_dataset(B, k, T, m, seed)`` followed by ``input_array(s)`` for every
sample (datasets.py:60-83): the same generator, the same RNG calls in the same order
(per-class rates U[0.01, 0.2], then per sample a label and a Bernoulli grid), so the
bits are identical -- checked against the reference in tests/test_oracle.py.
"""

from __future__ import annotations

import numpy as np


def poisson_batch(n_samples: int, n_channels: int, n_steps: int, n_classes: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    rates = rng.uniform(0.01, 0.2, size=(n_classes, n_channels))
    x = np.empty((n_samples, n_steps, n_channels), dtype=np.uint8)
    labels = np.empty(n_samples, dtype=np.int64)
    for s in range(n_samples):
        y = int(rng.integers(n_classes))
        labels[s] = y
        np.less(rng.random((n_steps, n_channels)), rates[y], out=x[s], casting="unsafe")
    return x, labels
