"""Golden fixtures for the rows next to the gradient path, produced by
running the REFERENCE itself in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_ext.py

* smooth_*.npz   -- ``eprop_sparse_gradient(..., smooth=True)`` and the smooth forward
                    raster of ``network_loss`` (gradients.py:132-185, 349-365)
* train_*.npz    -- ``training.train`` (training.py:116-166): per-update metrics and the
                    final weights, SGD and Adam, f32 and f64, LIF and ALIF
* ds_small.spikes, ds_pool.npz -- ``save_spike_dataset`` bytes and ``pool_channels``
                    output (datasets.py:86-159)
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from sparseprop.datasets import (generate_poisson_dataset, pool_channels,  # noqa: E402
                                 save_spike_dataset)
from sparseprop.gradients import eprop_sparse_gradient, network_loss  # noqa: E402
from sparseprop.training import NetworkSpec, init_network, train  # noqa: E402

SMOOTH = [
    # name, kind, n, k, m, T, B, precision, reset
    ("smooth_lif_f64", "lif", 32, 16, 2, 100, 8, "f64", False),
    ("smooth_alif_f64", "alif", 32, 16, 2, 100, 8, "f64", False),
    ("smooth_alif_f32", "alif", 32, 16, 2, 100, 8, "f32", False),
]

TRAIN = [
    # name, kind, n, k, m, precision, optimizer, lr, epochs, max_updates, (N, T, seed)
    ("train_lif_sgd_f64", "lif", 24, 20, 3, "f64", "sgd", 1e-4, 2, None, (8, 40, 0)),
    ("train_alif_adam_f64", "alif", 24, 20, 3, "f64", "adam", 1e-3, 2, None, (8, 40, 0)),
    ("train_lif_adam_f32", "lif", 24, 20, 3, "f32", "adam", 1e-3, 1, None, (8, 40, 1)),
    ("train_alif_sgd_f32", "alif", 24, 20, 3, "f32", "sgd", 1e-4, 1, 6, (8, 40, 1)),
]


def main():
    only = set(sys.argv[1:])
    for name, kind, n, k, m, T, B, prec, reset in SMOOTH:
        if only and name not in only:
            continue
        net = init_network(NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m,
                                       precision=prec, reset=reset, seed=0))
        ds = generate_poisson_dataset(B, k, T, m, seed=0)
        dtype = net.neuron.w.dtype
        gw, gwo, loss, rs, ras = [], [], [], [], []
        for s in range(B):
            x = ds.input_array(s, dtype=dtype)
            r = eprop_sparse_gradient(net, x, ds.label_of(s), smooth=True)
            _, _, raster = network_loss(net, x, ds.label_of(s), smooth=True)
            gw.append(r.grads["w"])
            gwo.append(r.grads["w_out"])
            loss.append(r.loss)
            rs.append(np.asarray(r.readout_sum, np.float64))
            ras.append(np.packbits(raster, axis=-1))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), kind=kind, n=n, k=k, m=m, T=T,
                            B=B, precision=prec, reset=reset, seed_net=0, seed_data=0,
                            eprop_w=np.stack(gw), eprop_w_out=np.stack(gwo),
                            loss=np.array(loss), readout_sum=np.stack(rs),
                            raster_packed=np.stack(ras))
        print(name, flush=True)
    for name, kind, n, k, m, prec, opt, lr, epochs, mu, (N, T, seed) in TRAIN:
        if only and name not in only:
            continue
        spec = NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m, precision=prec,
                           seed=seed)
        ds = generate_poisson_dataset(N, k, T, m, seed=seed)
        net, metrics = train(spec, ds, optimizer=opt, lr=lr, epochs=epochs, max_updates=mu)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), kind=kind, n=n, k=k, m=m,
                            precision=prec, optimizer=opt, lr=lr, epochs=epochs,
                            max_updates=-1 if mu is None else mu, N=N, T=T, seed=seed,
                            loss=np.array([r.loss for r in metrics]),
                            accuracy=np.array([r.accuracy for r in metrics]),
                            epoch=np.array([r.epoch for r in metrics]),
                            w=net.neuron.w, w_out=net.readout.w_out)
        print(name, len(metrics), flush=True)
    if not only or "ds" in only:
        ds = generate_poisson_dataset(4, 12, 15, 3, seed=2)
        save_spike_dataset(ds, os.path.join(HERE, "ds_small.spikes"))
        big = generate_poisson_dataset(3, 20, 15, 2, seed=5)
        pooled = pool_channels(big, 4)
        np.savez_compressed(os.path.join(HERE, "ds_pool.npz"),
                            events=np.array(big.events, dtype=np.int64),
                            labels=np.array(big.labels, dtype=np.int64),
                            pooled_events=np.array(pooled.events, dtype=np.int64),
                            pooled_weights=np.array(pooled.weights, dtype=np.float64),
                            pooled_input=np.stack([pooled.input_array(s) for s in range(3)]))
        print("ds", flush=True)


if __name__ == "__main__":
    main()
