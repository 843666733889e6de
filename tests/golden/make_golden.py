"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every number stored here comes from the unmodified reference package
``sparseprop`` 0.1.0 (``/root/reference/pkg/src/sparseprop``):

* inputs      -- ``datasets.generate_poisson_dataset`` (datasets.py:70-83) + ``input_array``
* weights     -- ``training.init_network`` (training.py:35-50)
* gradients   -- ``gradients.eprop_sparse_gradient`` (gradients.py:132-185) and
                 ``gradients.bptt_gradient`` (gradients.py:188-231)
* rasters     -- ``gradients.network_loss`` (gradients.py:349-365)

Inputs and weights are NOT stored; they are regenerated from the seeds by
``oracle.eprop_ref.poisson_batch`` / ``init_network_arrays``, and the stored
``x_checksum`` / ``w_checksum`` pin that the regeneration is bit-identical.  For the
large SHD/SSC-shaped cases only a fixed random subset of gradient entries plus
whole-tensor sums/norms are stored, to keep fixtures small.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from sparseprop.datasets import generate_poisson_dataset  # noqa: E402
from sparseprop.gradients import bptt_gradient, eprop_sparse_gradient, network_loss  # noqa: E402
from sparseprop.training import NetworkSpec, init_network  # noqa: E402

from oracle.eprop_ref import init_network_arrays, poisson_batch  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def grad_subset_idx(n, k, count, seed):
    rng = np.random.default_rng(seed)
    return rng.choice(n * k, size=min(count, n * k), replace=False)


CASES = [
    # name, kind, n, k, m, T, B, precision, reset, full, with_bptt, seed_net, seed_data
    ("c1_lif_f64", "lif", 32, 16, 2, 100, 8, "f64", False, True, True, 0, 0),
    ("c1_alif_f64", "alif", 32, 16, 2, 100, 8, "f64", False, True, True, 0, 0),
    ("c1_lif_f32", "lif", 32, 16, 2, 100, 8, "f32", False, True, True, 0, 0),
    ("c1_alif_f32", "alif", 32, 16, 2, 100, 8, "f32", False, True, True, 0, 0),
    ("c1_lif_reset_f64", "lif", 32, 16, 2, 100, 8, "f64", True, True, True, 1, 1),
    ("c1_alif_reset_f64", "alif", 32, 16, 2, 100, 8, "f64", True, True, True, 1, 1),
    ("mid_alif_f64", "alif", 96, 40, 5, 60, 4, "f64", False, True, True, 3, 3),
    ("c2_lif_f64", "lif", 256, 700, 20, 250, 2, "f64", False, False, False, 0, 0),
    ("c3_alif_f64", "alif", 1024, 700, 20, 250, 2, "f64", False, False, False, 0, 0),
    ("c4_alif_f64", "alif", 2048, 700, 35, 500, 1, "f64", False, False, False, 0, 0),
]


def main():
    only = set(sys.argv[1:])
    for (name, kind, n, k, m, T, B, prec, reset, full, with_bptt,
         seed_net, seed_data) in CASES:
        if only and name not in only:
            continue
        t0 = time.time()
        spec = NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m,
                           precision=prec, reset=reset, seed=seed_net)
        net = init_network(spec)
        dtype = net.neuron.w.dtype
        ds = generate_poisson_dataset(B, k, T, m, seed=seed_data)
        xs = np.stack([ds.input_array(s, dtype=dtype) for s in range(B)])
        labels = np.array([ds.label_of(s) for s in range(B)], dtype=np.int64)
        # pin the vectorised regenerators used by the tests
        xv, lv = poisson_batch(B, k, T, m, seed=seed_data)
        assert np.array_equal(xv.astype(dtype), xs) and np.array_equal(lv, labels)
        w, w_out = init_network_arrays(n, k, m, seed=seed_net, dtype=dtype)
        assert np.array_equal(w, net.neuron.w) and np.array_equal(w_out, net.readout.w_out)

        out = dict(kind=kind, n=n, k=k, m=m, T=T, B=B, precision=prec, reset=reset,
                   seed_net=seed_net, seed_data=seed_data,
                   x_checksum=sha(xv), w_checksum=sha(w), labels=labels)
        losses, rsums, rasters = [], [], []
        gw, gwo, bw, bwo = [], [], [], []
        idx = None if full else grad_subset_idx(n, k, 4096, 1234)
        gw_sum = np.zeros((n, k))
        gwo_sum = np.zeros((m, n))
        for s in range(B):
            res = eprop_sparse_gradient(net, xs[s], int(labels[s]))
            _, _, raster = network_loss(net, xs[s], int(labels[s]))
            losses.append(res.loss)
            rsums.append(np.asarray(res.readout_sum, dtype=np.float64))
            rasters.append(np.packbits(raster, axis=-1))
            gw_sum += res.grads["w"]
            gwo_sum += res.grads["w_out"]
            if full:
                gw.append(res.grads["w"])
                gwo.append(res.grads["w_out"])
            else:
                gw.append(res.grads["w"].ravel()[idx])
                gwo.append(res.grads["w_out"])
            if with_bptt:
                rb = bptt_gradient(net, xs[s], int(labels[s]))
                bw.append(rb.grads["w"])
                bwo.append(rb.grads["w_out"])
        out.update(loss=np.array(losses), readout_sum=np.stack(rsums),
                   raster_packed=np.stack(rasters), eprop_w=np.stack(gw),
                   eprop_w_out=np.stack(gwo), eprop_w_batch_sum=gw_sum if full else gw_sum.ravel()[idx],
                   eprop_w_out_batch_sum=gwo_sum,
                   eprop_w_batch_norm=np.linalg.norm(gw_sum),
                   eprop_w_batch_total=gw_sum.sum())
        if idx is not None:
            out["grad_idx"] = idx
        if with_bptt:
            out.update(bptt_w=np.stack(bw), bptt_w_out=np.stack(bwo))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(f"{name}: {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
