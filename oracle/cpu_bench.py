"""CPU baseline timing of the oracle port -- TEST/BENCH INFRASTRUCTURE ONLY.

``bench.py`` uses this for its ``cpu_baseline`` field and for ``--impl reference``:
the reference's algorithm (per-sample online e-prop, gradients.py:132-185, restated in
``oracle/eprop_ref.eprop_forward_mode``) timed on the host cores with one process per
core and single-threaded BLAS, following the reference's own timing conventions
(bench.py:77-99 of the reference: perf_counter around engine calls, inputs generated
outside the timed region).  The Python reference itself cannot travel to the GPU box,
so the port is what runs there ("kind": "port").
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np


def _task(args):
    kind, n, k, m, T_sub, seed = args
    from oracle import eprop_ref as O
    w, w_out = O.init_network_arrays(n, k, m, seed=0, dtype=np.float32)
    x, y = O.poisson_batch(1, k, T_sub, m, seed=seed)
    p = O.Params(alif=kind == "alif")
    xs = x[0].astype(np.float32)
    t0 = time.perf_counter()
    O.eprop_forward_mode(w, w_out, p, xs, int(y[0]))
    return T_sub, time.perf_counter() - t0


def _pool(procs):
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    return mp.get_context("spawn").Pool(procs)


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def time_cpu(kind, n, k, m, T_sub, tasks, procs=None, pool=None):
    """Run ``tasks`` single-sample e-prop computations of ``T_sub`` steps on ``procs``
    worker processes; return (sample*steps/s, wall seconds, procs)."""
    procs = procs or cores()
    own = pool is None
    pool = pool or _pool(procs)
    try:
        pool.map(_task, [(kind, n, k, m, 2, 10_000 + i) for i in range(procs)])  # warm
        t0 = time.perf_counter()
        res = pool.map(_task, [(kind, n, k, m, T_sub, i) for i in range(tasks)])
        wall = time.perf_counter() - t0
    finally:
        if own:
            pool.close()
            pool.join()
    steps = sum(r[0] for r in res)
    return steps / wall, wall, procs
