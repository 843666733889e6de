"""CPU baseline timing -- TEST/BENCH INFRASTRUCTURE ONLY.

``bench.py`` uses this for its ``cpu_baseline`` field and for ``--impl reference``.
Two CPU arms, both timed on the host cores with one process per core and
single-threaded BLAS, following the reference's own timing conventions (bench.py:77-99
of the reference: perf_counter around the engine call, inputs and weights generated
outside the timed region, f32 networks as in BenchConfig):

* ``impl="reference"`` -- the UNMODIFIED reference package (``sparseprop`` 0.1.0,
  installed into ``baseline/_ref`` with pip from /root/reference/pkg; git-ignored, it
  travels to the GPU box with the repo snapshot): ``ENGINES["eprop-sparse"]``
  (gradients.py:132-185, 436-441) on ``init_network(NetworkSpec(..., precision="f32",
  seed=0))`` and ``generate_poisson_dataset`` inputs (training.py:35-50,
  datasets.py:70-83).  This is the reference arm (``"kind": "reference"``).
* ``impl="port"`` -- the oracle's restatement of the same algorithm
  (``oracle/eprop_ref.eprop_forward_mode``), kept as a second, labelled number.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available() -> bool:
    return os.path.isfile(os.path.join(REF_DIR, "sparseprop", "gradients.py"))


def _task(args):
    impl, kind, n, k, m, T_sub, seed = args
    if impl == "reference":
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from sparseprop.datasets import generate_poisson_dataset
        from sparseprop.gradients import ENGINES
        from sparseprop.training import NetworkSpec, init_network
        net = init_network(NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m,
                                       precision="f32", seed=0))
        ds = generate_poisson_dataset(1, k, T_sub, m, seed=seed)
        x = ds.input_array(0, dtype=net.neuron.w.dtype)
        label = ds.label_of(0)
        engine = ENGINES["eprop-sparse"]
        t0 = time.perf_counter()
        engine(net, x, label)
        return T_sub, time.perf_counter() - t0
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


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def warm(pool, procs, kind, n, k, m, impl="port"):
    """One short call per worker: imports, the reference's lru-cached step graphs."""
    pool.map(_task, [(impl, kind, n, k, m, 2, 10_000 + i) for i in range(procs)], chunksize=1)


def time_cpu(kind, n, k, m, T_sub, tasks, procs=None, pool=None, impl="port", warmed=False):
    """Run ``tasks`` single-sample e-prop computations of ``T_sub`` steps on ``procs``
    worker processes; return (sample*steps/s, wall seconds, procs)."""
    procs = procs or cores()
    own = pool is None
    pool = pool or _pool(procs)
    try:
        if not warmed:
            warm(pool, procs, kind, n, k, m, impl)
        t0 = time.perf_counter()
        res = pool.map(_task, [(impl, kind, n, k, m, T_sub, i) for i in range(tasks)],
                       chunksize=1)
        wall = time.perf_counter() - t0
    finally:
        if own:
            pool.close()
            pool.join()
    steps = sum(r[0] for r in res)
    return steps / wall, wall, procs
