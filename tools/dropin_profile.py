"""Where the drop-in call's host time goes (eprop_batch_gradient at C3, numpy in/out)."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2501_11407_b200 as P  # noqa: E402
from paper_2501_11407_b200.datasets import poisson_batch  # noqa: E402
from paper_2501_11407_b200.gradients import eprop_batch_gradient  # noqa: E402

net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=1024, n_inputs=700, n_classes=20,
                                   precision="f32", seed=0))
x, y = poisson_batch(256, 700, 250, 20, seed=1000)
xb = np.packbits(x, axis=-1, bitorder="little")
for tag, xin, kw in (("packed", xb, {"packed": True}), ("counts", x, {})):
    for _ in range(3):
        eprop_batch_gradient(net, xin, y, **kw)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        eprop_batch_gradient(net, xin, y, **kw)
    print(tag, "ms/call", (time.perf_counter() - t0) * 100)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(10):
        eprop_batch_gradient(net, xin, y, **kw)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)
