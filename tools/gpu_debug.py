"""Quick GPU sanity run: C1-shaped ALIF/LIF through the engine vs the oracle (prints errors)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2501_11407_b200 as P
from paper_2501_11407_b200.datasets import poisson_batch
from oracle import eprop_ref as O

for kind, n, k, m, T, B, chunk in [("lif", 32, 16, 2, 100, 8, 32), ("alif", 32, 16, 2, 100, 8, 32),
                                   ("alif", 200, 90, 7, 77, 12, 16)]:
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m, precision="f64", seed=0))
    x, labels = poisson_batch(B, k, T, m, seed=0)
    t0 = time.time()
    r = P.eprop_batch_gradient(net, x, labels, chunk=chunk)
    torch.cuda.synchronize()
    ref = O.eprop_two_pass_batch(net.neuron.w, net.readout.w_out, O.Params(alif=kind == "alif"), x, labels)
    def rel(a, b): return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
    print(kind, n, k, "loss rel", rel(r.loss, ref.loss), "gw rel", rel(r.grads["w"], ref.grad_w),
          "gwo rel", rel(r.grads["w_out"], ref.grad_w_out), f"{time.time()-t0:.2f}s", flush=True)
