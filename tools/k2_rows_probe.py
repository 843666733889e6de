import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2501_11407_b200 as P
from paper_2501_11407_b200 import _lib
from paper_2501_11407_b200.engine import EpropEngine
from paper_2501_11407_b200.datasets import poisson_batch
B, n, k, T = 256, 1024, 700, 250
net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=n, n_inputs=k, n_classes=20, precision="f32"))
x, y = poisson_batch(B, k, T, 20, seed=1)
eng = EpropEngine(n, k, 20, B, alif=True, chunk=255)
eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()); torch.cuda.synchronize()
v = ctypes.c_void_p; st = v(torch.cuda.current_stream().cuda_stream)
for rep in range(3):
  for M in (B * eng.KR, B * T):
    ts = []
    for r in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("spb_input_proj_probe", v(eng.xq.data_ptr()), v(eng.wq.data_ptr()), v(eng.sexp.data_ptr()), M, n, eng.n_pad32, k, eng.Kpad, eng.P, v(eng.cur.data_ptr()), eng.sm_count, 1, 0, st)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(M, f"{np.median(ts[2:]):.4f} ms", flush=True)
