"""Time K21 (fused projection + dynamics) on the C3 shape with parts of the epilogue
switched off (FusedParams::probe) to locate the bottleneck.  GPU only."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2501_11407_b200 as P
from paper_2501_11407_b200 import _lib
from paper_2501_11407_b200.engine import EpropEngine
from paper_2501_11407_b200.datasets import poisson_batch

kind, n, k, m, T, B = "alif", 1024, 700, 20, 250, int(sys.argv[1]) if len(sys.argv) > 1 else 256
net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m, precision="f32"))
x, y = poisson_batch(B, k, T, m, seed=1)
eng = EpropEngine(n, k, m, B, alif=True, chunk=255, fused=True)
eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
xd = torch.from_numpy(x).cuda()
yd = torch.from_numpy(y).cuda()
eng.run(xd, yd, beta=0.8, rho=0.96)
torch.cuda.synchronize()
v = ctypes.c_void_p
st = v(torch.cuda.current_stream().cuda_stream)
for probe in (0, 2, 1, 3):
    for psi in (True, False):
        ts = []
        for rep in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.call("spb_fused_forward_probe", 0, v(eng.xq.data_ptr()), v(eng.wq.data_ptr()),
                      v(eng.sexp.data_ptr()), B, n, eng.n_pad32, eng.Kpad, eng.P, eng.Tc, eng.KR, T,
                      0, T, 0.95, 1.0, 10.0, 0.8, 0.96, 0.95, 0, 0, v(eng.u.data_ptr()),
                      v(eng.a.data_ptr()), v(eng.zbar.data_ptr()), v(eng.zsum.data_ptr()), None,
                      v(eng.psi.data_ptr()) if psi else None, eng.sm_count, probe, st)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"B={B} probe={probe} psi={psi}: {np.median(ts[1:]):.4f} ms", flush=True)
