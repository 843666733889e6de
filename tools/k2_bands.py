"""K2 (W-resident INT8 projection) at the C3 shape under different tile walks:
SPB_K2_BANDS row bands (TileWalk) and/or SPB_K2_PERSIST (MB of L2 persisting window on
the spike operand).  Prints the median CUDA-event time per setting and checks that the
currents are bitwise those of the default walk.
  python tools/k2_bands.py 1,2,4,8 [reps] [B n T]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2501_11407_b200 as P
from paper_2501_11407_b200 import _lib
from paper_2501_11407_b200.engine import EpropEngine
from paper_2501_11407_b200.datasets import poisson_batch

bands = [int(b) for b in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8").split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
B, n, k, T = 256, 1024, 700, 250
if len(sys.argv) > 5:
    B, n, T = int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
from paper_2501_11407_b200.engine import default_chunk
chunk = default_chunk(T, B, n, k, True)
net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=n, n_inputs=k, n_classes=20, precision="f32"))
x, y = poisson_batch(B, k, min(T, chunk), 20, seed=1)
eng = EpropEngine(n, k, 20, B, alif=True, chunk=chunk)
eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
torch.cuda.synchronize()
v = ctypes.c_void_p
st = v(torch.cuda.current_stream().cuda_stream)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def run():
    _lib.call("spb_input_proj", v(eng.xq.data_ptr()), v(eng.wq.data_ptr()), v(eng.sexp.data_ptr()),
              B * eng.KR, n, eng.n_pad32, k, eng.Kpad, eng.P, v(eng.cur.data_ptr()), eng.sm_count,
              1, st)


ref = None
for g in bands:
    os.environ["SPB_K2_BANDS"] = str(g)
    ts = []
    for rep in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    cur = eng.cur.clone()
    if ref is None:
        ref = cur
    same = bool(torch.equal(cur.view(torch.int64), ref.view(torch.int64)))
    print(f"B={B} n={n} KR={eng.KR} bands={g} persist={os.environ.get('SPB_K2_PERSIST', '0')}MB: "
          f"{float(np.median(ts[2:])):.4f} ms (min {min(ts[2:]):.4f}) bitwise_equal={same}", flush=True)
