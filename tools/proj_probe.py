"""Time K2 (W-resident INT8 projection) at the C3 shape with the epilogue and/or the
spike-operand loads switched off (spb_input_proj_probe) to locate its bottleneck
(bit 6 = 64: the stores go to tile-contiguous 32 KB blocks instead of the row layout)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2501_11407_b200 as P
from paper_2501_11407_b200 import _lib
from paper_2501_11407_b200.engine import EpropEngine
from paper_2501_11407_b200.datasets import poisson_batch

B, n, k, T = int(sys.argv[1]) if len(sys.argv) > 1 else 256, 1024, 700, 250
net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=n, n_inputs=k, n_classes=20, precision="f32"))
x, y = poisson_batch(B, k, T, 20, seed=1)
eng = EpropEngine(n, k, 20, B, alif=True, chunk=255)
eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
torch.cuda.synchronize()
v = ctypes.c_void_p
st = v(torch.cuda.current_stream().cuda_stream)
for binary, probe in ((1, 0), (1, 64), (1, 0), (1, 64), (1, 1), (1, 2), (1, 3), (1, 4), (1, 8), (1, 10), (1, 12), (1, 14), (1, 15)):
    ts = []
    for rep in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("spb_input_proj_probe", v(eng.xq.data_ptr()), v(eng.wq.data_ptr()),
                  v(eng.sexp.data_ptr()), B * eng.KR, n, eng.n_pad32, k, eng.Kpad, eng.P,
                  v(eng.cur.data_ptr()), eng.sm_count, binary, probe, st)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ops = 2.0 * eng.P * B * eng.KR * n * k
    ms = float(np.median(ts[2:]))
    print(f"binary={binary} probe={probe} (bit0: no epilogue, bit1: no x loads, bit2: no stores, bit3: no MMAs): {ms:.4f} ms, "
          f"{ops / ms / 1e9:.0f} TOPS issued", flush=True)

# issue-loop clock record (probe bit 5, with the stores off): SM cycles and ns per CTA
for probe, env in ((1 | 4 | 32, {}), (3 | 4 | 32, {}), (4 | 32, {}), (3 | 4 | 32, {"SPB_K2_BANDS": "1"}),
                   (3 | 4 | 32, {"SPB_K2_TAIL": "0"}), (3 | 4 | 32, {"SPB_K2_BANDS": "1", "SPB_K2_TAIL": "0"})):
    os.environ.pop("SPB_K2_BANDS", None)
    os.environ.pop("SPB_K2_TAIL", None)
    os.environ.update(env)
    _lib.call("spb_input_proj_probe", v(eng.xq.data_ptr()), v(eng.wq.data_ptr()),
              v(eng.sexp.data_ptr()), B * eng.KR, n, eng.n_pad32, k, eng.Kpad, eng.P,
              v(eng.cur.data_ptr()), eng.sm_count, 1, probe, st)
    torch.cuda.synchronize()
    rec = eng.cur.view(-1)[:3 * eng.sm_count].view(-1, 3).cpu().numpy()
    cyc, ns, tl = rec[:, 0], rec[:, 1], rec[:, 2]
    nmma = 24 if env.get("SPB_K2_TAIL") == "0" else 22
    print(f"probe={probe} {env}: issue loop {np.median(cyc):.0f} cycles (max {cyc.max():.0f}), "
          f"{np.median(ns) / 1e3:.1f} us -> {np.median(cyc / ns):.3f} GHz, {np.median(tl):.0f} tiles, "
          f"{np.median(cyc / tl / nmma):.1f} cycles per MMA", flush=True)
