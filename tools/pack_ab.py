"""A/B of the one-chunk pack at C3: device-resident uint8 spikes vs bit-packed spikes
(the e2e input format), whole update as a CUDA graph, CUDA events; plus the pack kernels
alone."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_11407_b200 as P  # noqa: E402
from paper_2501_11407_b200 import _lib  # noqa: E402
from paper_2501_11407_b200.datasets import poisson_batch  # noqa: E402
from paper_2501_11407_b200.engine import EpropEngine  # noqa: E402
from paper_2501_11407_b200.gradients import _neuron_kwargs  # noqa: E402

n, k, m, T, B = 1024, 700, 20, 250, 256
net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=n, n_inputs=k, n_classes=m,
                                   precision="f32", seed=0))
kw = _neuron_kwargs(net)
x, y = poisson_batch(B, k, T, m, seed=1000)
xd = torch.from_numpy(x).cuda()
xbits = torch.from_numpy(np.packbits(x, axis=-1, bitorder="little")).cuda()
yd = torch.from_numpy(y).cuda()
eng = EpropEngine(n, k, m, B, alif=True, chunk=255)
eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for name, xx, bits in (("bytes", xd, False), ("bits", xbits, True)):
    step = eng.graphed(xx, yd, static_inputs=True, bits=bits, binary=True, **kw)
    print(name, "update ms", round(timed(step), 4))
    v = ctypes.c_void_p
    st = v(torch.cuda.current_stream().cuda_stream)
    strideb = T * (xx.shape[-1])

    def pk():
        _lib.call("spb_pack_spikes_xh", v(xx.data_ptr()), strideb, B, k, int(bits), T, eng.KR,
                  eng.Kpad, eng.KR, v(eng.xq.data_ptr()), v(eng.xh.data_ptr()), st)
    print(name, "pack_xh ms", round(timed(pk), 4))
