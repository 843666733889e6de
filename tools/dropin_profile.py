"""Where the drop-in call's time goes (eprop_batch_gradient at C3, numpy in/out):
whole-call ms for uint8 counts (staged bit-packed), forced byte staging and packed=True
input, then the phases of one call timed apart (each followed by a device sync)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2501_11407_b200 as P  # noqa: E402
from paper_2501_11407_b200.datasets import poisson_batch  # noqa: E402
from paper_2501_11407_b200 import gradients as G  # noqa: E402

# python tools/dropin_profile.py [kind n B]   (default: C3 = alif 1024 256)
KIND = sys.argv[1] if len(sys.argv) > 1 else "alif"
N_H = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
BATCH = int(sys.argv[3]) if len(sys.argv) > 3 else 256
net = P.init_network(P.NetworkSpec(kind=KIND, n_hidden=N_H, n_inputs=700, n_classes=20,
                                   precision="f32", seed=0))
x, y = poisson_batch(BATCH, 700, 250, 20, seed=1000)
xb = np.packbits(x, axis=-1, bitorder="little")
eng = G.get_engine(net, BATCH, T=250)
st = G._staging(eng)


def timeit(f, n=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print("counts (bit-packed staging) ms/call %.3f" % timeit(lambda: G.eprop_batch_gradient(net, x, y)))
print("packed=True               ms/call %.3f" % timeit(
    lambda: G.eprop_batch_gradient(net, xb, y, packed=True)))
st.counts_nonbinary = True
print("counts (byte staging)     ms/call %.3f" % timeit(lambda: G.eprop_batch_gradient(net, x, y)))
st.counts_nonbinary = False
sync = torch.cuda.synchronize
print("phase: pack+H2D (counts)  %.3f" % timeit(lambda: (st.inputs_packed_from_counts(x, y), sync())))
print("phase: pack only (1 thr)  %.3f" % timeit(lambda: P._lib.load().spb_host_pack_bits(
    x.ctypes.data, BATCH * 250, 700, st.bufs[(BATCH, 250, 88)][0].numpy().ctypes.data)))
print("phase: copy+H2D (packed)  %.3f" % timeit(lambda: (st.inputs(xb, y), sync())))
print("phase: weights check      %.3f" % timeit(lambda: st.weights(net)))
kw = dict(smooth=False, bits=True, binary=True, **G._neuron_kwargs(net))
key = tuple(sorted(kw.items())) + (250,)
print("phase: graph replay       %.3f" % timeit(lambda: (st.run(key, **kw), sync())))


def outs():
    o = {"w": G._to_host(eng.grad_w(torch.float32)), "w_out": G._to_host(eng.grad_wout.to(torch.float32)),
         "loss": G._to_host(eng.loss), "s": G._to_host(eng.s), "correct": G._to_host(eng.correct)}
    sync()
    return o


print("phase: outputs D2H        %.3f" % timeit(outs))
print("phase: _check_batch       %.3f" % timeit(lambda: G._check_batch(net, x, y, False)))
for sp in (1, 2, 4, 8):
    G._STAGE_PARTS = sp
    print("packed=True stage parts %d: ms/call %.3f, copy+H2D %.3f" % (
        sp, timeit(lambda: G.eprop_batch_gradient(net, xb, y, packed=True)),
        timeit(lambda: (st.inputs(xb, y), sync()))))
for pp in (2, 4, 8, 16, 32):
    G._PACK_PARTS = pp
    print("counts pack parts %d: ms/call %.3f, pack+H2D %.3f" % (
        pp, timeit(lambda: G.eprop_batch_gradient(net, x, y)),
        timeit(lambda: (st.inputs_packed_from_counts(x, y), sync()))))
hb = st.bufs[(BATCH, 250, 88)]
print("H2D 5.6 MB pinned alone %.3f" % timeit(lambda: (hb[1].copy_(hb[0], non_blocking=True), sync())))
