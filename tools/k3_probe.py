"""K3 (spb_readout_loss) alone at the C3 shape: mean us per launch over back-to-back
launches.  With SPB_LIB pointing at a K3_PROBE build (tools/build_variant.sh) it times the
kernel with a phase switched off."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_11407_b200 import _lib

B, n, m = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (256, 1024, 20)))
d = torch.device("cuda")
g = torch.Generator(device=d).manual_seed(0)
wout = torch.randn(m, n, dtype=torch.float64, device=d, generator=g) * 0.05
zsum = torch.rand(B, n, dtype=torch.float64, device=d, generator=g) * 20
labels = torch.randint(0, m, (B,), device=d, generator=g)
s_out = torch.empty(B, m, dtype=torch.float64, device=d)
loss = torch.empty(B, dtype=torch.float64, device=d)
gg = torch.empty(B, m, dtype=torch.float64, device=d)
wsig = torch.empty(B, n, dtype=torch.float32, device=d)
corr = torch.empty(B, dtype=torch.int32, device=d)
v = ctypes.c_void_p
st = v(torch.cuda.current_stream().cuda_stream)


def launch():
    _lib.call("spb_readout_loss", v(wout.data_ptr()), v(zsum.data_ptr()), v(labels.data_ptr()),
              B, n, m, v(s_out.data_ptr()), v(loss.data_ptr()), v(gg.data_ptr()),
              v(wsig.data_ptr()), v(corr.data_ptr()), st)


for _ in range(20):
    launch()
torch.cuda.synchronize()
# 50 launches in one CUDA graph (no host launch cost in the timing)
N = 50
cs = torch.cuda.Stream()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=cs):
    st = v(cs.cuda_stream)
    for _ in range(N):
        launch()
gr.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
gr.replay()
e1.record()
torch.cuda.synchronize()
print(f"{os.environ.get('SPB_LIB') or 'default'}: K3 B={B} n={n} m={m}: "
      f"{1e3 * e0.elapsed_time(e1) / N:.2f} us/launch", flush=True)
