"""Two ranks (gloo, both on cuda:0) vs one rank on the whole batch.

The data-parallel path shards a global batch over the ranks (contiguous shards) and
combines the packed [grad W | grad W_out | loss sum | #correct] with ONE allreduce per
update (parallel.py).  Its result must equal one engine over the whole batch up to the
fp32 rounding of the packed payload; train() sharded over two ranks must follow the
single-rank train() to fp32 tolerance.  (One GPU per box: NCCL cannot put two ranks on
one device, so the collective here is gloo; the bench's NCCL path is the same code.)
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_two_ranks_equal_one_rank(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import dist_worker as W

    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import generate_poisson_dataset, poisson_batch
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    from paper_2501_11407_b200.training import train
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "dist_worker.py"), str(tmp_path)]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    d = np.load(tmp_path / "dist.npz")
    # one rank, whole batch
    net = P.init_network(P.NetworkSpec(**W.SPEC))
    x, y = poisson_batch(W.GB, 40, W.T, 5, seed=4)
    eng = EpropEngine(96, 40, 5, W.GB, alif=True, chunk=W.CHUNK)
    eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
    eng.run(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), **_neuron_kwargs(net))
    gw = eng.grad_w(torch.float64).cpu().numpy()
    assert _rel(d["gw"], gw) <= 2e-6
    assert _rel(d["gwo"], eng.grad_wout.cpu().numpy()) <= 1e-6
    assert float(d["loss_sum"]) == pytest.approx(float(eng.loss.sum().item()), rel=1e-6)
    assert float(d["correct"]) == float(eng.correct.sum().item())
    # train(): 2 epochs x 2 updates of 8 samples, sharded 4 + 4
    ds = generate_poisson_dataset(16, 40, 80, 5, seed=6)
    net1, rows = train(P.NetworkSpec(**W.SPEC), ds, batch_size=8, epochs=2, lr=0.05)
    assert np.array_equal(d["row_acc"], [r.accuracy for r in rows])
    np.testing.assert_allclose(d["row_loss"], [r.loss for r in rows], rtol=1e-5)
    # (the two-rank update applies the fp32 allreduce payload, one rank its fp64
    # accumulators directly: the weights agree to the fp32 rounding of 4 updates)
    assert _rel(d["w"], net1.neuron.w) <= 5e-5
    assert _rel(d["w_out"], net1.readout.w_out) <= 5e-5
    # recurrent extension (W_rec): sharded training = one rank on the whole batch
    net3, rows3 = train(P.NetworkSpec(**W.SPEC, recurrent=True), ds, batch_size=8, epochs=1,
                        lr=0.05)
    assert np.array_equal(d["rec_row_acc"], [r.accuracy for r in rows3])
    np.testing.assert_allclose(d["rec_row_loss"], [r.loss for r in rows3], rtol=1e-5)
    assert _rel(d["rec_w"], net3.neuron.w) <= 5e-5
    assert _rel(d["rec_w_out"], net3.readout.w_out) <= 5e-5
    assert _rel(d["rec_w_rec"], net3.neuron.w_rec) <= 5e-5
    assert _rel(d["rec_w_rec"], P.init_network(P.NetworkSpec(**W.SPEC, recurrent=True)).neuron.w_rec) > 0
