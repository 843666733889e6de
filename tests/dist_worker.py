"""Worker of tests/test_dist_gpu.py: one rank of a 2-rank gloo job sharing cuda:0.

Runs (1) one DataParallelEprop.step on this rank's contiguous shard of a global batch
and (2) train() with batch_size=8 sharded over the ranks, and writes rank 0's results
to <out>/dist.npz.  Launched by torch.distributed.run with MASTER_ADDR=127.0.0.1.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2501_11407_b200 as P  # noqa: E402
from paper_2501_11407_b200.datasets import generate_poisson_dataset, poisson_batch  # noqa: E402
from paper_2501_11407_b200.engine import EpropEngine  # noqa: E402
from paper_2501_11407_b200.gradients import _neuron_kwargs  # noqa: E402
from paper_2501_11407_b200.parallel import DataParallelEprop, shard_range  # noqa: E402
from paper_2501_11407_b200.training import train  # noqa: E402

SPEC = dict(kind="alif", n_hidden=96, n_inputs=40, n_classes=5, precision="f32", seed=3)
GB, T, CHUNK = 10, 150, 63          # 3 chunks: the per-synapse trace is carried


def main(out):
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    net = P.init_network(P.NetworkSpec(**SPEC))
    x, y = poisson_batch(GB, 40, T, 5, seed=4)
    lo, hi = shard_range(GB, rank, world)
    eng = EpropEngine(96, 40, 5, hi - lo, alif=True, chunk=CHUNK)
    eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
    dp = DataParallelEprop(eng)
    gw, gwo, ls, nc = dp.step(torch.from_numpy(x[lo:hi]).cuda(),
                              torch.from_numpy(y[lo:hi]).cuda(), **_neuron_kwargs(net))
    res = dict(gw=gw.cpu().numpy().copy(), gwo=gwo.cpu().numpy().copy(),
               loss_sum=float(ls.item()), correct=float(nc.item()))
    ds = generate_poisson_dataset(16, 40, 80, 5, seed=6)
    net2, rows = train(P.NetworkSpec(**SPEC), ds, batch_size=8, epochs=2, lr=0.05)
    res.update(w=net2.neuron.w, w_out=net2.readout.w_out,
               row_loss=np.array([r.loss for r in rows]),
               row_acc=np.array([r.accuracy for r in rows]))
    # the recurrent extension: grad W and grad W_rec travel in the one payload
    net3, rows3 = train(P.NetworkSpec(**SPEC, recurrent=True), ds, batch_size=8, epochs=1,
                        lr=0.05)
    res.update(rec_w=net3.neuron.w, rec_w_out=net3.readout.w_out, rec_w_rec=net3.neuron.w_rec,
               rec_row_loss=np.array([r.loss for r in rows3]),
               rec_row_acc=np.array([r.accuracy for r in rows3]))
    if rank == 0:
        np.savez(os.path.join(out, "dist.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
