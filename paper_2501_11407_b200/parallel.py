"""Data parallelism over the batch: one process per GPU, one NCCL allreduce per update.

Samples are independent in the reference (training.py:142-152 processes
them one at a time), so the batch is sharded in contiguous ranges, every rank keeps
its own traces and state (engine.py), and the only collective is a single sum
allreduce of the packed buffer

    [ grad W (n*k) | grad W_out (m*n) | sum of losses | #correct ]      (fp32 or fp64)

issued on the compute stream after the last chunk.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(batch: int, rank: int, world: int):
    """Contiguous shard [lo, hi) of a global batch for ``rank`` (sizes differ by <= 1)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


class GradPacker:
    """Packs the per-rank results into one flat fp32 buffer and unpacks the reduced sum."""

    def __init__(self, n: int, k: int, m: int, device, dtype=torch.float32):
        self.n, self.k, self.m = n, k, m
        self.size = n * k + m * n + 2
        # fp32 for throughput runs (as the reference's f32 grads); fp64 when training an
        # f64 network so the allreduce adds no rounding beyond the fp64 sum
        self.buf = torch.empty(self.size, dtype=dtype, device=device)

    def views(self):
        n, k, m = self.n, self.k, self.m
        gw = self.buf[: n * k].view(n, k)
        gwo = self.buf[n * k: n * k + m * n].view(m, n)
        return gw, gwo, self.buf[n * k + m * n], self.buf[n * k + m * n + 1]

    def pack(self, grad_w_acc, grad_wout, loss, correct):
        """grad_w_acc may be column-padded ([n, k_pad]); only [:, :k] is packed.  On CUDA
        one fused kernel (spb_pack_grads) does it; elsewhere (gloo tests) torch ops."""
        if (self.buf.is_cuda and grad_w_acc.dtype == torch.float64
                and grad_wout.dtype == torch.float64 and loss.dtype == torch.float64
                and correct.dtype == torch.int32 and grad_w_acc.stride(1) == 1
                and grad_wout.is_contiguous()):
            import ctypes
            from . import _lib
            v = ctypes.c_void_p
            _lib.call("spb_pack_grads", v(grad_w_acc.data_ptr()), self.n, self.k,
                      grad_w_acc.stride(0), v(grad_wout.data_ptr()), self.m,
                      v(loss.data_ptr()), v(correct.data_ptr()), int(loss.shape[0]),
                      v(self.buf.data_ptr()), int(self.buf.dtype == torch.float64),
                      v(torch.cuda.current_stream(self.buf.device).cuda_stream))
            return self.buf
        gw, gwo, ls, nc = self.views()
        gw.copy_(grad_w_acc[:, : self.k])
        gwo.copy_(grad_wout)
        ls.copy_(loss.sum())
        nc.copy_(correct.sum())
        return self.buf

    def allreduce(self, group=None):
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.buf, op=dist.ReduceOp.SUM, group=group)
        return self.views()


class DataParallelEprop:
    """Engine + packer: ``step`` runs the local update and the single allreduce."""

    def __init__(self, engine, group=None):
        self.engine = engine
        self.group = group
        self.packer = GradPacker(engine.n, engine.k, engine.m, engine.device)

    def step(self, x, labels, **neuron_kwargs):
        eng = self.engine
        eng.run(x, labels, **neuron_kwargs)
        self.packer.pack(eng.grad_w_acc, eng.grad_wout, eng.loss, eng.correct)
        return self.packer.allreduce(self.group)
