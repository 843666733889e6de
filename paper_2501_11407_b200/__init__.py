"""sparseprop-b200: B200-native (sm_100a) e-prop training step of arXiv 2501.11407.

Drop-in for the reference package's neuron-model and gradient entry points
(/root/reference/pkg/src/sparseprop/{neurons,gradients}.py).  The compute path is the
hand-written CUDA in ``csrc/`` behind the C-ABI ``include/sparseprop_b200.h``.
"""

from .errors import (KernelError, LabelOutOfRange, ResourceLimit, ShapeMismatch,
                     SparsePropError, StructureFallback)
from .neurons import ALIFParams, LIFParams, Network, ReadoutParams
from .training import NetworkSpec, init_network

__version__ = "0.1.0"


def __getattr__(name):
    # the compute entry points need torch + the CUDA library; import lazily
    if name in ("eprop_sparse_gradient", "eprop_batch_gradient", "ENGINES", "GradResult",
                "BatchGradResult", "softmax_cross_entropy", "gradient_deviation_stats",
                "network_loss", "DeviationStats", "TraceState", "initial_trace",
                "eprop_trace_update", "learning_signal", "accumulate_param_grad"):
        from . import gradients
        return getattr(gradients, name)
    if name == "EpropEngine":
        from .engine import EpropEngine
        return EpropEngine
    raise AttributeError(name)
