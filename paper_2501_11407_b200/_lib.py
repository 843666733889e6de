"""ctypes binding of the C-ABI library ``libsparseprop_b200.so`` (include/sparseprop_b200.h).

The library is built in-tree by ``make`` (``__graft_entry__.build()``).  There is no CPU
or Python fallback: if the library is missing, importing the compute path raises.
"""

from __future__ import annotations

import ctypes
import os

from .errors import KernelError, ShapeMismatch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPB_LIB: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("SPB_LIB") or os.path.join(_HERE, "libsparseprop_b200.so")

P = ctypes.c_void_p
I = ctypes.c_int
LL = ctypes.c_longlong
D = ctypes.c_double

# name -> argtypes (every function returns int status)
SIGNATURES = {
    "spb_slice_weights": [P, I, I, I, I, I, I, P, P, P],
    "spb_pack_spikes": [P, LL, I, I, I, I, I, I, I, P, P],
    "spb_pack_spikes_xh": [P, LL, I, I, I, I, I, I, I, P, P, P],
    "spb_input_proj": [P, P, P, I, I, I, I, I, I, P, I, I, P],
    "spb_input_proj_rows": [P, P, P, I, I, I, I, I, I, I, I, P, I, I, P],
    "spb_input_proj_probe": [P, P, P, I, I, I, I, I, I, P, I, I, I, P],
    "spb_forward_chunk": [I, P, I, I, I, I, I, I, I, D, D, D, D, D, D, I, I, I,
                          P, P, P, P, P, P, P, P, P, P, P, P, P, I, P, P, P],
    "spb_xbar_chunk": [P, LL, LL, I, I, I, I, I, I, D, P, P, P, P],
    "spb_xbar_chunk_seg": [P, LL, LL, I, I, I, I, I, I, D, P, P, P, P],
    "spb_xbar_chunk_raw": [P, LL, LL, I, I, I, I, I, I, D, P, P, P, P, P],
    "spb_readout_loss": [P, P, P, I, I, I, P, P, P, P, P, P],
    "spb_readout_grad": [P, P, I, I, I, P, P],
    "spb_grad_gemm_partials": [P, P, I, P, P, I, I, I, I, I, P, I, LL, P],
    "spb_grad_gemm_simt": [P, P, I, P, P, I, I, I, I, P, I, P],
    "spb_alif_carry_chunk": [P, P, I, P, P, P, P, P, I, I, I, I, I, I, I, I, I, I, I, P, P,
                             P],
    "spb_reset_carry_chunk": [P, P, P, P, I, P, P, P, P, P, I, I, I, I, I, I, I, I, I, I,
                              I, P],
    "spb_reduce_partials": [P, I, I, I, I, I, P, P],
    "spb_finalize_grad": [P, I, I, I, P, I, P],
    "spb_pack_grads": [P, I, I, I, P, I, P, P, I, P, I, P],
    "spb_copy_chunk_h2d": [P, LL, P, LL, LL, I, P],
    "spb_host_pack_bits": [P, LL, I, P],
    "spb_pack_real": [P, I, LL, I, I, I, I, I, P, P, P],
    "spb_sgd_slice_update": [P, I, I, I, P, I, I, D, D, I, I, I, P, P, P],
    "spb_sgd_update": [P, I, I, I, P, I, I, D, D, P, P],
    "spb_adam_update": [P, P, P, I, I, I, P, I, I, D, D, D, D, D, I, P, P],
    "spb_poisson_bits": [P, P, I, I, I, I, ctypes.c_ulonglong, P, LL, P],
    "spb_forward_rec_chunk": [I, P, P, I, I, I, I, I, I, I, I, D, D, D, D, D, D, I, I, I,
                              P, P, P, P, P, P, P, P],
    "spb_pack_rec": [P, LL, LL, P, I, I, I, I, I, I, I, P, P],
    "spb_version": [],
    "spb_device_sm": [],
}

_lib = None


def load():
    """Load the library once; raise ImportError (never fall back) if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not built; run `make` (or __graft_entry__.build()). "
            "sparseprop-b200 has no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.spb_last_error.argtypes = []
    lib.spb_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


def call(name, *args):
    """Invoke a C-ABI entry point and translate its status code into an exception."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.spb_last_error().decode(errors="replace")
        if rc == 2:
            raise ShapeMismatch(msg)
        raise KernelError(f"{name}: {msg} (rc={rc})")
    return rc
