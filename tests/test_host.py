"""Host-side tests (CPU only): the C-ABI library loads and exports every declared entry
point, the ctypes signatures match include/sparseprop_b200.h, the engine's launch
sequence is well-formed (dry run with a recording stub), API validation errors."""

import ctypes
import os
import re

XB = ("spb_xbar_chunk", "spb_xbar_chunk_seg", "spb_xbar_chunk_raw")  # K4 entry points

import numpy as np
import pytest
import torch

import paper_2501_11407_b200 as P
from paper_2501_11407_b200 import _lib
from paper_2501_11407_b200.engine import EpropEngine, default_chunk, readout_gains

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sparseprop_b200.h")


def _header_decls():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    decls = {}
    for m in re.finditer(r"\b(?:int|const char\*)\s+(spb_\w+)\s*\(([^)]*)\)\s*;", txt):
        args = [a.strip() for a in m.group(2).split(",") if a.strip() and a.strip() != "void"]
        decls[m.group(1)] = args
    return decls


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    decls = _header_decls()
    assert len(decls) >= 12
    for name in decls:
        assert hasattr(lib, name), name


def test_ctypes_signatures_match_header():
    decls = _header_decls()
    for name, args in _lib.SIGNATURES.items():
        assert name in decls, name
        hargs = decls[name]
        assert len(args) == len(hargs), (name, len(args), len(hargs))
        for ct, h in zip(args, hargs):
            is_ptr = "*" in h or "cudaStream_t" in h
            if is_ptr:
                assert ct is ctypes.c_void_p, (name, h)
            elif "double" in h:
                assert ct is ctypes.c_double, (name, h)
            elif "unsigned long long" in h:
                assert ct is ctypes.c_ulonglong, (name, h)
            elif "long long" in h:
                assert ct is ctypes.c_longlong, (name, h)
            else:
                assert ct is ctypes.c_int, (name, h)


def test_version_and_error_text():
    lib = _lib.load()
    assert lib.spb_version() == 1
    assert isinstance(lib.spb_last_error(), bytes)


def test_bad_arguments_are_rejected_without_gpu():
    # argument validation happens before any CUDA call -> works on a CPU-only host
    with pytest.raises(P.ShapeMismatch):
        _lib.call("spb_forward_chunk", 2, None, 1, 1, 63, 64, 1, 0, 1,
                  0.95, 1.0, 10.0, 0.0, 0.0, 0.95, 0, 0, 0, None, None, None, None, None, None, None, None,
                  None, None, None, None, None, 8, None, None, None)
    with pytest.raises(P.ShapeMismatch):
        _lib.call("spb_input_proj", None, None, None, 1, 1, 32, 100, 100, 7, None, 148, 0, None)
    with pytest.raises(P.ShapeMismatch):
        _lib.call("spb_alif_carry_chunk", None, None, 8, None, None, None, None, None, 1, 1, 100,
                  1, 4, 128, 64, 1, 0, 0, 0, None, None, None)


class _Recorder:
    def __init__(self):
        self.calls = []

    def __call__(self, name, *args):
        sig = _lib.SIGNATURES[name]
        assert len(args) == len(sig), (name, len(args), len(sig))
        for a, t in zip(args, sig):
            if t is ctypes.c_void_p:
                assert a is None or isinstance(a, (ctypes.c_void_p, int)), (name, a)
            elif t is ctypes.c_double:
                assert isinstance(a, float), (name, a)
            else:
                assert isinstance(a, (int, np.integer)) and not isinstance(a, bool) or \
                    isinstance(a, bool), (name, a)
        self.calls.append((name, args))
        return 0


@pytest.mark.parametrize("alif,T,chunk", [(True, 300, 63), (False, 150, 63), (True, 127, 127),
                                          (True, 128, 127)])
def test_engine_launch_sequence_dry_run(monkeypatch, alif, T, chunk):
    rec = _Recorder()
    monkeypatch.setattr(_lib, "call", rec)
    monkeypatch.setattr(torch.cuda, "current_stream", lambda *a, **k: type("S", (), {"cuda_stream": 0})())
    eng = EpropEngine(40, 30, 3, 6, alif=alif, chunk=chunk, device="cpu", sm_count=148)
    x = torch.zeros((6, T, 30), dtype=torch.uint8)
    y = torch.zeros(6, dtype=torch.int64)
    eng.run(x, y)
    names = [c[0] for c in rec.calls]
    nch = (T + chunk - 1) // chunk
    assert names.count("spb_forward_chunk") == 2 * nch
    # a single chunk reuses pass A's packed spikes and current in pass B
    # one chunk: the pack also writes K5's raw-spike operand (spb_pack_spikes_xh, no K4)
    packs = names.count("spb_pack_spikes") + names.count("spb_pack_spikes_xh")
    assert packs == (2 * nch if nch > 1 else 1)
    pack_xh = nch == 1 and 30 % 4 == 0          # byte rows must be 4-byte aligned (k = 30)
    assert names.count("spb_pack_spikes_xh") == (1 if pack_xh else 0)
    assert names.count("spb_input_proj") == (2 * nch if nch > 1 else 1)
    assert names.count("spb_slice_weights") == 0
    assert sum(names.count(x) for x in XB) == (0 if pack_xh else nch)
    # K5 per chunk, plus the K = B GEMM of the carried filter state for chunks after the first
    assert names.count("spb_grad_gemm_partials") == nch + (nch - 1)
    carries = [c[1] for c in rec.calls if c[0] == "spb_alif_carry_chunk"]
    if alif:
        # no carry launch for a single chunk; chunk 0 only carries, the last only adds M E0
        assert len(carries) == (nch if nch > 1 else 0)
        if carries:
            flags = [(e[16], e[17], e[18]) for e in carries]   # do_mma, load_eps, store_eps
            assert flags[0] == (1, 0, 1)
            assert flags[-1] == (0, 1, 0)
            assert all(f == (1, 1, 1) for f in flags[1:-1])
    else:
        assert not carries
    assert names.count("spb_readout_loss") == 1
    # spb_forward_chunk pass B launches two kernels (dynamics + chunk scan)
    passb = sum(1 for c in rec.calls if c[0] == "spb_forward_chunk" and c[1][0] == 1)
    if nch == 1:  # pass A parks psi, pass B runs the scan only, input filter folded in
        assert [c[1][0] for c in rec.calls if c[0] == "spb_forward_chunk"] == [0, 3]
        # the raw-spike operand: written by the pack, K5 gets no B-lo
        gm = [c[1] for c in rec.calls if c[0] == "spb_grad_gemm_partials"]
        assert all(a[4] is None for a in gm)
    assert eng.launches == len(rec.calls) + passb


@pytest.mark.parametrize("compact", ["1", "0"])
def test_engine_compact_rows_dry_run(monkeypatch, compact):
    """One chunk with the raw-spike operand folded into the pack: xq holds only the live
    steps (pack rows-per-sample = len) and K2 maps input row b*len + s to current row
    b*KR + s (spb_input_proj_rows); SPB_COMPACT_ROWS=0 keeps the KR-row layout."""
    monkeypatch.setenv("SPB_COMPACT_ROWS", compact)
    rec = _Recorder()
    monkeypatch.setattr(_lib, "call", rec)
    monkeypatch.setattr(torch.cuda, "current_stream", lambda *a, **k: type("S", (), {"cuda_stream": 0})())
    eng = EpropEngine(40, 32, 3, 6, alif=True, chunk=127, device="cpu", sm_count=148)
    eng.run(torch.zeros((6, 100, 32), dtype=torch.uint8), torch.zeros(6, dtype=torch.int64))
    packs = [c[1] for c in rec.calls if c[0] == "spb_pack_spikes_xh"]
    assert len(packs) == 1 and packs[0][5] == 100                  # len
    assert packs[0][6] == (100 if compact == "1" else eng.KR)      # xq rows per sample
    rows = [c[1] for c in rec.calls if c[0] == "spb_input_proj_rows"]
    plain = [c[1] for c in rec.calls if c[0] == "spb_input_proj"]
    if compact == "1":
        assert not plain and len(rows) == 1 and rows[0][3:6] == (6, 100, eng.KR)
    else:
        assert not rows and len(plain) == 1 and plain[0][3] == 6 * eng.KR


@pytest.mark.parametrize("alif", [False, True])
def test_engine_reset_dry_run(monkeypatch, alif):
    """reset=True: raw-input operand (K4 alpha = 0, fresh every chunk), the reset scan
    and one (LIF: G_u) or two (ALIF: G_u, G_a) carried traces."""
    rec = _Recorder()
    monkeypatch.setattr(_lib, "call", rec)
    eng = EpropEngine(40, 30, 3, 6, alif=alif, chunk=63, device="cpu", sm_count=148, reset=True)
    x = torch.zeros((6, 200, 30), dtype=torch.uint8)
    with pytest.raises(ValueError):
        eng.run(x, torch.zeros(6, dtype=torch.int64), reset=False)
    eng.run(x, torch.zeros(6, dtype=torch.int64), reset=True)
    xb = [c[1] for c in rec.calls if c[0] in XB]
    assert xb and all(a[8] == 1 and a[9] == 0.0 for a in xb)      # fresh, alpha = 0
    fw = [c[1] for c in rec.calls if c[0] == "spb_forward_chunk"]
    assert all(a[15] == 1 for a in fw)                              # reset flag
    carry = "spb_reset_carry_chunk" if alif else "spb_alif_carry_chunk"
    other = "spb_alif_carry_chunk" if alif else "spb_reset_carry_chunk"
    names = [c[0] for c in rec.calls]
    assert names.count(carry) == 4 and names.count(other) == 0     # 4 chunks
    assert eng.mdt.shape[-1] == (8 if alif else 2)


def test_engine_recurrent_dry_run(monkeypatch):
    """Recurrent engines: K1rec instead of K1 in both passes, the x~ = [x, z_{t-1}]
    operand (spb_pack_rec) before K4, eligibility buffers over k + n columns."""
    rec = _Recorder()
    monkeypatch.setattr(_lib, "call", rec)
    eng = EpropEngine(40, 30, 3, 6, alif=True, chunk=63, device="cpu", sm_count=148,
                      recurrent=True)
    assert eng.kx == 70 and eng.kp == 128 and eng.xbar_state.shape == (6, 70)
    eng.run(torch.zeros((6, 150, 30), dtype=torch.uint8), torch.zeros(6, dtype=torch.int64))
    names = [c[0] for c in rec.calls]
    assert names.count("spb_forward_rec_chunk") == 6          # 3 chunks x 2 passes
    assert names.count("spb_pack_rec") == 3 and sum(names.count(x) for x in XB) == 3
    fw = [c[1] for c in rec.calls if c[0] == "spb_forward_chunk"]
    assert fw and all(a[0] == 2 for a in fw)                  # scans only
    xb = [c[1] for c in rec.calls if c[0] in XB]
    assert all(a[4] == 70 for a in xb)                        # filters k + n columns
    with pytest.raises(P.ShapeMismatch):
        eng.set_weights(torch.zeros(40, 30), torch.zeros(3, 40))   # w_rec missing


def test_engine_forward_only_dry_run(monkeypatch):
    rec = _Recorder()
    monkeypatch.setattr(_lib, "call", rec)
    eng = EpropEngine(40, 30, 3, 6, alif=True, chunk=63, device="cpu", sm_count=148)
    eng.run(torch.zeros((6, 150, 30), dtype=torch.uint8), torch.zeros(6, dtype=torch.int64),
            forward_only=True, smooth=True)
    names = [c[0] for c in rec.calls]
    assert names.count("spb_forward_chunk") == 3 and names.count("spb_input_proj") == 3
    assert names[-1] == "spb_readout_loss"
    for n in ("spb_xbar_chunk", "spb_xbar_chunk_seg", "spb_grad_gemm_partials", "spb_alif_carry_chunk",
              "spb_readout_grad"):
        assert n not in names
    # smooth flag reaches the kernel (argument after `alif`)
    assert all(c[1][17] == 1 for c in rec.calls if c[0] == "spb_forward_chunk")


def test_engine_rejects_bad_inputs():
    eng = EpropEngine(8, 5, 2, 3, alif=False, chunk=63, device="cpu", sm_count=148)
    with pytest.raises(P.ShapeMismatch):
        eng.run(torch.zeros((3, 10, 4), dtype=torch.uint8), torch.zeros(3, dtype=torch.int64))
    with pytest.raises(P.ShapeMismatch):
        eng.run(torch.zeros((3, 10, 5), dtype=torch.int32), torch.zeros(3, dtype=torch.int64))
    with pytest.raises(P.ShapeMismatch):
        eng.run(torch.zeros((3, 10, 4), dtype=torch.float32), torch.zeros(3, dtype=torch.int64))
    with pytest.raises(ValueError):   # real-valued inputs: one chunk on a CUDA engine only
        eng.run(torch.zeros((3, 10, 5), dtype=torch.float32), torch.zeros(3, dtype=torch.int64))
    with pytest.raises(ValueError):
        eng.run(torch.zeros((3, 10, 5), dtype=torch.uint8), torch.zeros(3, dtype=torch.int64),
                reset=True)
    with pytest.raises(ValueError):
        EpropEngine(8, 5, 2, 3, alif=True, chunk=24, device="cpu")
    with pytest.raises(ValueError):
        EpropEngine(8, 5, 2, 3, alif=False, chunk=64, device="cpu")


def test_readout_gains_match_bptt_recurrence():
    c = readout_gains(6, 0.9)
    acc, ref = 0.0, []
    for _ in range(6):
        acc = 1.0 + 0.9 * acc
        ref.append(acc)
    assert np.allclose(c, ref[::-1])


def test_param_validation_mirrors_reference():
    with pytest.raises(ValueError):
        P.LIFParams(np.zeros((1, 1)), alpha=1.5)
    with pytest.raises(ValueError):
        P.LIFParams(np.zeros((1, 1)), theta=0.0)
    with pytest.raises(ValueError):
        P.ALIFParams(np.zeros((1, 1)), beta=-0.1)
    with pytest.raises(ValueError):
        P.ALIFParams(np.zeros((1, 1)), rho=1.0)
    with pytest.raises(ValueError):
        P.ReadoutParams(np.zeros((1, 1)), kappa=0.0)


def test_init_network_matches_oracle_and_reference_seed_stream():
    from oracle.eprop_ref import init_network_arrays
    net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=17, n_inputs=9, n_classes=4,
                                       precision="f32", seed=3))
    w, wo = init_network_arrays(17, 9, 4, seed=3, dtype=np.float32)
    assert np.array_equal(net.neuron.w, w) and np.array_equal(net.readout.w_out, wo)
    assert net.is_alif and net.n == 17 and net.k == 9 and net.m == 4


def test_input_count_conversion():
    """Integer-valued inputs in [0, 255] go the exact INT8 way as uint8 counts; anything
    else real-valued is kept as float64 (the fp64-projection path); non-numbers raise."""
    from paper_2501_11407_b200.gradients import _as_counts, _as_inputs
    x = np.array([[0.0, 1.0, 3.0]])
    assert _as_counts(x).dtype == np.uint8
    assert _as_inputs(x)[1] is False and _as_inputs(x)[0].dtype == np.uint8
    for v in (0.5, -1.0, 300.0):
        assert _as_counts(np.array([[v]])) is None
        xr, real = _as_inputs(np.array([[v]], dtype=np.float32))
        assert real and xr.dtype == np.float64 and xr[0, 0] == v
    with pytest.raises(P.ShapeMismatch):
        _as_inputs(np.array([["a"]]))


def test_default_chunk():
    assert default_chunk(10) == 63 and default_chunk(100) == 127 and default_chunk(250) == 255
    assert default_chunk(500) == 511 and default_chunk(10_000) == 2047
    assert default_chunk(2000) == 2047 and default_chunk(1000) == 1023
    # the chunk buffers are sized by Tc only; a budget caps Tc for huge layers
    from paper_2501_11407_b200.engine import chunk_bytes
    assert default_chunk(500, 128, 2048, 700) == 511
    big = default_chunk(10_000, 256, 8192, 700, budget=8 << 30)
    assert big < 511 and chunk_bytes(big, 256, 8192, 700) <= 8 << 30


def test_engine_label_and_mode_checks():
    """Labels must be int64 [B] on the engine's device; a grad=False engine (evaluate)
    allocates no pass-B buffers and refuses gradient runs."""
    eng = EpropEngine(8, 5, 2, 3, alif=True, chunk=63, device="cpu", sm_count=148)
    x = torch.zeros((3, 10, 5), dtype=torch.uint8)
    for bad in (torch.zeros(3, dtype=torch.int32), torch.zeros(4, dtype=torch.int64),
                torch.zeros((3, 1), dtype=torch.int64)):
        with pytest.raises(P.ShapeMismatch):
            eng.run(x, bad)
    fwd = EpropEngine(8, 5, 2, 3, alif=True, chunk=63, device="cpu", sm_count=148, grad=False)
    assert fwd.eps is None and fwd.psi is None and fwd.grad_w_acc is None
    with pytest.raises(ValueError):
        fwd.run(x, torch.zeros(3, dtype=torch.int64))


def test_train_and_evaluate_reject_bad_labels_before_any_kernel():
    from paper_2501_11407_b200.datasets import generate_poisson_dataset
    from paper_2501_11407_b200.training import evaluate, train
    ds = generate_poisson_dataset(4, 6, 10, 3, seed=0)
    ds.labels[2] = (2, 7)     # class 7 of 3
    spec = P.NetworkSpec(kind="lif", n_hidden=4, n_inputs=6, n_classes=3, seed=0)
    with pytest.raises(P.LabelOutOfRange):
        train(spec, ds)
    with pytest.raises(P.LabelOutOfRange):
        evaluate(P.init_network(spec), ds)


@pytest.mark.parametrize("k", [1, 7, 8, 16, 700, 701])
def test_host_pack_bits_matches_numpy_packbits(k):
    """The drop-in's native packer (host code, no GPU) = np.packbits(bitorder='little'),
    and it reports counts > 1 anywhere in a row (full words and the tail bytes)."""
    rng = np.random.default_rng(k)
    x = (rng.random((5, 9, k)) < 0.3).astype(np.uint8)
    kb = (k + 7) // 8
    out = np.zeros((5, 9, kb), np.uint8)
    lib = _lib.load()
    assert lib.spb_host_pack_bits(x.ctypes.data, 45, k, out.ctypes.data) == 0
    np.testing.assert_array_equal(out, np.packbits(x, axis=-1, bitorder="little"))
    for j in {0, k // 2, k - 1}:
        y = x.copy()
        y[3, 4, j] = 2
        assert lib.spb_host_pack_bits(y.ctypes.data, 45, k, out.ctypes.data) == 1
    assert lib.spb_host_pack_bits(x.ctypes.data, 45, 0, out.ctypes.data) == 2
