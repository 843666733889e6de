"""GPU parity tests: the B200 kernels (through the C-ABI) against the reference's own
outputs (tests/golden, produced by the unmodified reference) and the CPU oracle.

Tolerances (north_star / SURVEY.md 8(c)):
  * spikes   -- bit-exact rasters vs the f64 reference over the full horizon T
  * gradients-- batch-summed relative L2 <= 1e-4 and cosine >= 0.9999 vs the f64
               reference e-prop (and vs BPTT on the exact-gradient task C1)
  * losses   -- relative 1e-9 (fp64 forward and readout)
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from conftest import load_golden  # noqa: E402
from oracle import eprop_ref as O  # noqa: E402

REL_TOL = 1e-4
COS_TOL = 0.9999


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _cos(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(a @ b / max(np.linalg.norm(a) * np.linalg.norm(b), 1e-300))


def _net_from_golden(g):
    import paper_2501_11407_b200 as P
    spec = P.NetworkSpec(kind=str(g["kind"]), n_hidden=int(g["n"]), n_inputs=int(g["k"]),
                         n_classes=int(g["m"]), precision=str(g["precision"]),
                         reset=bool(g["reset"]), seed=int(g["seed_net"]))
    return P.init_network(spec)


def _inputs(g):
    from paper_2501_11407_b200.datasets import poisson_batch
    return poisson_batch(int(g["B"]), int(g["k"]), int(g["T"]), int(g["m"]), int(g["seed_data"]))


def _run_engine(net, x, labels, chunk=None, raster=False):
    from paper_2501_11407_b200.gradients import _neuron_kwargs, get_engine
    B, T, k = x.shape
    eng = get_engine(net, B, chunk=chunk, T=T)
    xd = torch.from_numpy(x).cuda()
    ld = torch.from_numpy(labels).cuda()
    eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
    r = None
    if raster:
        r = torch.zeros((B, T, (net.n + 31) // 32), dtype=torch.int32, device="cuda")
    eng.run(xd, ld, raster=r, **_neuron_kwargs(net))
    torch.cuda.synchronize()
    return eng, r


def _unpack_raster(r, n):
    r = r.cpu().numpy().view(np.uint32)
    B, T, nw = r.shape
    bits = ((r[..., None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool)
    return bits.reshape(B, T, nw * 32)[..., :n]


def _golden_raster(g):
    B, T, n = int(g["B"]), int(g["T"]), int(g["n"])
    return np.unpackbits(g["raster_packed"], axis=-1)[..., :n].astype(bool).reshape(B, T, n)


SMALL = ["c1_lif_f64", "c1_alif_f64", "c1_lif_f32", "c1_alif_f32", "mid_alif_f64"]


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("chunk", [63, 127, 511])
def test_small_configs_vs_reference(name, chunk):
    _need_gpu()
    g = load_golden(name)
    net = _net_from_golden(g)
    x, labels = _inputs(g)
    eng, r = _run_engine(net, x, labels, chunk=chunk, raster=True)
    f64 = str(g["precision"]) == "f64"
    # spikes bit-exact over the whole horizon vs the f64 reference (for f32 nets: the
    # f64 evaluation of the same f32 weights -- the f32 reference integrates in f32)
    if f64:
        want = _golden_raster(g)
    else:
        p = O.Params(alif=str(g["kind"]) == "alif")
        want = np.stack([O.network_loss(net.neuron.w.astype(np.float64),
                                        net.readout.w_out.astype(np.float64), p,
                                        x[b].astype(np.float64), int(labels[b]))[2]
                         for b in range(x.shape[0])])
    assert np.array_equal(_unpack_raster(r, net.n), want)
    # losses / readouts
    assert np.allclose(eng.loss.cpu().numpy(), g["loss"], rtol=1e-9 if f64 else 1e-4, atol=1e-12)
    # batch-summed gradients vs reference e-prop and vs BPTT (exact-gradient task)
    gw = eng.grad_w(torch.float64).cpu().numpy()
    gwo = eng.grad_wout.cpu().numpy()
    for ref_w, ref_wo in ((g["eprop_w"].sum(0), g["eprop_w_out"].sum(0)),
                          (g["bptt_w"].sum(0), g["bptt_w_out"].sum(0))):
        assert _rel(gw, ref_w) <= REL_TOL, _rel(gw, ref_w)
        assert _cos(gw, ref_w) >= COS_TOL
        assert _rel(gwo, ref_wo) <= (1e-9 if f64 else 1e-5)


@pytest.mark.parametrize("name", ["c1_lif_f64", "c1_alif_f64"])
def test_drop_in_single_sample_api(name):
    """eprop_sparse_gradient(net, x_seq, label) per sample, like the reference call."""
    _need_gpu()
    import paper_2501_11407_b200 as P
    g = load_golden(name)
    net = _net_from_golden(g)
    x, labels = _inputs(g)
    for b in range(int(g["B"])):
        res = P.eprop_sparse_gradient(net, x[b].astype(np.float64), int(labels[b]))
        assert res.grads["w"].dtype == net.neuron.w.dtype
        assert res.loss == pytest.approx(float(g["loss"][b]), rel=1e-9, abs=1e-12)
        ref = g["eprop_w"][b]
        gnorm = np.linalg.norm(ref)
        if gnorm > 1e-8:  # saturated softmax => g ~ 0 (SURVEY.md TL;DR 8)
            assert _rel(res.grads["w"], ref) <= REL_TOL
        assert np.allclose(res.readout_sum, g["readout_sum"][b], rtol=1e-12)
        assert res.prediction == int(np.argmax(g["readout_sum"][b]))


@pytest.mark.parametrize("name", ["c2_lif_f64", "c3_alif_f64", "c4_alif_f64"])
@pytest.mark.parametrize("chunk", [127, None])   # None = the engine's default (255 / 511)
def test_shd_ssc_shapes_vs_reference(name, chunk):
    _need_gpu()
    g = load_golden(name)
    net = _net_from_golden(g)
    x, labels = _inputs(g)
    eng, r = _run_engine(net, x, labels, chunk=chunk, raster=True)
    assert np.array_equal(_unpack_raster(r, net.n), _golden_raster(g))
    assert np.allclose(eng.loss.cpu().numpy(), g["loss"], rtol=1e-9)
    gw = eng.grad_w(torch.float64).cpu().numpy()
    idx = g["grad_idx"]
    ref = g["eprop_w_batch_sum"]
    assert _rel(gw.ravel()[idx], ref) <= REL_TOL
    assert _cos(gw.ravel()[idx], ref) >= COS_TOL
    assert abs(np.linalg.norm(gw) - float(g["eprop_w_batch_norm"])) <= \
        REL_TOL * float(g["eprop_w_batch_norm"])


@pytest.mark.parametrize("kind,n,k,m,T,B,chunk", [
    ("alif", 200, 90, 7, 177, 12, 63),
    ("lif", 300, 130, 5, 150, 10, 63),
    ("alif", 130, 700, 20, 300, 33, 127),
    ("alif", 64, 40, 3, 520, 5, 255),
    ("alif", 96, 60, 4, 1300, 4, 511),      # 3 chunks of 511 (the long-sequence default)
    ("alif", 333, 45, 3, 130, 5, 127),      # odd n: unaligned current rows
    ("lif", 70, 50, 3, 600, 6, 511),
    ("alif", 33, 9, 2, 1, 3, 63),           # a single time step
    ("alif", 40, 20, 3, 64, 2, 63),         # two chunks, the last one step long
    ("lif", 1, 1, 2, 20, 1, 63),            # one neuron, one input, one sample
    ("alif", 257, 129, 4, 255, 3, 255),     # T exactly one chunk, n / k one past a tile
])
def test_batched_vs_two_pass_oracle(kind, n, k, m, T, B, chunk):
    """Ragged shapes (n, k not tile multiples, T not a chunk multiple) vs the numpy oracle."""
    _need_gpu()
    import paper_2501_11407_b200 as P
    net = P.init_network(P.NetworkSpec(kind=kind, n_hidden=n, n_inputs=k, n_classes=m,
                                       precision="f32", seed=7))
    from paper_2501_11407_b200.datasets import poisson_batch
    x, labels = poisson_batch(B, k, T, m, seed=11)
    eng, r = _run_engine(net, x, labels, chunk=chunk, raster=True)
    p = O.Params(alif=kind == "alif")
    ref = O.eprop_two_pass_batch(net.neuron.w.astype(np.float64),
                                 net.readout.w_out.astype(np.float64), p, x, labels)
    assert np.array_equal(_unpack_raster(r, n), ref.raster)
    gw = eng.grad_w(torch.float64).cpu().numpy()
    assert _rel(gw, ref.grad_w) <= REL_TOL
    assert _cos(gw, ref.grad_w) >= COS_TOL
    assert _rel(eng.grad_wout.cpu().numpy(), ref.grad_w_out) <= 1e-9
    assert np.allclose(eng.loss.cpu().numpy(), ref.loss, rtol=1e-9)


@pytest.mark.parametrize("blo,M,N,K", [(True, 300, 320, 1024), (False, 1024, 768, 2048),
                                        (False, 130, 128, 96)])
def test_pair_gemm_slices_vs_cuda_core_gemm(blo, M, N, K):
    """K5 on CTA pairs at the geometries the pair tiling makes special -- a half pair
    past the partial slice (M = 300 over 384 rows, M = 130), the raw exact-bf16 B operand
    (bl = NULL), several splits -- against the CUDA-core GEMM on the same operands and the
    exact product; nothing is written past the last slice."""
    _need_gpu()
    import ctypes
    from paper_2501_11407_b200 import _lib
    torch.manual_seed(1)
    lda = (M + 7) // 8 * 8
    mp = (M + 127) // 128 * 128
    at = torch.zeros(K, lda, device="cuda")
    at[:, :M] = torch.randn(K, M, device="cuda")
    ah = at.to(torch.bfloat16); al = (at - ah.float()).to(torch.bfloat16)
    if blo:
        bt = torch.randn(K, N, device="cuda")
    else:
        bt = (torch.rand(K, N, device="cuda") < 0.1).float()
    bh = bt.to(torch.bfloat16); bl = (bt - bh.float()).to(torch.bfloat16)
    v = ctypes.c_void_p
    splits = 3
    part = torch.full((splits + 1, mp, N), 7.0, device="cuda")   # +1: guard slice
    _lib.call("spb_grad_gemm_partials", v(ah.data_ptr()), v(al.data_ptr()), lda,
              v(bh.data_ptr()), v(bl.data_ptr()) if blo else None, N, M, N, K, splits,
              v(part.data_ptr()), N, mp * N, None)
    ref = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    zl = torch.zeros_like(bl)
    _lib.call("spb_grad_gemm_simt", v(ah.data_ptr()), v(al.data_ptr()), lda, v(bh.data_ptr()),
              v((bl if blo else zl).data_ptr()), N, M, N, K, v(ref.data_ptr()), N, None)
    torch.cuda.synchronize()
    assert bool((part[splits] == 7.0).all())        # nothing written past the slices
    got = part[:splits, :M].double().sum(0)
    assert float((got - ref).norm() / ref.norm()) < 1e-5
    exact = at[:, :M].double().t() @ bt.double()
    assert float((got - exact).norm() / exact.norm()) < 1e-4


@pytest.mark.parametrize("k", [20, 60, 64, 65, 129, 700, 768])
def test_projection_tail_block_is_bitwise_the_padded_block(k, monkeypatch):
    """K2 runs the last <= 64 inputs past a 128-byte K block as a 64-byte SWIZZLE_64B
    block; integer MMA accumulation is exact, so the fp64 currents equal the zero-padded
    full-block path bit for bit (k = 20: the tail is the whole K; 768: no tail)."""
    _need_gpu()
    import ctypes
    from paper_2501_11407_b200.engine import EpropEngine
    rng = np.random.default_rng(k)
    B, T, n = 3, 40, 96
    w = (rng.uniform(-1, 1, (n, k)) / np.sqrt(k)).astype(np.float32)
    x = (rng.random((B, T, k)) < 0.2).astype(np.uint8)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("SPB_K2_TAIL", flag)
        eng = EpropEngine(n, k, 3, B, alif=False, w_f64=False, chunk=63)
        eng.set_weights(torch.from_numpy(w), torch.zeros((3, n), dtype=torch.float64))
        xd = torch.from_numpy(x).cuda()
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        eng._pack(xd.data_ptr(), T * k, False, T, st)
        eng.cur.zero_()
        eng._project(T, st, binary=True)
        torch.cuda.synchronize()
        out[flag] = eng.cur.cpu().numpy().reshape(B, eng.KR, n)[:, :T].copy()
    assert np.array_equal(out["1"], out["0"])
    exact = np.einsum("btk,nk->btn", x.astype(np.longdouble), w.astype(np.longdouble))
    assert np.max(np.abs(out["1"] - exact.astype(np.float64))) <= 2.3e-16 * np.max(np.abs(exact))


@pytest.mark.parametrize("B,T,n,k,binary", [(40, 250, 1024, 700, True), (7, 300, 200, 90, True),
                                              (5, 120, 96, 700, False), (64, 250, 2048, 130, True)])
def test_projection_banded_walk_is_bitwise_the_plain_walk(B, T, n, k, binary, monkeypatch):
    """K2's banded tile walk (TileWalk: row bands, odd bands reversed, one weight reload per
    band) visits every (row, neuron) tile exactly once: the currents equal the one-band walk
    bit for bit for any band count (also more bands than row tiles, which are clamped)."""
    _need_gpu()
    import ctypes
    from paper_2501_11407_b200.engine import EpropEngine
    rng = np.random.default_rng(n + k)
    w = (rng.uniform(-1, 1, (n, k)) / np.sqrt(k)).astype(np.float32)
    x = (rng.random((B, T, k)) < 0.1).astype(np.uint8)
    if not binary:
        x[0, :, :5] = 3
    eng = EpropEngine(n, k, 3, B, alif=False, w_f64=False, chunk=255 if T < 256 else 511)
    eng.set_weights(torch.from_numpy(w), torch.zeros((3, n), dtype=torch.float64))
    xd = torch.from_numpy(x).cuda()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    eng._pack(xd.data_ptr(), T * k, False, T, st)
    out = {}
    for bands in ("1", "2", "3", "7", "1000", None):
        if bands is None:
            monkeypatch.delenv("SPB_K2_BANDS", raising=False)   # the default band count
        else:
            monkeypatch.setenv("SPB_K2_BANDS", bands)
        eng.cur.fill_(float("nan"))
        eng._project(T, st, binary=binary)
        torch.cuda.synchronize()
        out[bands] = eng.cur.cpu().numpy().reshape(B, eng.KR, n)[:, :T].copy()
    for bands, cur in out.items():
        assert np.isfinite(cur).all(), bands
        assert np.array_equal(cur.view(np.int64), out["1"].view(np.int64)), bands


@pytest.mark.parametrize("B,T,n,k,binary", [(40, 250, 1024, 700, True), (64, 250, 2048, 130, True),
                                              (5, 120, 96, 700, False), (2, 50, 64, 700, True),
                                              (3, 100, 128, 700, False), (1, 20, 64, 64, True)])
def test_projection_pair_multicast_is_bitwise_single_cta(B, T, n, k, binary, monkeypatch):
    """K2 on CTA pairs (each loads half of every spike stage and multicasts it to both;
    a stage is refilled once both CTAs' MMAs released it) gives the single-CTA kernel's
    currents bit for bit -- also with a single cluster, fewer pair tiles than clusters,
    odd band counts, and an odd neuron-tile count (which takes the single-CTA kernel)."""
    _need_gpu()
    import ctypes
    from paper_2501_11407_b200.engine import EpropEngine
    rng = np.random.default_rng(7 * n + k)
    w = (rng.uniform(-1, 1, (n, k)) / np.sqrt(k)).astype(np.float32)
    x = (rng.random((B, T, k)) < 0.1).astype(np.uint8)
    if not binary:
        x[0, :, :5] = 3
    eng = EpropEngine(n, k, 3, B, alif=False, w_f64=False, chunk=255 if T < 256 else 511)
    eng.set_weights(torch.from_numpy(w), torch.zeros((3, n), dtype=torch.float64))
    xd = torch.from_numpy(x).cuda()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    eng._pack(xd.data_ptr(), T * k, False, T, st)
    out = {}
    for mc, bands in (("0", None), ("1", None), ("1", "1"), ("1", "3"), ("1", "1000")):
        monkeypatch.setenv("SPB_K2_MC", mc)
        if bands is None:
            monkeypatch.delenv("SPB_K2_BANDS", raising=False)
        else:
            monkeypatch.setenv("SPB_K2_BANDS", bands)
        eng.cur.fill_(float("nan"))
        eng._project(T, st, binary=binary)
        torch.cuda.synchronize()
        out[(mc, bands)] = eng.cur.cpu().numpy().reshape(B, eng.KR, n)[:, :T].copy()
    ref = out[("0", None)]
    assert np.isfinite(ref).all()
    for key, cur in out.items():
        assert np.array_equal(cur.view(np.int64), ref.view(np.int64)), key
    exact = np.einsum("btk,nk->btn", x.astype(np.longdouble), w.astype(np.longdouble))
    assert np.max(np.abs(ref - exact.astype(np.float64))) <= 2.3e-16 * np.max(np.abs(exact))


@pytest.mark.parametrize("B,T,n,k,binary,chunk,w64", [(40, 250, 1024, 700, True, 255, False),
                                                        (5, 20, 96, 700, False, 63, False),
                                                        (3, 31, 64, 128, True, 63, False),
                                                        (2, 127, 200, 64, False, 127, False),
                                                        (7, 33, 2048, 132, True, 63, False),
                                                        (6, 45, 160, 900, True, 63, False),
                                                        (4, 50, 96, 300, True, 63, True)])
def test_projection_compact_rows_is_bitwise_kr_rows(B, T, n, k, binary, chunk, w64):
    """K2 over the chunk's live steps only (xq rows b*len + s, spb_input_proj_rows, the
    one-chunk default) writes the same currents to rows b*KR + s as the projection over
    all KR rows per sample -- bit for bit, incl. len < 32 (a quarter tile spanning several
    samples), the generic (non-binary / f64 weights, P = 8) epilogue and the streaming
    kernel of K > 768 (k = 900)."""
    _need_gpu()
    import ctypes
    from paper_2501_11407_b200.engine import EpropEngine
    rng = np.random.default_rng(B * T + n)
    w = (rng.uniform(-1, 1, (n, k)) / np.sqrt(k)).astype(np.float64 if w64 else np.float32)
    x = (rng.random((B, T, k)) < 0.1).astype(np.uint8)
    if not binary:
        x[0, :, :5] = 3
    eng = EpropEngine(n, k, 3, B, alif=False, w_f64=w64, chunk=chunk)
    eng.set_weights(torch.from_numpy(w), torch.zeros((3, n), dtype=torch.float64))
    xd = torch.from_numpy(x).cuda()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    out = {}
    for compact in (False, True):
        eng.xq.zero_()
        eng._pack(xd.data_ptr(), T * k, False, T, st, xh=True, compact=compact)
        eng.cur.fill_(float("nan"))
        eng._project(T, st, binary=binary, compact=compact)
        torch.cuda.synchronize()
        out[compact] = eng.cur.cpu().numpy().reshape(B, eng.KR, n)[:, :T].copy()
    assert np.isfinite(out[False]).all() and np.isfinite(out[True]).all()
    assert np.array_equal(out[True].view(np.int64), out[False].view(np.int64))
    exact = np.einsum("btk,nk->btn", x.astype(np.longdouble), w.astype(np.longdouble))
    assert np.max(np.abs(out[True] - exact.astype(np.float64))) <= 2.3e-16 * np.max(np.abs(exact))


def test_label_out_of_range_raises():
    _need_gpu()
    import paper_2501_11407_b200 as P
    net = P.init_network(P.NetworkSpec(kind="lif", n_hidden=8, n_inputs=4, n_classes=3))
    with pytest.raises(P.LabelOutOfRange):
        P.eprop_sparse_gradient(net, np.zeros((5, 4)), 3)
    with pytest.raises(P.ShapeMismatch):
        P.eprop_sparse_gradient(net, np.zeros((5, 5)), 0)


def test_pooled_count_inputs_vs_oracle():
    """Integer event counts (pool_channels, datasets.py:138-159) through the drop-in API."""
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    x, labels = poisson_batch(6, 700, 45, 5, seed=3)
    xp = x.reshape(6, 45, 140, 5).sum(-1).astype(np.float64)   # factor-5 pooling, counts <= 5
    assert xp.max() > 1
    net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=160, n_inputs=140, n_classes=5,
                                       precision="f64", seed=2))
    r = P.eprop_batch_gradient(net, xp, labels, chunk=63)
    ref = O.eprop_two_pass_batch(net.neuron.w, net.readout.w_out, O.Params(alif=True), xp, labels)
    assert _rel(r.grads["w"], ref.grad_w) <= REL_TOL
    assert np.allclose(r.loss, ref.loss, rtol=1e-9)


@pytest.mark.parametrize("w_f64", [False, True])
def test_int8_tensor_core_projection_is_exact(w_f64):
    """K2: cur = W x_t from sliced INT8 tcgen05 MMAs equals the exactly-rounded sum."""
    _need_gpu()
    import ctypes
    from paper_2501_11407_b200.engine import EpropEngine
    rng = np.random.default_rng(0)
    B, T, k, n = 5, 16, 700, 100
    w = rng.uniform(-1, 1, (n, k)) / np.sqrt(k)
    w[3, :] *= 1e-6                        # tiny row: per-neuron exponent
    w[7, 5] = 0.0
    w = w.astype(np.float64 if w_f64 else np.float32)
    x = (rng.random((B, T, k)) < 0.1).astype(np.uint8)
    x[0, 0, :10] = 7                       # pooled counts
    eng = EpropEngine(n, k, 3, B, alif=False, w_f64=w_f64, chunk=63)
    eng.set_weights(torch.from_numpy(w), torch.zeros((3, n), dtype=torch.float64))
    xd = torch.from_numpy(x).cuda()
    v = ctypes.c_void_p
    st = v(torch.cuda.current_stream().cuda_stream)
    eng._pack(xd.data_ptr(), T * k, False, T, st)
    eng._project(T, st)
    torch.cuda.synchronize()
    got = eng.cur.cpu().numpy().reshape(B, eng.KR, n)[:, :T]
    exact = np.einsum("btk,nk->btn", x.astype(np.longdouble), w.astype(np.longdouble))
    err = np.abs(got.astype(np.longdouble) - exact)
    # one fp64 rounding of the exact sum (half an ulp) + the digit truncation: every
    # weight is represented to within 2^(s_i - 7P) (s_i = exponent of the row maximum)
    P = eng.P                                   # 6 radix-256 digits (f32) / 8 radix-128 (f64)
    F = {6: 46, 7: 48, 8: 55}[P]                # csrc/digits.cuh
    rowmax = np.abs(w.astype(np.float64)).max(axis=1)
    s_i = np.frexp(rowmax)[1]
    trunc = np.ldexp(1.0, s_i - F - 1)                          # [n]
    cnt = x.astype(np.float64).sum(-1)                           # [B, T]
    bound = 1.12e-16 * np.abs(exact) + cnt[..., None] * trunc[None, None, :]
    assert float(np.max(err - bound)) <= 0.0


@pytest.mark.parametrize("k", [700, 2000])   # W-resident and streamed-W kernels
def test_binary_recombination_is_bitwise_the_two_part_path(k):
    """K2 with binary=1 (one int64 per output) gives the same bits as binary=0."""
    _need_gpu()
    import ctypes
    from paper_2501_11407_b200.engine import EpropEngine
    rng = np.random.default_rng(1)
    B, T, n = 6, 40, 200
    w = (rng.uniform(-1, 1, (n, k)) / np.sqrt(k)).astype(np.float32)
    w[5, :] *= 1e-5
    x = (rng.random((B, T, k)) < 0.15).astype(np.uint8)
    eng = EpropEngine(n, k, 3, B, alif=False, chunk=63)
    eng.set_weights(torch.from_numpy(w), torch.zeros((3, n), dtype=torch.float64))
    xd = torch.from_numpy(x).cuda()
    v = ctypes.c_void_p
    st = v(torch.cuda.current_stream().cuda_stream)
    eng._pack(xd.data_ptr(), T * k, False, T, st)
    outs = []
    for binary in (False, True):
        eng.cur.zero_()
        eng._project(T, st, binary=binary)
        torch.cuda.synchronize()
        outs.append(eng.cur.cpu().numpy().copy())
    assert np.array_equal(outs[0], outs[1])
    exact = np.einsum("btk,nk->btn", x.astype(np.longdouble), w.astype(np.longdouble))
    got = outs[1].reshape(B, eng.KR, n)[:, :T]
    assert np.max(np.abs(got - exact.astype(np.float64))) <= 2.3e-16 * np.max(np.abs(exact))


def test_streamed_inputs_match_resident_and_memory_is_flat_in_T():
    """Streaming x chunk by chunk from pinned host memory gives bitwise the same update as
    resident inputs, and peak device memory does not grow with T."""
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=256, n_inputs=700, n_classes=20,
                                       precision="f32", seed=0))
    kw = _neuron_kwargs(net)
    B = 16
    x, y = poisson_batch(B, 700, 300, 20, seed=5)
    yd = torch.from_numpy(y).cuda()
    res = {}
    for mode in ("resident", "streamed"):
        eng = EpropEngine(256, 700, 20, B, alif=True, chunk=127)
        eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
        xin = torch.from_numpy(x).cuda() if mode == "resident" else torch.from_numpy(x).pin_memory()
        eng.run(xin, yd, **kw)
        torch.cuda.synchronize()
        res[mode] = (eng.grad_w(torch.float64).cpu().numpy(), eng.loss.cpu().numpy(),
                     eng.grad_wout.cpu().numpy())
    for a, b in zip(res["resident"], res["streamed"]):
        assert np.array_equal(a, b)
    del eng, xin  # measure the next engines from a clean base
    import gc
    gc.collect()
    peaks = []
    for T in (300, 3000):
        x, y = poisson_batch(B, 700, T, 20, seed=6)
        xh = torch.from_numpy(x).pin_memory()
        yd = torch.from_numpy(y).cuda()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        eng = EpropEngine(256, 700, 20, B, alif=True, chunk=127)
        eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
        eng.run(xh, yd, **kw)
        torch.cuda.synchronize()
        peaks.append(torch.cuda.max_memory_allocated() - base)
        del eng
    assert peaks[1] <= 1.05 * peaks[0], peaks


@pytest.mark.parametrize("k,T", [(700, 300), (37, 70)])
def test_bit_packed_inputs_match_byte_inputs(k, T):
    """Binary spikes given bit-packed (8x less H2D) give bitwise the same update."""
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=160, n_inputs=k, n_classes=5,
                                       precision="f32", seed=1))
    B = 6
    x, y = poisson_batch(B, k, T, 5, seed=9)
    xbits = np.packbits(x, axis=-1, bitorder="little")
    yd = torch.from_numpy(y).cuda()
    outs = []
    for xin, bits in ((torch.from_numpy(x).cuda(), False), (torch.from_numpy(xbits).cuda(), True),
                      (torch.from_numpy(xbits).pin_memory(), True)):
        eng = EpropEngine(160, k, 5, B, alif=True, chunk=63)
        eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
        eng.run(xin, yd, bits=bits, **_neuron_kwargs(net))
        torch.cuda.synchronize()
        outs.append((eng.grad_w(torch.float64).cpu().numpy(), eng.loss.cpu().numpy()))
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])


@pytest.mark.parametrize("bits", [False, True])
def test_one_chunk_streamed_inputs_match_resident(bits):
    """One chunk (the pack also writes K5's raw operand) from pinned host memory, bytes and
    bit-packed: bitwise the resident-input update."""
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    from paper_2501_11407_b200.engine import EpropEngine
    from paper_2501_11407_b200.gradients import _neuron_kwargs
    net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=256, n_inputs=700, n_classes=20,
                                       precision="f32", seed=2))
    B = 12
    x, y = poisson_batch(B, 700, 100, 20, seed=7)
    xin = np.packbits(x, axis=-1, bitorder="little") if bits else x
    yd = torch.from_numpy(y).cuda()
    outs = []
    for dev_in in (torch.from_numpy(xin).cuda(), torch.from_numpy(xin).pin_memory()):
        eng = EpropEngine(256, 700, 20, B, alif=True, chunk=127)
        eng.set_weights(torch.from_numpy(net.neuron.w), torch.from_numpy(net.readout.w_out))
        eng.run(dev_in, yd, bits=bits, **_neuron_kwargs(net))
        torch.cuda.synchronize()
        outs.append((eng.grad_w_acc.cpu().numpy().copy(), eng.loss.cpu().numpy().copy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_dropin_binary_counts_travel_bit_packed():
    """uint8 0/1 counts through the drop-in are bit-packed on the host (spb_host_pack_bits)
    and give bitwise the update of packed=True input and of the byte-staged path; a count
    > 1 falls back to byte staging."""
    _need_gpu()
    import paper_2501_11407_b200 as P
    from paper_2501_11407_b200.datasets import poisson_batch
    from paper_2501_11407_b200.gradients import _staging, get_engine
    net = P.init_network(P.NetworkSpec(kind="alif", n_hidden=160, n_inputs=700, n_classes=5,
                                       precision="f32", seed=4))
    B, T = 64, 120   # 5.4 MB of counts: the threaded, sliced packing path
    x, y = poisson_batch(B, 700, T, 5, seed=11)
    r_counts = P.eprop_batch_gradient(net, x, y)
    st = _staging(get_engine(net, B, T=T))
    assert not st.counts_nonbinary and len(st.bufs) == 1 and \
        next(iter(st.bufs))[2] == 88                       # staged bit-packed
    r_packed = P.eprop_batch_gradient(net, np.packbits(x, axis=-1, bitorder="little"), y,
                                      packed=True)
    st.counts_nonbinary = True                               # force the byte staging
    r_bytes = P.eprop_batch_gradient(net, x, y)
    for r in (r_packed, r_bytes):
        assert np.array_equal(r.grads["w"], r_counts.grads["w"])
        assert np.array_equal(r.grads["w_out"], r_counts.grads["w_out"])
        assert np.array_equal(r.loss, r_counts.loss)
    st.counts_nonbinary = False
    x2 = x.copy()
    x2[B - 1, T - 1, 699] = 2
    r2 = P.eprop_batch_gradient(net, x2, y)
    assert st.counts_nonbinary
    ref = O.eprop_two_pass_batch(net.neuron.w, net.readout.w_out, O.Params(alif=True), x2, y)
    assert _rel(r2.grads["w"], ref.grad_w) <= REL_TOL
