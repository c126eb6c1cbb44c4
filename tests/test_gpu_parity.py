"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle.

Bars (BASELINE.json north_star): codes / packed bytes / scales / folded are
BIT-EXACT; GEMM outputs have normwise relative error
max|Y - Y_ref| / max|Y_ref| <= 1e-3 against the fp32 dequantize-then-matmul
(and, where the reference's own test uses it, the elementwise bound
gemm_tolerance = 4 eps32 K max|W_hat| max|X|, gemm.py:118-122).
"""

import hashlib
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_2312_08583_b200 as L  # noqa: E402
from oracle import lpqt_oracle as O  # noqa: E402  (checker only)
from tests.conftest import names  # noqa: E402

CGQ = L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP6_E3M2)
REL_TOL = 1e-3


def normwise_rel(Y, Yref):
    Y = np.asarray(Y, np.float64)
    Yref = np.asarray(Yref, np.float64)
    den = np.max(np.abs(Yref))
    return float(np.max(np.abs(Y - Yref)) / den) if den else float(np.max(np.abs(Y)))


# ---------------------------------------------------------------- quantize
def test_quantize_bit_exact_vs_reference(golden):
    for name in names(golden, "q_names"):
        W = golden[f"q/{name}/W"]
        if name.startswith("bf16"):
            Win = torch.from_numpy(W).to(torch.bfloat16).cuda()
            q = L.quantize_tensor(Win, CGQ, bias_shift=True)
            scales, folded = q.scales.cpu().numpy(), q.folded_scales.cpu().numpy()
            seg4, seg2 = q.payload.seg4.cpu().numpy(), q.payload.seg_tail.cpu().numpy()
        else:
            q = L.quantize_tensor(W, CGQ, bias_shift=True)
            scales, folded, seg4, seg2 = q.scales, q.folded_scales, q.payload.seg4, q.payload.seg_tail
        assert np.array_equal(scales.view(np.uint16), golden[f"q/{name}/scales"]), name
        assert np.array_equal(folded.view(np.uint16), golden[f"q/{name}/folded"]), name
        assert np.array_equal(seg4, golden[f"q/{name}/seg4"]), name
        assert np.array_equal(seg2, golden[f"q/{name}/seg2"]), name
        deq = L.dequantize_tensor(q, "bias_shift")
        deq = deq.cpu().numpy() if torch.is_tensor(deq) else deq
        assert np.array_equal(deq, golden[f"q/{name}/deq"]), name
        naive = L.dequantize_tensor(q, "naive")
        naive = naive.cpu().numpy() if torch.is_tensor(naive) else naive
        assert np.array_equal(naive, golden[f"q/{name}/deq"]), name


def test_quantize_error_cases_vs_reference(golden):
    for name in names(golden, "e_names"):
        W = golden[f"e/{name}/W"]
        bs = bool(golden[f"e/{name}/bias_shift"])
        want = str(golden[f"e/{name}/result"])
        try:
            q = L.quantize_tensor(W, CGQ, bias_shift=bs)
            got = "ok"
            assert np.array_equal(q.scales.view(np.uint16), golden[f"e/{name}/scales"])
        except L.LpqtError as exc:
            got = type(exc).__name__
        assert got == want, name


@pytest.mark.parametrize("dtype", [np.float64, np.float32, np.float16])
@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (17, 40), (128, 264), (257, 1000)])
def test_quantize_random_vs_oracle(dtype, shape):
    rng = np.random.default_rng(hash((shape, np.dtype(dtype).name)) % 2**32)
    W = (rng.standard_normal(shape) * rng.choice([1e-3, 0.02, 1.0, 30.0])).astype(dtype)
    W[rng.random(shape) < 0.05] = 0
    q = L.quantize_tensor(W, CGQ, bias_shift=True)
    o = O.quantize_tensor(W, bias_shift=True)
    assert np.array_equal(q.scales.view(np.uint16), o["scales"].view(np.uint16))
    assert np.array_equal(q.folded_scales.view(np.uint16), o["folded"].view(np.uint16))
    assert np.array_equal(q.payload.seg4, o["seg4"])
    assert np.array_equal(q.payload.seg_tail, o["seg2"])


def test_quantize_llama_shape_codes_match_oracle():
    # full-row property at a realistic size: codes of every row equal the oracle's
    rng = np.random.default_rng(7)
    W = (rng.standard_normal((512, 4096)) * 0.02).astype(np.float16)
    q = L.quantize_tensor(torch.from_numpy(W).cuda(), CGQ, bias_shift=True)
    o = O.quantize_tensor(W, bias_shift=True)
    assert np.array_equal(q.payload.seg4.cpu().numpy(), o["seg4"])
    assert np.array_equal(q.payload.seg_tail.cpu().numpy(), o["seg2"])


_TORCH_DT = {"f64": torch.float64, "f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}


def _planes_then_prepack(Wt):
    q = L.quantize_tensor(Wt, CGQ, bias_shift=True)
    n, k = Wt.shape
    return L.Fp6Weight.from_planes(q.payload.seg4, q.payload.seg_tail, q.scales, n, k, q.folded_scales), q


def _oracle_of(Wt):
    # bf16 / f16 / f32 widen to f64 exactly; the reference quantizes in f64
    return O.quantize_tensor(Wt.double().cpu().numpy(), bias_shift=True)


@pytest.mark.parametrize("dt", ["f16", "bf16", "f32", "f64"])
@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (130, 300), (129, 1000), (256, 4096)])
def test_quantize_tiles_equals_prepacked_planes(dt, shape):
    """lpqt_fp6_quantize_tiles == prepack(lpqt_fp6_quantize_pack) byte for
    byte, and both agree with the oracle (quantizer.py:189-248)."""
    g = torch.Generator().manual_seed(hash((dt, shape)) % 2**31)
    Wt = (torch.randn(shape, generator=g, dtype=torch.float64) * 0.05).to(_TORCH_DT[dt])
    Wt[torch.rand(shape, generator=g) < 0.03] = 0
    Wt = Wt.cuda()
    fused = L.Fp6Weight.quantize(Wt)
    ref, q = _planes_then_prepack(Wt)
    assert torch.equal(fused.tiles, ref.tiles)
    assert torch.equal(fused.scales.view(torch.int16), ref.scales.view(torch.int16))
    assert torch.equal(fused.folded.view(torch.int16), q.folded_scales.view(torch.int16))
    o = _oracle_of(Wt)
    assert np.array_equal(q.scales.cpu().numpy().view(np.uint16), o["scales"].view(np.uint16))
    assert np.array_equal(q.payload.seg4.cpu().numpy(), o["seg4"])
    assert np.array_equal(q.payload.seg_tail.cpu().numpy(), o["seg2"])


def _adversarial_rows(dt):
    """Rows whose scale is pinned (peak = 28 * S0 exactly) and whose entries
    sit exactly on every grid midpoint m_i * S0, one ulp of the input dtype
    either side of it, on -0.0, on tiny negatives and near saturation."""
    tdt = _TORCH_DT[dt]
    ibits = {torch.float16: torch.int16, torch.bfloat16: torch.int16,
             torch.float32: torch.int32, torch.float64: torch.int64}[tdt]
    rows = []
    for s0 in (2.0 ** -7, 1.5 * 2 ** -9, 1.25 * 2 ** -3, 1.75 * 2 ** -12, 0.0123, 3.0e-5):
        s0 = float(np.float16(s0))
        row = [28.0 * s0, -28.0 * s0, -0.0, 0.0, -1e-30, 1e-30, 27.9 * s0, -26.0 * s0]
        for m in O.grid_midpoints():
            v = torch.tensor([m * s0], dtype=torch.float64).to(tdt)
            b = v.view(ibits)
            for x in (v, (b + 1).view(tdt), (b - 1).view(tdt)):
                row += [float(x), -float(x)]
        rows.append(row)
    W = torch.zeros((len(rows), max(len(r) for r in rows)), dtype=torch.float64)
    for i, r in enumerate(rows):
        W[i, :len(r)] = torch.tensor(r, dtype=torch.float64)
    return W.to(tdt)


@pytest.mark.parametrize("dt", ["f16", "bf16", "f32", "f64"])
def test_quantize_midpoint_ties_and_signs_vs_oracle(dt):
    Wt = _adversarial_rows(dt).cuda()
    fused = L.Fp6Weight.quantize(Wt)
    ref, q = _planes_then_prepack(Wt)
    o = _oracle_of(Wt)
    assert np.array_equal(q.scales.cpu().numpy().view(np.uint16), o["scales"].view(np.uint16))
    assert np.array_equal(q.payload.seg4.cpu().numpy(), o["seg4"])
    assert np.array_equal(q.payload.seg_tail.cpu().numpy(), o["seg2"])
    assert torch.equal(fused.tiles, ref.tiles)
    assert torch.equal(fused.codes().cpu(), torch.from_numpy(O.unpack(o["seg4"], o["seg2"], Wt.numel())
                                                             .reshape(Wt.shape)))


@pytest.mark.parametrize("offset", [0, 8, 3])
def test_quantize_tiles_strided_rows(offset):
    """ldw > K and 16-byte-misaligned rows go through the scalar path with
    the same result."""
    n, k, ldw = 200, 520, 600
    g = torch.Generator().manual_seed(5)
    big = (torch.randn((n, ldw), generator=g) * 0.1).half().cuda()
    view = big[:, offset:offset + k]
    want = L.Fp6Weight.quantize(view.contiguous())
    from paper_2312_08583_b200 import _lib
    lib = _lib.load()
    tiles = torch.empty(lib.lpqt_fp6_tiles_bytes(n, k), dtype=torch.uint8, device="cuda")
    scales = torch.empty(n, dtype=torch.float16, device="cuda")
    flags = _lib.Flags()
    st = lib.lpqt_fp6_quantize_tiles(view.data_ptr(), _lib.F16, n, k, ldw, 0, scales.data_ptr(), None,
                                     tiles.data_ptr(), flags.ptr, _lib.stream_ptr())
    assert st == 0
    flags.raise_if_set()
    assert torch.equal(tiles, want.tiles)
    assert torch.equal(scales.view(torch.int16), want.scales.view(torch.int16))


def test_quantize_tiles_errors():
    W = torch.ones((4, 8), dtype=torch.float16, device="cuda")
    W[1, 3] = float("nan")
    with pytest.raises(L.InvalidInput):
        L.Fp6Weight.quantize(W)
    W = torch.full((2, 8), 3.0e38, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(L.InvalidInput):
        L.Fp6Weight.quantize(W)   # S = peak / 28 overflows binary16
    W = torch.full((2, 8), 60000.0, dtype=torch.float16, device="cuda")
    with pytest.raises(L.ScaleOverflow):
        L.Fp6Weight.quantize(W)   # S * 2^12 > 65504 (bias shift)
    assert L.Fp6Weight.quantize(W, bias_shift=False).folded is None


def test_empty_inputs():
    q = L.quantize_tensor(np.zeros((0, 5)), CGQ, bias_shift=True)
    assert q.scales.size == 0 and q.payload.code_count == 0
    q = L.quantize_tensor(np.zeros((3, 0)), CGQ)
    Y = L.gemm_quantized(q, np.zeros((0, 2), np.float32))
    assert Y.shape == (3, 2) and not Y.any()


# ---------------------------------------------------------------- codec / packing / fold
def test_encode_vs_reference(golden):
    assert np.array_equal(L.encode_rtn_array(L.FP6_E3M2, golden["enc/x"]), golden["enc/codes"])
    with pytest.raises(L.InvalidInput):
        L.encode_rtn_array(L.FP6_E3M2, np.array([1.0, np.inf]))
    assert L.encode_rtn(L.FP6_E3M2, 26.0) == 0b011110


def test_pack_unpack_vs_reference(golden):
    for n in golden["p_lens"]:
        c = golden[f"p/{n}/codes"]
        seg = L.pack(L.FP6_E3M2, c)
        assert np.array_equal(seg.seg4, golden[f"p/{n}/seg4"]), n
        assert np.array_equal(seg.seg_tail, golden[f"p/{n}/seg2"]), n
        assert np.array_equal(L.unpack(L.FP6_E3M2, seg), c)
    seg = L.pack(L.FP6_E3M2, [0b011111, 0b001100, 0, 0b100001])
    assert list(seg.seg4) == [0x37, 0x80, 0, 0] and list(seg.seg_tail) == [0x43, 0, 0, 0]
    with pytest.raises(L.InvalidCode):
        L.pack(L.FP6_E3M2, [64])
    with pytest.raises(L.PayloadMismatch):
        L.unpack(L.FP6_E3M2, L.PackedSegments(seg.seg4[:-1], seg.seg_tail, 4))


def test_fold_and_exhaustive_bias_shift_sweep(golden):
    s = golden["fold/scales"].view(np.float16)
    f = L.fold_scale_array(L.FP6_E3M2, s)
    assert np.array_equal(f.view(np.uint16), golden["fold/folded"])
    codes = np.arange(64, dtype=np.uint8)
    sweep = L.dequant_bias_shift_array(L.FP6_E3M2, codes[:, None], f[None, :])
    naive = L.dequant_naive_array(L.FP6_E3M2, codes[:, None], s[None, :])
    assert np.array_equal(sweep.view(np.uint16), naive.view(np.uint16))
    assert hashlib.sha256(sweep.view(np.uint16).tobytes()).hexdigest() == str(golden["fold/sweep_sha256"])
    with pytest.raises(L.ScaleOverflow):
        L.fold_scale(L.FP6_E3M2, np.float16(16.0))
    with pytest.raises(L.InvalidInput):
        L.fold_scale_array(L.FP6_E3M2, np.array([0.0], np.float16))


# ---------------------------------------------------------------- tile layout + transform
@pytest.mark.parametrize("shape", [(1, 1), (5, 33), (128, 128), (130, 300), (384, 1024)])
def test_prepack_roundtrip_and_register_transform(shape):
    rng = np.random.default_rng(11)
    n, k = shape
    codes = rng.integers(0, 64, size=n * k, dtype=np.uint8)
    seg4, seg2 = O.pack(codes)
    scales = (rng.uniform(1e-4, 15.9, size=n)).astype(np.float16)
    folded = O.fold_scale_array(scales)
    w = L.Fp6Weight.from_planes(torch.from_numpy(seg4).cuda(), torch.from_numpy(seg2).cuda(),
                                torch.from_numpy(scales).cuda(), n, k, torch.from_numpy(folded).cuda())
    assert np.array_equal(w.codes().cpu().numpy().ravel(), codes)
    # the GEMM's register rebuild (hardware e3m2 converter) x S in binary16 ==
    # the reference's bias-shift dequant (and its naive path) bit for bit
    deq = w.dequantize_f16().cpu().numpy()
    ref = O.dequant_bias_shift_array(codes.reshape(n, k), folded[:, None])
    assert np.array_equal(deq.view(np.uint16), ref.view(np.uint16))
    ref_naive = O.dequant_naive_array(codes.reshape(n, k), scales[:, None])
    assert np.array_equal(deq.view(np.uint16), ref_naive.view(np.uint16))


# ---------------------------------------------------------------- GEMM
def test_gemm_vs_reference_golden(golden):
    for name in names(golden, "g_names"):
        W, X = golden[f"g/{name}/W"], golden[f"g/{name}/X"]
        q = L.quantize_tensor(W, CGQ, bias_shift=True)
        Y = L.gemm_quantized(q, X)
        assert Y.dtype == np.float32 and Y.shape == golden[f"g/{name}/Y"].shape
        assert normwise_rel(Y, golden[f"g/{name}/Y"]) <= REL_TOL, name
        # the reference's own elementwise f32-vs-f64 bound (tests/test_gemm.py:100-107)
        assert np.max(np.abs(Y - golden[f"g/{name}/Yf64"])) <= float(golden[f"g/{name}/tol"]) + 1e-30, name
        if name.startswith("grid_exact"):
            assert np.array_equal(Y.astype(np.float64), golden[f"g/{name}/Yf64"])


def test_gemm_identity_weights_exact():
    # pkg/tests/test_gemm.py:59-64: identity stored with unit scale
    n = 130
    codes = np.zeros((n, n), np.uint8)
    codes[np.arange(n), np.arange(n)] = 0b001100
    s4, s2 = O.pack(codes.ravel())
    q = L.QuantizedTensor(n, n, CGQ, np.ones(n, np.float16), None, L.PackedSegments(s4, s2, n * n))
    X = np.random.default_rng(31).standard_normal((n, 5)).astype(np.float16)
    assert np.array_equal(L.gemm_quantized(q, X), X.astype(np.float32))


def test_gemm_subnormal_codes_one_hot():
    # composed values of codes 1-3 are binary16 subnormals (dequant.py:40):
    # one-hot activation columns must reproduce every weight exactly
    rng = np.random.default_rng(5)
    n, k = 256, 128
    codes = rng.choice(np.array([1, 2, 3, 33, 34, 35, 0, 31, 63], np.uint8), size=(n, k))
    scales = rng.uniform(1e-3, 15.0, size=n).astype(np.float16)
    s4, s2 = O.pack(codes.ravel())
    q = L.QuantizedTensor(n, k, CGQ, scales, None, L.PackedSegments(s4, s2, n * k))
    X = np.eye(k, dtype=np.float16)
    Y = L.gemm_quantized(q, X)
    ref = O.dequantize_tensor(codes.ravel(), n, k, scales=scales, path="naive").astype(np.float32)
    assert np.array_equal(Y, ref)


SHAPES = [(4096, 4096, 1), (4096, 4096, 16), (1024, 2048, 7), (512, 640, 33), (256, 1024, 129),
          (384, 512, 300), (256, 384, 600),
          # long K (many ring wraps per CTA) at every MMA width
          (1024, 8192, 3), (2048, 8192, 24), (1024, 8192, 48), (2048, 8192, 100), (1024, 8192, 600)]


@pytest.mark.parametrize("n,k,m", SHAPES)
def test_gemm_llama_like_vs_dequant_matmul(n, k, m):
    g = torch.Generator(device="cuda").manual_seed(n * 7 + k * 3 + m)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    X = torch.randn(k, m, generator=g, device="cuda").half()
    q = L.quantize_tensor(W, CGQ, bias_shift=True)
    W_hat = L.dequantize_tensor(q, "bias_shift")       # f64, exact
    Y = L.gemm_quantized(q, X)
    Y_ref = (W_hat @ X.double()).float()                  # dequantize-then-matmul (f64)
    assert normwise_rel(Y.cpu().numpy(), Y_ref.cpu().numpy()) <= REL_TOL


@pytest.mark.parametrize("split_k", [1, 2, 3, 7])
def test_gemm_split_k_variants_agree(split_k):
    g = torch.Generator(device="cuda").manual_seed(3)
    W = (torch.randn(512, 3072, generator=g, device="cuda") * 0.02).half()
    X = torch.randn(3072, 16, generator=g, device="cuda").half()
    q = L.quantize_tensor(W, CGQ, bias_shift=True)
    Y = L.gemm_quantized(q, X, split_k=split_k, sched="streamk")
    Y_ref = (L.dequantize_tensor(q, "bias_shift") @ X.double()).float()
    assert normwise_rel(Y.cpu().numpy(), Y_ref.cpu().numpy()) <= REL_TOL
    Y2 = L.gemm_quantized(q, X, split_k=split_k, sched="streamk")
    assert torch.equal(Y.view(torch.int32), Y2.view(torch.int32))   # deterministic


@pytest.mark.parametrize("cluster", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("n,k,m", [(512, 3072, 16), (1280, 1000, 5), (4096, 4096, 1), (640, 11008, 32)])
def test_gemm_cluster_split_k(n, k, m, cluster):
    """Cluster split-K (DSMEM reduction) against the dequantize-then-matmul
    oracle, bit-identical on repeat, and consistent with stream-K."""
    g = torch.Generator(device="cuda").manual_seed(n + k + m + cluster)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    X = torch.randn(k, m, generator=g, device="cuda").half()
    q = L.quantize_tensor(W, CGQ, bias_shift=True)
    p = L.plan(m, n, k, cluster, sched="cluster")
    assert p["schedule"] == "cluster" and p["cluster"] == min(cluster, (k + 127) // 128)
    Y = L.gemm_quantized(q, X, split_k=cluster, sched="cluster")
    Y_ref = (L.dequantize_tensor(q, "bias_shift") @ X.double()).float()
    assert normwise_rel(Y.cpu().numpy(), Y_ref.cpu().numpy()) <= REL_TOL
    Y2 = L.gemm_quantized(q, X, split_k=cluster, sched="cluster")
    assert torch.equal(Y.view(torch.int32), Y2.view(torch.int32))   # deterministic
    Y3 = L.gemm_quantized(q, X, sched="streamk")
    assert normwise_rel(Y.cpu().numpy(), Y3.cpu().numpy()) <= REL_TOL


def test_w6a16_linear_torch_layout():
    g = torch.Generator(device="cuda").manual_seed(9)
    W = (torch.randn(1000, 520, generator=g, device="cuda") * 0.05).half()
    lin = L.Fp6Linear.from_dense(W)
    for m in (1, 5, 16, 40):
        x = torch.randn(m, 520, generator=g, device="cuda").half()
        y = lin(x)
        assert y.shape == (m, 1000) and y.dtype == torch.float16
        q = L.quantize_tensor(W, CGQ, bias_shift=True)
        ref = (L.dequantize_tensor(q, "bias_shift") @ x.double().T).T
        assert normwise_rel(y.float().cpu().numpy(), ref.cpu().numpy()) <= REL_TOL


def test_w6a16_linear_input_forms_and_device_check():
    """3-D / strided / bf16 activations give the same product as the plain
    fp16 matrix; a host tensor is refused before any launch (the kernel reads
    x by address)."""
    g = torch.Generator(device="cuda").manual_seed(19)
    W = (torch.randn(384, 640, generator=g, device="cuda") * 0.05).half()
    w = L.Fp6Weight.quantize(W)
    x = torch.randn(2, 3, 640, generator=g, device="cuda").half()
    y = L.w6a16_linear(x, w, out_dtype=torch.float32)
    assert y.shape == (2, 3, 384)
    y2 = L.w6a16_linear(x.reshape(6, 640), w, out_dtype=torch.float32)
    assert torch.equal(y.reshape(6, 384), y2)
    xs = torch.randn(640, 6, generator=g, device="cuda").half().t()      # non-contiguous view
    assert torch.equal(L.w6a16_linear(xs, w, out_dtype=torch.float32),
                       L.w6a16_linear(xs.contiguous(), w, out_dtype=torch.float32))
    xb = x.reshape(6, 640).to(torch.bfloat16)                            # cast once to fp16
    assert torch.equal(L.w6a16_linear(xb, w, out_dtype=torch.float32),
                       L.w6a16_linear(xb.half(), w, out_dtype=torch.float32))
    with pytest.raises(L.InvalidInput):
        L.w6a16_linear(x.cpu(), w)
    with pytest.raises(L.ShapeError):
        L.w6a16_linear(torch.zeros(4, 641, device="cuda").half(), w)


def test_workspace_reuse_across_shapes():
    # a split-K call with many tiles after one with few must not read the
    # previous call's partials as tile counters (regression)
    g = torch.Generator(device="cuda").manual_seed(21)
    outs = []
    for n, k in [(4096, 11008), (10240, 8192), (1024, 4096), (10240, 8192)]:
        W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
        lin = L.Fp6Linear.from_dense(W)
        x = torch.randn(3, k, generator=g, device="cuda").half()
        y = lin(x).float()
        q = L.quantize_tensor(W, CGQ, bias_shift=True)
        ref = (L.dequantize_tensor(q, "bias_shift") @ x.double().T).T
        assert torch.isfinite(y).all()
        assert normwise_rel(y.cpu().numpy(), ref.cpu().numpy()) <= REL_TOL
        outs.append(y)


@pytest.mark.parametrize("y_dtype", [torch.float16, torch.bfloat16, torch.float32])
@pytest.mark.parametrize("n,k,m", [(4096, 4096, 16), (1000, 2048, 3), (22016, 1024, 16), (512, 1024, 32)])
def test_linear_output_dtypes_and_layouts(n, k, m, y_dtype):
    """Both output layouts and all output dtypes, with and without the TMA
    tensor-store epilogue (unaligned row strides fall back to direct stores)."""
    g = torch.Generator(device="cuda").manual_seed(n + k + m)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    lin = L.Fp6Linear.from_dense(W)
    q = L.quantize_tensor(W, CGQ, bias_shift=True)
    W_hat = L.dequantize_tensor(q, "bias_shift")
    x = torch.randn(m, k, generator=g, device="cuda").half()
    ref = (W_hat @ x.double().T).T                       # [M, N]
    y = L.w6a16_linear(x, lin.weight, out_dtype=y_dtype)    # torch layout [M, N]
    assert y.dtype == y_dtype and y.shape == (m, n)
    assert normwise_rel(y.double().cpu().numpy(), ref.cpu().numpy()) <= 1e-3 + (8e-3 if y_dtype == torch.bfloat16 else 0)
    from paper_2312_08583_b200.linear import gemm_nm, stage_activations
    xt, kp = stage_activations(x.T.contiguous(), k)
    ynm = gemm_nm(lin.weight, xt, kp, m)                  # reference layout [N, M] f32
    assert normwise_rel(ynm.T.double().cpu().numpy(), ref.cpu().numpy()) <= 1e-3


def test_chained_layers_read_previous_output():
    """A GEMM whose activations are the previous GEMM's output, launched back
    to back (programmatic dependent launch): the consumer must see the
    producer's complete output (TMA-stored tiles included)."""
    g = torch.Generator(device="cuda").manual_seed(5)
    W1 = (torch.randn(4096, 4096, generator=g, device="cuda") * 0.02).half()
    W2 = (torch.randn(2048, 4096, generator=g, device="cuda") * 0.02).half()
    l1, l2 = L.Fp6Linear.from_dense(W1), L.Fp6Linear.from_dense(W2)
    x = torch.randn(16, 4096, generator=g, device="cuda").half()
    for _ in range(3):
        y1 = l1(x)
        y2 = l2(y1)
        torch.cuda.synchronize()
        r1 = (L.dequantize_tensor(L.quantize_tensor(W1, CGQ, bias_shift=True), "bias_shift") @ x.double().T).T
        assert normwise_rel(y1.double().cpu().numpy(), r1.cpu().numpy()) <= 1e-3
        r2 = (L.dequantize_tensor(L.quantize_tensor(W2, CGQ, bias_shift=True), "bias_shift") @ y1.double().T).T
        assert normwise_rel(y2.double().cpu().numpy(), r2.cpu().numpy()) <= 1e-3


def test_prefill_large_x_weight_row_fastest_order():
    """M x K x 2 B > 40 MB switches the tile order (weight-row tiles of one
    batch tile back to back); results must not change."""
    g = torch.Generator(device="cuda").manual_seed(17)
    n, k, m = 640, 8192, 2600
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    X = torch.randn(k, m, generator=g, device="cuda").half()
    q = L.quantize_tensor(W, CGQ, bias_shift=True)
    Y = L.gemm_quantized(q, X)
    Y_ref = (L.dequantize_tensor(q, "bias_shift") @ X.double()).float()
    assert normwise_rel(Y.cpu().numpy(), Y_ref.cpu().numpy()) <= REL_TOL


def test_prefill_round_robin_tiles_match_stream_k():
    """X > 40 MB with >= 2 waves of tiles: whole tiles round-robin over the
    CTAs (plan schedule "roundrobin"); same result as forced stream-K within
    the fp32 summation tolerance, and within REL_TOL of the f64 reference."""
    g = torch.Generator(device="cuda").manual_seed(23)
    n, k, m = 4096, 8192, 2600
    assert L.plan(m, n, k, sched="single")["schedule"] == "roundrobin"   # (auto: the CTA-pair kernel)
    w = L.Fp6Weight.quantize((torch.randn(n, k, generator=g, device="cuda") * 0.02).half())
    x = torch.randn(m, k, generator=g, device="cuda").half()
    y = L.w6a16_linear(x, w, out_dtype=torch.float32, sched="single")
    y_sk = L.w6a16_linear(x, w, out_dtype=torch.float32, sched="streamk")
    assert normwise_rel(y.cpu().numpy(), y_sk.cpu().numpy()) <= 1e-5
    y_pair = L.w6a16_linear(x, w, out_dtype=torch.float32)
    assert L.plan(m, n, k)["schedule"] == "pair"
    assert normwise_rel(y_pair.cpu().numpy(), y_sk.cpu().numpy()) <= 1e-5
    ref = (x.double() @ w.dequantize_f16().double().t())
    assert normwise_rel(y.cpu().numpy(), ref.cpu().numpy()) <= REL_TOL


@pytest.mark.parametrize("m", [1, 16, 512])
def test_prefetch_next_linear_is_transparent(m):
    """lpqt_w6a16_linear_pf: naming the next launch's weight (stream-K and
    cluster-split next plans, any depth) leaves every result bit-identical."""
    g = torch.Generator(device="cuda").manual_seed(3)
    shapes = [(12288, 4096), (4096, 4096), (4096, 11008), (640, 256)]
    ws = [L.Fp6Weight.quantize((torch.randn(n, k, device="cuda", generator=g) * 0.02).half()) for n, k in shapes]
    xs = [torch.randn(m, k, device="cuda", generator=g).half() for _, k in shapes]
    want = [L.w6a16_linear(x, w) for x, w in zip(xs, ws)]
    for depth in (0, 16, 12288, 1 << 20):
        for i, (x, w) in enumerate(zip(xs, ws)):
            nxt = ws[(i + 1) % len(ws)]
            got = L.w6a16_linear(x, w, prefetch=nxt, prefetch_bytes=depth)
            assert torch.equal(got, want[i]), (i, depth)
    torch.cuda.synchronize()


@pytest.mark.parametrize("n,k,m", [(4096, 11008, 16), (4096, 11008, 1), (1024, 16384, 8), (4096, 11008, 32)])
def test_streamk_fixup_paths_bit_identical(n, k, m):
    """Stream-K tiles shared by 2..N CTAs close through whichever path the
    timing picks (last-arriver peek + bulk gather, two-contributor fast path,
    publish + atomic): every path sums the contributors in k order, so
    repeated launches are bit-identical and match the oracle within tolerance."""
    g = torch.Generator(device="cuda").manual_seed(9)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    w = L.Fp6Weight.quantize(W)
    x = torch.randn(m, k, generator=g, device="cuda").half()
    ys = [L.w6a16_linear(x, w, out_dtype=torch.float32, sched="streamk") for _ in range(20)]
    for y in ys[1:]:
        assert torch.equal(y.view(torch.int32), ys[0].view(torch.int32))
    ref = (w.dequantize_f16().double() @ x.double().t()).t()
    assert normwise_rel(ys[0].cpu().numpy(), ref.cpu().numpy()) <= REL_TOL


def test_split_k_workspace_shared_across_shapes_is_exact():
    """Launches of different shapes back to back (PDL) reuse the same split-K
    workspace slots; every result must equal its own first run bit for bit
    (partials are read through L2 only — an L1 line left by the previous
    shape's launch must never be seen)."""
    g = torch.Generator(device="cuda").manual_seed(31)
    shapes = [(4096, 11008, 1), (640, 256, 1), (4096, 11008, 16), (1024, 8192, 3), (8192, 8192, 128),
              (4096, 4096, 300), (2048, 4096, 40), (1024, 8192, 24), (4096, 11008, 64)]
    blocks = [0, 0, 0, 128, 0, 256, 0, 128, 0]     # FGQ launches interleaved with CGQ ones
    ws = [L.Fp6Weight.quantize((torch.randn(n, k, device="cuda", generator=g) * 0.02).half(), block=b)
          for (n, k, _), b in zip(shapes, blocks)]
    xs = [torch.randn(m, k, device="cuda", generator=g).half() for _, k, m in shapes]
    want = [L.w6a16_linear(x, w, out_dtype=torch.float32) for x, w in zip(xs, ws)]
    for r in range(30):
        for i in (range(len(shapes)) if r % 2 else reversed(range(len(shapes)))):
            y = L.w6a16_linear(xs[i], ws[i], out_dtype=torch.float32, prefetch=ws[(i + 1) % len(ws)])
            assert torch.equal(y, want[i]), (r, shapes[i])


# ---------------------------------------------------------------- FGQ x FP6
FGQ_GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_fgq.npz")


def test_fgq_quantize_dequantize_vs_reference():
    """FGQ quantize on the GPU == the reference's bytes for every block size
    (16, 7, 64, 128, 256, ragged last blocks, an all-zero block)."""
    g = np.load(FGQ_GOLD)
    for name in [str(s) for s in g["f_names"]]:
        W, b = g[f"f/{name}/W"], int(g[f"f/{name}/block"])
        q = L.quantize_tensor(W, L.QuantScheme(L.Granularity.FGQ, L.TensorFormat.FP6_E3M2, b), bias_shift=True)
        assert np.array_equal(q.scales.view(np.uint16), g[f"f/{name}/scales"]), name
        assert np.array_equal(q.folded_scales.view(np.uint16), g[f"f/{name}/folded"]), name
        assert np.array_equal(q.payload.seg4, g[f"f/{name}/seg4"]), name
        assert np.array_equal(q.payload.seg_tail, g[f"f/{name}/seg2"]), name
        for path in ("naive", "bias_shift"):
            assert np.array_equal(L.dequantize_tensor(q, path), g[f"f/{name}/deq"]), (name, path)
        if b % 128 == 0 or b >= W.shape[1]:
            Y = L.gemm_quantized(q, g[f"f/{name}/X"])
            assert normwise_rel(Y, g[f"f/{name}/Y"]) <= REL_TOL, name


@pytest.mark.parametrize("dt", ["f16", "bf16", "f32"])
@pytest.mark.parametrize("n,k,block", [(300, 1000, 128), (256, 4096, 256), (130, 640, 384), (129, 777, 40)])
def test_fgq_quantize_tiles_equals_prepacked_planes(dt, n, k, block):
    gen = torch.Generator().manual_seed(n + k + block)
    Wt = (torch.randn((n, k), generator=gen, dtype=torch.float64) * 0.05).to(_TORCH_DT[dt]).cuda()
    scheme = L.QuantScheme(L.Granularity.FGQ, L.TensorFormat.FP6_E3M2, block)
    q = L.quantize_tensor(Wt, scheme, bias_shift=True)
    fused = L.Fp6Weight.quantize(Wt, block=block)
    ref = L.Fp6Weight.from_planes(q.payload.seg4, q.payload.seg_tail, q.scales, n, k, q.folded_scales, block=block)
    assert torch.equal(fused.tiles, ref.tiles)
    assert torch.equal(fused.scales.view(torch.int16), q.scales.view(torch.int16))
    o = O.quantize_tensor_fgq(Wt.double().cpu().numpy(), block, bias_shift=True)
    assert np.array_equal(q.scales.cpu().numpy().view(np.uint16), o["scales"].view(np.uint16))
    assert np.array_equal(q.payload.seg4.cpu().numpy(), o["seg4"])


@pytest.mark.parametrize("m", [1, 16, 33, 300])
@pytest.mark.parametrize("n,k,block", [(512, 1024, 128), (1000, 4096, 512), (384, 1000, 256), (4096, 4096, 128)])
def test_fgq_gemm_vs_oracle(n, k, block, m):
    """Block scales applied to the rebuilt binary16 weights before the MMA:
    within the fp32 tolerance of the reference's block-partial GEMM
    (gemm.py:96-110) on the same fp16 activations, for every batch-tile
    width (BN 16 / 32 / 64 / 192) and ragged last blocks."""
    gen = torch.Generator(device="cuda").manual_seed(n * 7 + k + m)
    W = (torch.randn(n, k, generator=gen, device="cuda") * 0.02).half()
    w = L.Fp6Weight.quantize(W, block=block)
    x = torch.randn(m, k, generator=gen, device="cuda").half()
    y = L.w6a16_linear(x, w, out_dtype=torch.float32)
    codes = w.codes().cpu().numpy()
    Yo = O.gemm_quantized_fgq(codes.ravel(), w.scales.cpu().numpy(), n, k, block, x.t().float().cpu().numpy())
    assert normwise_rel(y.t().cpu().numpy(), Yo) <= REL_TOL
    y2 = L.w6a16_linear(x, w, out_dtype=torch.float32, sched="streamk", split_k=3)
    assert normwise_rel(y2.cpu().numpy(), y.cpu().numpy()) <= 1e-5


@pytest.mark.parametrize("m", [1, 16, 32, 33, 300])
@pytest.mark.parametrize("n,k,block", [(512, 2048, 128), (384, 4096, 256), (1024, 8192, 128)])
def test_fgq_block_magnitudes_1e6_to_1_per_row(n, k, block, m):
    """block magnitudes spanning 1e-6 .. 1 inside every row.
    Decode widths (M <= 32) scale each 128-k partial in fp32 (the reference's
    FGQ order, gemm.py:96-110); wider batches rebuild v * S'_b in binary16 with
    the row's power-of-two factor applied in fp32 (no binary16 underflow).
    Checked ELEMENTWISE per row against the oracle's block-partial GEMM on the
    same fp16 activations: |y - y_ref| <= 1e-3 * max_row |y_ref| for every
    row, and within the reference's own f32 bound (gemm.py:118-122, with the
    2^-11 binary16-rebuild term for M > 32) of the f64 product of the
    oracle's W_hat."""
    rng = np.random.default_rng(n + k + block + m)
    nb = -(-k // block)
    mag = 10.0 ** rng.uniform(-6, 0, size=(n, nb))
    Wn = rng.standard_normal((n, k)) * np.repeat(mag, block, axis=1)[:, :k]
    W = torch.from_numpy(Wn.astype(np.float32)).cuda()
    w = L.Fp6Weight.quantize(W, block=block)
    o = O.quantize_tensor_fgq(Wn.astype(np.float32), block, True)
    codes = w.codes().cpu().numpy()
    assert np.array_equal(codes.ravel(), o["codes"]) and np.array_equal(
        w.scales.cpu().numpy().view(np.uint16), o["scales"].view(np.uint16))
    x = torch.randn(m, k, device="cuda", generator=torch.Generator(device="cuda").manual_seed(m)).half()
    X = x.t().float().cpu().numpy()
    y = L.w6a16_linear(x, w, out_dtype=torch.float32).t().cpu().numpy().astype(np.float64)
    Yo = O.gemm_quantized_fgq(o["codes"], o["scales"], n, k, block, X).astype(np.float64)
    row_max = np.maximum(np.abs(Yo).max(axis=1, keepdims=True), 1e-30)
    assert np.all(np.abs(y - Yo) <= 1e-3 * row_max)
    W_hat = O.value_table()[o["codes"].reshape(n, k)] * O.block_scale_per_element(o["scales"], n, k, block)
    Yf64 = W_hat @ X.astype(np.float64)
    extra = 2.0 ** -11 if m > 32 else 0.0
    tol = (4 * np.finfo(np.float32).eps + extra) * k * np.abs(W_hat).max(axis=1, keepdims=True) * np.abs(X).max()
    assert np.all(np.abs(y - Yf64) <= tol)


# ---------------------------------------------------------------- FP5 e3m1 (4 + 1)
FP5_GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_fp5.npz")


def test_fp5_codec_pack_dequant_vs_reference():
    g = np.load(FP5_GOLD)
    F5 = L.FP5_E3M1
    assert np.array_equal(L.encode_rtn_array(F5, g["enc/x"]), g["enc/codes"])
    for n in g["p_lens"]:
        seg = L.pack(F5, g[f"p/{n}/codes"])
        assert np.array_equal(seg.seg4, g[f"p/{n}/seg4"]) and np.array_equal(seg.seg_tail, g[f"p/{n}/seg1"]), n
        assert np.array_equal(L.unpack(F5, seg), g[f"p/{n}/codes"]), n
    s = g["dq/scales"].view(np.float16)
    codes = np.arange(32, dtype=np.uint8)
    f = L.fold_scale_array(F5, s)
    assert np.array_equal(L.dequant_bias_shift_array(F5, codes[:, None], f[None, :]).view(np.uint16), g["dq/bias"])
    assert np.array_equal(L.dequant_naive_array(F5, codes[:, None], s[None, :]).view(np.uint16), g["dq/naive"])


def test_fp5_quantize_dequantize_gemm_container_vs_reference():
    """FP5 CGQ / FGQ quantize on the GPU == the reference's scales, folded
    scales, 4 + 1 planes and .lpqt bytes; dequantize exact; the GEMM (through
    the FP6 tile layout) within the normwise bar of the reference's GEMM."""
    g = np.load(FP5_GOLD)
    for name in [str(s) for s in g["q_names"]]:
        W, b = g[f"q/{name}/W"], int(g[f"q/{name}/block"])
        gran = L.Granularity.FGQ if b else L.Granularity.CGQ
        q = L.quantize_tensor(W, L.QuantScheme(gran, L.TensorFormat.FP5_E3M1, b), bias_shift=True)
        assert np.array_equal(q.scales.view(np.uint16), g[f"q/{name}/scales"]), name
        assert np.array_equal(q.folded_scales.view(np.uint16), g[f"q/{name}/folded"]), name
        assert np.array_equal(q.payload.seg4, g[f"q/{name}/seg4"]), name
        assert np.array_equal(q.payload.seg_tail, g[f"q/{name}/seg1"]), name
        assert L.write_lpqt(q) == g[f"q/{name}/container"].tobytes(), name
        for path in ("naive", "bias_shift"):
            assert np.array_equal(L.dequantize_tensor(q, path), g[f"q/{name}/deq"]), (name, path)
        if b == 0 or b % 128 == 0:
            Y = L.gemm_quantized(q, g[f"q/{name}/X"])
            assert normwise_rel(Y, g[f"q/{name}/Y"]) <= REL_TOL, name
            w = L.load_lpqt(g[f"q/{name}/container"].tobytes())
            y = L.w6a16_linear(torch.from_numpy(g[f"q/{name}/X"].T.copy()).cuda().half(), w, out_dtype=torch.float32)
            assert normwise_rel(y.t().cpu().numpy(), g[f"q/{name}/Y"]) <= REL_TOL, name


@pytest.mark.parametrize("n,k,m", [(512, 1024, 16), (1000, 4096, 300), (4096, 4096, 1)])
def test_fp5_gemm_vs_oracle_large(n, k, m):
    rng = np.random.default_rng(n + k + m)
    W = (rng.standard_normal((n, k)) * 0.02).astype(np.float16)
    X = rng.standard_normal((k, m)).astype(np.float16)
    q = L.quantize_tensor(W, L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP5_E3M1), bias_shift=True)
    o = O.quantize_tensor_fp5(W, True)
    assert np.array_equal(q.payload.seg4, o["seg4"]) and np.array_equal(q.payload.seg_tail, o["seg1"])
    Y = L.gemm_quantized(q, X)
    What = O.fp5_value_table()[o["codes"].reshape(n, k)] * o["scales"].astype(np.float64)[:, None]
    assert normwise_rel(Y, What @ X.astype(np.float64)) <= REL_TOL


# ---------------------------------------------------------------- INT4 comparator
INT4_GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_int4.npz")


def test_int4_quantize_pack_dequant_gemm_vs_reference():
    """INT4 asymmetric CGQ / FGQ (any block size) on the GPU == the
    reference's zero points, scales, nibbles, container bytes and f64
    dequant; the comparator GEMM within the normwise bar."""
    g = np.load(INT4_GOLD)
    assert np.array_equal(L.pack_int4(g["p/levels"]), g["p/nibbles"])
    assert np.array_equal(L.unpack_int4(g["p/nibbles"], g["p/levels"].size), g["p/levels"])
    with pytest.raises(L.InvalidCode):
        L.pack_int4([3, 16])
    for name in [str(s) for s in g["q_names"]]:
        W, b = g[f"q/{name}/W"], int(g[f"q/{name}/block"])
        gran = L.Granularity.FGQ if b else L.Granularity.CGQ
        q = L.quantize_tensor(W, L.QuantScheme(gran, L.TensorFormat.INT4_ASYM, b))
        assert np.array_equal(q.scales.view(np.uint16), g[f"q/{name}/scales"]), name
        assert np.array_equal(q.zero_points.view(np.uint16), g[f"q/{name}/zeros"]), name
        assert np.array_equal(q.payload, g[f"q/{name}/nibbles"]), name
        assert L.write_lpqt(q) == g[f"q/{name}/container"].tobytes(), name
        assert np.array_equal(L.dequantize_tensor(q), g[f"q/{name}/deq"]), name
        assert normwise_rel(L.gemm_quantized(q, g[f"q/{name}/X"]), g[f"q/{name}/Y"]) <= REL_TOL, name
    with pytest.raises(L.InvalidScheme):
        L.quantize_tensor(np.ones((2, 4)), L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.INT4_ASYM), bias_shift=True)


@pytest.mark.parametrize("n,k,m,block", [(128, 128, 1, 0), (1000, 3000, 16, 0), (4096, 4096, 16, 128),
                                         (4224, 1024, 96, 256), (640, 8192, 300, 0), (2048, 2048, 2, 512)])
def test_w4a16_gemm_vs_oracle(n, k, m, block):
    """Fused W4A16 tcgen05 GEMM (INT4 tiles, per-row / per-128k-block zero
    points and scales): within the normwise bar of the reference f64 product,
    and within 1e-5 of the f64 product of its own binary16 rebuild; ragged
    N / K, every BN bucket; bit-identical on relaunch."""
    rng = np.random.default_rng(n * 7 + k + m + block)
    W = (rng.standard_normal((n, k)) * 0.02 + rng.standard_normal((n, 1)) * 0.01).astype(np.float32)
    X = rng.standard_normal((k, m)).astype(np.float16)
    gran = L.Granularity.FGQ if block else L.Granularity.CGQ
    q = L.quantize_tensor(W, L.QuantScheme(gran, L.TensorFormat.INT4_ASYM, block))
    o = O.quantize_tensor_int4(W, block)
    assert np.array_equal(q.payload, o["nibbles"]) and np.array_equal(q.scales.view(np.uint16),
                                                                        o["scales"].view(np.uint16))
    Y = L.gemm_quantized(q, X, exact=False)       # force the W4A16 kernel (auto: reference-order kernel)
    assert np.array_equal(Y, L.gemm_quantized(q, X, exact=False))
    deq = O.dequantize_int4(o["levels"], o["scales"], o["zeros"], n, k, block)
    assert normwise_rel(Y, deq @ X.astype(np.float64)) <= REL_TOL
    # the kernel's binary16 weight RN_f16(Z + S * level): one rounding (HFMA2) of the exact f64 value
    W16 = deq.astype(np.float16).astype(np.float64)
    assert normwise_rel(Y, W16 @ X.astype(np.float64)) <= 1e-5
    # torch-facing call with fp16 output through the same weight
    w = L.Int4Weight.from_quantized(q)
    y = L.w6a16_linear(torch.from_numpy(X.T.copy()).cuda(), w, out_dtype=torch.float32)
    assert torch.equal(y.t().cpu(), torch.from_numpy(Y))


@pytest.mark.parametrize("sched,split_k", [("streamk", 0), ("streamk", 3), ("cluster", 1), ("cluster", 2),
                                           ("cluster", 3), ("cluster", 4)])
@pytest.mark.parametrize("fmt", ["fp6_fgq", "int4_cgq", "int4_fgq"])
def test_block_params_every_schedule(fmt, sched, split_k):
    """Stage-ordered block parameters (FGQ scales, INT4 scale | zero) under
    stream-K and cluster split-K, ragged K (odd k-tile counts split unevenly
    over the cluster ranks): within 1e-5 of the f64 product of the weights
    the kernel multiplies — the exact v * S_b for FGQ FP6 at decode widths
    (block scales applied to fp32 per-tile partials), the binary16 rebuild
    otherwise — and deterministic."""
    n, k = 1000, 3000 if fmt != "fp6_fgq" else 3072
    rng = np.random.default_rng(hash((fmt, sched, split_k)) % 2**32)
    W = (rng.standard_normal((n, k)) * 0.02).astype(np.float16)
    for m in (1, 16, 24):
        x = torch.from_numpy(rng.standard_normal((m, k)).astype(np.float16)).cuda()
        if fmt == "fp6_fgq":
            w = L.Fp6Weight.quantize(torch.from_numpy(W).cuda(), block=256)
            q = L.quantize_tensor(torch.from_numpy(W).cuda(), L.QuantScheme(L.Granularity.FGQ,
                                                                           L.TensorFormat.FP6_E3M2, 256))
            Wh = L.dequantize_tensor(q) if m <= 32 else w.dequantize_f16().double()
        else:
            block = 256 if fmt == "int4_fgq" else 0
            gran = L.Granularity.FGQ if block else L.Granularity.CGQ
            q = L.quantize_tensor(W, L.QuantScheme(gran, L.TensorFormat.INT4_ASYM, block))
            w = L.Int4Weight.from_quantized(q)
            Wh = torch.from_numpy(np.asarray(L.dequantize_tensor(q)).astype(np.float16).astype(np.float64)).cuda()
        y = L.w6a16_linear(x, w, out_dtype=torch.float32, split_k=split_k, sched=sched)
        assert torch.equal(y, L.w6a16_linear(x, w, out_dtype=torch.float32, split_k=split_k, sched=sched))
        ref = x.double() @ Wh.t()
        assert normwise_rel(y.cpu().numpy(), ref.cpu().numpy()) <= 1e-5, (m, fmt, sched, split_k)


def test_random_shape_fuzz():
    """Seeded fuzz over shapes / batch / scheme: every launch within the
    normwise bar of the f64 product of the kernel's own binary16 weights,
    bit-identical on relaunch (whatever path the timing picks)."""
    rng = np.random.default_rng(20261017)
    for _ in range(int(os.environ.get("LPQT_FUZZ_ITERS", "40"))):
        n = int(rng.choice([128, 256, 384, 640, 1000, 2048, 4224]))
        k = int(rng.choice([128, 256, 520, 1024, 3000, 4096, 8192]))
        m = int(rng.choice([1, 2, 5, 16, 17, 31, 32, 40, 64, 96, 128, 129, 200, 300]))
        block = int(rng.choice([0, 0, 128, 256])) if k > 256 else 0
        w = L.Fp6Weight.quantize((torch.randn(n, k, device="cuda") * 0.02).half(), block=block)
        x = torch.randn(m, k, device="cuda").half()
        y = L.w6a16_linear(x, w, out_dtype=torch.float32)
        assert torch.equal(y, L.w6a16_linear(x, w, out_dtype=torch.float32)), (n, k, m, block)
        ref = x.double() @ w.dequantize_f16().double().t()
        assert normwise_rel(y.cpu().numpy(), ref.cpu().numpy()) <= REL_TOL, (n, k, m, block)


@pytest.mark.parametrize("m", [1, 8, 16, 32])
@pytest.mark.parametrize("n,k,block", [(512, 1024, 64), (384, 1000, 32), (256, 2048, 16), (1024, 4096, 64)])
def test_fgq_sub_tile_blocks_vs_oracle(n, k, block, m):
    """FGQ blocks narrower than a 128-k tile (16 / 32 / 64 columns) at decode
    widths: one tensor-core partial per block, scaled by the block's raw f16
    scale in fp32 and summed in k order (the reference's FGQ loop,
    gemm.py:96-110).  Block magnitudes 1e-6 .. 1 inside every row; checked
    elementwise per row against the oracle's block-partial GEMM on the same
    fp16 activations, and bit-identical across stream-K / cluster schedules
    is not required (fp32 summation order) but within 1e-5 normwise."""
    rng = np.random.default_rng(n + k + block + m)
    nb = -(-k // block)
    mag = 10.0 ** rng.uniform(-6, 0, size=(n, nb))
    Wn = rng.standard_normal((n, k)) * np.repeat(mag, block, axis=1)[:, :k]
    w = L.Fp6Weight.quantize(torch.from_numpy(Wn.astype(np.float32)).cuda(), block=block)
    o = O.quantize_tensor_fgq(Wn.astype(np.float32), block, True)
    assert np.array_equal(w.codes().cpu().numpy().ravel(), o["codes"])
    x = torch.randn(m, k, device="cuda", generator=torch.Generator(device="cuda").manual_seed(m)).half()
    X = x.t().float().cpu().numpy()
    Yo = O.gemm_quantized_fgq(o["codes"], o["scales"], n, k, block, X).astype(np.float64)
    # the reference's own f32 bound (gemm.py:118-122) per row: 4 eps32 K max_row|W_hat| max|X|
    W_hat = O.value_table()[o["codes"].reshape(n, k)] * O.block_scale_per_element(o["scales"], n, k, block)
    tol = 4 * np.finfo(np.float32).eps * k * np.abs(W_hat).max(axis=1, keepdims=True) * np.abs(X).max()
    for sched in ("auto", "streamk", "cluster"):
        y = L.w6a16_linear(x, w, out_dtype=torch.float32, sched=sched).t().cpu().numpy().astype(np.float64)
        assert np.all(np.abs(y - Yo) <= tol), sched
    with pytest.raises(L.InvalidScheme):   # prefill widths keep whole-tile blocks
        L.w6a16_linear(torch.zeros(33, k, device="cuda").half(), w)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_division_free_encode_exhaustive(dtype):
    """The quantizer's division-free RTN quotient (RN(1/S) once per row, then
    q0 = RN(a Y), R = a - S q0, q = RN(q0 + R Y)) gives the same e3m2 code as
    the __fdiv_rn quotient (the path pinned to the reference's golden vectors)
    for EVERY positive finite binary16 scale and every positive finite
    binary16 / bfloat16 weight with |w| <= 29 S (the quantizer's whole domain:
    |w| <= peak <= 28 S (1 + 2^-11)); for binary16 weights even the f32
    quotients are identical."""
    import ctypes
    from paper_2312_08583_b200 import _lib
    out = (ctypes.c_ulonglong * 3)()
    code = _lib.F16 if dtype == "f16" else _lib.BF16
    _lib.check(_lib.load().lpqt_selftest_fp6_encode(code, out), "selftest")
    bad_codes, bad_quot, pairs = out[0], out[1], out[2]
    assert pairs > 10 ** 8
    assert bad_codes == 0, (bad_codes, bad_quot, pairs)
    if dtype == "f16":   # (bf16 weights: 0.26 % of the quotients differ by an ulp, never across a code boundary)
        assert bad_quot == 0, (bad_codes, bad_quot, pairs)


def test_w4a16_schedule_flags():
    """The W4A16 comparator runs the single-SM kernel only: sched="single" is
    the automatic path, sched="pair" is refused (no CTA-pair W4A16 kernel)."""
    g = torch.Generator(device="cuda").manual_seed(41)
    W = (torch.randn(512, 1024, generator=g, device="cuda") * 0.02).half()
    q = L.quantize_tensor(W, L.QuantScheme(L.Granularity.FGQ, L.TensorFormat.INT4_ASYM, 128))
    w = L.Int4Weight.from_quantized(q)
    for m in (7, 200):
        x = torch.randn(m, 1024, generator=g, device="cuda").half()
        assert torch.equal(L.w6a16_linear(x, w, out_dtype=torch.float32, sched="single"),
                           L.w6a16_linear(x, w, out_dtype=torch.float32))
        with pytest.raises(L.InvalidInput):
            L.w6a16_linear(x, w, sched="pair")
