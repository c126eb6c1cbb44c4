"""The CTA-pair prefill kernel (prefill2sm.cu: tcgen05 cta_group::2, M = 256 x
N = 256 MMAs, A rebuilt in each SM's TMEM, X split between the pair):
against the dequantize-then-matmul f64 product of the same weights (normwise
bar), against the single-SM kernel (fp32 summation-order differences only),
every output layout / dtype, ragged K / M / N, deterministic, and the
fallback for an odd number of 128-row tiles."""

from __future__ import annotations

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2312_08583_b200 as L  # noqa: E402

CGQ = L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP6_E3M2)


def _rel(a, b):
    return float((a.double() - b.double()).abs().max() / b.double().abs().max())


@pytest.mark.parametrize("n,k,m", [(512, 1024, 300), (1024, 3000, 129), (2048, 4096, 512), (256, 640, 1000),
                                   (8192, 8192, 2048), (1024, 8192, 4100)])
def test_pair_kernel_vs_reference_and_single_sm(n, k, m):
    g = torch.Generator(device="cuda").manual_seed(n + k + m)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    x = torch.randn(m, k, generator=g, device="cuda").half()
    w = L.Fp6Weight.quantize(W)
    q = L.quantize_tensor(W, CGQ, bias_shift=True)
    ref = x.double() @ L.dequantize_tensor(q).t()
    y2 = L.w6a16_linear(x, w, out_dtype=torch.float32, sched="pair")
    y1 = L.w6a16_linear(x, w, out_dtype=torch.float32, sched="single")
    assert _rel(y2, ref) <= 1e-3
    assert _rel(y2, y1) <= 1e-5
    assert torch.equal(y2, L.w6a16_linear(x, w, out_dtype=torch.float32, sched="pair"))


@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16, torch.float32])
def test_pair_kernel_layouts_and_dtypes(dt):
    n, k, m = 1024, 2048, 700
    W = (torch.randn(n, k, device="cuda") * 0.02).half()
    X = torch.randn(k, m, device="cuda").half()
    w = L.Fp6Weight.quantize(W)
    y_mn = L.w6a16_linear(X.t().contiguous(), w, out_dtype=dt, sched="pair")
    y_ref = L.w6a16_linear(X.t().contiguous(), w, out_dtype=torch.float32, sched="single")
    assert _rel(y_mn.float(), y_ref) <= (1e-5 if dt == torch.float32 else 1e-2)
    # reference layout Y[N, M] (gemm_quantized) takes the pair kernel automatically at this size
    assert L.plan(m, n, k, sched="pair")["schedule"] == "pair"
    Y = L.gemm_quantized(L.quantize_tensor(W, CGQ), X)
    assert _rel(Y, y_ref.t()) <= 1e-5


@pytest.mark.parametrize("dt", [torch.float16, torch.float32])
@pytest.mark.parametrize("m", [512, 777])
def test_pair_kernel_reference_layout(dt, m):
    """Y[N, M] (the reference layout, gemm_nm): the TMA-store epilogue when the
    row stride allows it (m = 512), element stores otherwise (m = 777)."""
    from paper_2312_08583_b200.linear import gemm_nm, _launch
    from paper_2312_08583_b200 import _lib
    n, k = 2048, 4096
    W = (torch.randn(n, k, device="cuda") * 0.02).half()
    x = torch.randn(m, k, device="cuda").half()
    w = L.Fp6Weight.quantize(W)
    ref = L.w6a16_linear(x, w, out_dtype=torch.float32, sched="single").t()
    y = torch.empty(n, m, dtype=dt, device="cuda")
    _launch(w, x, k, m, y, _lib.F32 if dt == torch.float32 else _lib.F16, _lib.Y_NM, m, 0, "pair")
    assert _rel(y.float(), ref) <= (1e-5 if dt == torch.float32 else 1e-2)


def test_odd_tile_count_falls_back():
    n, k, m = 1100, 1024, 600          # 9 row tiles: no pairs
    W = (torch.randn(n, k, device="cuda") * 0.02).half()
    x = torch.randn(m, k, device="cuda").half()
    w = L.Fp6Weight.quantize(W)
    assert L.plan(m, n, k, sched="pair")["schedule"] != "pair"
    y = L.w6a16_linear(x, w, out_dtype=torch.float32, sched="pair")
    assert _rel(y, L.w6a16_linear(x, w, out_dtype=torch.float32, sched="single")) <= 1e-5


@pytest.mark.parametrize("n,k,m,force", [(2048, 8192, 512, 0), (10240, 8192, 512, 0), (1024, 8192, 300, 0),
                                         (1024, 4096, 1000, 0), (8192, 4096, 1280, 2), (2048, 4096, 8192, 2),
                                         (2048, 4096, 8192, 1), (1024, 4096, 600, 2)])
def test_pair_stream_k(n, k, m, force):
    """Whole rounds + a stream-K wave over the pairs (units cut between pairs,
    partials reduced by the unit's head pair in k order), whole units only
    (force 1), grouped rasterization at M x K x 2 > 40 MB: against the f64
    product of the same dequantized weights, the single-SM kernel, and
    bit-identical on repeat.  force: 0 = the planner's choice (stream-K at
    these shapes), 1 / 2 = split_k hook forcing whole units / stream-K."""
    plan = L.plan(m, n, k, split_k=force, sched="pair")
    assert plan["schedule"] == "pair" and plan["splits"] == (1 if force == 1 else 2), plan
    g = torch.Generator(device="cuda").manual_seed(n + k + m)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    x = torch.randn(m, k, generator=g, device="cuda").half()
    w = L.Fp6Weight.quantize(W)
    ref = x.double() @ w.dequantize_f16().double().t()
    run = lambda dt: L.w6a16_linear(x, w, out_dtype=dt, sched="pair", split_k=force)
    y2 = run(torch.float32)
    y1 = L.w6a16_linear(x, w, out_dtype=torch.float32, sched="single")
    assert _rel(y2, ref) <= 1e-3
    assert _rel(y2, y1) <= 3e-5   # (a unit may be cut over several pairs: more partial sums)
    for _ in range(3):
        assert torch.equal(y2, run(torch.float32))
    assert _rel(run(torch.float16).float(), y1) <= 1e-2
    if force == 0:  # the reference layout Y[N, M] through the same schedule
        Y = L.gemm_quantized(L.quantize_tensor(W, CGQ), x.t().contiguous())
        assert _rel(Y, y1.t()) <= 3e-5
