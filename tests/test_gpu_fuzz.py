"""Seeded random shapes through every GEMM path the planner can pick (decode
stream-K / cluster split-K, single-SM prefill, CTA-pair whole units / stream-K
wave, FGQ whole-tile and sub-tile blocks, native FP5 tiles): each result
against the f64 product of the SAME weights' binary16 dequant (the oracle's
dequant is pinned separately), fp32 accumulation bar 1e-3 normwise, and
bit-identical on repeat (every schedule is deterministic)."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2312_08583_b200 as L  # noqa: E402

RNG = np.random.default_rng(20241017)
CASES = []
for i in range(96):
    n = int(RNG.choice([128, 256, 384, 1000, 1536, 2048, 4096, 5120]))
    k = int(RNG.choice([128, 256, 640, 1024, 2000, 3072, 4096]))
    m = int(RNG.choice([1, 3, 8, 16, 17, 32, 33, 64, 65, 100, 128, 200, 256, 300, 512, 700]))
    kind = ["cgq", "cgq", "fgq128", "fgq64", "fgq32", "fp5"][i % 6]
    sched = ["auto", "auto", "streamk", "cluster", "pair", "single"][int(RNG.integers(6))]
    CASES.append((n, k, m, kind, sched))


def _weight(W, kind, k):
    if kind == "cgq":
        return L.Fp6Weight.quantize(W)
    if kind.startswith("fgq"):
        b = int(kind[3:])
        return L.Fp6Weight.quantize(W, block=b) if b < k else L.Fp6Weight.quantize(W)
    q = L.quantize_tensor(W, L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP5_E3M1), bias_shift=True)
    return L.Fp6Weight.from_quantized(q)


@pytest.mark.parametrize("n,k,m,kind,sched", CASES)
def test_fuzz_paths(n, k, m, kind, sched):
    if sched == "cluster" and m > 32:
        sched = "auto"
    g = torch.Generator(device="cuda").manual_seed(n * 131 + k * 7 + m)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    x = torch.randn(m, k, generator=g, device="cuda").half()
    w = _weight(W, kind, k)
    sub = w.block and w.block % 128
    if sub and m > 32:
        with pytest.raises(L.InvalidScheme):
            L.w6a16_linear(x, w, out_dtype=torch.float32, sched=sched)
        return
    y = L.w6a16_linear(x, w, out_dtype=torch.float32, sched=sched)
    ref = x.double() @ w.dequantize_f16().double().t()
    err = float((y.double() - ref).abs().max() / ref.abs().max().clamp_min(1e-30))
    # binary16 rebuild of v * S'_b at prefill widths for FGQ: + 2^-11
    bar = 2e-3 if (w.block and m > 32) else 1e-3
    assert err <= bar, (err, L.plan(m, n, k, sched=sched))
    assert torch.equal(y, L.w6a16_linear(x, w, out_dtype=torch.float32, sched=sched))
