"""Stream-K tiles cut into many contributors: the reducer stages the other
contributors' fp32 partials in its drained weight ring (one bulk copy each)
while they fit, else reads them from L2.  Forced splits walk every batch-tile
width (BN 16 / 32 / 64) across the ring's capacity, where an off-by-one once
wrote one partial past the ring (5120 x 13824 at M = 33: 4 others x 32 KB in a
144 KB ring); each result against the f64 product of the same weights'
binary16 dequant (1e-3 normwise, the fuzz suite's bar) and bit-identical on
repeat."""

from __future__ import annotations

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2312_08583_b200 as L  # noqa: E402

_W = {}


def _weight(n, k):
    if (n, k) not in _W:
        g = torch.Generator(device="cuda").manual_seed(n + 7 * k)
        W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
        w = L.Fp6Weight.quantize(W)
        _W[(n, k)] = (w, w.dequantize_f16().double())
    return _W[(n, k)]


def _check(n, k, m, split_k=0):
    w, wd = _weight(n, k)
    g = torch.Generator(device="cuda").manual_seed(m + 31 * split_k)
    x = torch.randn(m, k, generator=g, device="cuda").half()
    y = L.w6a16_linear(x, w, out_dtype=torch.float32, split_k=split_k, sched="streamk")
    torch.cuda.synchronize()
    ref = x.double() @ wd.t()
    err = float((y.double() - ref).abs().max() / ref.abs().max())
    assert err <= 1e-3, (err, L.plan(m, n, k, split_k, sched="streamk"))
    assert torch.equal(y, L.w6a16_linear(x, w, out_dtype=torch.float32, split_k=split_k, sched="streamk"))


@pytest.mark.parametrize("m", [16, 32, 33, 64])
@pytest.mark.parametrize("split_k", [3, 4, 5, 6, 7, 8, 10, 12])
def test_forced_splits_across_ring_capacity(m, split_k):
    _check(1024, 8192, m, split_k)


@pytest.mark.parametrize("n,k,m", [(5120, 13824, 33), (5120, 13824, 64), (1024, 28672, 48),
                                   (1280, 8192, 40), (2560, 8192, 32), (3072, 8192, 24)])
def test_auto_plans_with_many_contributors(n, k, m):
    _check(n, k, m)


@pytest.mark.parametrize("block", [128, 32])
@pytest.mark.parametrize("n,k", [(1536, 13900), (1536, 28000), (3000, 28000), (1000, 11000)])
@pytest.mark.parametrize("m", [1, 16, 32])
def test_fgq_partials_over_ragged_stages(n, k, m, block):
    """FGQ at decode widths (one fp32 partial per block in a TMEM slot ring):
    an odd k-tile count leaves each tile's last two-tile stage ragged; the
    missing tile's partial ordinals must still pass through their slots, or a
    later parity wait aliases an old phase (1536 x 13900 once read stale
    partials: 0.1 normwise).  Against the f64 product of the exact v * S_b."""
    g = torch.Generator(device="cuda").manual_seed(n + k + block)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    w = L.Fp6Weight.quantize(W, block=block)
    q = L.quantize_tensor(W, L.QuantScheme(L.Granularity.FGQ, L.TensorFormat.FP6_E3M2, block))
    d = L.dequantize_tensor(q)
    wd = (d if torch.is_tensor(d) else torch.from_numpy(d)).cuda().double()
    x = torch.randn(m, k, generator=g, device="cuda").half()
    y = L.w6a16_linear(x, w, out_dtype=torch.float32)
    ref = x.double() @ wd.t()
    err = float((y.double() - ref).abs().max() / ref.abs().max())
    assert err <= 1e-5, (err, L.plan(m, n, k))
    assert torch.equal(y, L.w6a16_linear(x, w, out_dtype=torch.float32))
