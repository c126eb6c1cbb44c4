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
