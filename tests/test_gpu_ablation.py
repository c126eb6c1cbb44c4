"""The paper's Bias-Shift ablation kernels ("the same FP6
kernel without Bias-Shift"): the decode GEMM with the software bias-shift
rebuild x folded scale (dequant.py:33-43, 82-86) and with the naive two-step
cast x S (dequant.py:72-79), both applying the per-weight binary16 scale of
the reference's dequant paths.  Checked against the oracle's binary16
dequant (dequant_naive_array / dequant_bias_shift_array) times X in f64,
against each other (bit-identical, tests/test_dequant.py:93-102 of the
reference) and against the product kernel (hardware e3m2 rebuild, fp32 scale)."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2312_08583_b200 as L  # noqa: E402
from oracle import lpqt_oracle as O  # noqa: E402  (checker only)


def _rel(a, b):
    return float((a.double() - b.double()).abs().max() / b.double().abs().max())


@pytest.mark.parametrize("n,k,m", [(256, 512, 8), (384, 1000, 3), (640, 2048, 16)])
def test_ablation_rebuilds_vs_oracle_dequant(n, k, m):
    rng = np.random.default_rng(n + k + m)
    W = (rng.standard_normal((n, k)) * 0.02).astype(np.float16)
    W[0, :8] = [0, -0.0, 1e-7, -1e-7, 3e-6, 0.0625, -0.5, 1.0]   # zero / subnormal / normal codes
    o = O.quantize_tensor(W, bias_shift=True)
    w16 = O.dequant_naive_array(o["codes"], np.repeat(o["scales"], k)).reshape(n, k)
    assert np.array_equal(w16.view(np.uint16),
                          O.dequant_bias_shift_array(o["codes"], np.repeat(o["folded"], k)).reshape(n, k).view(np.uint16))
    x = torch.from_numpy(rng.standard_normal((m, k)).astype(np.float16)).cuda()
    ref = x.double() @ torch.from_numpy(w16.astype(np.float64)).cuda().t()
    w = L.Fp6Weight.quantize(torch.from_numpy(W).cuda())
    ys = {rb: L.w6a16_linear(x, w, out_dtype=torch.float32, rebuild=rb) for rb in ("cvt", "bias_shift", "naive")}
    assert torch.equal(ys["bias_shift"], ys["naive"])
    assert _rel(ys["naive"], ref) <= 1e-6          # fp32 summation order only
    assert _rel(ys["cvt"], ref) <= 1e-3            # the product path scales in fp32 (no binary16 rounding of V*S)


@pytest.mark.parametrize("n,k", [(5504, 2048), (2048, 5504), (13824, 5120), (8192, 22016)])
@pytest.mark.parametrize("sched", ["auto", "streamk", "cluster"])
def test_ablation_paper_presets(n, k, sched):
    """The paper's FFN presets at its batch 8, every decode schedule."""
    g = torch.Generator(device="cuda").manual_seed(n + k)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    x = torch.randn(8, k, generator=g, device="cuda").half()
    w = L.Fp6Weight.quantize(W)
    ref = x.double() @ w.dequantize_f16().double().t()
    yb = L.w6a16_linear(x, w, out_dtype=torch.float32, sched=sched, rebuild="bias_shift")
    yn = L.w6a16_linear(x, w, out_dtype=torch.float32, sched=sched, rebuild="naive")
    assert torch.equal(yb, yn)
    assert _rel(yn, ref) <= 4e-7 * k ** 0.5    # fp32 summation order (normwise)


def test_ablation_outside_decode_is_refused():
    w = L.Fp6Weight.quantize((torch.randn(256, 512, device="cuda") * 0.02).half())
    with pytest.raises(L.LpqtError):
        L.w6a16_linear(torch.randn(17, 512, device="cuda").half(), w, rebuild="naive")
    with pytest.raises(ValueError):
        L.w6a16_linear(torch.randn(4, 512, device="cuda").half(), w, rebuild="other")
