"""FP5 e3m1 in its own 4+1 tile layout (0.625 B per weight; common.cuh
fp5x32_*, prepack.cu lpqt_fp5n_*; the reference's 4+1 split,
packing.py:84-85): the tiles hold the oracle's codes, the rebuild gives the
oracle's binary16 dequant bit for bit, and the GEMM on native tiles equals the
GEMM on the FP6-widened tiles of the same weights (identical MMA operands)
bit for bit, for every schedule."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2312_08583_b200 as L  # noqa: E402
from paper_2312_08583_b200.linear import prepack  # noqa: E402
from oracle import lpqt_oracle as O  # noqa: E402  (checker only)

CGQ5 = L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP5_E3M1)


def _weights(n, k, seed):
    rng = np.random.default_rng(seed)
    W = (rng.standard_normal((n, k)) * 0.02).astype(np.float16)
    q = L.quantize_tensor(W, CGQ5, bias_shift=True)
    o = O.quantize_tensor_fp5(W, True)
    w5 = L.Fp6Weight.from_quantized(q)
    s4 = torch.from_numpy(np.asarray(q.payload.seg4)).cuda()
    s1 = torch.from_numpy(np.asarray(q.payload.seg_tail)).cuda()
    sc = torch.from_numpy(np.asarray(q.scales)).cuda()
    w6 = L.Fp6Weight(prepack(s4, s1, n, k, "fp5"), sc, n, k, static=True)   # FP6-widened tiles
    return W, q, o, w5, w6


@pytest.mark.parametrize("n,k", [(256, 512), (300, 1000), (1024, 4096)])
def test_native_fp5_tiles_codes_and_dequant(n, k):
    W, q, o, w5, w6 = _weights(n, k, n + k)
    assert w5.wbits == 5 and w6.wbits == 6
    assert w5.tiles.numel() == -(-n // 128) * -(-k // 128) * 10240
    assert np.array_equal(w5.codes().cpu().numpy().reshape(-1), o["codes"])
    deq = (O.fp5_value_table()[o["codes"]].reshape(n, k).astype(np.float16) *
           o["scales"][:, None]).astype(np.float16)
    assert np.array_equal(w5.dequantize_f16().cpu().numpy().view(np.uint16), deq.view(np.uint16))
    assert torch.equal(w5.dequantize_f16(), w6.dequantize_f16())
    assert w5.stream_bytes() < w6.stream_bytes() and abs(w5.stream_bytes() / (n * k) - 0.625) < 0.02


@pytest.mark.parametrize("m", [1, 8, 16, 32, 100, 300])
@pytest.mark.parametrize("sched", ["auto", "streamk", "cluster"])
def test_native_fp5_gemm_equals_widened(m, sched):
    n, k = 2048, 3072
    if sched == "cluster" and m > 32:
        pytest.skip("cluster split-K is a decode schedule")
    W, q, o, w5, w6 = _weights(n, k, 7 + m)
    x = torch.from_numpy(np.random.default_rng(m).standard_normal((m, k)).astype(np.float16)).cuda()
    s = sched if sched != "auto" or m < 65 else "single"   # (the widened tiles would take the pair kernel)
    y5 = L.w6a16_linear(x, w5, out_dtype=torch.float32, sched=s)
    y6 = L.w6a16_linear(x, w6, out_dtype=torch.float32, sched=s)
    assert torch.equal(y5, y6)
    ref = x.double() @ (torch.from_numpy(O.fp5_value_table()[o["codes"]].reshape(n, k)).cuda() *
                        torch.from_numpy(o["scales"].astype(np.float64)).cuda()[:, None]).t()
    assert float((y5.double() - ref).abs().max() / ref.abs().max()) <= 1e-3


def test_native_fp5_reference_api_and_container():
    n, k, m = 1024, 2048, 8
    W, q, o, w5, _ = _weights(n, k, 3)
    X = np.random.default_rng(1).standard_normal((k, m)).astype(np.float16)
    Y = L.gemm_quantized(q, X)    # through the cached native-FP5 weight
    What = O.fp5_value_table()[o["codes"].reshape(n, k)] * o["scales"].astype(np.float64)[:, None]
    ref = What @ X.astype(np.float64)
    assert np.max(np.abs(Y - ref)) / np.max(np.abs(ref)) <= 1e-3
    wl = L.load_lpqt(L.write_lpqt(q))
    assert wl.wbits == 5 and torch.equal(wl.tiles, w5.tiles)


@pytest.mark.parametrize("m", [65, 300, 700])
def test_native_fp5_pair_kernel_equals_widened(m):
    """Prefill on the CTA-pair kernel: native FP5 tiles rebuild the same MMA
    operands as the FP6-widened tiles, so Y is bit-identical (same schedule)."""
    n, k = 2048, 4096
    W, q, o, w5, w6 = _weights(n, k, 100 + m)
    assert L.plan(m, n, k)["schedule"] == "pair"
    x = torch.from_numpy(np.random.default_rng(m).standard_normal((m, k)).astype(np.float16)).cuda()
    y5 = L.w6a16_linear(x, w5, out_dtype=torch.float32)
    y6 = L.w6a16_linear(x, w6, out_dtype=torch.float32)
    assert torch.equal(y5, y6)
