"""Parity at the BASELINE.json configurations, against the ORACLE's own
quantization (never the product's dequant).

* configs[0] end to end: 4096 x 4096, M = 1 — GPU quantize bit-exact with the
  oracle on the whole tensor, the W6A16 GEMM within the normwise bar of the
  oracle's gemm_quantized and within the reference's elementwise f32-vs-f64
  bound (gemm.py:118-122) of the f64 product of the oracle's W_hat.
* configs[1-4]: every LLaMA-2-7B / 13B, StarCoder-15B and LLaMA-2-70B layer
  shape, whole (P = 1) and as the last rank's column shard at TP = 2 / 4 / 8,
  at M = 1, 16 and 512 (decode and prefill kernels).  CGQ quantization is
  per row, so the oracle quantizes a sample of rows (one per row tile, at a
  varying offset, plus the shard's first and last rows) and the GPU result
  for exactly those rows must match: codes and scales bit for bit, and the
  GEMM output rows within 1e-3 normwise of W_hat_oracle @ X (f64, on the GPU).
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2312_08583_b200 as L  # noqa: E402
from oracle import lpqt_oracle as O  # noqa: E402  (checker only)
from paper_2312_08583_b200.tp import shard_rows  # noqa: E402

REL_TOL = 1e-3
CGQ = L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP6_E3M2)

MODELS = {
    "llama2-7b": [(12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008)],
    "llama2-13b": [(15360, 5120), (5120, 5120), (27648, 5120), (5120, 13824)],
    "starcoder-15b": [(6400, 6144), (6144, 6144), (24576, 6144), (6144, 24576)],
    "llama2-70b": [(10240, 8192), (8192, 8192), (57344, 8192), (8192, 28672)],
}
CASES = [(model, n, k) for model, shapes in MODELS.items() for n, k in shapes]


def normwise_rel(Y, Yref):
    d = float(np.max(np.abs(np.asarray(Y, np.float64) - Yref)))
    s = float(np.max(np.abs(Yref)))
    return d / s if s else d


def test_config0_4096x4096_m1_end_to_end():
    rng = np.random.default_rng(0)
    n = k = 4096
    W = (rng.standard_normal((n, k), dtype=np.float32) * 0.02).astype(np.float16)
    X = np.random.default_rng(1).standard_normal((k, 1)).astype(np.float16)
    q = L.quantize_tensor(W, CGQ, bias_shift=True)
    o = O.quantize_tensor(W, bias_shift=True)
    assert np.array_equal(q.payload.seg4, o["seg4"]) and np.array_equal(q.payload.seg_tail, o["seg2"])
    assert np.array_equal(q.scales.view(np.uint16), o["scales"].view(np.uint16))
    assert np.array_equal(q.folded_scales.view(np.uint16), o["folded"].view(np.uint16))
    Y = L.gemm_quantized(q, X)
    Yo = O.gemm_quantized(o["codes"], o["scales"], n, k, X)
    assert normwise_rel(Y, Yo) <= REL_TOL
    W_hat = O.dequantize_tensor(o["codes"], n, k, scales=o["scales"], path="naive")
    Yf64 = (torch.from_numpy(W_hat).cuda() @ torch.from_numpy(X.astype(np.float64)).cuda()).cpu().numpy()
    tol = O.gemm_tolerance(k, W_hat, X)
    assert np.max(np.abs(Y - Yf64)) <= tol
    assert np.max(np.abs(Yo - Yf64)) <= tol       # the oracle meets its own bound too


def _sample_rows(n: int) -> np.ndarray:
    tiles = (n + 127) // 128
    rows = {0, n - 1}
    for t in range(tiles):
        rows.add(min(n - 1, t * 128 + (t * 37 + 5) % 128))
    return np.array(sorted(rows), dtype=np.int64)


@pytest.mark.parametrize("model,n,k", CASES, ids=[f"{m}-{n}x{k}" for m, n, k in CASES])
def test_layer_shapes_and_tp_shards_vs_oracle(model, n, k):
    g = torch.Generator(device="cuda").manual_seed(n * 31 + k)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    gx = torch.Generator(device="cuda").manual_seed(k)
    xs = {m: torch.randn(m, k, generator=gx, device="cuda").half() for m in (1, 16, 512)}
    for P in (1, 2, 4, 8):
        a, b = shard_rows(n, P, P - 1)
        w = L.Fp6Weight.quantize(W[a:b], bias_shift=True)
        rows = _sample_rows(b - a)
        Wr = W[a:b][torch.from_numpy(rows).cuda()].cpu().numpy()
        o = O.quantize_tensor(Wr, bias_shift=True)
        codes = w.codes()[torch.from_numpy(rows).cuda()].cpu().numpy()
        assert np.array_equal(codes, o["codes"].reshape(len(rows), k)), (P, "codes")
        assert np.array_equal(w.scales[torch.from_numpy(rows).cuda()].cpu().numpy().view(np.uint16),
                              o["scales"].view(np.uint16)), (P, "scales")
        W_hat = torch.from_numpy(O.dequantize_tensor(o["codes"], len(rows), k, scales=o["scales"],
                                                     path="naive")).cuda()
        for m, x in xs.items():
            y = L.w6a16_linear(x, w, out_dtype=torch.float32)           # [m, N/P]
            y_rows = y[:, torch.from_numpy(rows).cuda()].double()
            ref = x.double() @ W_hat.T
            err = float((y_rows - ref).abs().max() / ref.abs().max())
            assert err <= REL_TOL, (P, m, err)
        del w
    torch.cuda.empty_cache()
