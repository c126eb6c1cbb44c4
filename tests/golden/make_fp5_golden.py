"""FP5 (e3m1, 4 + 1) fixtures from the REFERENCE (codec, packing, quantizer
CGQ / FGQ, dequant, gemm).  Run here (the only place /root/reference exists):

    python tests/golden/make_fp5_golden.py      -> tests/golden/golden_fp5.npz
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import lpqt as ref  # noqa: E402  (the reference, read-only)

HERE = os.path.dirname(os.path.abspath(__file__))
F5 = ref.FP5_E3M1


def main() -> None:
    rng = np.random.default_rng(2312 + 5)
    out = {}
    # encode KATs: grid, midpoints +- 1 ulp, signs, saturation
    grid = np.array([ref.decode(F5, c) for c in range(16)])
    mids = (grid[:-1] + grid[1:]) / 2
    x = np.concatenate([grid, -grid, mids, -mids, np.nextafter(mids, 0), np.nextafter(mids, 99),
                        [0.0, -0.0, 30.0, -1e-9, 1e-9, 24.0, 23.99, 22.0, 20.0], rng.standard_normal(200) * 8])
    out["enc/x"] = x
    out["enc/codes"] = ref.encode_rtn_array(F5, x)
    for n in (0, 1, 7, 8, 9, 31, 1000):
        c = rng.integers(0, 32, size=n).astype(np.uint8)
        seg = ref.pack(F5, c)
        out[f"p/{n}/codes"], out[f"p/{n}/seg4"], out[f"p/{n}/seg1"] = c, seg.seg4, seg.seg_tail
    out["p_lens"] = np.array([0, 1, 7, 8, 9, 31, 1000])
    names = []
    for (n, k, block, scale) in [(3, 40, 0, 1.0), (5, 33, 0, 0.02), (4, 256, 128, 0.02), (6, 300, 128, 3.0),
                                 (2, 512, 0, 0.5), (7, 130, 16, 1e-3), (1, 1, 0, 1.0)]:
        W = (rng.standard_normal((n, k)) * scale).astype(np.float32)
        W[rng.random((n, k)) < 0.05] = 0
        gran = ref.Granularity.FGQ if block else ref.Granularity.CGQ
        q = ref.quantize_tensor(W, ref.QuantScheme(gran, ref.TensorFormat.FP5_E3M1, block), bias_shift=True)
        X = rng.integers(-2, 3, size=(k, 3)).astype(np.float32)
        name = f"{n}x{k}_b{block}"
        out[f"q/{name}/W"], out[f"q/{name}/block"] = W, np.array(block)
        out[f"q/{name}/scales"] = q.scales.view(np.uint16)
        out[f"q/{name}/folded"] = q.folded_scales.view(np.uint16)
        out[f"q/{name}/seg4"], out[f"q/{name}/seg1"] = q.payload.seg4, q.payload.seg_tail
        out[f"q/{name}/deq"] = ref.dequantize_tensor(q, "bias_shift")
        out[f"q/{name}/X"], out[f"q/{name}/Y"] = X, ref.gemm_quantized(q, X)
        out[f"q/{name}/container"] = np.frombuffer(ref.write_lpqt(q), dtype=np.uint8)
        names.append(name)
    out["q_names"] = np.array(names)
    codes = np.arange(32, dtype=np.uint8)
    s = np.array([0.5, 1.0, 0.03570556640625, 6.0e-8, 15.9921875], dtype=np.float16)
    f = ref.fold_scale_array(F5, s)
    out["dq/bias"] = ref.dequant_bias_shift_array(F5, codes[:, None], f[None, :]).view(np.uint16)
    out["dq/naive"] = ref.dequant_naive_array(F5, codes[:, None], s[None, :]).view(np.uint16)
    out["dq/scales"] = s.view(np.uint16)
    np.savez_compressed(os.path.join(HERE, "golden_fp5.npz"), **out)
    print(f"wrote {len(names)} FP5 quantize cases")


if __name__ == "__main__":
    main()
