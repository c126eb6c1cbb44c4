"""INT4 asymmetric (CGQ / FGQ) fixtures from the REFERENCE.  Run here:

    python tests/golden/make_int4_golden.py      -> tests/golden/golden_int4.npz
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import lpqt as ref  # noqa: E402  (the reference, read-only)

HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    rng = np.random.default_rng(2312 + 4)
    out, names = {}, []
    for (n, k, block, scale) in [(3, 40, 0, 1.0), (5, 33, 0, 0.02), (4, 256, 128, 0.02), (6, 300, 128, 3.0),
                                 (7, 130, 32, 1e-3), (2, 64, 7, 1.0), (1, 1, 0, 1.0)]:
        W = (rng.standard_normal((n, k)) * scale + rng.choice([0.0, 0.5])).astype(np.float32)
        if k >= 8:
            W[0, :8] = 0.25                    # a constant block start (scale 1.0 when the block is constant)
        gran = ref.Granularity.FGQ if block else ref.Granularity.CGQ
        q = ref.quantize_tensor(W, ref.QuantScheme(gran, ref.TensorFormat.INT4_ASYM, block))
        X = rng.integers(-2, 3, size=(k, 3)).astype(np.float32)
        name = f"{n}x{k}_b{block}"
        out[f"q/{name}/W"], out[f"q/{name}/block"] = W, np.array(block)
        out[f"q/{name}/scales"] = q.scales.view(np.uint16)
        out[f"q/{name}/zeros"] = q.zero_points.view(np.uint16)
        out[f"q/{name}/nibbles"] = np.asarray(q.payload, np.uint8)
        out[f"q/{name}/deq"] = ref.dequantize_tensor(q)
        out[f"q/{name}/X"], out[f"q/{name}/Y"] = X, ref.gemm_quantized(q, X)
        out[f"q/{name}/container"] = np.frombuffer(ref.write_lpqt(q), dtype=np.uint8)
        names.append(name)
    out["q_names"] = np.array(names)
    lv = rng.integers(0, 16, size=1001).astype(np.uint8)
    out["p/levels"], out["p/nibbles"] = lv, ref.pack_int4(lv)
    np.savez_compressed(os.path.join(HERE, "golden_int4.npz"), **out)
    print(f"wrote {len(names)} INT4 cases")


if __name__ == "__main__":
    main()
