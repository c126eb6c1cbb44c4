"""FGQ x FP6 fixtures from the REFERENCE (quantizer.py FGQ blocks, gemm.py
:96-110).  Run here (the only place /root/reference exists):

    python tests/golden/make_fgq_golden.py      -> tests/golden/golden_fgq.npz
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
    rng = np.random.default_rng(2312 + 6)
    out, names = {}, []
    for (n, k, block, scale) in [(3, 40, 16, 1.0), (5, 33, 7, 0.02), (4, 256, 128, 0.02), (6, 300, 128, 3.0),
                                 (2, 512, 256, 0.5), (7, 384, 128, 1e-3), (1, 1, 1, 1.0), (3, 129, 64, 1.0)]:
        W = (rng.standard_normal((n, k)) * scale).astype(np.float32)
        W[rng.random((n, k)) < 0.05] = 0
        if k >= 16:
            W[0, :min(block, k)] = 0          # an all-zero block (scale 1.0)
        q = ref.quantize_tensor(W, ref.QuantScheme(ref.Granularity.FGQ, ref.TensorFormat.FP6_E3M2, block),
                                bias_shift=True)
        name = f"{n}x{k}_b{block}"
        X = rng.integers(-2, 3, size=(k, 3)).astype(np.float32)      # fp16-exact activations
        out[f"f/{name}/W"] = W
        out[f"f/{name}/block"] = np.array(block)
        out[f"f/{name}/scales"] = q.scales.view(np.uint16)
        out[f"f/{name}/folded"] = q.folded_scales.view(np.uint16)
        out[f"f/{name}/seg4"] = q.payload.seg4
        out[f"f/{name}/seg2"] = q.payload.seg_tail
        out[f"f/{name}/deq"] = ref.dequantize_tensor(q, "bias_shift")
        out[f"f/{name}/X"] = X
        out[f"f/{name}/Y"] = ref.gemm_quantized(q, X)
        names.append(name)
    out["f_names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "golden_fgq.npz"), **out)
    print(f"wrote {len(names)} FGQ cases")


if __name__ == "__main__":
    main()
