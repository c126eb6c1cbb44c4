"""Reference GEMM outputs for the reference-order kernels (exact.cu), from the
REFERENCE itself (gemm.py:28-110).  Activations are float32 / float64 values
binary16 cannot hold, blocks of any width, every format — the calls the A16
tcgen05 kernel does not serve.  Run here (the only place /root/reference
exists):

    python tests/golden/make_exact_golden.py     -> tests/golden/golden_exact.npz
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import lpqt as ref  # noqa: E402  (the reference, read-only)

HERE = os.path.dirname(os.path.abspath(__file__))

FMTS = {"fp6": ref.TensorFormat.FP6_E3M2, "fp5": ref.TensorFormat.FP5_E3M1, "int4": ref.TensorFormat.INT4_ASYM}


def main() -> None:
    rng = np.random.default_rng(2312 + 8)
    out, names = {}, []
    cases = [("fp6", 0, 8, 64, 5), ("fp6", 16, 13, 40, 3), ("fp6", 7, 5, 33, 4), ("fp6", 128, 9, 300, 2),
             ("fp6", 24, 64, 64, 8), ("fp5", 0, 7, 50, 3), ("fp5", 24, 6, 70, 5), ("int4", 0, 9, 45, 4),
             ("int4", 16, 12, 48, 8), ("int4", 7, 4, 29, 3), ("fp6", 40, 130, 520, 17), ("int4", 128, 136, 384, 16)]
    for i, (fmt, block, n, k, m) in enumerate(cases):
        W = rng.standard_normal((n, k)) * (10.0 ** rng.uniform(-3, 1, size=(n, 1)))
        if block:
            # block magnitudes spanning 1e-6 .. 1 inside a row
            nb = -(-k // block)
            W = W * np.repeat(10.0 ** rng.uniform(-6, 0, size=(n, nb)), block, axis=1)[:, :k]
        gran = ref.Granularity.FGQ if block else ref.Granularity.CGQ
        q = ref.quantize_tensor(W, ref.QuantScheme(gran, FMTS[fmt], block), bias_shift=False)
        X = rng.standard_normal((k, m)) * (4.0 if i % 2 else 1.0)
        if i % 3 == 0:
            X = X.astype(np.float32)          # float32 (not binary16-exact)
        name = f"{fmt}_b{block}_{n}x{k}x{m}"
        names.append(name)
        out[f"e/{name}/W"] = W
        out[f"e/{name}/fmt"] = np.array(fmt)
        out[f"e/{name}/block"] = np.array(block)
        out[f"e/{name}/X"] = X
        out[f"e/{name}/Y"] = ref.gemm_quantized(q, X)
        W_hat = ref.dequantize_tensor(q)
        out[f"e/{name}/Yd"] = ref.gemm_dense(W_hat, X)
        out[f"e/{name}/Yr"] = ref.gemm_reference(W_hat, X)
        out[f"e/{name}/tol"] = np.array(ref.gemm_tolerance(k, W_hat, X))
    out["e_names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "golden_exact.npz"), **out)
    print(f"{len(names)} cases -> golden_exact.npz")


if __name__ == "__main__":
    main()
