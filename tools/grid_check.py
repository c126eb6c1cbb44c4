"""Correctness sweep over (n, k, m, split_k) (dev tool): normwise rel err of
w6a16_linear (fp32 out) vs the f64 dequantize-then-matmul."""
import itertools
import sys

import torch

sys.path.insert(0, ".")
import paper_2312_08583_b200 as L  # noqa: E402

CGQ = L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP6_E3M2)
ns = [int(v) for v in sys.argv[1].split(",")]
ks = [int(v) for v in sys.argv[2].split(",")]
ms = [int(v) for v in sys.argv[3].split(",")]
splits = [int(v) for v in sys.argv[4].split(",")] if len(sys.argv) > 4 else [0]
for n, k in itertools.product(ns, ks):
    W = (torch.randn(n, k, device="cuda") * 0.02).half()
    lin = L.Fp6Linear.from_dense(W)
    q = L.quantize_tensor(W, CGQ, bias_shift=True)
    Wd = L.dequantize_tensor(q, "bias_shift")
    for m, sp in itertools.product(ms, splits):
        x = torch.randn(m, k, device="cuda").half()
        y = L.w6a16_linear(x, lin.weight, out_dtype=torch.float32, split_k=sp)
        ref = (Wd @ x.double().T).T
        err = float((y.double() - ref).abs().max() / ref.abs().max())
        bad = (y.double() - ref).abs().amax(dim=0) > 1e-3 * ref.abs().max()
        rows = bad.nonzero().flatten()
        info = f" bad_rows={rows.numel()} first={rows[:4].tolist()}" if err > 1e-3 else ""
        print(f"n={n} k={k} m={m} split={sp} plan={L.plan(m, n, k, sp)} err={err:.2e}{info}", flush=True)
