"""One W6A16 call on (n, k, m) vs the fp16 matmul of the unquantized W (dev tool)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2312_08583_b200 as L  # noqa: E402

n, k, m = (int(v) for v in sys.argv[1:4])
W = (torch.randn(n, k, device="cuda") * 0.02).half()
lin = L.Fp6Linear.from_dense(W)
x = torch.randn(m, k, device="cuda").half()
print("plan", L.plan(m, n, k), flush=True)
y = lin(x)
torch.cuda.synchronize()
q = L.quantize_tensor(W, L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP6_E3M2), bias_shift=True)
ref = (L.dequantize_tensor(q, "bias_shift") @ x.double().T).T
print(n, k, m, "normwise rel err vs dequantized", float((y.double() - ref).abs().max() / ref.abs().max()), flush=True)
