"""One FP6 CGQ, one FP6 FGQ-128 and one INT4 CGQ launch at a 70B decode shape,
for an ncu capture (`-k regex:w6a16 -s 3 -c 3`).  Dev tool."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

n, k, m = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (57344, 8192, 16)))
W = (torch.randn(n, k, device="cuda") * 0.02).half()
ws = [L.Fp6Weight.quantize(W), L.Fp6Weight.quantize(W, block=128),
      L.Int4Weight.from_quantized(L.quantize_tensor(W, L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.INT4_ASYM)))]
x = torch.randn(m, k, device="cuda").half()
for w in ws:          # warm-up: one launch each (skipped by -s 3)
    L.w6a16_linear(x, w)
torch.cuda.synchronize()
for w in ws:
    L.w6a16_linear(x, w)
torch.cuda.synchronize()
