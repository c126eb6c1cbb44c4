"""Repro (dev tool): W6A16 at M = 33-64 on 5120 x 13824 (BN 64, stream-K, 5 splits)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L
n, k = int(sys.argv[1]), int(sys.argv[2])
ms = [int(v) for v in sys.argv[3].split(",")]
W = (torch.randn(n, k, device="cuda") * 0.02).half()
w = L.Fp6Weight.quantize(W)
Wd = w.dequantize_f16().float()
torch.cuda.synchronize()
print("quantize ok", flush=True)
for m in ms:
    x = torch.randn(m, k, device="cuda").half()
    y = L.w6a16_linear(x, w, out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref = x.float() @ Wd.t()
    print(m, L.plan(m, n, k), float((y - ref).abs().max() / ref.abs().max()), flush=True)
