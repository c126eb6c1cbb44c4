import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2312_08583_b200 as L
n, k, m = 57344, 8192, 16
W = (torch.randn(n, k, device="cuda") * 0.02).half()
q = L.quantize_tensor(W, L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.INT4_ASYM, 0))
w = L.Int4Weight.from_quantized(q)
x = torch.randn(m, k, device="cuda").half()
for _ in range(3):
    y = L.w6a16_linear(x, w)
torch.cuda.synchronize()
