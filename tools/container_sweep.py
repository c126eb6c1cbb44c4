"""Container sweep (dev tool): quantize on the GPU -> write_lpqt -> read_lpqt /
load_lpqt at LLaMA-size and ragged shapes for every scheme: the bytes round
trip, and the loaded weight's GEMM equals the directly built weight's."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

G, T = L.Granularity, L.TensorFormat
schemes = [("cgq_fp6", L.QuantScheme(G.CGQ, T.FP6_E3M2), True), ("fgq128_fp6", L.QuantScheme(G.FGQ, T.FP6_E3M2, 128), False),
           ("fgq32_fp6", L.QuantScheme(G.FGQ, T.FP6_E3M2, 32), False), ("cgq_fp5", L.QuantScheme(G.CGQ, T.FP5_E3M1), True),
           ("fgq128_int4", L.QuantScheme(G.FGQ, T.INT4_ASYM, 128), False)]
bad = []
for n, k in [(4096, 11008), (1536, 13900), (12288, 4096), (1000, 3000)]:
    g = torch.Generator(device="cuda").manual_seed(n + k)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    x = torch.randn(16, k, generator=g, device="cuda").half()
    for name, sch, bs in schemes:
        q = L.quantize_tensor(W, sch, bias_shift=bs)
        data = L.write_lpqt(q)
        rt = L.write_lpqt(L.read_lpqt(data)) == data
        w = L.load_lpqt(data)
        direct = (L.Int4Weight if "int4" in name else L.Fp6Weight).from_quantized(q)
        same = torch.equal(L.w6a16_linear(x, w, out_dtype=torch.float32), L.w6a16_linear(x, direct, out_dtype=torch.float32))
        rec = {"n": n, "k": k, "scheme": name, "bytes": len(data), "roundtrip": rt, "gemm_equal": same}
        print(json.dumps(rec), flush=True)
        if not (rt and same):
            bad.append(rec)
print(json.dumps({"bad": bad}), flush=True)
