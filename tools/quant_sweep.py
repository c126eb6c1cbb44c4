"""Quantizer consistency sweep (dev tool): the fused tile quantizer
(Fp6Weight.quantize, FP6 straight into the GEMM tile layout) against the
canonical path (quantize_tensor -> 4+2 planes -> prepack) on ragged and large
shapes, every input dtype, CGQ and FGQ blocks: identical codes and scales."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

shapes = [(1000, 11000), (1536, 13900), (4224, 5000), (3000, 28000), (640, 8200), (5000, 3000), (57344, 8192),
          (8192, 28672), (7, 33), (129, 17000), (3, 16385)]
bad = []
for n, k in shapes:
    for dt in (torch.float16, torch.bfloat16, torch.float32):
        for block in (0, 128, 32):
            if block and n * k > 2e8:
                continue
            g = torch.Generator(device="cuda").manual_seed(n * 7 + k)
            W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).to(dt)
            w = L.Fp6Weight.quantize(W, block=block) if block else L.Fp6Weight.quantize(W)
            scheme = (L.QuantScheme(L.Granularity.FGQ, L.TensorFormat.FP6_E3M2, block) if block
                      else L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP6_E3M2))
            q = L.quantize_tensor(W, scheme, bias_shift=not block)
            w2 = L.Fp6Weight.from_quantized(q)
            same_codes = torch.equal(w.codes(), w2.codes())
            same_deq = torch.equal(w.dequantize_f16(), w2.dequantize_f16())
            rec = {"n": n, "k": k, "dtype": str(dt)[6:], "block": block, "codes": same_codes, "dequant": same_deq}
            print(json.dumps(rec), flush=True)
            if not (same_codes and same_deq):
                bad.append(rec)
            del W, w, w2, q
            torch.cuda.empty_cache()
print(json.dumps({"bad": bad}), flush=True)
