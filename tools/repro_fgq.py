"""Bisect (dev tool): FGQ decode (per-block partials) across K / N / split_k."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L
block = int(sys.argv[1]) if len(sys.argv) > 1 else 128
cases = []
for n in (128, 256, 1536):
    for k in (13824, 13952, 13900, 3072, 3200, 3100, 6144, 6272, 28000):
        cases.append((n, k))
for n, k in cases:
    g = torch.Generator(device="cuda").manual_seed(n + k)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    w = L.Fp6Weight.quantize(W, block=block)
    q = L.quantize_tensor(W, L.QuantScheme(L.Granularity.FGQ, L.TensorFormat.FP6_E3M2, block))
    wd = L.dequantize_tensor(q)
    wd = (wd if torch.is_tensor(wd) else torch.from_numpy(wd)).cuda().double()
    res = {}
    for sched, sp in (("auto", 0), ("streamk", 1), ("streamk", 2), ("streamk", 4), ("streamk", 8), ("cluster", 1), ("cluster", 2)):
        x = torch.randn(1, k, generator=g, device="cuda").half()
        try:
            y = L.w6a16_linear(x, w, out_dtype=torch.float32, sched=sched, split_k=sp)
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            res[f"{sched}{sp}"] = "ERR " + repr(e)[:60]
            print(json.dumps({"n": n, "k": k, "res": res}), flush=True)
            sys.exit(1)
        ref = x.double() @ wd.t()
        res[f"{sched}{sp}"] = float(f"{float((y.double() - ref).abs().max() / ref.abs().max()):.2g}")
    print(json.dumps({"n": n, "k": k, "k_tiles": -(-k // 128), "plan": L.plan(1, n, k), "res": res}), flush=True)
