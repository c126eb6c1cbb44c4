"""Large random fuzz (dev tool): random N / K (up to 28672, ragged) / M / scheme /
schedule / split / output dtype, each against the f64 product of the same
weights (binary16 dequant; INT4 its binary16 rebuild) and bit-identical on repeat."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 150
G, T = L.Granularity, L.TensorFormat
bad = []
for it in range(iters):
    n = int(rng.choice([128, 256, 640, 1000, 1536, 2304, 3000, 4096, 5120, 7168]))
    k = int(rng.choice([512, 1000, 2048, 3100, 4096, 5000, 8192, 11008, 13900, 16500, 28672]))
    m = int(rng.choice([1, 2, 7, 16, 17, 31, 32, 33, 50, 64, 65, 100, 128, 200, 256, 333, 512, 777]))
    kind = str(rng.choice(["cgq", "cgq", "fgq128", "fgq64", "fgq16", "fp5", "int4", "int4_128"]))
    sched = str(rng.choice(["auto", "auto", "streamk", "cluster", "pair", "single"]))
    split = int(rng.choice([0, 0, 2, 3, 5, 8]))
    odt = [torch.float32, torch.float16, torch.bfloat16][int(rng.integers(3))]
    if sched == "cluster" and m > 32:
        sched = "auto"
    g = torch.Generator(device="cuda").manual_seed(it)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    x = torch.randn(m, k, generator=g, device="cuda").half()
    if kind == "cgq":
        w = L.Fp6Weight.quantize(W); wd = w.dequantize_f16().double()
    elif kind.startswith("fgq"):
        w = L.Fp6Weight.quantize(W, block=int(kind[3:])); wd = w.dequantize_f16().double()
        if w.block and w.block % 128 and m > 32:
            continue
    elif kind == "fp5":
        q = L.quantize_tensor(W, L.QuantScheme(G.CGQ, T.FP5_E3M1), bias_shift=True)
        w = L.Fp6Weight.from_quantized(q); wd = w.dequantize_f16().double()
    else:
        b = 128 if kind == "int4_128" else 0
        q = L.quantize_tensor(W, L.QuantScheme(G.FGQ if b else G.CGQ, T.INT4_ASYM, b))
        w = L.Int4Weight.from_quantized(q)
        d = L.dequantize_tensor(q)
        wd = (d if torch.is_tensor(d) else torch.from_numpy(np.asarray(d))).cuda().half().double()
    rec = {"it": it, "n": n, "k": k, "m": m, "kind": kind, "sched": sched, "split": split, "out": str(odt)[6:]}
    try:
        y = L.w6a16_linear(x, w, out_dtype=odt, sched=sched, split_k=split)
        torch.cuda.synchronize()
        y2 = L.w6a16_linear(x, w, out_dtype=odt, sched=sched, split_k=split)
        torch.cuda.synchronize()
    except L.LpqtError as e:  # refused combinations are fine; report them
        rec["refused"] = type(e).__name__
        print(json.dumps(rec), flush=True)
        continue
    ref = x.double() @ wd.t()
    err = float((y.double() - ref).abs().max() / ref.abs().max())
    bar = (2e-3 if (getattr(w, "block", 0) and m > 32) else 1e-3) + {torch.float32: 0, torch.float16: 2 ** -11, torch.bfloat16: 2 ** -8}[odt]
    rec.update(err=float(f"{err:.3g}"), repeat_equal=bool(torch.equal(y, y2)))
    print(json.dumps(rec), flush=True)
    if err > bar or not rec["repeat_equal"]:
        bad.append(rec)
print(json.dumps({"iters": iters, "bad": bad}), flush=True)
