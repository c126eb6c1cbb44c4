"""Correctness sweep (dev tool): every BASELINE layer shape (7B, 13B,
StarCoder-15B, 70B and its TP 2 / 4 / 8 shards) at batch sizes across every
schedule boundary, automatic plan, against the f64 product of the same
weights' binary16 dequant; prints one JSON line per shape and a summary.

python tools/sweep_check.py [--ms 1,8,...]
"""
import argparse, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402
from tools.probe import SHAPES  # noqa: E402

# ragged K (not a multiple of 128; odd k-tile counts) and N not a multiple of 128
SHAPES = dict(SHAPES, ragged=[(1000, 11000), (1536, 13900), (4224, 5000), (3000, 28000), (640, 8200), (5000, 3000)])

ap = argparse.ArgumentParser()
ap.add_argument("--ms", default="1,8,16,17,24,32,33,48,64,65,96,128,192,256,384,512,1024")
ap.add_argument("--sets", default="7b,13b,sc15b,70b,70b_tp2,70b_tp4,70b_tp8")
ap.add_argument("--kind", default="cgq", help="cgq / fgq128 / fgq64 / fgq32 / fgq16 / fp5")
ap.add_argument("--sched", default="auto", help="auto / streamk / cluster / single / pair")
ap.add_argument("--splits", default="0", help="comma list of forced split_k values")
ap.add_argument("--out", default="f32", help="f32 / f16 / bf16 output (bar + the output rounding)")
ap.add_argument("--rebuild", default="cvt", help="cvt / bias_shift / naive (the ablation rebuilds, CGQ FP6, M <= 16)")
ap.add_argument("--layout", default="mn", help="mn (torch layout, w6a16_linear) / nm (reference layout, gemm_nm)")
a = ap.parse_args()
ms = [int(v) for v in a.ms.split(",")]
ODT = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[a.out]
OUT_BAR = {"f32": 0.0, "f16": 2.0 ** -11, "bf16": 2.0 ** -8}[a.out]
shapes = []
for s in a.sets.split(","):
    for sh in SHAPES[s]:
        if sh not in shapes:
            shapes.append(sh)
worst, bad = 0.0, []
for n, k in shapes:
    g = torch.Generator(device="cuda").manual_seed(n + 3 * k)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    if a.kind == "cgq":
        w = L.Fp6Weight.quantize(W)
    elif a.kind.startswith("fgq"):
        w = L.Fp6Weight.quantize(W, block=int(a.kind[3:]))
    elif a.kind.startswith("int4"):  # int4 = per row, int4_128 = blocks of 128 (the comparator)
        b = int(a.kind[5:]) if "_" in a.kind else 0
        q = L.quantize_tensor(W, L.QuantScheme(L.Granularity.FGQ if b else L.Granularity.CGQ,
                                               L.TensorFormat.INT4_ASYM, b))
        w = L.Int4Weight.from_quantized(q)
    else:
        q = L.quantize_tensor(W, L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP5_E3M1), bias_shift=True)
        w = L.Fp6Weight.from_quantized(q)
    del W
    if a.kind.startswith("int4"):  # the kernel's binary16 weight RN_f16(Z + S * level)
        d = L.dequantize_tensor(q)
        wd = (d if torch.is_tensor(d) else torch.from_numpy(np.asarray(d))).cuda().half().double()
    else:
        wd = w.dequantize_f16().double()
    errs = {}
    sub = w.block and w.block % 128
    for m, sp in ((m, int(sp)) for m in ms for sp in a.splits.split(",")):
        if sub and m > 32:
            continue  # (sub-tile blocks run at decode widths only: InvalidScheme above)
        if a.sched == "cluster" and m > 32:
            continue  # (cluster split-K is the decode schedule)
        x = torch.randn(m, k, generator=g, device="cuda").half()
        try:
            if a.layout == "nm":
                from paper_2312_08583_b200.linear import gemm_nm
                kp = -(-k // 8) * 8  # (the staged B operand: row stride a multiple of 8, as gemm_quantized stages it)
                xt = torch.zeros(m, kp, dtype=torch.float16, device="cuda")
                xt[:, :k] = x
                y = gemm_nm(w, xt, kp, m, split_k=sp, sched=a.sched).t()
            else:
                y = L.w6a16_linear(x, w, out_dtype=ODT, sched=a.sched, split_k=sp, rebuild=a.rebuild)
            torch.cuda.synchronize()
            ref = x.double() @ wd.t()
            e = float((y.double() - ref).abs().max() / ref.abs().max())
        except Exception as exc:  # noqa: BLE001
            print(json.dumps({"n": n, "k": k, "m": m, "split_k": sp, "error": repr(exc)[:200]}), flush=True)
            sys.exit(1)
        errs[f"{m}/{sp}"] = e
        worst = max(worst, e)
        if e > (2e-3 if (w.block and m > 32) else 1e-3) + OUT_BAR:
            bad.append((n, k, m, sp, e, L.plan(m, n, k, sp, sched=a.sched)))
    print(json.dumps({"n": n, "k": k, "max_err": max(errs.values()),
                      "errs": {m: float(f"{e:.3g}") for m, e in errs.items()}}), flush=True)
    del wd, w
    torch.cuda.empty_cache()
print(json.dumps({"kind": a.kind, "sched": a.sched, "splits": a.splits, "shapes": len(shapes), "ms": ms, "worst": worst, "bad": bad}), flush=True)
