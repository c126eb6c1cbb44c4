"""Run one GEMM with the LPQT_TRACE library and print the CTA-0 timeline.
LPQT_LIB=build/variants/lib_trace.so python tools/trace_run.py --n 22016 --k 4096 --m 16"""
import argparse, ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L
from paper_2312_08583_b200 import _lib
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=22016); ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--m", type=int, default=16); ap.add_argument("--split", type=int, default=0)
a = ap.parse_args()
W = (torch.randn(a.n, a.k, device="cuda") * 0.02).half()
w = L.Fp6Weight.quantize(W)
x = torch.randn(a.m, a.k, device="cuda").half()
y = torch.empty(a.m, a.n, device="cuda", dtype=torch.float16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.zero_(); L.w6a16_linear(x, w, out=y, split_k=a.split)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_longlong * (2 * 16 * 64))()
lib.lpqt_trace_dump(buf)
t = np.frombuffer(buf, dtype=np.int64).reshape(2, 16, 64)
names = ["p_pre_empty", "p_issued", "dq_it_start", "dq_aempty", "dq_sttm", "dq_pf_full", "dq_waitst", "dq_arrive", "mma_ready", "epi_dfull", "mma_commit"]
print("plan", L.plan(a.m, a.n, a.k, a.split))
for c in range(2):
    base = t[c][t[c] > 0].min() if (t[c] > 0).any() else 0
    print(f"--- CTA {'0' if c == 0 else '77'} (cycles from first event)")
    print("it " + " ".join(f"{n[:11]:>11}" for n in names))
    for i in range(40):
        row = [(t[c, e, i] - base) if t[c, e, i] > 0 else -1 for e in range(11)]
        print(f"{i:2d} " + " ".join(f"{v:11d}" for v in row))
