"""One W6A16 launch with a forced schedule, a few times (ncu target, dev tool).
python tools/profile_pair.py --n 8192 --k 8192 --m 2048 --sched pair"""
import argparse, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192); ap.add_argument("--k", type=int, default=8192)
ap.add_argument("--m", type=int, default=2048); ap.add_argument("--sched", default="pair")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
w = L.Fp6Weight.quantize((torch.randn(a.n, a.k, device="cuda") * 0.02).half())
x = torch.randn(a.m, a.k, device="cuda").half()
y = torch.empty(a.m, a.n, device="cuda", dtype=torch.float16)
for _ in range(a.iters):
    L.w6a16_linear(x, w, out=y, sched=a.sched)
torch.cuda.synchronize()
print(L.plan(a.m, a.n, a.k, sched=a.sched))
