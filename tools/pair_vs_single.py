"""Standalone vs chained timing of the pair / single-SM prefill kernels (dev tool)."""
import os, sys, statistics
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

def timeit(fn, flush=None, iters=20):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(iters):
        if flush is not None:
            flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return round(statistics.median(ts), 1)

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for n, k, m in [(8192, 8192, 512), (57344, 8192, 512), (8192, 8192, 2048)]:
    w = L.Fp6Weight.quantize((torch.randn(n, k, device="cuda") * 0.02).half())
    x = torch.randn(m, k, device="cuda").half()
    y = torch.empty(m, n, device="cuda", dtype=torch.float16)
    W16 = (torch.randn(n, k, device="cuda") * 0.02).half()
    res = {}
    for sched in ("pair", "single"):
        f = lambda: L.w6a16_linear(x, w, out=y, sched=sched)
        res[sched] = {"flush": timeit(f, flush), "noflush": timeit(f)}
        # chain of 4 in one graph
        def chain():
            for _ in range(4):
                L.w6a16_linear(x, w, out=y, sched=sched)
        res[sched]["chain4_per"] = round(timeit(chain) / 4, 1)
    cb = lambda: torch.matmul(x, W16.t(), out=y)
    res["cublas"] = {"flush": timeit(cb, flush), "noflush": timeit(cb)}
    print(n, k, m, res, flush=True)
