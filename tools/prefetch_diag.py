"""Mimic test_prefetch_next_linear_is_transparent and report mismatches (dev tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = torch.Generator(device="cuda").manual_seed(3)
shapes = [(12288, 4096), (4096, 4096), (4096, 11008), (640, 256)]
ws = [L.Fp6Weight.quantize((torch.randn(n, k, device="cuda", generator=g) * 0.02).half()) for n, k in shapes]
xs = [torch.randn(m, k, device="cuda", generator=g).half() for _, k in shapes]
want = [L.w6a16_linear(x, w, out_dtype=torch.float32) for x, w in zip(xs, ws)]
for i, (n, k) in enumerate(shapes):
    print(i, L.plan(m, n, k))
for rep in range(3):
    for depth in (None, 0, 16, 12288, 1 << 20):
        for i, (x, w) in enumerate(zip(xs, ws)):
            kw = {} if depth is None else {"prefetch": ws[(i + 1) % len(ws)], "prefetch_bytes": depth}
            got = L.w6a16_linear(x, w, out_dtype=torch.float32, **kw)
            if not torch.equal(got, want[i]):
                d = (got - want[i]).abs()
                nz = torch.nonzero(d)
                rows = sorted({int(c) // 128 for c in nz[:, 1].tolist()})
                mt = sorted({int(r) // 192 for r in nz[:, 0].tolist()})
                rel = float(d.max() / want[i].abs().max())
                print(f"rep {rep} depth {depth} layer {i}: {nz.shape[0]} elems, n-tiles {rows[:12]}, m-tiles {mt}, "
                      f"max rel {rel:.3g}")
