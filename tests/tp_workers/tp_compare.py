"""torchrun worker (one rank per GPU): NCCL-gather column-parallel linear,
fused-gather linear and the single-GPU GEMM must agree.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/tp_workers/tp_compare.py

Used by tests/test_tp_nccl.py (marked multigpu: runs when >= 2 GPUs exist).
Every rank prints one line "rank r ok <max_err_nccl> <max_err_fused>".
"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_08583_b200 as L  # noqa: E402
from paper_2312_08583_b200 import tp  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    errs = []
    for n, k, m in [(8192, 8192, 16), (10240, 8192, 1), (4096, 11008, 5)]:
        g = torch.Generator(device="cuda").manual_seed(n + k)
        W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()    # same on every rank
        X = torch.randn(k, m, generator=g, device="cuda").half()
        full = L.Fp6Weight.quantize(W)
        y_ref = L.w6a16_linear(X.t().contiguous(), full, out_dtype=torch.float32).t()   # [n, m]
        lin = tp.ColumnParallelFp6Linear.quantize_shard(W)
        y_nccl = lin(X)
        fused = tp.FusedColumnParallelFp6Linear.quantize_shard(W, m_max=m, out_dtype=torch.float32)
        y_fused = fused(X.t().contiguous()).t()
        torch.cuda.synchronize()
        # shard GEMMs run their own split-K plans: equal up to fp32 summation order
        s = y_ref.abs().max().item()
        e1, e2 = (y_nccl.float() - y_ref).abs().max().item() / s, (y_fused - y_ref).abs().max().item() / s
        errs.append((e1, e2))
        assert e1 <= 1e-5 and e2 <= 1e-5, (n, k, m, e1, e2)
    print(f"rank {rank} ok {max(e[0] for e in errs)} {max(e[1] for e in errs)}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
