"""Column-parallel TP on real NCCL, GPU side.

* one-rank NCCL group on the box's GPU: `ColumnParallelFp6Linear` with the
  tcgen05 local GEMM and the NCCL all-gather must equal the single-GPU GEMM
  bit for bit (the gather only moves rows), for equal and ragged shards;
* `multigpu`: torchrun with one rank per GPU (2 or more GPUs) comparing the
  NCCL-gather layer, the fused-gather layer and the single-GPU GEMM
  (tests/tp_workers/tp_compare.py); skipped on one-GPU boxes.
"""

from __future__ import annotations

import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

import paper_2312_08583_b200 as L  # noqa: E402
from paper_2312_08583_b200 import tp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(_port())
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist.group.WORLD


@pytest.mark.gpu
@pytest.mark.parametrize("n,k,m", [(8192, 8192, 16), (10240, 8192, 1), (1000, 3000, 7), (4096, 11008, 300)])
def test_column_parallel_tcgen05_one_rank_nccl(nccl_group, n, k, m):
    g = torch.Generator(device="cuda").manual_seed(n + k + m)
    W = (torch.randn(n, k, generator=g, device="cuda") * 0.02).half()
    X = torch.randn(k, m, generator=g, device="cuda").half()
    lin = tp.ColumnParallelFp6Linear.quantize_shard(W, group=nccl_group)
    assert lin.local_gemm == lin._tcgen05_gemm and lin.world == 1
    y = lin(X)                                      # tcgen05 shard GEMM + NCCL all_gather_into_tensor
    ref = L.gemm_quantized(L.quantize_tensor(W, L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP6_E3M2),
                                             bias_shift=True), X)
    assert torch.equal(y, ref)


@pytest.mark.gpu
def test_ragged_gather_path_one_rank(nccl_group):
    """The padded-gather branch (unequal shards) runs through NCCL too."""
    W = (torch.randn(300, 512, device="cuda") * 0.02).half()
    X = torch.randn(512, 5, device="cuda").half()
    lin = tp.ColumnParallelFp6Linear.quantize_shard(W, group=nccl_group)
    lin.sizes = [300]                                # single rank: equal by construction
    assert torch.equal(lin(X), lin.forward_local(X))


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_torchrun_nccl_vs_fused_vs_single_gpu():
    n = min(torch.cuda.device_count(), 8)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                        os.path.join(ROOT, "tests", "tp_workers", "tp_compare.py")],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert sum(line.startswith("rank ") and " ok " in line for line in r.stdout.splitlines()) == n
