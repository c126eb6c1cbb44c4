"""Fused GEMM + all-gather (`lpqt_w6a16_linear_gather`, tp.FusedColumnParallelFp6Linear).

The round's GPU boxes have one B200, so two "ranks" run on one GPU: each
rank's launch goes to its own stream (the kernels run concurrently: one
rank's last CTA waits for the other's signal while the other computes), the
"peer" Y buffers and flag arrays are ordinary device buffers.  That
exercises the epilogue fan-out, the system-scope fence / counter / flag
barrier, ragged shards, both Y layouts and epoch reuse; on a multi-GPU node
the same pointers come from torch symmetric memory (P2P over NVLink).
Host-side layout logic is checked on CPU.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2312_08583_b200 as L
from paper_2312_08583_b200 import _lib
from paper_2312_08583_b200 import tp


def test_block_offsets_tile_the_output():
    for n, world, m in [(2048, 2, 16), (1920, 2, 3), (8192, 8, 5), (1000, 3, 7)]:
        sizes = tp.shard_sizes(n, world)
        for layout, unit in (("nm", m), ("mn", 1)):
            offs = [tp.block_offset(sizes, r, m, layout) for r in range(world)]
            assert offs[0] == 0
            for r in range(1, world):
                assert offs[r] - offs[r - 1] == sizes[r - 1] * unit


@pytest.mark.gpu
@pytest.mark.parametrize("n,k,m,layout,dt", [(2048, 4096, 16, "nm", "f32"), (1920, 3000, 3, "mn", "f16"),
                                             (4096, 1024, 64, "mn", "bf16"), (1024, 8192, 1, "mn", "f16"),
                                             (2048, 2048, 200, "nm", "f16"), (1536, 13900, 16, "mn", "f16"),
                                             (3000, 28000, 4, "nm", "f32")])
def test_fused_gather_two_ranks_one_gpu(n, k, m, layout, dt):
    import torch
    tdt = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[dt]
    code = {"f32": _lib.F32, "f16": _lib.F16, "bf16": _lib.BF16}[dt]
    rng = np.random.default_rng(n + k + m)
    W = torch.from_numpy((rng.standard_normal((n, k)) * 0.02).astype(np.float16)).cuda()
    world = 2
    rows = [tp.shard_rows(n, world, r) for r in range(world)]
    ws_ = [L.Fp6Weight.quantize(W[a:b]) for a, b in rows]
    shape = (n, m) if layout == "nm" else (m, n)
    ldy = m if layout == "nm" else n
    Y = [torch.zeros(shape, dtype=tdt, device="cuda") for _ in range(world)]
    flags = [torch.zeros(_lib.MAX_PEERS, dtype=torch.int32, device="cuda") for _ in range(world)]
    done = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(world)]
    scratch = [torch.zeros(8 << 20, dtype=torch.uint8, device="cuda") for _ in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    for epoch in (1, 2, 3):
        x = torch.from_numpy(rng.standard_normal((m, k)).astype(np.float16)).cuda()
        kp = (k + 7) // 8 * 8
        xt = torch.zeros((m, kp), dtype=torch.float16, device="cuda")
        xt[:, :k] = x
        for y in Y:
            y.fill_(float("nan"))
        torch.cuda.synchronize()
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                tp.gather_linear(ws_[r], xt, kp, m, [y.data_ptr() for y in Y], [f.data_ptr() for f in flags], r,
                                 epoch, done[r], code, layout, ldy, rows[r][0], workspace=scratch[r])
        torch.cuda.synchronize()
        ref = torch.cat([L.w6a16_linear(x, w, out_dtype=tdt) for w in ws_], dim=1)   # [m, n]
        if layout == "nm":
            ref = ref.t()
        for r in range(world):
            assert torch.equal(Y[r], ref), (epoch, r)
        assert all(int(d.item()) == 0 for d in done)
        assert all(int(f[q].item()) == epoch for f in flags for q in range(world))


@pytest.mark.gpu
def test_fused_gather_single_rank_is_a_plain_launch():
    import torch
    w = L.Fp6Weight.quantize((torch.randn(1024, 2048, device="cuda") * 0.02).half())
    x = torch.randn(16, 2048, device="cuda").half()
    y = torch.empty(16, 1024, dtype=torch.float16, device="cuda")
    flags = torch.zeros(_lib.MAX_PEERS, dtype=torch.int32, device="cuda")
    done = torch.zeros(1, dtype=torch.int32, device="cuda")
    for epoch in range(1, 4):
        tp.gather_linear(w, x, 2048, 16, [y.data_ptr()], [flags.data_ptr()], 0, epoch, done, _lib.F16, "mn", 1024, 0)
        assert torch.equal(y, L.w6a16_linear(x, w))
    with pytest.raises(L.InvalidInput):
        tp.gather_linear(w, x, 2048, 16, [y.data_ptr()], [flags.data_ptr()], 1, 4, done, _lib.F16, "mn", 1024, 0)
    # decode tiles leave by per-peer TMA stores: a Y row stride the tensor map
    # cannot describe (reference layout Y[N, 1] in fp16: 2-byte rows) is refused
    y1 = torch.empty(1024, 1, dtype=torch.float16, device="cuda")
    with pytest.raises(L.ShapeError):
        tp.gather_linear(w, x[:1], 2048, 1, [y1.data_ptr()], [flags.data_ptr()], 0, 5, done, _lib.F16, "nm", 1, 0)


@pytest.mark.gpu
def test_fused_layer_world1_symmetric_memory():
    """FusedColumnParallelFp6Linear end to end on a one-rank NCCL group:
    torch symmetric memory for y and the flags, four calls (both output
    buffers twice), equal to the plain launch."""
    import os
    import socket

    import torch
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        W = (torch.randn(2048, 4096, device="cuda") * 0.02).half()
        layer = tp.FusedColumnParallelFp6Linear.quantize_shard(W, m_max=32)
        for m in (1, 16, 32, 5):
            x = torch.randn(m, 4096, device="cuda").half()
            y = layer(x)
            assert torch.equal(y, L.w6a16_linear(x, layer.weight)), m
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_fused_gather_refuses_unaligned_rows():
    """Decode tiles reach the peers only by TMA tensor stores: Y[N, M] f32 at
    M = 1 (4-byte rows) cannot be described and is refused before the launch."""
    import torch
    w = L.Fp6Weight.quantize((torch.randn(256, 1024, device="cuda") * 0.02).half())
    xt = torch.randn(1, 1024, device="cuda").half()
    Y = torch.zeros(512, 1, dtype=torch.float32, device="cuda")
    flags = torch.zeros(_lib.MAX_PEERS, dtype=torch.int32, device="cuda")
    done = torch.zeros(1, dtype=torch.int32, device="cuda")
    scratch = torch.zeros(8 << 20, dtype=torch.uint8, device="cuda")
    with pytest.raises(L.ShapeError):
        tp.gather_linear(w, xt, 1024, 1, [Y.data_ptr(), Y.data_ptr()], [flags.data_ptr(), flags.data_ptr()], 0, 1,
                         done, _lib.F32, "nm", 1, 0, workspace=scratch)
