"""world_size-2 gloo tests (CPU) of the column-parallel host logic: shard
bounds, per-shard quantization == slice of the whole-tensor quantization
(SURVEY.md 8e), and the all-gather assembly of Y.  The local compute is the
CPU oracle here (test-only); on GPUs it is the tcgen05 kernel."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_08583_b200.tp import ColumnParallelFp6Linear, shard_rows, shard_sizes


def test_shard_rows_cover_and_align():
    for n in (1, 7, 128, 1000, 4096, 22016, 57344):
        for world in (1, 2, 4, 8):
            if n < world:
                continue
            spans = [shard_rows(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert sum(shard_sizes(n, world)) == n
            if n % (128 * world) == 0:
                assert all((b - a) % 128 == 0 for a, b in spans)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, k, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import lpqt_oracle as O
        rng = np.random.default_rng(0)
        W = (rng.standard_normal((n, k)) * 0.02).astype(np.float16)
        X = rng.standard_normal((k, m)).astype(np.float16)
        a, b = shard_rows(n, world, rank)
        shard = O.quantize_tensor(W[a:b], bias_shift=True)
        full = O.quantize_tensor(W, bias_shift=True)
        # per-shard quantization is the byte slice of the whole-tensor result
        assert np.array_equal(shard["scales"], full["scales"][a:b])
        assert np.array_equal(shard["codes"], full["codes"][a * k:b * k])
        if k % 4 == 0:
            assert np.array_equal(shard["seg4"][: (b - a) * k // 2], full["seg4"][a * k // 2: b * k // 2])
            assert np.array_equal(shard["seg2"][: (b - a) * k // 4], full["seg2"][a * k // 4: b * k // 4])

        def local_gemm(w, Xl):
            return torch.from_numpy(O.gemm_quantized(w["codes"], w["scales"], b - a, k, Xl))

        lin = ColumnParallelFp6Linear(shard, n, k, local_gemm=local_gemm)
        Y = lin(X)
        Y_ref = O.gemm_quantized(full["codes"], full["scales"], n, k, X)
        assert np.array_equal(Y.numpy(), Y_ref)
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,k,m", [(256, 64, 3), (300, 40, 2)])
def test_column_parallel_gather_gloo(n, k, m):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, k, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(results) == [(0, "ok"), (1, "ok")], results
