"""Column-sharded tensor parallelism for the W6A16 linear.

CGQ scales are per output row and quantization never crosses rows
(quantizer.py:95-96, :118-130), so quantizing row shard p of W on rank p
gives exactly rows [p*N/P, (p+1)*N/P) of the whole-tensor result — codes,
planes, scales and folded scales are bit-identical per shard.  Each rank runs
its shard's GEMM into Y_p (reference N x M layout: a contiguous row block)
and one NCCL all-gather (torch.distributed, ProcessGroupNCCL over NVLink /
NVSwitch) assembles Y = [Y_0; ...; Y_{P-1}] with no permute.

The per-rank compute is pluggable (`local_gemm`) so the sharding + gather
logic is exercised by world_size-2 gloo tests on CPU with the oracle as the
local compute; the product path uses the tcgen05 kernel.
"""

from __future__ import annotations

from typing import Callable

from . import _lib


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) of rank's output rows: equal blocks, remainder to the
    first ranks; blocks are rounded to multiples of 128 (one GEMM row tile)
    when n allows, so no tile straddles two ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    unit = 128 if n % (128 * world) == 0 else 1
    blocks = n // unit
    base, extra = divmod(blocks, world)
    start = (rank * base + min(rank, extra)) * unit
    stop = start + (base + (1 if rank < extra else 0)) * unit
    if rank == world - 1:
        stop = n
    return start, stop


def shard_sizes(n: int, world: int) -> list[int]:
    return [b - a for a, b in (shard_rows(n, world, r) for r in range(world))]


class ColumnParallelFp6Linear:
    """Y[N, M] = W_hat[N, K] @ X[K, M] with W's rows sharded over the group.

    `local_gemm(weight_shard, X) -> Y_shard[N_p, M]` is the per-rank compute
    (default: the tcgen05 kernel via `linear.gemm_nm`).  `weight_shard` is
    whatever the caller built for this rank (default: an Fp6Weight).
    """

    def __init__(self, weight_shard, n: int, k: int, group=None,
                 local_gemm: Callable | None = None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n, self.k = int(n), int(k)
        self.rows = shard_rows(self.n, self.world, self.rank)
        self.sizes = shard_sizes(self.n, self.world)
        self.weight = weight_shard
        self.local_gemm = local_gemm or self._tcgen05_gemm

    @classmethod
    def quantize_shard(cls, W_full, group=None, bias_shift: bool = True):
        """Build this rank's Fp6Weight from the full matrix (rows sliced
        before quantization; per-shard result == whole-tensor slice)."""
        import torch.distributed as dist
        from .linear import Fp6Weight
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        n, k = int(W_full.shape[0]), int(W_full.shape[1])
        a, b = shard_rows(n, world, rank)
        return cls(Fp6Weight.quantize(W_full[a:b], bias_shift), n, k, group)

    @staticmethod
    def _tcgen05_gemm(weight, X):
        from .linear import gemm_nm, stage_activations
        xt, kp = stage_activations(X, weight.k)
        return gemm_nm(weight, xt, kp, int(X.shape[1]))

    def forward_local(self, X):
        return self.local_gemm(self.weight, X)

    def __call__(self, X, out=None):
        """X[K, M] replicated on every rank -> Y[N, M] on every rank."""
        t = _lib.torch()
        y_local = self.forward_local(X).contiguous()
        m = int(y_local.shape[1])
        if out is None:
            out = t.empty((self.n, m), dtype=y_local.dtype, device=y_local.device)
        if len(set(self.sizes)) == 1:
            self.dist.all_gather_into_tensor(out, y_local, group=self.group)
            return out
        # ragged shards: gather equal padded blocks, then compact
        mx = max(self.sizes)
        padded = t.zeros((mx, m), dtype=y_local.dtype, device=y_local.device)
        padded[: y_local.shape[0]] = y_local
        buf = t.empty((self.world * mx, m), dtype=y_local.dtype, device=y_local.device)
        self.dist.all_gather_into_tensor(buf, padded, group=self.group)
        a = 0
        for r, sz in enumerate(self.sizes):
            out[a:a + sz] = buf[r * mx: r * mx + sz]
            a += sz
        return out
