"""Column-sharded tensor parallelism for the W6A16 linear.

CGQ scales are per output row and quantization never crosses rows
(quantizer.py:95-96, :118-130), so quantizing row shard p of W on rank p
gives exactly rows [p*N/P, (p+1)*N/P) of the whole-tensor result — codes,
planes, scales and folded scales are bit-identical per shard.  Each rank runs
its shard's GEMM into Y_p (reference N x M layout: a contiguous row block)
and one NCCL all-gather (torch.distributed, ProcessGroupNCCL over NVLink /
NVSwitch) assembles Y = [Y_0; ...; Y_{P-1}] with no permute.

`FusedColumnParallelFp6Linear` is the B200 variant with no collective call:
the GEMM's epilogue stores each rank's block straight into every peer's
symmetric-memory Y and the same kernel ends with a flag barrier
(`lpqt_w6a16_linear_gather`, SURVEY §8e "fused variant").

The per-rank compute is pluggable (`local_gemm`) so the sharding + gather
logic is exercised by world_size-2 gloo tests on CPU with the oracle as the
local compute; the product path uses the tcgen05 kernel.
"""

from __future__ import annotations

import ctypes
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


# ---------------------------------------------------------------- fused all-gather
def block_offset(sizes: list[int], rank: int, m: int, layout: str) -> int:
    """Element offset of `rank`'s output block inside the full Y: rows
    [row0, row0 + N_p) of Y[N, M] ("nm", ldy = M) or columns of Y[M, N]
    ("mn", ldy = N)."""
    row0 = sum(sizes[:rank])
    return row0 * m if layout == "nm" else row0


def gather_linear(weight, xt, ldx: int, m: int, peer_y: list[int], peer_flags: list[int], rank: int, epoch: int,
                  done, y_dtype: int, layout: str, ldy: int, row0: int, split_k: int = 0, sched: str = "auto",
                  workspace=None) -> None:
    """One fused GEMM + all-gather launch (`lpqt_w6a16_linear_gather`): this
    rank's shard GEMM stores its block straight into every peer's Y
    (`peer_y[p]` = peer p's Y base address; the block offset is added here)
    and the same kernel completes only when every peer's block has landed in
    this GPU's Y (flag barrier, `peer_flags[p]` = peer p's flag array).
    All ranks must call it with the same epoch.  row0: this rank's first
    output row (`shard_rows`).  workspace: split-K scratch (default: the
    per-device one; launches that may run concurrently need their own)."""
    from .linear import _sched_flags
    lib = _lib.load()
    npeers = len(peer_y)
    if not 1 <= npeers <= _lib.MAX_PEERS or len(peer_flags) != npeers:
        raise ValueError(f"1..{_lib.MAX_PEERS} peers with one flag array each")
    es = 4 if y_dtype == _lib.F32 else 2
    off = row0 * m if layout == "nm" else row0
    po = _lib.PeerOut()
    for p in range(npeers):
        po.y[p] = int(peer_y[p]) + off * es
        po.flags[p] = int(peer_flags[p])
    po.npeers, po.rank, po.epoch, po.done = npeers, rank, epoch & 0xFFFFFFFF, done.data_ptr()
    ws_bytes = int(lib.lpqt_w6a16_workspace_bytes(m, weight.n, weight.k, split_k))
    ws = workspace if workspace is not None else (_lib.Workspace.get(ws_bytes) if ws_bytes else None)
    if ws is not None and ws.numel() < ws_bytes:
        raise ValueError(f"workspace of {ws.numel()} B, the plan needs {ws_bytes}")
    flags = (_lib.LAUNCH_PDL if weight.static else 0) | _sched_flags(sched)
    _lib.check(lib.lpqt_w6a16_linear_gather(
        weight.tiles.data_ptr(), weight.gemm_scales().data_ptr(), weight.block, xt.data_ptr(), ldx, m, weight.n,
        weight.k, y_dtype, _lib.Y_NM if layout == "nm" else _lib.Y_MN, ldy, split_k, _lib.ptr(ws),
        ws.numel() if ws is not None else 0, flags, ctypes.byref(po), _lib.stream_ptr()), "w6a16_linear_gather")


def _peer_ptrs(handle, local, rank: int) -> list[int]:
    """Every peer's address of `local` (a tensor inside a symmetric
    allocation): the peer's allocation base plus this tensor's offset in it."""
    base = list(handle.buffer_ptrs)
    off = local.data_ptr() - base[rank]
    return [b + off for b in base]


class FusedColumnParallelFp6Linear:
    """y[M, N] = x[M, K] @ W_hat^T with W's rows sharded over the group and
    the all-gather fused into the GEMM: every rank's epilogue writes its
    columns of y straight into every peer's symmetric-memory copy of y over
    NVLink / NVSwitch, and the kernel's last CTA runs a flag barrier with the
    peers (no NCCL call on the data path).  Buffers come from
    `torch.distributed._symmetric_memory` (P2P-mapped on every peer); three
    output buffers rotate.  Lifetime of a returned y (epoch e): a peer can
    overwrite this buffer only in its epoch e + 3 launch, which starts after
    its e + 2 kernel finished, which waits for THIS rank's e + 2 kernel's
    signal — and that kernel ends only after everything enqueued on this
    rank's stream before it.  So y stays valid for every reader enqueued on
    the stream before this rank's call after next (e + 2); clone it to keep
    it longer.  (With two buffers a peer's e + 2 stores could land while
    readers enqueued after this rank's e + 1 call still ran.)"""

    NBUF = 3

    def __init__(self, weight_shard, n: int, k: int, m_max: int, group=None, out_dtype=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        t = _lib.torch()
        self.group = group or dist.group.WORLD
        self.world, self.rank = dist.get_world_size(self.group), dist.get_rank(self.group)
        if self.world > _lib.MAX_PEERS:
            raise ValueError(f"at most {_lib.MAX_PEERS} ranks")
        self.n, self.k, self.m_max = int(n), int(k), int(m_max)
        self.sizes = shard_sizes(self.n, self.world)
        self.weight = weight_shard
        self.dtype = out_dtype or t.float16
        dev = weight_shard.tiles.device
        gname = self.group.group_name
        self.bufs = [symm.empty((self.m_max, self.n), dtype=self.dtype, device=dev) for _ in range(self.NBUF)]
        self.buf_h = [symm.rendezvous(b, gname) for b in self.bufs]
        self.flag_t = symm.empty((_lib.MAX_PEERS,), dtype=t.int32, device=dev)
        self.flag_t.zero_()
        self.flag_h = symm.rendezvous(self.flag_t, gname)
        self.done = t.zeros(1, dtype=t.int32, device=dev)
        self.epoch = 0
        dist.barrier(group=self.group)   # every rank's flags are zero before the first signal

    @classmethod
    def quantize_shard(cls, W_full, m_max: int, group=None, bias_shift: bool = True, out_dtype=None):
        import torch.distributed as dist
        from .linear import Fp6Weight
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        n, k = int(W_full.shape[0]), int(W_full.shape[1])
        a, b = shard_rows(n, world, rank)
        return cls(Fp6Weight.quantize(W_full[a:b], bias_shift), n, k, m_max, group, out_dtype)

    def __call__(self, x):
        """x[M, K] fp16, replicated on every rank -> y[M, N] on every rank."""
        t = _lib.torch()
        m = int(x.shape[0])
        if m > self.m_max:
            raise ValueError(f"batch {m} exceeds m_max {self.m_max}")
        x2 = x if (x.dtype == t.float16 and x.is_contiguous() and self.k % 8 == 0) else None
        if x2 is None:
            kp = (self.k + 7) // 8 * 8
            x2 = t.zeros((m, kp), dtype=t.float16, device=x.device)
            x2[:, :self.k] = x
        ldx = int(x2.shape[1])
        self.epoch += 1
        i = self.epoch % self.NBUF
        code = {t.float32: _lib.F32, t.float16: _lib.F16, t.bfloat16: _lib.BF16}[self.dtype]
        gather_linear(self.weight, x2, ldx, m, _peer_ptrs(self.buf_h[i], self.bufs[i], self.rank),
                      _peer_ptrs(self.flag_h, self.flag_t, self.rank), self.rank, self.epoch, self.done, code, "mn",
                      self.n, sum(self.sizes[:self.rank]))
        return self.bufs[i][:m]
