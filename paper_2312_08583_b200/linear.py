"""Device-resident FP6 weights and the W6A16 linear (the B200 hot path).

`Fp6Weight` holds a weight matrix the way the GEMM streams it: the B200 tile
layout (128 x 128 tiles of 12288 B, `lpqt_fp6_prepack`) plus the f16 row
scales.  `w6a16_linear` is the torch-facing call (x[M, K] fp16 -> y[M, N]);
`gemm_nm` is the reference-layout call used by `gemm.gemm_quantized`
(X[K, M] -> Y[N, M] f32, gemm.py:65-94).  Both launch the tcgen05 kernel
`lpqt_w6a16_linear`; nothing here computes on the CPU.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import InvalidInput, ShapeError
from .packing import seg4_length

TILE = 128


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def sub_tile_block(block: int) -> bool:
    """FGQ blocks narrower than a 128-k tile that the decode GEMM scales per
    block partial (16 / 32 / 64 columns; gemm.py:96-110 order)."""
    return bool(block) and block % 16 == 0 and TILE % block == 0


def stage_params(scales, zeros, n: int, k: int, block: int):
    """Row-major per-block f16 scales (and INT4 zero points) -> the GEMM's
    stage-ordered block parameters (`lpqt_fgq_stage_params`): built once per
    weight, read by the W producer next to each stage's weight bytes."""
    t = _lib.torch()
    lib = _lib.load()
    out = t.empty(int(lib.lpqt_fgq_stage_bytes(n, k, int(zeros is not None))), dtype=t.uint8, device=scales.device)
    _lib.check(lib.lpqt_fgq_stage_params(scales.data_ptr(), _lib.ptr(zeros), n, k, block, out.data_ptr(),
                                         _lib.stream_ptr()), "fgq_stage_params")
    return out


def prepack(seg4, seg2, n: int, k: int, fmt: str = "fp6"):
    """Canonical planes (CUDA uint8) -> tile layout (CUDA uint8).
    fmt "fp6": 4 + 2 planes -> FP6 tiles (0.75 B per weight);
    "fp5n": 4 + 1 planes -> native FP5 tiles (0.625 B per weight, CGQ GEMM);
    "fp5": 4 + 1 planes -> FP6 tiles (every e3m1 value is an e3m2 value; the
    FGQ FP5 GEMM streams these at 0.75 B per weight)."""
    t = _lib.torch()
    lib = _lib.load()
    nbytes = int(lib.lpqt_fp5n_tiles_bytes(n, k) if fmt == "fp5n" else lib.lpqt_fp6_tiles_bytes(n, k))
    tiles = t.empty(nbytes, dtype=t.uint8, device=seg4.device)
    fn = {"fp6": lib.lpqt_fp6_prepack, "fp5": lib.lpqt_fp5_prepack, "fp5n": lib.lpqt_fp5n_prepack}[fmt]
    _lib.check(fn(seg4.data_ptr(), seg2.data_ptr(), n, k, tiles.data_ptr(), _lib.stream_ptr()), "prepack")
    return tiles


class Fp6Weight:
    """An N x K FP6 (e3m2) weight resident in HBM in the GEMM's tile layout
    (wbits 6), or an FP5 (e3m1) CGQ weight in the native 5-bit tile layout
    (wbits 5, `lpqt_fp5n_prepack`; the GEMM runs with LPQT_WEIGHTS_FP5)."""

    def __init__(self, tiles, scales, n: int, k: int, folded=None, static: bool = False, block: int = 0,
                 wbits: int = 6):
        self.tiles = tiles
        self.wbits = int(wbits)
        # f16 scales: one per row (CGQ, block 0; the GEMM multiplies the fp32
        # accumulator by S) or one per (row, block of `block` columns), FGQ,
        # row-major (the GEMM scales the rebuilt weights per 128-k tile)
        self.scales = scales
        self.folded = folded          # f16 or None (bias-shift artifact, API parity)
        self.n = int(n)
        self.k = int(k)
        self.block = int(block) if block and int(block) < int(k) else 0
        # FGQ: the GEMM's stage-ordered copy of the block scales (built once here)
        # (blocks that are not whole 128-k tiles dequantize but do not run the GEMM)
        self._stage = (stage_params(scales, None, self.n, self.k, self.block)
                       if self.block and self.block % TILE == 0 else None)
        # static: tiles/scales are complete and never rewritten, so the GEMM
        # may be launched with programmatic dependent launch (it prefetches
        # weights before the preceding kernel on the stream has finished).
        self.static = bool(static)

    # -- construction -------------------------------------------------------
    @classmethod
    def from_planes(cls, seg4, seg2, scales, n: int, k: int, folded=None, block: int = 0,
                    fmt: str = "fp6") -> "Fp6Weight":
        cgq = not block or int(block) >= int(k)
        if fmt == "fp5" and cgq:
            fmt = "fp5n"  # CGQ FP5 streams its own 5-bit tiles
        tiles = prepack(seg4, seg2, n, k, fmt)
        # one-time: the weights are complete before any GEMM can overlap them
        _lib.torch().cuda.current_stream().synchronize()
        return cls(tiles, scales, n, k, folded, static=True, block=block, wbits=5 if fmt == "fp5n" else 6)

    @classmethod
    def quantize(cls, W, bias_shift: bool = True, block: int = 0) -> "Fp6Weight":
        """RTN FP6 quantize on the GPU (quantizer.py:189-248) straight into
        the tile layout (`lpqt_fp6_quantize_tiles_blocks`; byte-identical to
        prepack of the canonical planes).  block: 0 = one scale per row
        (CGQ), else FGQ blocks of `block` columns."""
        from .quantizer import _weights_to_device
        w, _ = _weights_to_device(W)
        n, k = (int(v) for v in w.shape)
        block = int(block) if block and int(block) < k else 0
        nb = n * (-(-k // block) if block else 1)
        t = _lib.torch()
        dev = w.device
        tiles = t.empty(int(_lib.load().lpqt_fp6_tiles_bytes(n, k)), dtype=t.uint8, device=dev)
        scales = t.empty(nb, dtype=t.float16, device=dev)
        folded = t.empty(nb, dtype=t.float16, device=dev) if bias_shift else None
        flags = _lib.Flags()
        _lib.check(_lib.load().lpqt_fp6_quantize_tiles_blocks(
            w.data_ptr(), _lib.dtype_code(w.dtype), n, k, int(w.stride(0)) if n else k, block,
            int(bool(bias_shift)), scales.data_ptr(), _lib.ptr(folded), tiles.data_ptr(), flags.ptr,
            _lib.stream_ptr()), "quantize_tiles")
        flags.raise_if_set()
        return cls(tiles, scales, n, k, folded, static=True, block=block)

    @classmethod
    def from_quantized(cls, q) -> "Fp6Weight":
        from .quantizer import _require_path, cache_of, device_planes, scale_block
        _require_path(q.scheme)
        s4, s2, sc = device_planes(q)   # validates lengths / code_count first
        cache = cache_of(q)
        if cache is not None and "weight" in cache:
            return cache["weight"]
        fmt = "fp5" if q.scheme.fmt.minifloat.mantissa_bits == 1 else "fp6"
        w = cls.from_planes(s4, s2, sc, q.rows, q.cols, block=scale_block(q.scheme), fmt=fmt)
        if cache is not None:
            cache["weight"] = w
        return w

    def gemm_scales(self):
        """The scale operand of the GEMM: the per-row scales (CGQ), the
        stage-ordered block scales (FGQ, whole tiles) or the row-major block
        scales (FGQ blocks of 16 / 32 / 64)."""
        return self._stage if self._stage is not None else self.scales

    # -- inspection -----------------------------------------------------------
    @property
    def nbytes(self) -> int:
        return int(self.tiles.numel() + 2 * self.scales.numel())

    def stream_bytes(self) -> int:
        """Algorithmic weight bytes per GEMM: 0.75 B/weight (FP5 native: 0.625)
        + 2 B per scale (cli.py:75-80)."""
        nk = self.n * self.k
        tail = (self.wbits - 4) * nk
        return seg4_length(nk) + _round_up((tail + 7) // 8, 4) + 2 * int(self.scales.numel())

    def codes(self):
        """Row-major codes [N, K] recovered from the tile layout (test hook):
        e3m2 codes of FP6 tiles, e3m1 codes of native FP5 tiles."""
        t = _lib.torch()
        out = t.empty((self.n, self.k), dtype=t.uint8, device=self.tiles.device)
        lib = _lib.load()
        fn = lib.lpqt_fp5n_unprepack if self.wbits == 5 else lib.lpqt_fp6_unprepack
        _lib.check(fn(self.tiles.data_ptr(), self.n, self.k, out.data_ptr(), _lib.stream_ptr()), "unprepack")
        return out

    def dequantize_f16(self):
        """[N, K] binary16 via the GEMM's register rebuild: value_f16[c] * S
        (dequant.py:72-79), bit-identical to the bias-shift path
        compose[c] * folded (dequant.py:82-86)."""
        t = _lib.torch()
        out = t.empty((self.n, self.k), dtype=t.float16, device=self.tiles.device)
        if self.wbits == 5:
            _lib.check(_lib.load().lpqt_fp5n_tiles_dequant(self.tiles.data_ptr(), self.scales.data_ptr(), self.n,
                                                           self.k, out.data_ptr(), _lib.stream_ptr()), "tiles_dequant")
            return out
        _lib.check(_lib.load().lpqt_fp6_tiles_dequant_blocks(self.tiles.data_ptr(), self.scales.data_ptr(), self.n,
                                                             self.k, self.block, out.data_ptr(), _lib.stream_ptr()),
                   "tiles_dequant")
        return out


class Int4Weight:
    """An N x K INT4 asymmetric weight (the paper's comparator format,
    quantizer.py:232-244) in the W4A16 tile layout (128 x 128 tiles of 8192 B,
    `lpqt_int4_prepack`) with f16 scales and zero points per row (CGQ) or per
    block of `block` columns (FGQ, a multiple of 128).  The GEMM rebuilds
    Z + S * level in binary16 and runs the FP6 kernel's tcgen05 pipeline."""

    static = True

    def __init__(self, tiles, scales, zeros, n: int, k: int, block: int = 0):
        self.tiles = tiles
        self.scales = scales
        self.zeros = zeros
        self.n = int(n)
        self.k = int(k)
        self.block = int(block) if block and int(block) < int(k) else 0
        # (blocks that are not whole 128-k tiles dequantize but do not run the GEMM)
        self.params = (stage_params(scales, zeros, self.n, self.k, self.block)
                       if self.n and self.k and self.block % TILE == 0 else None)

    @classmethod
    def from_quantized(cls, q) -> "Int4Weight":
        from .errors import InvalidScheme, PayloadMismatch
        from .quantizer import cache_of, scale_block
        block = scale_block(q.scheme)
        if block and block < q.cols and block % TILE:
            raise InvalidScheme(f"FGQ block_size {block} is not a multiple of 128: outside the B200 GEMM path")
        cache = cache_of(q)
        if cache is not None and "weight" in cache:
            return cache["weight"]
        t = _lib.torch()
        nib = _lib.to_device(q.payload if _lib.is_torch(q.payload) else np.asarray(q.payload, np.uint8))
        nib = nib.reshape(-1).to(t.uint8)
        if nib.numel() != (q.rows * q.cols + 1) // 2:
            raise PayloadMismatch("payload does not hold rows*cols levels")

        def f16(a):
            return _lib.to_device(a if _lib.is_torch(a) else np.asarray(a, np.float16)).reshape(-1).to(t.float16)

        w = cls.from_nibbles(nib, f16(q.scales), f16(q.zero_points), q.rows, q.cols, block)
        if cache is not None:
            cache["weight"] = w
        return w

    @classmethod
    def from_nibbles(cls, nib, scales, zeros, n: int, k: int, block: int = 0) -> "Int4Weight":
        """CUDA nibble payload (packing.py INT4 order) + f16 scales / zero
        points -> tile layout (`lpqt_int4_prepack`)."""
        t = _lib.torch()
        lib = _lib.load()
        tiles = t.empty(int(lib.lpqt_int4_tiles_bytes(n, k)), dtype=t.uint8, device=nib.device)
        _lib.check(lib.lpqt_int4_prepack(nib.data_ptr(), n, k, tiles.data_ptr(), _lib.stream_ptr()), "int4_prepack")
        w = cls(tiles, scales, zeros, n, k, block)
        t.cuda.current_stream().synchronize()
        return w

    @property
    def nbytes(self) -> int:
        return int(self.tiles.numel() + 2 * self.scales.numel() + 2 * self.zeros.numel())

    def stream_bytes(self) -> int:
        """Algorithmic weight bytes per GEMM: 0.5 B/weight + 4 B per block."""
        return (self.n * self.k + 1) // 2 + 4 * int(self.scales.numel())


_SCHED_FLAGS = {"auto": 0, "streamk": 2, "cluster": 4, "single": 8, "pair": 16}
# weight rebuild in the GEMM: "cvt" = the hardware e3m2 converter (the product
# path); "bias_shift" / "naive" = the paper's software rebuilds with the
# per-weight binary16 scale (the Bias-Shift ablation; M <= 16)
_REBUILD_FLAGS = {"cvt": 0, "bias_shift": 32, "naive": 64}


def _sched_flags(sched: str) -> int:
    if sched not in _SCHED_FLAGS:
        raise ValueError(f"sched must be one of {sorted(_SCHED_FLAGS)}")
    return _SCHED_FLAGS[sched]


def plan(m: int, n: int, k: int, split_k: int = 0, sched: str = "auto") -> dict:
    """The launch plan the library picks: block_n (MMA N), splits (CTAs per
    tile), grid, stages, schedule ("streamk" / "cluster") and cluster size."""
    import ctypes
    out = (ctypes.c_int * 6)()
    _lib.check(_lib.load().lpqt_w6a16_plan_ex(m, n, k, split_k, _sched_flags(sched), out, 6), "plan")
    return {"block_n": out[0], "splits": out[1], "grid": out[2], "stages": out[3],
            "schedule": {0: "streamk", 1: "cluster", 2: "roundrobin", 3: "pair"}[out[4]], "cluster": out[5]}


def _launch(weight: Fp6Weight, xt, ldx: int, m: int, y, y_dtype: int, y_layout: int, ldy: int, split_k: int,
            sched: str = "auto", prefetch: "Fp6Weight | None" = None, prefetch_bytes: int = 0, workspace=None,
            rebuild: str = "cvt"):
    lib = _lib.load()
    ws_bytes = int(lib.lpqt_w6a16_workspace_bytes(m, weight.n, weight.k, split_k))
    if workspace is not None:
        # caller-owned: zero-initialised once by the caller, never shared
        # between concurrently running GEMMs (the tile counters self-reset)
        if workspace.numel() * workspace.element_size() < ws_bytes:
            from .errors import LpqtError
            raise LpqtError(f"workspace too small: {ws_bytes} bytes needed")
        ws = workspace.view(_lib.torch().uint8) if ws_bytes else None
    else:
        ws = _lib.Workspace.get(ws_bytes) if ws_bytes else None
    if rebuild not in _REBUILD_FLAGS:
        raise ValueError(f"rebuild must be one of {sorted(_REBUILD_FLAGS)}")
    flags = (_lib.LAUNCH_PDL if weight.static else 0) | _sched_flags(sched) | _REBUILD_FLAGS[rebuild]
    if getattr(weight, "wbits", 6) == 5:
        flags |= _lib.WEIGHTS_FP5
    if weight.block and weight.block % TILE and (isinstance(weight, Int4Weight) or not sub_tile_block(weight.block)
                                                 or m > 32):
        from .errors import InvalidScheme
        raise InvalidScheme(f"FGQ block_size {weight.block}: the B200 GEMM takes multiples of 128, or 16 / 32 / 64 "
                            f"at decode batches (M <= 32, FP6)")
    if isinstance(weight, Int4Weight):
        _lib.check(lib.lpqt_w4a16_linear_blocks(
            weight.tiles.data_ptr(), weight.params.data_ptr(), weight.block, xt.data_ptr(),
            ldx, m, weight.n, weight.k, y.data_ptr(), y_dtype, y_layout, ldy, split_k, _lib.ptr(ws),
            ws.numel() if ws is not None else 0, flags, _lib.stream_ptr()), "w4a16_linear")
        return
    nxt = None
    if prefetch is not None and getattr(prefetch, "wbits", 6) == 6:
        # the next launch is assumed to use the same batch and the automatic schedule
        nxt = _lib.NextLinear(prefetch.tiles.data_ptr(), m, prefetch.n, prefetch.k, 0, 0, int(prefetch_bytes))
    _lib.check(lib.lpqt_w6a16_linear_blocks(
        weight.tiles.data_ptr(), weight.gemm_scales().data_ptr(), weight.block, xt.data_ptr(), ldx, m, weight.n,
        weight.k,
        y.data_ptr(), y_dtype, y_layout, ldy, split_k, _lib.ptr(ws), ws.numel() if ws is not None else 0,
        flags, None if nxt is None else ctypes.byref(nxt), _lib.stream_ptr()), "w6a16_linear")


def stage_activations(X, k: int):
    """Reference-layout activations X[K, M] (any float dtype, numpy or CUDA)
    -> Xt[M, round_up(K, 8)] fp16 on the GPU (lpqt_stage_activations)."""
    t = _lib.torch()
    xd = X if _lib.is_torch(X) else np.asarray(X)
    if not _lib.is_torch(xd) and xd.dtype not in (np.float64, np.float32, np.float16):
        xd = xd.astype(np.float64)
    xd = _lib.to_device(xd)
    if xd.dtype not in (t.float64, t.float32, t.float16, t.bfloat16):
        xd = xd.to(t.float64)
    m = int(xd.shape[1])
    kp = _round_up(max(k, 1), 8)
    xt = t.empty((m, kp), dtype=t.float16, device=xd.device)
    _lib.check(_lib.load().lpqt_stage_activations(xd.data_ptr(), _lib.dtype_code(xd.dtype), k, m, m,
                                                  xt.data_ptr(), kp, _lib.stream_ptr()), "stage_activations")
    return xt, kp


def gemm_nm(weight: Fp6Weight, xt, ldx: int, m: int, out=None, split_k: int = 0, sched: str = "auto"):
    """Y[N, M] f32 = W_hat @ X in the reference layout (gemm.py:65-94)."""
    t = _lib.torch()
    y = out if out is not None else t.empty((weight.n, m), dtype=t.float32, device=xt.device)
    if m and weight.n:
        _launch(weight, xt, ldx, m, y, _lib.F32, _lib.Y_NM, m, split_k, sched)
    return y


def workspace_bytes(m: int, weight, split_k: int = 0) -> int:
    """Bytes of zeroed scratch a call at batch `m` needs (0: none)."""
    return int(_lib.load().lpqt_w6a16_workspace_bytes(m, weight.n, weight.k, split_k))


def w6a16_linear(x, weight: Fp6Weight, out=None, out_dtype=None, split_k: int = 0, sched: str = "auto",
                 prefetch: "Fp6Weight | None" = None, prefetch_bytes: int = 0, workspace=None, rebuild: str = "cvt"):
    """y = x @ W_hat^T for x[..., K] (CUDA, fp16 preferred) -> y[..., N].

    x is the K-major B operand as is when it is contiguous fp16 with K % 8 ==
    0; otherwise it is cast / padded once.  out_dtype: fp16 (default for
    fp16 x), bf16 or fp32; a given `out` must be a contiguous CUDA tensor of
    shape [..., N] and its dtype decides the output type.  prefetch: the
    weight of the linear that runs next on this stream (same batch); this
    launch's drain pulls its first bytes into L2 (lpqt_w6a16_linear_pf).
    workspace: optional caller-owned zeroed uint8 CUDA buffer of at least
    `workspace_bytes(m, weight)` bytes (default: one per stream, _lib.Workspace).
    rebuild: "cvt" (default, hardware e3m2 converter, S applied in fp32 after
    the contraction) or the paper's ablation rebuilds "bias_shift" / "naive"
    (software rebuild x per-weight binary16 scale; CGQ FP6, M <= 16).
    """
    t = _lib.torch()
    if x.shape[-1] != weight.k:
        raise ShapeError(f"inner dimensions differ: weights K={weight.k}, activations K={x.shape[-1]}")
    if not (_lib.is_torch(x) and x.is_cuda and x.device == weight.tiles.device):
        # (the kernel reads x by address: a host or other-device tensor must not reach it)
        raise InvalidInput(f"activations must be a CUDA tensor on the weight's device {weight.tiles.device}")
    lead = tuple(x.shape[:-1])
    x2 = x.reshape(-1, weight.k)
    m = int(x2.shape[0])
    if x2.dtype != t.float16:
        x2 = x2.to(t.float16)
    if weight.k % 8 or not x2.is_contiguous() or x2.data_ptr() % 16:
        kp = _round_up(weight.k, 8)
        xp = t.zeros((m, kp), dtype=t.float16, device=x2.device)
        xp[:, : weight.k] = x2
        x2, ldx = xp, kp
    else:
        ldx = weight.k
    codes = {t.float32: _lib.F32, t.float16: _lib.F16, t.bfloat16: _lib.BF16}
    if out is not None:
        if out.dtype not in codes:
            raise ShapeError(f"out dtype {out.dtype} unsupported (fp16, bf16, fp32)")
        if out_dtype is not None and out_dtype != out.dtype:
            raise ShapeError(f"out dtype {out.dtype} differs from out_dtype {out_dtype}")
        if tuple(out.shape) not in ((m, weight.n), lead + (weight.n,)) or not out.is_contiguous() \
                or out.device != x2.device:
            raise ShapeError(f"out must be a contiguous {tuple(lead) + (weight.n,)} tensor on {x2.device}, "
                             f"got {tuple(out.shape)}")
        odt = out.dtype
        y = out.view(m, weight.n)
    else:
        odt = out_dtype or (x.dtype if x.dtype in codes else t.float16)
        if odt not in codes:
            raise ShapeError(f"out_dtype {odt} unsupported (fp16, bf16, fp32)")
        y = t.empty((m, weight.n), dtype=odt, device=x2.device)
    if m and weight.n:
        if weight.k == 0:
            y.zero_()
        else:
            _launch(weight, x2, ldx, m, y, codes[odt], _lib.Y_MN, weight.n, split_k, sched, prefetch,
                    prefetch_bytes, workspace, rebuild)
    return y.reshape(*lead, weight.n)


class Fp6Linear:
    """torch.nn.Linear-style callable over an Fp6Weight (no bias)."""

    def __init__(self, weight: Fp6Weight):
        self.weight = weight
        self.in_features = weight.k
        self.out_features = weight.n

    @classmethod
    def from_dense(cls, W, bias_shift: bool = True) -> "Fp6Linear":
        return cls(Fp6Weight.quantize(W, bias_shift))

    def __call__(self, x, out=None):
        return w6a16_linear(x, self.weight, out=out)
