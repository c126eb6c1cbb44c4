"""Per-output-channel FP6 quantization — reference quantizer.py:1-320.

`quantize_tensor` for CGQ x FP6_E3M2 (the north-star path: RTN, one scale per
weight row) runs as one fused GPU kernel (`lpqt_fp6_quantize_pack`): row
max|w|, S = RN_f16(peak/28), fold S*2^12, RTN codes of W/S and the canonical
4+2 planes, bit-exact with the reference for f64/f32/f16/bf16 input.
`dequantize_tensor` is the GPU `lpqt_fp6_dequantize_tensor` (f64 exact).
FP6 (4+2) and FP5 (4+1) quantize under CGQ (one scale per output row) or FGQ
(one per block of block_size columns; the GEMM needs blocks of whole 128-k
tiles); INT4 asymmetric (the paper's comparator) quantizes per row or block
too, with zero points, and runs the fused W4A16 GEMM (`linear.Int4Weight`).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .codec import FP5_E3M1, FP6_E3M2, MiniFloatFormat, kernel_prefix
from .errors import (InvalidInput, InvalidScheme, PathUnavailable, PayloadMismatch,
                     ShapeError)
from .packing import PackedSegments, seg4_length, tail_length


class Granularity(Enum):
    CGQ = "cgq"
    FGQ = "fgq"


class TensorFormat(Enum):
    FP6_E3M2 = "fp6"
    FP5_E3M1 = "fp5"
    INT4_ASYM = "int4"

    @property
    def minifloat(self) -> MiniFloatFormat | None:
        if self is TensorFormat.FP6_E3M2:
            return FP6_E3M2
        if self is TensorFormat.FP5_E3M1:
            return FP5_E3M1
        return None


@dataclass(frozen=True)
class QuantScheme:
    """Granularity + format; `block_size` is FGQ-only (quantizer.py:46-52)."""

    granularity: Granularity
    fmt: TensorFormat
    block_size: int = 0


@dataclass(frozen=True)
class BlockParams:
    scale: np.float16
    zero_point: np.float16 | None = None


@dataclass(frozen=True)
class ErrorReport:
    mse: float
    max_abs_error: float
    sqnr_db: float


@dataclass(frozen=True)
class QuantizedTensor:
    """Reference fields (quantizer.py:70-83) plus a private device cache."""

    rows: int
    cols: int
    scheme: QuantScheme
    scales: object
    zero_points: object
    payload: object
    bias_shift: bool = False
    folded_scales: object = None
    device_cache: dict | None = field(default=None, compare=False, repr=False)

    @property
    def num_blocks(self) -> int:
        s = self.scales
        return int(s.numel() if _lib.is_torch(s) else np.asarray(s).size)


CGQ_FP6 = QuantScheme(Granularity.CGQ, TensorFormat.FP6_E3M2)


def _validate_scheme(scheme: QuantScheme) -> None:
    if scheme.granularity is Granularity.FGQ and scheme.block_size < 1:
        raise InvalidScheme(f"FGQ requires block_size >= 1, got {scheme.block_size}")


def _require_path(scheme: QuantScheme) -> None:
    """CGQ or FGQ x FP6_E3M2 / FP5_E3M1 (the formats this library runs on the GPU)."""
    _validate_scheme(scheme)
    if scheme.fmt.minifloat is None:
        raise InvalidScheme(
            f"{scheme.granularity.name} x {scheme.fmt.name} is outside the B200 path (FP6 / FP5, CGQ or FGQ)")


def scale_block(scheme: QuantScheme) -> int:
    """Columns per scale for the kernels: 0 = one scale per row (CGQ)."""
    return scheme.block_size if scheme.granularity is Granularity.FGQ else 0


def _require_gemm_path(scheme: QuantScheme, cols: int) -> None:
    """The GEMM applies FGQ scales per 128-k weight tile: blocks must be
    whole tiles (or span the row)."""
    _require_path(scheme)
    b = scale_block(scheme)
    if b and b < cols and b % 128:
        raise InvalidScheme(f"FGQ block_size {b} is not a multiple of 128: outside the B200 GEMM path")


def blocks_per_row(cols: int, scheme: QuantScheme) -> int:
    _validate_scheme(scheme)
    if cols == 0:
        return 0
    if scheme.granularity is Granularity.CGQ:
        return 1
    return -(-cols // scheme.block_size)


def block_widths(cols: int, scheme: QuantScheme) -> np.ndarray:
    """Widths of the blocks inside one row (quantizer.py:100-109)."""
    bpr = blocks_per_row(cols, scheme)
    if scheme.granularity is Granularity.CGQ:
        return np.array([cols] * bpr, dtype=np.int64)
    d = scheme.block_size
    w = np.full(bpr, d, dtype=np.int64)
    if bpr and cols % d:
        w[-1] = cols % d
    return w


def num_blocks(rows: int, cols: int, scheme: QuantScheme) -> int:
    if rows == 0 or cols == 0:
        return 0
    return rows * blocks_per_row(cols, scheme)


def partition_blocks(rows: int, cols: int, scheme: QuantScheme) -> list[tuple[int, int, int]]:
    """(row, col_start, col_end) per block, row-major (quantizer.py:118-130)."""
    if rows < 0 or cols < 0:
        raise InvalidScheme("dimensions must be non-negative")
    _validate_scheme(scheme)
    widths = block_widths(cols, scheme)
    bounds = np.concatenate([[0], np.cumsum(widths)])
    return [(r, int(bounds[j]), int(bounds[j + 1]))
            for r in range(rows if cols else 0) for j in range(len(widths))]


# ---------------------------------------------------------------------------
def _weights_to_device(W):
    """-> (2-D CUDA tensor in a kernel dtype, torch_in)."""
    t = _lib.torch()
    if _lib.is_torch(W):
        if W.dim() != 2:
            raise ShapeError(f"expected a 2-D matrix, got shape {tuple(W.shape)}")
        w = W
        if w.dtype not in (t.float64, t.float32, t.float16, t.bfloat16):
            w = w.to(t.float64)
        return w.to(_lib.device()).contiguous(), True
    a = np.asarray(W)
    if a.ndim != 2:
        raise ShapeError(f"expected a 2-D matrix, got shape {a.shape}")
    if a.dtype not in (np.float64, np.float32, np.float16):
        a = a.astype(np.float64)
    return _lib.to_device(a), False


def quantize_device(w, bias_shift: bool = True, block: int = 0, fmt: MiniFloatFormat = FP6_E3M2):
    """GPU quantize of a 2-D CUDA tensor -> dict of CUDA tensors
    {scales, folded, seg4, seg2} (canonical planes, flat index r*K + k;
    scales one per row, or per block of `block` columns row-major)."""
    t = _lib.torch()
    n, k = (int(v) for v in w.shape)
    dev = w.device
    nb = n * (-(-k // block) if block and block < k else 1)
    scales = t.empty(nb, dtype=t.float16, device=dev)
    folded = t.empty(nb, dtype=t.float16, device=dev) if bias_shift else None
    nk = n * k
    seg4 = t.empty(seg4_length(nk), dtype=t.uint8, device=dev)
    seg2 = t.empty(tail_length(fmt, nk), dtype=t.uint8, device=dev)
    if seg4.numel():
        seg4[-4:].zero_()
        seg2[-4:].zero_()
    flags = _lib.Flags()
    _lib.check(getattr(_lib.load(), kernel_prefix(fmt) + "_quantize_pack_blocks")(
        w.data_ptr(), _lib.dtype_code(w.dtype), n, k, k, int(block), int(bool(bias_shift)), scales.data_ptr(),
        _lib.ptr(folded), seg4.data_ptr(), seg2.data_ptr(), flags.ptr, _lib.stream_ptr()), "quantize_tensor")
    flags.raise_if_set()
    return {"scales": scales, "folded": folded, "seg4": seg4, "seg2": seg2}


def quantize_tensor(W, scheme: QuantScheme, bias_shift: bool = False) -> QuantizedTensor:
    """Quantize a dense N x K matrix (quantizer.py:189-248) on the GPU.

    numpy / array-like in -> numpy fields (the reference's types); a torch
    tensor in -> CUDA tensor fields.  Errors: ShapeError (not 2-D),
    InvalidInput (non-finite, scale overflows binary16), ScaleOverflow
    (bias_shift and S * 2^12 > 65504), InvalidScheme (outside CGQ x FP6).
    """
    _validate_scheme(scheme)
    if bias_shift and scheme.fmt.minifloat is None:
        raise InvalidScheme("bias shift applies to minifloat formats only")
    if scheme.fmt is TensorFormat.INT4_ASYM:
        return _quantize_int4(W, scheme)
    _require_path(scheme)
    w, torch_in = _weights_to_device(W)
    n, k = (int(v) for v in w.shape)
    t = _lib.torch()
    if n == 0 or k == 0:
        if torch_in:
            e16 = t.zeros(0, dtype=t.float16, device=w.device)
            e8 = t.zeros(0, dtype=t.uint8, device=w.device)
            return QuantizedTensor(n, k, scheme, e16, None, PackedSegments(e8, e8.clone(), 0), bias_shift,
                                   e16.clone() if bias_shift else None)
        e16 = np.zeros(0, dtype=np.float16)
        e8 = np.zeros(0, dtype=np.uint8)
        return QuantizedTensor(n, k, scheme, e16, None, PackedSegments(e8, e8.copy(), 0), bias_shift,
                               e16.copy() if bias_shift else None)
    d = quantize_device(w, bias_shift, scale_block(scheme), scheme.fmt.minifloat)
    if torch_in:
        payload = PackedSegments(d["seg4"], d["seg2"], n * k)
        q = QuantizedTensor(n, k, scheme, d["scales"], None, payload, bias_shift, d["folded"], {})
    else:
        payload = PackedSegments(_frozen(d["seg4"]), _frozen(d["seg2"]), n * k)
        q = QuantizedTensor(n, k, scheme, _frozen(d["scales"]), None, payload, bias_shift,
                            None if d["folded"] is None else _frozen(d["folded"]), {})
    _bind_cache(q, {"scales": d["scales"], "seg4": d["seg4"], "seg2": d["seg2"]})
    return q


def _frozen(t):
    """CUDA tensor -> read-only numpy copy: the reference's QuantizedTensor is
    frozen, and the device cache below relies on host fields never changing
    in place (callers copy before editing, as the reference tests do)."""
    a = t.cpu().numpy()
    a.setflags(write=False)
    return a


def _fields_key(q: QuantizedTensor) -> tuple:
    """Identity (and, for torch fields, in-place version) of every field the
    device cache was derived from.  dataclasses.replace() shares the cache
    dict with the new tensor; its fields differ, so the key does too."""
    p = q.payload
    objs = (q.scales, q.zero_points, p, getattr(p, "seg4", None), getattr(p, "seg_tail", None))
    return (tuple((id(o), getattr(o, "_version", None) if _lib.is_torch(o) else None) for o in objs),
            q.rows, q.cols, q.scheme, getattr(p, "code_count", None))


def _bind_cache(q: QuantizedTensor, entries: dict) -> None:
    c = q.device_cache
    c.clear()
    c.update(entries)
    c["_key"] = _fields_key(q)
    # the key holds ids: keep the objects alive so an id cannot be reused
    c["_refs"] = (q.scales, q.zero_points, q.payload)


def cache_of(q: QuantizedTensor) -> dict | None:
    """The device cache of `q` if it still describes q's fields, else None
    (a replaced or in-place-modified tensor never sees stale device data)."""
    c = q.device_cache
    if c is None or c.get("_key") != _fields_key(q):
        return None
    return c


def compute_scale_fp(values, fmt: MiniFloatFormat) -> BlockParams:
    """Max-abs scale of one block (quantizer.py:156-163), via the GPU quantizer."""
    kernel_prefix(fmt)
    v = np.asarray(values, dtype=np.float64).ravel()
    if v.size == 0:
        raise InvalidInput("block must be non-empty")
    tf = TensorFormat.FP6_E3M2 if fmt == FP6_E3M2 else TensorFormat.FP5_E3M1
    q = quantize_tensor(v.reshape(1, -1), QuantScheme(Granularity.CGQ, tf), bias_shift=False)
    return BlockParams(scale=np.float16(q.scales[0]))


def _quantize_int4(W, scheme: QuantScheme) -> QuantizedTensor:
    """INT4 asymmetric (quantizer.py:232-244) on the GPU: per block zero
    point / scale, levels packed two per byte — the paper's comparator."""
    w, torch_in = _weights_to_device(W)
    n, k = (int(v) for v in w.shape)
    t = _lib.torch()
    block = scale_block(scheme)
    nb = num_blocks(n, k, scheme)
    scales = t.empty(nb, dtype=t.float16, device=w.device)
    zeros = t.empty(nb, dtype=t.float16, device=w.device)
    nib = t.zeros((n * k + 1) // 2, dtype=t.uint8, device=w.device)
    if n and k:
        flags = _lib.Flags()
        _lib.check(_lib.load().lpqt_int4_quantize_blocks(
            w.data_ptr(), _lib.dtype_code(w.dtype), n, k, k, block, scales.data_ptr(), zeros.data_ptr(),
            nib.data_ptr(), flags.ptr, _lib.stream_ptr()), "quantize_tensor")
        flags.raise_if_set()
    if torch_in:
        q = QuantizedTensor(n, k, scheme, scales, zeros, nib, False, None, {})
    else:
        q = QuantizedTensor(n, k, scheme, _frozen(scales), _frozen(zeros), _frozen(nib), False, None, {})
    _bind_cache(q, {})
    return q


def compute_affine_params_int4(values) -> BlockParams:
    """Zero point / scale of one INT4 block (quantizer.py:166-177), via the GPU quantizer."""
    v = np.asarray(values, dtype=np.float64).ravel()
    if v.size == 0:
        raise InvalidInput("block must be non-empty")
    q = _quantize_int4(v.reshape(1, -1), QuantScheme(Granularity.CGQ, TensorFormat.INT4_ASYM))
    return BlockParams(scale=np.float16(q.scales[0]), zero_point=np.float16(q.zero_points[0]))


def device_planes(q: QuantizedTensor):
    """(seg4, seg2, scales) of `q` as CUDA tensors (cached when built here)."""
    n = q.rows * q.cols
    if not isinstance(q.payload, PackedSegments) or q.payload.code_count != n:
        raise PayloadMismatch("payload does not hold rows*cols codes")
    c = cache_of(q)
    if c is not None and "seg4" in c:
        return c["seg4"], c["seg2"], c["scales"]
    s4 = _lib.to_device(q.payload.seg4).reshape(-1)
    s2 = _lib.to_device(q.payload.seg_tail).reshape(-1)
    if s4.numel() != seg4_length(n) or s2.numel() != tail_length(q.scheme.fmt.minifloat, n):
        raise PayloadMismatch("segment lengths inconsistent with rows*cols")
    t = _lib.torch()
    sc = q.scales if _lib.is_torch(q.scales) else np.asarray(q.scales, dtype=np.float16)
    sc = _lib.to_device(sc).reshape(-1).to(t.float16)
    return s4, s2, sc


def dequantize_tensor(q: QuantizedTensor, path: str = "naive"):
    """f64-exact reconstruction (quantizer.py:269-299) on the GPU."""
    torch_in = _lib.is_torch(q.scales)
    t = _lib.torch()
    if q.rows == 0 or q.cols == 0:
        return t.zeros((q.rows, q.cols), dtype=t.float64, device=_lib.device()) if torch_in \
            else np.zeros((q.rows, q.cols), dtype=np.float64)
    if q.num_blocks != num_blocks(q.rows, q.cols, q.scheme):
        raise PayloadMismatch("block parameter count does not match the scheme")
    if q.scheme.fmt is TensorFormat.INT4_ASYM:   # zero_point + scale * level, f64 (quantizer.py:296-298)
        nib = q.payload if _lib.is_torch(q.payload) else np.asarray(q.payload, dtype=np.uint8)
        if (nib.numel() if _lib.is_torch(nib) else nib.size) != (q.rows * q.cols + 1) // 2:
            raise PayloadMismatch("payload does not hold rows*cols levels")
        dn = _lib.to_device(nib).reshape(-1).to(t.uint8)
        ds = _lib.to_device(q.scales if _lib.is_torch(q.scales) else np.asarray(q.scales, np.float16)).to(t.float16)
        dz = _lib.to_device(q.zero_points if _lib.is_torch(q.zero_points)
                            else np.asarray(q.zero_points, np.float16)).to(t.float16)
        out = t.empty((q.rows, q.cols), dtype=t.float64, device=dn.device)
        _lib.check(_lib.load().lpqt_int4_dequantize_blocks(
            dn.data_ptr(), ds.data_ptr(), dz.data_ptr(), q.rows, q.cols, scale_block(q.scheme), out.data_ptr(),
            _lib.stream_ptr()), "dequantize_tensor")
        return out if torch_in else out.cpu().numpy()
    _require_path(q.scheme)
    if path == "naive":
        s4, s2, row_scale = device_planes(q)
        p = 0
    elif path == "bias_shift":
        if q.folded_scales is None:
            raise PathUnavailable("tensor carries no folded scales")
        s4, s2, _ = device_planes(q)
        f = q.folded_scales if _lib.is_torch(q.folded_scales) else np.asarray(q.folded_scales, np.float16)
        row_scale = _lib.to_device(f).reshape(-1).to(t.float16)
        p = 1
    else:
        raise ValueError(f"unknown dequantization path {path!r}")
    out = t.empty((q.rows, q.cols), dtype=t.float64, device=s4.device)
    _lib.check(getattr(_lib.load(), kernel_prefix(q.scheme.fmt.minifloat) + "_dequantize_tensor_blocks")(
        s4.data_ptr(), s2.data_ptr(), row_scale.data_ptr(), p, q.rows, q.cols, scale_block(q.scheme), out.data_ptr(),
        _lib.F64, _lib.stream_ptr()), "dequantize_tensor")
    return out if torch_in else out.cpu().numpy()


def error_report(W, W_hat) -> ErrorReport:
    """MSE / max-abs / SQNR between a tensor and its proxy (quantizer.py:302-320).
    A metrics utility, not on the compute path."""
    if _lib.is_torch(W):
        W = W.detach().cpu().numpy()
    if _lib.is_torch(W_hat):
        W_hat = W_hat.detach().cpu().numpy()
    W = np.asarray(W, dtype=np.float64)
    W_hat = np.asarray(W_hat, dtype=np.float64)
    if W.shape != W_hat.shape:
        raise ShapeError(f"shape mismatch: {W.shape} vs {W_hat.shape}")
    if W.size == 0:
        return ErrorReport(0.0, 0.0, float("inf"))
    err = W - W_hat
    mse = float(np.mean(err * err))
    sig = float(np.mean(W * W))
    sqnr = float("inf") if mse == 0.0 else (float("-inf") if sig == 0.0 else 10.0 * float(np.log10(sig / mse)))
    return ErrorReport(mse, float(np.max(np.abs(err))), sqnr)
