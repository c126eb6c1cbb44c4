"""`.lpqt` container: byte-exact serialization of quantized tensors and the
device loader that puts a container's FP6 weight straight into the GEMM's
tile layout.

Wire format (the reference's, container.py:1-19; little-endian, every
section zero-padded to 8 bytes):

    header   "LPQT" | version u16 | format u8 | granularity u8 | block u32 |
             rows u64 | cols u64 | bias_shift u8 | 7 zero bytes   (36 -> 40)
    scales   binary16 per block
    zeros    binary16 per block                     (INT4 only)
    folded   binary16 per block                     (bias_shift only)
    payload  minifloat: u64 len + seg4, u64 len + tail;  INT4: u64 len + nibbles

`write_lpqt` / `read_lpqt` / `read_raw` keep the reference's signatures,
return types and exceptions (container.py:50-200).  Parsing is host work on
a few header fields; `load_lpqt` then moves the whole stream to the GPU in
one copy and runs the prepack kernel on the payload in place
(`lpqt_fp6_prepack`), so a stored model never round-trips through numpy
code arrays.
"""

from __future__ import annotations

import struct

import numpy as np

from . import _lib
from .errors import (BadMagic, InvalidInput, InvariantViolation, LengthMismatch, TruncatedPayload,
                     UnsupportedVersion)
from .packing import PackedSegments, seg4_length, tail_length
from .quantizer import Granularity, QuantizedTensor, QuantScheme, TensorFormat, num_blocks

MAGIC = b"LPQT"
VERSION = 1
_HDR = struct.Struct("<4sHBBIQQB7s")          # 36 bytes, section padding -> 40
_FMT_CODE = {TensorFormat.FP6_E3M2: 0, TensorFormat.FP5_E3M1: 1, TensorFormat.INT4_ASYM: 2}
_GRAN_CODE = {Granularity.CGQ: 0, Granularity.FGQ: 1}
_CODE_FMT = {c: f for f, c in _FMT_CODE.items()}
_CODE_GRAN = {c: g for g, c in _GRAN_CODE.items()}
_RAW = {"f32le": np.dtype("<f4"), "f16le": np.dtype("<f2")}


def _pad(n: int) -> int:
    return -n % 8


def _host(a) -> np.ndarray:
    """numpy view of a field (torch CUDA tensors are copied to the host)."""
    if _lib.is_torch(a):
        return a.detach().cpu().numpy()
    return np.asarray(a)


# ------------------------------------------------------------------ writer
def write_lpqt(q: QuantizedTensor) -> bytes:
    """Serialize `q` to the canonical byte layout (container.py:50-77)."""
    scheme = q.scheme
    parts = [_HDR.pack(MAGIC, VERSION, _FMT_CODE[scheme.fmt], _GRAN_CODE[scheme.granularity],
                       scheme.block_size if scheme.granularity is Granularity.FGQ else 0,
                       q.rows, q.cols, int(bool(q.bias_shift)), bytes(7))]

    sections = [np.ascontiguousarray(_host(q.scales), dtype="<f2").tobytes()]
    if scheme.fmt is TensorFormat.INT4_ASYM:
        sections.append(np.ascontiguousarray(_host(q.zero_points), dtype="<f2").tobytes())
    if q.bias_shift:
        sections.append(np.ascontiguousarray(_host(q.folded_scales), dtype="<f2").tobytes())
    if isinstance(q.payload, PackedSegments):
        payload = [_host(q.payload.seg4).astype(np.uint8, copy=False).tobytes(),
                   _host(q.payload.seg_tail).astype(np.uint8, copy=False).tobytes()]
    else:
        payload = [_host(q.payload).astype(np.uint8, copy=False).tobytes()]
    out = bytearray(parts[0])
    out += bytes(_pad(len(out)))
    for raw in sections:
        out += raw
        out += bytes(_pad(len(out)))
    for raw in payload:
        out += struct.pack("<Q", len(raw)) + raw
        out += bytes(_pad(len(out)))
    return bytes(out)


# ------------------------------------------------------------------ reader
class _Cursor:
    """Sequential reader: short reads raise TruncatedPayload, section padding
    must be zero (container.py:80-101)."""

    def __init__(self, data: bytes):
        self.buf = memoryview(data)
        self.pos = 0

    def bytes(self, n: int) -> memoryview:
        have = len(self.buf) - self.pos
        if n > have:
            raise TruncatedPayload(f"need {n} bytes at offset {self.pos}, have {have}")
        view = self.buf[self.pos:self.pos + n]
        self.pos += n
        return view

    def pad(self) -> None:
        if any(self.bytes(_pad(self.pos))):
            raise InvariantViolation("section padding is not zero")

    def u64(self) -> int:
        return struct.unpack("<Q", self.bytes(8))[0]

    def f16(self, count: int) -> tuple[int, np.ndarray]:
        off = self.pos
        arr = np.frombuffer(self.bytes(2 * count), dtype="<f2")
        self.pad()
        return off, arr


def _parse(data: bytes):
    """Validate a container and locate its sections -> (header dict, views,
    byte offsets).  Checks and their order follow container.py:108-185."""
    cur = _Cursor(data)
    magic, version, fcode, gcode, block, rows, cols, bias, reserved = _HDR.unpack(cur.bytes(_HDR.size))
    if magic != MAGIC:
        raise BadMagic(f"bad container magic {bytes(magic)!r}")
    if version != VERSION:
        raise UnsupportedVersion(f"container version {version} not supported")
    if fcode not in _CODE_FMT:
        raise InvariantViolation(f"unknown format code {fcode}")
    if gcode not in _CODE_GRAN:
        raise InvariantViolation(f"unknown granularity code {gcode}")
    if bias not in (0, 1):
        raise InvariantViolation(f"bias_shift flag must be 0 or 1, got {bias}")
    if any(reserved):
        raise InvariantViolation("reserved header bytes are not zero")
    cur.pad()
    fmt, gran = _CODE_FMT[fcode], _CODE_GRAN[gcode]
    if gran is Granularity.CGQ and block != 0:
        raise InvariantViolation("CGQ containers must store block_size 0")
    if gran is Granularity.FGQ and block < 1:
        raise InvariantViolation("FGQ containers need block_size >= 1")
    if fmt is TensorFormat.INT4_ASYM and bias:
        raise InvariantViolation("bias shift is not defined for INT4 payloads")
    scheme = QuantScheme(granularity=gran, fmt=fmt, block_size=block)
    nb = num_blocks(rows, cols, scheme)

    def positive_finite(a: np.ndarray) -> bool:
        b = a.view(np.uint16)
        return bool(np.all(((b & 0x8000) == 0) & ((b & 0x7FFF) != 0) & ((b & 0x7C00) != 0x7C00)))

    off = {}
    off["scales"], scales = cur.f16(nb)
    if nb and not positive_finite(scales):
        raise InvariantViolation("scales must be positive and finite")
    zeros = folded = None
    if fmt is TensorFormat.INT4_ASYM:
        off["zeros"], zeros = cur.f16(nb)
        if nb and not np.all((zeros.view(np.uint16) & 0x7C00) != 0x7C00):
            raise InvariantViolation("zero points must be finite")
    if bias:
        off["folded"], folded = cur.f16(nb)
        if nb and not positive_finite(folded):
            raise InvariantViolation("folded scales must be positive and finite")
    n = rows * cols
    mf = fmt.minifloat
    if mf is not None:
        want = {"seg4": seg4_length(n), "tail": tail_length(mf, n)}
        noun = "codes"
    else:
        want = {"nibbles": (n + 1) // 2}
        noun = "levels"
    payload = {}
    for key, length in want.items():
        got = cur.u64()
        if got != length:
            label = {"seg4": "seg4", "tail": "tail", "nibbles": "nibble"}[key]
            raise InvariantViolation(f"{label} length {got} does not match {n} {noun}")
        off[key] = cur.pos
        payload[key] = np.frombuffer(cur.bytes(length), dtype=np.uint8)
        cur.pad()
    if cur.pos != len(data):
        raise InvariantViolation(f"{len(data) - cur.pos} trailing bytes after payload")
    hdr = {"rows": rows, "cols": cols, "scheme": scheme, "bias_shift": bool(bias)}
    return hdr, {"scales": scales, "zeros": zeros, "folded": folded, **payload}, off


def read_lpqt(data: bytes) -> QuantizedTensor:
    """Parse and validate a container (exact inverse of write_lpqt;
    container.py:108-185).  Fields are fresh numpy arrays."""
    hdr, v, _ = _parse(data)
    if "seg4" in v:
        payload = PackedSegments(v["seg4"].copy(), v["tail"].copy(), hdr["rows"] * hdr["cols"])
    else:
        payload = v["nibbles"].copy()
    return QuantizedTensor(rows=hdr["rows"], cols=hdr["cols"], scheme=hdr["scheme"], scales=v["scales"].copy(),
                           zero_points=None if v["zeros"] is None else v["zeros"].copy(), payload=payload,
                           bias_shift=hdr["bias_shift"],
                           folded_scales=None if v["folded"] is None else v["folded"].copy())


def read_raw(data: bytes, rows: int, cols: int, dtype: str) -> np.ndarray:
    """Headerless row-major dense tensor -> f64 [rows, cols] (container.py:191-200)."""
    if dtype not in _RAW:
        raise InvalidInput(f"unknown raw dtype {dtype!r}")
    dt = _RAW[dtype]
    if len(data) != rows * cols * dt.itemsize:
        raise LengthMismatch(f"raw stream of {len(data)} bytes does not hold {rows}x{cols} {dtype}")
    return np.frombuffer(data, dtype=dt).astype(np.float64).reshape(rows, cols)


# ------------------------------------------------------------------ device loader
def load_lpqt(data: bytes):
    """Container stream -> weight resident in HBM in the GEMM's tile layout.

    The stream is validated on the host (header fields, section lengths, the
    reference's scale checks), copied to the GPU once from pinned memory, and
    the prepack kernel reads the payload in place from the device copy:
    FP6 / FP5 (CGQ or FGQ) -> `Fp6Weight` (`lpqt_fp6_prepack` /
    `lpqt_fp5_prepack`), INT4 -> `Int4Weight` (`lpqt_int4_prepack`).
    """
    from .linear import Fp6Weight, Int4Weight
    from .quantizer import _require_path, scale_block
    hdr, _, off = _parse(data)
    scheme = hdr["scheme"]
    t = _lib.torch()
    rows, cols = hdr["rows"], hdr["cols"]
    nb = num_blocks(rows, cols, scheme)
    host = t.frombuffer(bytearray(data), dtype=t.uint8).pin_memory()
    blob = host.to(_lib.device(), non_blocking=True)
    # scales / zeros / folded are kept as views into the device copy of the
    # stream; the payload is only read by the prepack
    scales = blob[off["scales"]:off["scales"] + 2 * nb].view(t.float16)
    if scheme.fmt is TensorFormat.INT4_ASYM:
        zeros = blob[off["zeros"]:off["zeros"] + 2 * nb].view(t.float16)
        nib = blob[off["nibbles"]:off["nibbles"] + (rows * cols + 1) // 2]
        return Int4Weight.from_nibbles(nib, scales, zeros, rows, cols, block=scale_block(scheme))
    _require_path(scheme)
    folded = blob[off["folded"]:off["folded"] + 2 * nb].view(t.float16) if hdr["bias_shift"] else None
    seg4 = blob[off["seg4"]:off["seg4"] + seg4_length(rows * cols)]
    tail = blob[off["tail"]:off["tail"] + tail_length(scheme.fmt.minifloat, rows * cols)]
    fmt = "fp5" if scheme.fmt.minifloat.mantissa_bits == 1 else "fp6"
    return Fp6Weight.from_planes(seg4, tail, scales, rows, cols, folded, block=scale_block(scheme), fmt=fmt)
