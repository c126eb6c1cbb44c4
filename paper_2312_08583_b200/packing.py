"""Canonical 4+2 bit-split planes — reference packing.py:24-141.

`pack`/`unpack` run on the GPU (`lpqt_fp6_pack` / `lpqt_fp6_unpack`) and are
byte-identical to the reference: code i puts c>>2 in nibble i of `seg4`
(even index low) and c&3 in 2-bit lane i of `seg_tail`, both zero-padded to a
4-byte multiple.  The GEMM's own tile layout is derived from these planes by
`linear.prepack`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .codec import FP6_E3M2, MiniFloatFormat, kernel_prefix
from .errors import InvalidCode, InvalidScheme, PayloadMismatch


def _align4(n: int) -> int:
    return (n + 3) // 4 * 4


def seg4_length(code_count: int) -> int:
    """Bytes of the 4-bit plane (packing.py:28-30)."""
    return _align4((code_count + 1) // 2)


def tail_length(fmt: MiniFloatFormat, code_count: int) -> int:
    """Bytes of the tail plane (packing.py:33-36)."""
    return _align4((code_count * fmt.mantissa_bits + 7) // 8)


@dataclass(frozen=True)
class PackedSegments:
    """The two planes holding one code stream (packing.py:39-45).  Arrays
    are numpy on the numpy API and CUDA tensors on the torch API."""

    seg4: object
    seg_tail: object
    code_count: int


def split_code(fmt: MiniFloatFormat, code: int) -> tuple[int, int]:
    """(sign+exponent nibble, mantissa bits) of one code (packing.py:48-53)."""
    code = int(code)
    if not 0 <= code < fmt.code_count:
        raise InvalidCode(f"code {code:#x} does not fit {fmt.total_bits} bits")
    return code >> fmt.mantissa_bits, code & fmt.mantissa_mask


def _codes_to_device(fmt: MiniFloatFormat, codes):
    t = _lib.torch()
    if _lib.is_torch(codes):
        c = codes.reshape(-1)
        if c.dtype != t.uint8:
            if c.numel() and (int(c.min()) < 0 or int(c.max()) >= fmt.code_count):
                raise InvalidCode(f"codes must fit {fmt.total_bits} bits")
            c = c.to(t.uint8)
        return c.to(_lib.device()).contiguous(), True
    a = np.asarray(codes).reshape(-1)
    if a.dtype != np.uint8:
        if a.size and (a.min() < 0 or a.max() >= fmt.code_count):
            raise InvalidCode(f"codes must fit {fmt.total_bits} bits")
        a = a.astype(np.uint8)
    return _lib.to_device(a), False


def pack_device(codes_dev, n: int, fmt: MiniFloatFormat = FP6_E3M2):
    """codes (uint8 CUDA tensor, n) -> (seg4, tail) CUDA tensors."""
    t = _lib.torch()
    seg4 = t.empty(seg4_length(n), dtype=t.uint8, device=codes_dev.device)
    tail = t.empty(tail_length(fmt, n), dtype=t.uint8, device=codes_dev.device)
    if tail.numel():
        flags = _lib.Flags()
        _lib.check(getattr(_lib.load(), kernel_prefix(fmt) + "_pack")(
            codes_dev.data_ptr(), n, seg4.data_ptr(), tail.data_ptr(), flags.ptr, _lib.stream_ptr()), "pack")
        if flags.value():
            raise InvalidCode(f"codes must fit {fmt.total_bits} bits")
    return seg4, tail


def unpack_device(seg4, tail, n: int, fmt: MiniFloatFormat = FP6_E3M2):
    t = _lib.torch()
    codes = t.empty(n, dtype=t.uint8, device=seg4.device)
    if n:
        _lib.check(getattr(_lib.load(), kernel_prefix(fmt) + "_unpack")(
            seg4.data_ptr(), tail.data_ptr(), n, codes.data_ptr(), _lib.stream_ptr()), "unpack")
    return codes


def pack(fmt: MiniFloatFormat, codes) -> PackedSegments:
    """Pack a code stream into the canonical planes (packing.py:63-90)."""
    kernel_prefix(fmt)
    c, torch_in = _codes_to_device(fmt, codes)
    n = c.numel()
    seg4, seg2 = pack_device(c, n, fmt)
    if torch_in:
        return PackedSegments(seg4, seg2, n)
    return PackedSegments(seg4.cpu().numpy(), seg2.cpu().numpy(), n)


def unpack(fmt: MiniFloatFormat, segments: PackedSegments):
    """Recover the first `code_count` codes; pad bits ignored (packing.py:93-118)."""
    kernel_prefix(fmt)
    n = int(segments.code_count)
    torch_in = _lib.is_torch(segments.seg4)
    s4 = segments.seg4 if torch_in else np.asarray(segments.seg4, dtype=np.uint8)
    s2 = segments.seg_tail if torch_in else np.asarray(segments.seg_tail, dtype=np.uint8)
    n4 = s4.numel() if torch_in else s4.size
    n2 = s2.numel() if torch_in else s2.size
    if n4 != seg4_length(n) or n2 != tail_length(fmt, n):
        raise PayloadMismatch(f"segment lengths ({n4}, {n2}) inconsistent with code count {n}")
    d4 = _lib.to_device(s4).reshape(-1)
    d2 = _lib.to_device(s2).reshape(-1)
    codes = unpack_device(d4, d2, n, fmt)
    return codes if torch_in else codes.cpu().numpy()


def pack_int4(levels):
    """INT4 levels -> nibbles, two per byte, even index in the low nibble
    (packing.py:121-129), on the GPU.  InvalidCode outside [0, 15]."""
    t = _lib.torch()
    torch_in = _lib.is_torch(levels)
    if torch_in:
        lv = levels.reshape(-1)
        if lv.numel() and (int(lv.min()) < 0 or int(lv.max()) > 15):
            raise InvalidCode("INT4 levels must lie in [0, 15]")
        lv = lv.to(_lib.device()).to(t.uint8).contiguous()
    else:
        a = np.asarray(levels).reshape(-1)
        if a.size and (a.min() < 0 or a.max() > 15):
            raise InvalidCode("INT4 levels must lie in [0, 15]")
        lv = _lib.to_device(a.astype(np.uint8))
    n = lv.numel()
    out = t.empty((n + 1) // 2, dtype=t.uint8, device=lv.device)
    if n:
        flags = _lib.Flags()
        _lib.check(_lib.load().lpqt_int4_pack(lv.data_ptr(), n, out.data_ptr(), flags.ptr, _lib.stream_ptr()),
                   "pack_int4")
        if flags.value():
            raise InvalidCode("INT4 levels must lie in [0, 15]")
    return out if torch_in else out.cpu().numpy()


def unpack_int4(data, count: int):
    """Recover `count` INT4 levels from a nibble array (packing.py:132-141)."""
    t = _lib.torch()
    torch_in = _lib.is_torch(data)
    d = data.reshape(-1) if torch_in else np.asarray(data, dtype=np.uint8).reshape(-1)
    size = d.numel() if torch_in else d.size
    if size != (count + 1) // 2:
        raise PayloadMismatch(f"nibble array of {size} bytes cannot hold {count} levels")
    dd = _lib.to_device(d).to(t.uint8).contiguous()
    out = t.empty(count, dtype=t.uint8, device=dd.device)
    if count:
        _lib.check(_lib.load().lpqt_int4_unpack(dd.data_ptr(), count, out.data_ptr(), _lib.stream_ptr()),
                   "unpack_int4")
    return out if torch_in else out.cpu().numpy()
