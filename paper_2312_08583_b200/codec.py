"""FP6 (e3m2) and FP5 (e3m1) code spaces — reference codec.py:20-151.

Format descriptors and the value tables are static metadata and are built
here; the RTN encoder (`encode_rtn_array`, the quantizer's inner loop,
codec.py:116-132) runs on the GPU (`lpqt_fp6_encode_rtn` / `lpqt_fp5_encode_rtn`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib
from .errors import InvalidCode, InvalidInput, InvalidScheme


@dataclass(frozen=True)
class MiniFloatFormat:
    """Static description of a low-bit minifloat (codec.py:20-45)."""

    name: str
    exponent_bits: int
    mantissa_bits: int
    stored_bias: int
    total_bits: int
    max_value: float

    @property
    def code_count(self) -> int:
        return 1 << self.total_bits

    @property
    def sign_shift(self) -> int:
        return self.total_bits - 1

    @property
    def mantissa_mask(self) -> int:
        return (1 << self.mantissa_bits) - 1

    @property
    def exponent_mask(self) -> int:
        return (1 << self.exponent_bits) - 1


FP6_E3M2 = MiniFloatFormat("FP6_E3M2", 3, 2, 3, 6, 28.0)
FP5_E3M1 = MiniFloatFormat("FP5_E3M1", 3, 1, 3, 5, 24.0)
MINIFLOAT_FORMATS = (FP6_E3M2, FP5_E3M1)


def kernel_prefix(fmt: MiniFloatFormat) -> str:
    """C-ABI family of a format: lpqt_fp6_* (4 + 2) or lpqt_fp5_* (4 + 1)."""
    if fmt == FP6_E3M2:
        return "lpqt_fp6"
    if fmt == FP5_E3M1:
        return "lpqt_fp5"
    raise InvalidScheme(f"{fmt.name} is not a format of this library (FP6_E3M2, FP5_E3M1)")



def decode(fmt: MiniFloatFormat, code: int) -> float:
    """Exact value of a code: normal (1 + M/2^m) 2^(E-b), subnormal
    (M/2^m) 2^(1-b), sign kept on zero (codec.py:63-82)."""
    code = int(code)
    if not 0 <= code < fmt.code_count:
        raise InvalidCode(f"code {code:#x} does not fit {fmt.total_bits} bits")
    neg = (code >> fmt.sign_shift) & 1
    e = (code >> fmt.mantissa_bits) & fmt.exponent_mask
    m = code & fmt.mantissa_mask
    frac = m / (1 << fmt.mantissa_bits)
    mag = math.ldexp(frac, 1 - fmt.stored_bias) if e == 0 else math.ldexp(1.0 + frac, e - fmt.stored_bias)
    return -mag if neg else mag


@lru_cache(maxsize=None)
def value_table(fmt: MiniFloatFormat) -> np.ndarray:
    """All decoded values indexed by code, float64 (codec.py:99-105)."""
    t = np.array([decode(fmt, c) for c in range(fmt.code_count)], dtype=np.float64)
    t.setflags(write=False)
    return t


@lru_cache(maxsize=None)
def value_table_f16(fmt: MiniFloatFormat) -> np.ndarray:
    """Same table in binary16 — exact (codec.py:108-113)."""
    t = value_table(fmt).astype(np.float16)
    t.setflags(write=False)
    return t


def codebook(fmt: MiniFloatFormat) -> list[tuple[int, float]]:
    """(code, value) pairs ordered by code bits (codec.py:149-151)."""
    return [(c, decode(fmt, c)) for c in range(fmt.code_count)]


def encode_rtn_array(fmt: MiniFloatFormat, x):
    """Round-to-nearest encode on the GPU (codec.py:116-132).

    Ties go to the even magnitude index, values beyond the format's max_value
    (28 FP6, 24 FP5) saturate, -0.0
    encodes to code 0.  numpy / array-like in -> numpy uint8 out; a torch
    tensor in -> a uint8 tensor on the GPU.  Non-finite input raises
    InvalidInput.
    """
    prefix = kernel_prefix(fmt)
    t = _lib.torch()
    torch_in = _lib.is_torch(x)
    if torch_in:
        src = x
        if src.dtype not in (t.float64, t.float32, t.float16, t.bfloat16):
            src = src.to(t.float64)
        shape = tuple(src.shape)
        src = src.to(_lib.device()).contiguous()
    else:
        a = np.asarray(x)
        if a.dtype not in (np.float64, np.float32, np.float16):
            a = a.astype(np.float64)
        shape = a.shape
        src = _lib.to_device(a)
    n = src.numel()
    codes = t.empty(n, dtype=t.uint8, device=src.device)
    if n:
        flags = _lib.Flags()
        _lib.check(getattr(_lib.load(), prefix + "_encode_rtn")(
            src.data_ptr(), _lib.dtype_code(src.dtype), n, codes.data_ptr(), flags.ptr, _lib.stream_ptr()),
            "encode_rtn_array")
        if flags.value():
            raise InvalidInput("cannot encode non-finite values")
    codes = codes.reshape(shape)
    return codes if torch_in else codes.cpu().numpy()


def encode_rtn(fmt: MiniFloatFormat, x: float) -> int:
    """Scalar form of :func:`encode_rtn_array` (codec.py:135-146)."""
    if not math.isfinite(x):
        raise InvalidInput(f"cannot encode non-finite value {x!r}")
    return int(encode_rtn_array(fmt, np.array([x], dtype=np.float64))[0])
