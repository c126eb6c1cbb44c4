"""Bias-shift dequantization — reference dequant.py:1-115.

The fold (S * 2^12, exact or ScaleOverflow) and both elementwise dequant
paths run on the GPU.  `compose_table_f16` is the static 64-entry bit table
sign<<15 | E<<10 | M<<8 (dequant.py:33-43) the kernels implement in-register.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

from . import _lib
from .codec import MiniFloatFormat, kernel_prefix
from .errors import InvalidInput
from .packing import PackedSegments, unpack

FOLD_SHIFT = 12  # binary16 bias 15 - stored bias 3 (dequant.py:30)


@lru_cache(maxsize=None)
def compose_table_f16(fmt: MiniFloatFormat) -> np.ndarray:
    """binary16 patterns of every code padded into the f16 fields (dequant.py:33-43)."""
    c = np.arange(fmt.code_count, dtype=np.uint16)
    sign = (c >> fmt.sign_shift) & 1
    e = (c >> fmt.mantissa_bits) & fmt.exponent_mask
    m = c & fmt.mantissa_mask
    t = ((sign << 15) | (e << 10) | (m << (10 - fmt.mantissa_bits))).astype(np.uint16).view(np.float16)
    t.setflags(write=False)
    return t


def _as_f16_device(x):
    t = _lib.torch()
    if _lib.is_torch(x):
        return x.to(_lib.device()).to(t.float16).contiguous(), True
    return _lib.to_device(np.asarray(x, dtype=np.float16)), False


def fold_scale_array(fmt: MiniFloatFormat, scales):
    """folded = S * 2^12 exactly; InvalidInput for non-positive / non-finite
    scales, ScaleOverflow above 65504 (dequant.py:61-69; the fold constant is
    2^12 for both formats: bias 15 - 3)."""
    kernel_prefix(fmt)
    t = _lib.torch()
    s, torch_in = _as_f16_device(scales)
    shape = tuple(s.shape)
    s = s.reshape(-1)
    out = t.empty_like(s)
    if s.numel():
        flags = _lib.Flags()
        _lib.check(_lib.load().lpqt_fp6_fold_scales(s.data_ptr(), s.numel(), out.data_ptr(), flags.ptr,
                                                    _lib.stream_ptr()), "fold_scale_array")
        flags.raise_if_set()
    out = out.reshape(shape)
    return out if torch_in else out.cpu().numpy()


def fold_scale(fmt: MiniFloatFormat, scale) -> np.float16:
    """Scalar :func:`fold_scale_array` (dequant.py:46-58)."""
    s = np.float16(scale)
    if not (float(s) > 0.0 and np.isfinite(float(s))):
        raise InvalidInput(f"scale must be a positive finite binary16, got {scale!r}")
    return np.float16(fold_scale_array(fmt, np.array([s], dtype=np.float16))[0])


def _elementwise(fn_name: str, codes, scale):
    t = _lib.torch()
    torch_in = _lib.is_torch(codes) or _lib.is_torch(scale)
    c = codes if _lib.is_torch(codes) else _lib.to_device(np.asarray(codes, dtype=np.uint8))
    c = c.to(_lib.device()).to(t.uint8)
    s, _ = _as_f16_device(scale)
    c, s = t.broadcast_tensors(c, s)
    c = c.contiguous()
    s = s.contiguous()
    out = t.empty(c.shape, dtype=t.float16, device=c.device)
    if out.numel():
        _lib.check(getattr(_lib.load(), fn_name)(c.data_ptr(), s.data_ptr(), out.numel(), out.data_ptr(),
                                                 _lib.stream_ptr()), fn_name)
    return out if torch_in else out.cpu().numpy()


def dequant_naive_array(fmt: MiniFloatFormat, codes, scale):
    """value_f16[c] * S in binary16 (dequant.py:72-79); broadcasts."""
    return _elementwise(kernel_prefix(fmt) + "_dequant_naive", codes, scale)


def dequant_bias_shift_array(fmt: MiniFloatFormat, codes, folded):
    """compose[c] * folded in binary16 (dequant.py:82-86); broadcasts."""
    return _elementwise(kernel_prefix(fmt) + "_dequant_bias_shift", codes, folded)


def dequant_naive(fmt: MiniFloatFormat, code: int, scale) -> np.float16:
    return np.float16(dequant_naive_array(fmt, np.array([code]), np.float16(scale))[0])


def dequant_bias_shift(fmt: MiniFloatFormat, code: int, folded) -> np.float16:
    return np.float16(dequant_bias_shift_array(fmt, np.array([code]), np.float16(folded))[0])


def dequant_block(fmt: MiniFloatFormat, segments: PackedSegments, scale, path: str = "naive",
                  folded_scale=None):
    """Dequantize one packed block to binary16 (dequant.py:100-115)."""
    codes = unpack(fmt, segments)
    if path == "naive":
        return dequant_naive_array(fmt, codes, np.float16(scale))
    if path == "bias_shift":
        folded = fold_scale(fmt, scale) if folded_scale is None else np.float16(folded_scale)
        return dequant_bias_shift_array(fmt, codes, folded)
    raise ValueError(f"unknown dequantization path {path!r}")
