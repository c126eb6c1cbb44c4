"""W6A16 GEMM API — reference gemm.py:1-122.

`gemm_quantized(wq, X)` (gemm.py:65-110) keeps the reference contract —
W_hat (N x K) times X (K x M) -> float32 N x M.  FP6 / FP5 per-row-scaled
weights with binary16-exact X run the tcgen05 W6A16 kernel (equal to the
reference up to fp32 summation order); every other call runs the
reference-order kernel (exact.cu), bit-identical to the reference.

`gemm_reference` / `gemm_dense` (f64 / f32 dense oracles, gemm.py:28-51) run
the same reference-order loop on the GPU (bit-identical);
`gemm_tolerance` / `compare_outputs` are the reference's error bounds.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import PayloadMismatch, ShapeError
from .linear import Fp6Weight, Int4Weight, gemm_nm, stage_activations
from .packing import unpack_device
from .quantizer import (ErrorReport, QuantizedTensor, TensorFormat, _require_gemm_path, _require_path,
                        device_planes, error_report, num_blocks, scale_block)


def _check_activation(X, k: int) -> None:
    if X.ndim != 2:
        raise ShapeError(f"activations must be 2-D, got shape {tuple(X.shape)}")
    if X.shape[0] != k:
        raise ShapeError(f"inner dimensions differ: weights K={k}, activations K={X.shape[0]}")


def _x32(X):
    """The reference's activation conversion, np.asarray(X, float32)
    (gemm.py:69): numpy stays on the host, torch on its device."""
    if _lib.is_torch(X):
        return X.to(_lib.torch().float32)
    return np.asarray(X, dtype=np.float32)


def _f16_exact(X32) -> bool:
    """Every activation is a binary16 value (then the A16 kernel sees
    exactly the reference's operands)."""
    if _lib.is_torch(X32):
        return bool((X32.half().float() == X32).all()) if X32.numel() else True
    return bool(np.array_equal(X32.astype(np.float16).astype(np.float32), X32))


def a16_path(wq: QuantizedTensor) -> bool:
    """Schemes the tcgen05 W6A16 kernel reproduces within the reference's
    tolerance: FP6 / FP5 with one scale per row (CGQ, or FGQ blocks spanning
    the row).  (INT4 and FGQ blocks run the reference-order kernel.)"""
    if wq.scheme.fmt.minifloat is None:
        return False
    b = scale_block(wq.scheme)
    return not b or b >= wq.cols


def gemm_quantized(wq: QuantizedTensor, X, split_k: int = 0, sched: str = "auto", exact: bool | None = None):
    """Y = W_hat @ X for a quantized N x K tensor and X (K x M) -> f32 (N x M),
    the reference contract (gemm.py:65-110).

    Two GPU kernels serve it:
    * the tcgen05 W6A16 GEMM (the product path): FP6 / FP5 with per-row
      scales and binary16-exact activations — Y = S * sum(value * x) with fp32
      tensor-core accumulation, equal to the reference up to summation order;
    * the reference-order kernel (`lpqt_gemm_exact_quantized`, exact.cu) for
      every other call — float32 activations that binary16 cannot hold, FGQ
      blocks of any width (block partials scaled in fp32, gemm.py:96-110),
      INT4 (S * sum(level x) + Z * sum(x)) — bit-identical to the reference.
    `exact`: None = pick as above; True / False force a kernel (False rounds
    X to binary16 and needs a tcgen05-capable scheme).  `split_k` / `sched`
    tune the tcgen05 schedule (same result up to fp32 summation order)."""
    if wq.num_blocks != num_blocks(wq.rows, wq.cols, wq.scheme):
        raise PayloadMismatch("block parameter count does not match the scheme")
    torch_in = _lib.is_torch(X)
    Xa = X if torch_in else np.asarray(X)
    _check_activation(Xa, wq.cols)
    n, k, m = wq.rows, wq.cols, int(Xa.shape[1])
    t = _lib.torch()
    if n == 0 or k == 0 or m == 0:
        if torch_in:
            return t.zeros((n, m), dtype=t.float32, device=_lib.device())
        return np.zeros((n, m), dtype=np.float32)
    int4 = wq.scheme.fmt is TensorFormat.INT4_ASYM
    if not int4:
        _require_path(wq.scheme)
    X32 = None
    if exact is None:
        X32 = _x32(Xa)
        exact = not (a16_path(wq) and _f16_exact(X32))
    if exact:
        y = _gemm_exact(wq, X32 if X32 is not None else _x32(Xa))
        return y if torch_in else y.cpu().numpy()
    if not int4:
        _require_gemm_path(wq.scheme, wq.cols)
    weight = Int4Weight.from_quantized(wq) if int4 else Fp6Weight.from_quantized(wq)
    xt, kp = stage_activations(Xa, k)
    y = gemm_nm(weight, xt, kp, m, split_k=split_k, sched=sched)
    return y if torch_in else y.cpu().numpy()


def _device_codes(wq: QuantizedTensor):
    """Row-major codes (INT4: levels) of `wq` as a uint8 CUDA tensor [N*K]."""
    t = _lib.torch()
    nk = wq.rows * wq.cols
    if wq.scheme.fmt is TensorFormat.INT4_ASYM:
        nib = wq.payload if _lib.is_torch(wq.payload) else np.asarray(wq.payload, np.uint8)
        if (nib.numel() if _lib.is_torch(nib) else nib.size) != (nk + 1) // 2:
            raise PayloadMismatch("payload does not hold rows*cols levels")
        d = _lib.to_device(nib).reshape(-1).to(t.uint8)
        out = t.empty(nk, dtype=t.uint8, device=d.device)
        _lib.check(_lib.load().lpqt_int4_unpack(d.data_ptr(), nk, out.data_ptr(), _lib.stream_ptr()), "int4_unpack")
        return out
    s4, s2, _ = device_planes(wq)
    return unpack_device(s4, s2, nk, wq.scheme.fmt.minifloat)


def _gemm_exact(wq: QuantizedTensor, X32):
    """gemm.py:65-110 operation for operation (`lpqt_gemm_exact_quantized`)."""
    t = _lib.torch()
    codes = _device_codes(wq)
    xd = _lib.to_device(X32).to(t.float32).contiguous()
    sc = _lib.to_device(wq.scales if _lib.is_torch(wq.scales) else np.asarray(wq.scales, np.float16))
    sc = sc.reshape(-1).to(t.float16).contiguous()
    int4 = wq.scheme.fmt is TensorFormat.INT4_ASYM
    zp = None
    if int4:
        zp = _lib.to_device(wq.zero_points if _lib.is_torch(wq.zero_points)
                            else np.asarray(wq.zero_points, np.float16)).reshape(-1).to(t.float16).contiguous()
    fmt = 2 if int4 else (1 if wq.scheme.fmt is TensorFormat.FP5_E3M1 else 0)
    m = int(xd.shape[1])
    y = t.empty((wq.rows, m), dtype=t.float32, device=xd.device)
    _lib.check(_lib.load().lpqt_gemm_exact_quantized(
        codes.data_ptr(), fmt, sc.data_ptr(), _lib.ptr(zp), wq.rows, wq.cols, scale_block(wq.scheme), xd.data_ptr(),
        m, y.data_ptr(), _lib.stream_ptr()), "gemm_exact")
    return y


def _dense(W, X, dtype):
    """gemm.py:28-51: W [N, K] @ X [K, M] in `dtype` (float32 / float64), k
    ascending with separately rounded products and sums
    (`lpqt_gemm_exact_dense`): bit-identical to the reference's loop."""
    t = _lib.torch()
    torch_in = _lib.is_torch(W) or _lib.is_torch(X)
    npd = np.float32 if dtype == t.float32 else np.float64
    Wd = _lib.to_device(W if _lib.is_torch(W) else np.asarray(W, dtype=npd)).to(dtype).contiguous()
    Xd = _lib.to_device(X if _lib.is_torch(X) else np.asarray(X, dtype=npd)).to(dtype).contiguous()
    if Wd.dim() != 2:
        raise ShapeError(f"weights must be 2-D, got shape {tuple(Wd.shape)}")
    _check_activation(Xd, Wd.shape[1])
    n, k, m = int(Wd.shape[0]), int(Wd.shape[1]), int(Xd.shape[1])
    Y = t.empty((n, m), dtype=dtype, device=Wd.device)
    if n and m:
        if k == 0:
            Y.zero_()
        else:
            _lib.check(_lib.load().lpqt_gemm_exact_dense(Wd.data_ptr(), Xd.data_ptr(),
                                                         _lib.F32 if dtype == t.float32 else _lib.F64, n, k, m,
                                                         Y.data_ptr(), _lib.stream_ptr()), "gemm_dense")
    return Y if torch_in else Y.cpu().numpy()


def gemm_reference(W, X):
    """float64 dense product, k ascending (gemm.py:28-38)."""
    return _dense(W, X, _lib.torch().float64)


def gemm_dense(W, X):
    """float32 dense product, k ascending (gemm.py:41-51)."""
    return _dense(W, X, _lib.torch().float32)


def compare_outputs(Y, Y_ref) -> ErrorReport:
    """Elementwise comparison report (gemm.py:113-115)."""
    return error_report(Y_ref, Y)


def gemm_tolerance(k: int, W_hat, X) -> float:
    """4 * eps32 * K * max|W_hat| * max|X| (gemm.py:118-122)."""
    def peak(a):
        if _lib.is_torch(a):
            return float(a.abs().max()) if a.numel() else 0.0
        a = np.asarray(a)
        return float(np.max(np.abs(a))) if a.size else 0.0
    return 4.0 * float(np.finfo(np.float32).eps) * k * peak(W_hat) * peak(X)
