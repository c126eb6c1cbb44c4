"""W6A16 GEMM API — reference gemm.py:1-122.

`gemm_quantized(wq, X)` (gemm.py:65-94) keeps the reference contract —
W_hat (N x K, CGQ FP6) times X (K x M) -> float32 N x M — and runs the
tcgen05 kernel.  Activations are rounded to binary16 (A16) before the GEMM;
with fp16-exact X the result equals the reference's up to fp32 summation
order (normwise relative error <= 1e-3 is the parity bar, tests/).

`gemm_reference` / `gemm_dense` (f64 / f32 dense oracles, gemm.py:28-51) run
as GPU matmuls (TF32 off); `gemm_tolerance` / `compare_outputs` are the
reference's error bounds.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import PayloadMismatch, ShapeError
from .linear import Fp6Weight, Int4Weight, gemm_nm, stage_activations
from .quantizer import (ErrorReport, QuantizedTensor, TensorFormat, _require_gemm_path, dequantize_tensor,
                        error_report, num_blocks)


def _check_activation(X, k: int) -> None:
    if X.ndim != 2:
        raise ShapeError(f"activations must be 2-D, got shape {tuple(X.shape)}")
    if X.shape[0] != k:
        raise ShapeError(f"inner dimensions differ: weights K={k}, activations K={X.shape[0]}")


def gemm_quantized(wq: QuantizedTensor, X, split_k: int = 0, sched: str = "auto"):
    """Y = W_hat @ X for an FP6 / FP5 / INT4 tensor (N x K; CGQ, or FGQ with
    blocks of whole 128-k tiles) and X (K x M) -> f32 (N x M).  INT4 runs the
    W4A16 variant of the kernel: W_hat = Z + S * level rebuilt in binary16
    (one rounding; the reference sums S * sum(level x) + Z * sum(x) in fp32).

    `split_k` / `sched` are B200 tuning hooks (default: automatic schedule);
    the result is the same up to fp32 summation order (FGQ: the block scale
    is applied to the binary16 rebuilt weight, gemm.py:96-110 applies it to
    the fp32 block partial)."""
    if wq.num_blocks != num_blocks(wq.rows, wq.cols, wq.scheme):
        raise PayloadMismatch("block parameter count does not match the scheme")
    int4 = wq.scheme.fmt is TensorFormat.INT4_ASYM
    if int4:
        b = wq.scheme.block_size if wq.scheme.granularity.name == "FGQ" else 0
        if b and b < wq.cols and b % 128:
            return _gemm_int4_comparator(wq, X)
    else:
        _require_gemm_path(wq.scheme, wq.cols)
    torch_in = _lib.is_torch(X)
    Xa = X if torch_in else np.asarray(X)
    _check_activation(Xa, wq.cols)
    n, k, m = wq.rows, wq.cols, int(Xa.shape[1])
    t = _lib.torch()
    if n == 0 or k == 0 or m == 0:
        if torch_in:
            return t.zeros((n, m), dtype=t.float32, device=_lib.device())
        return np.zeros((n, m), dtype=np.float32)
    weight = Int4Weight.from_quantized(wq) if int4 else Fp6Weight.from_quantized(wq)
    xt, kp = stage_activations(Xa, k)
    y = gemm_nm(weight, xt, kp, m, split_k=split_k, sched=sched)
    return y if torch_in else y.cpu().numpy()


def _dense(W, X, dtype):
    t = _lib.torch()
    torch_in = _lib.is_torch(W) or _lib.is_torch(X)
    Wd = _lib.to_device(W if _lib.is_torch(W) else np.asarray(W, dtype=np.float64)).to(dtype)
    Xd = _lib.to_device(X if _lib.is_torch(X) else np.asarray(X, dtype=np.float64)).to(dtype)
    if Wd.dim() != 2:
        raise ShapeError(f"weights must be 2-D, got shape {tuple(Wd.shape)}")
    _check_activation(Xd, Wd.shape[1])
    prev = t.backends.cuda.matmul.allow_tf32
    t.backends.cuda.matmul.allow_tf32 = False
    try:
        Y = Wd @ Xd
    finally:
        t.backends.cuda.matmul.allow_tf32 = prev
    return Y if torch_in else Y.cpu().numpy()


def _gemm_int4_comparator(wq: QuantizedTensor, X):
    """INT4 with FGQ blocks that are not whole 128-k tiles: the GPU
    dequantizes (Z + S * level, exact f64) and a library fp32 GEMM multiplies
    (gemm.py:84-110 INT4 terms).  CGQ and tile-aligned FGQ INT4 run the fused
    W4A16 tcgen05 kernel (`Int4Weight`)."""
    torch_in = _lib.is_torch(X)
    Xa = X if torch_in else np.asarray(X)
    _check_activation(Xa, wq.cols)
    W_hat = dequantize_tensor(wq)
    Y = _dense(W_hat, Xa, _lib.torch().float32)
    return Y


def gemm_reference(W, X):
    """float64 dense product (gemm.py:28-38)."""
    return _dense(W, X, _lib.torch().float64)


def gemm_dense(W, X):
    """float32 dense product (gemm.py:41-51); TF32 disabled."""
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
