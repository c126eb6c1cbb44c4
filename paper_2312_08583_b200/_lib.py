"""ctypes binding of liblpqt_b200.so (the C ABI in include/lpqt_b200.h).

PyTorch is used only as plumbing: device memory, the current CUDA stream and
host<->device copies.  Every compute step on the path is a call into the
in-tree CUDA library; there is no CPU fallback — without a CUDA device or
without the built library every call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import (InvalidCode, InvalidInput, LpqtError, PayloadMismatch,
                     ScaleOverflow, ShapeError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LPQT_LIB") or os.path.join(_HERE, "liblpqt_b200.so")

# dtype / layout codes (lpqt_b200.h)
F64, F32, F16, BF16 = 0, 1, 2, 3
Y_NM, Y_MN = 0, 1

# status codes
OK = 0
E_INVALID_INPUT, E_SHAPE, E_SCALE_OVERFLOW, E_PAYLOAD = -1, -2, -3, -4
E_INVALID_CODE, E_UNSUPPORTED, E_WORKSPACE, E_CUDA = -5, -6, -7, -100
LAUNCH_PDL = 1
WEIGHTS_FP5 = 128   # LPQT_WEIGHTS_FP5: native 5-bit tiles
SCHED_STREAMK, SCHED_CLUSTER = 2, 4

# device flag bits
F_NONFINITE, F_SCALE_INF, F_FOLD_OVERFLOW, F_BAD_SCALE, F_BAD_CODE = 1, 2, 4, 8, 16

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int



MAX_PEERS = 8


class PeerOut(ctypes.Structure):
    """lpqt_peer_out (include/lpqt_b200.h): fused GEMM + all-gather targets."""
    _fields_ = [("y", ctypes.c_void_p * MAX_PEERS), ("flags", ctypes.c_void_p * MAX_PEERS),
                ("npeers", ctypes.c_int), ("rank", ctypes.c_int), ("epoch", ctypes.c_uint32),
                ("done", ctypes.c_void_p)]


class NextLinear(ctypes.Structure):
    """lpqt_next_linear (include/lpqt_b200.h): the launch that follows on the stream."""
    _fields_ = [("tiles", ctypes.c_void_p), ("M", ctypes.c_int64), ("N", ctypes.c_int64), ("K", ctypes.c_int64),
                ("split_k", ctypes.c_int), ("flags", ctypes.c_int), ("bytes_per_cta", ctypes.c_int64)]


# name -> (restype, argtypes); every symbol declared in include/lpqt_b200.h
SIGNATURES = {
    "lpqt_strerror": (ctypes.c_char_p, [_I32]),
    "lpqt_abi_version": (_I32, []),
    "lpqt_fp6_encode_rtn": (_I32, [_P, _I32, _I64, _P, _P, _P]),
    "lpqt_fp6_pack": (_I32, [_P, _I64, _P, _P, _P, _P]),
    "lpqt_fp6_unpack": (_I32, [_P, _P, _I64, _P, _P]),
    "lpqt_fp6_seg4_length": (_I64, [_I64]),
    "lpqt_fp6_tail_length": (_I64, [_I64]),
    "lpqt_fp6_fold_scales": (_I32, [_P, _I64, _P, _P, _P]),
    "lpqt_fp6_dequant_bias_shift": (_I32, [_P, _P, _I64, _P, _P]),
    "lpqt_fp6_dequant_naive": (_I32, [_P, _P, _I64, _P, _P]),
    "lpqt_fp6_quantize_pack": (_I32, [_P, _I32, _I64, _I64, _I64, _I32, _P, _P, _P, _P, _P, _P, _P]),
    "lpqt_fp6_dequantize_tensor": (_I32, [_P, _P, _P, _I32, _I64, _I64, _P, _I32, _P]),
    "lpqt_fp6_tiles_bytes": (_I64, [_I64, _I64]),
    "lpqt_fp6_prepack": (_I32, [_P, _P, _I64, _I64, _P, _P]),
    "lpqt_fp6_quantize_tiles": (_I32, [_P, _I32, _I64, _I64, _I64, _I32, _P, _P, _P, _P, _P]),
    "lpqt_fp6_unprepack": (_I32, [_P, _I64, _I64, _P, _P]),
    "lpqt_fp6_tiles_dequant": (_I32, [_P, _P, _I64, _I64, _P, _P]),
    "lpqt_stage_activations": (_I32, [_P, _I32, _I64, _I64, _I64, _P, _I64, _P]),
    "lpqt_w6a16_workspace_bytes": (_I64, [_I64, _I64, _I64, _I32]),
    "lpqt_w6a16_plan": (_I32, [_I64, _I64, _I64, _I32, _P, _P, _P, _P]),
    "lpqt_w6a16_plan_ex": (_I32, [_I64, _I64, _I64, _I32, _I32, _P, _I32]),
    "lpqt_w6a16_linear": (_I32, [_P, _P, _P, _I64, _I64, _I64, _I64, _P, _I32, _I32, _I64, _I32, _P, _I64, _P]),
    "lpqt_w6a16_linear_ex": (_I32, [_P, _P, _P, _I64, _I64, _I64, _I64, _P, _I32, _I32, _I64, _I32, _P, _I64, _I32,
                                    _P]),
    "lpqt_w6a16_linear_pf": (_I32, [_P, _P, _P, _I64, _I64, _I64, _I64, _P, _I32, _I32, _I64, _I32, _P, _I64, _I32,
                                    ctypes.POINTER(NextLinear), _P]),
    "lpqt_fp6_quantize_pack_blocks": (_I32, [_P, _I32, _I64, _I64, _I64, _I64, _I32, _P, _P, _P, _P, _P, _P]),
    "lpqt_fp6_quantize_tiles_blocks": (_I32, [_P, _I32, _I64, _I64, _I64, _I64, _I32, _P, _P, _P, _P, _P]),
    "lpqt_fp6_dequantize_tensor_blocks": (_I32, [_P, _P, _P, _I32, _I64, _I64, _I64, _P, _I32, _P]),
    "lpqt_fp6_tiles_dequant_blocks": (_I32, [_P, _P, _I64, _I64, _I64, _P, _P]),
    "lpqt_w6a16_linear_blocks": (_I32, [_P, _P, _I64, _P, _I64, _I64, _I64, _I64, _P, _I32, _I32, _I64, _I32, _P,
                                        _I64, _I32, ctypes.POINTER(NextLinear), _P]),
    "lpqt_fp5_tail_length": (_I64, [_I64]),
    "lpqt_fp5_encode_rtn": (_I32, [_P, _I32, _I64, _P, _P, _P]),
    "lpqt_fp5_pack": (_I32, [_P, _I64, _P, _P, _P, _P]),
    "lpqt_fp5_unpack": (_I32, [_P, _P, _I64, _P, _P]),
    "lpqt_fp5_quantize_pack_blocks": (_I32, [_P, _I32, _I64, _I64, _I64, _I64, _I32, _P, _P, _P, _P, _P, _P]),
    "lpqt_fp5_dequantize_tensor_blocks": (_I32, [_P, _P, _P, _I32, _I64, _I64, _I64, _P, _I32, _P]),
    "lpqt_fp5_dequant_bias_shift": (_I32, [_P, _P, _I64, _P, _P]),
    "lpqt_fp5_dequant_naive": (_I32, [_P, _P, _I64, _P, _P]),
    "lpqt_fp5_prepack": (_I32, [_P, _P, _I64, _I64, _P, _P]),
    "lpqt_fp5n_tiles_bytes": (_I64, [_I64, _I64]),
    "lpqt_selftest_fp6_encode": (_I32, [_I32, _P]),
    "lpqt_fp5n_prepack": (_I32, [_P, _P, _I64, _I64, _P, _P]),
    "lpqt_fp5n_unprepack": (_I32, [_P, _I64, _I64, _P, _P]),
    "lpqt_fp5n_tiles_dequant": (_I32, [_P, _P, _I64, _I64, _P, _P]),
    "lpqt_int4_quantize_blocks": (_I32, [_P, _I32, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P]),
    "lpqt_int4_pack": (_I32, [_P, _I64, _P, _P, _P]),
    "lpqt_int4_unpack": (_I32, [_P, _I64, _P, _P]),
    "lpqt_int4_dequantize_blocks": (_I32, [_P, _P, _P, _I64, _I64, _I64, _P, _P]),
    "lpqt_int4_tiles_bytes": (_I64, [_I64, _I64]),
    "lpqt_int4_prepack": (_I32, [_P, _I64, _I64, _P, _P]),
    "lpqt_w4a16_linear_blocks": (_I32, [_P, _P, _I64, _P, _I64, _I64, _I64, _I64, _P, _I32, _I32, _I64, _I32, _P,
                                        _I64, _I32, _P]),
    "lpqt_fgq_stage_bytes": (_I64, [_I64, _I64, _I32]),
    "lpqt_w6a16_linear_gather": (_I32, [_P, _P, _I64, _P, _I64, _I64, _I64, _I64, _I32, _I32, _I64, _I32, _P,
                                        _I64, _I32, _P, _P]),
    "lpqt_fgq_stage_params": (_I32, [_P, _P, _I64, _I64, _I64, _P, _P]),
    "lpqt_gemm_exact_quantized": (_I32, [_P, _I32, _P, _P, _I64, _I64, _I64, _P, _I64, _P, _P]),
    "lpqt_gemm_exact_dense": (_I32, [_P, _P, _I32, _I64, _I64, _I64, _P, _P]),
    "lpqt_launch_count": (_I64, []),
}

_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with "
                        "`python -m paper_2312_08583_b200._build` (no CPU fallback exists)")
                lib = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = lib
    return _lib


def check(status: int, what: str = "") -> None:
    """Map a host-side status code to the reference's exception types."""
    if status == OK:
        return
    msg = load().lpqt_strerror(status).decode()
    if what:
        msg = f"{what}: {msg}"
    exc = {E_INVALID_INPUT: InvalidInput, E_SHAPE: ShapeError,
           E_SCALE_OVERFLOW: ScaleOverflow, E_PAYLOAD: PayloadMismatch,
           E_INVALID_CODE: InvalidCode}.get(status)
    if exc is not None:
        raise exc(msg)
    raise LpqtError(msg)


# ---------------------------------------------------------------------------
# torch plumbing
# ---------------------------------------------------------------------------
def torch():
    import torch as _t
    return _t


def device():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("a CUDA device is required: the B200 path has no CPU fallback")
    return t.device("cuda", t.cuda.current_device())


def stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def dtype_code(tdtype) -> int:
    t = torch()
    m = {t.float64: F64, t.float32: F32, t.float16: F16, t.bfloat16: BF16}
    if tdtype not in m:
        raise InvalidInput(f"unsupported dtype {tdtype}")
    return m[tdtype]


def is_torch(x) -> bool:
    try:
        import torch as _t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, _t.Tensor)


def to_device(x, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (no copy when already there)."""
    t = torch()
    if is_torch(x):
        y = x
    else:
        a = np.asarray(x)
        if a.dtype == np.float16:
            y = t.from_numpy(np.ascontiguousarray(a))
        elif a.dtype.kind == "f":
            y = t.from_numpy(np.ascontiguousarray(a))
        else:
            y = t.from_numpy(np.ascontiguousarray(a))
    if dtype is not None and y.dtype != dtype:
        y = y.to(dtype)
    return y.to(device(), non_blocking=False).contiguous()


class Flags:
    """Device error word for data-dependent errors (LPQT_F_* bits)."""

    def __init__(self):
        self.t = torch().zeros(1, dtype=torch().int32, device=device())

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def value(self) -> int:
        return int(self.t.item()) & 0xFFFFFFFF

    def raise_if_set(self, order=("nonfinite", "scale_inf", "bad_scale", "bad_code", "fold")):
        v = self.value()
        if not v:
            return
        if v & F_NONFINITE:
            raise InvalidInput("input contains non-finite values")
        if v & F_SCALE_INF:
            raise InvalidInput("block magnitude too large for a binary16 scale")
        if v & F_BAD_SCALE:
            raise InvalidInput("scales must be positive finite binary16 values")
        if v & F_BAD_CODE:
            raise InvalidCode("codes must fit 6 bits")
        if v & F_FOLD_OVERFLOW:
            raise ScaleOverflow("folded scale exceeds binary16 range")


class Workspace:
    """GEMM workspace (split-K partials + self-resetting tile counters),
    zero-initialised, one grow-only buffer per (device, stream).

    * Streams never share a buffer, so split-K GEMMs running concurrently on
      two streams cannot race on each other's tile counters / partials.
    * A buffer that is outgrown is retired, never freed: a CUDA graph captured
      earlier keeps pointing at valid, still-zeroed memory.
    * Inside a graph capture nothing is resized: an adequate buffer of the
      capturing stream is used as is, else the default stream's (a graph is
      replayed on the launching stream, normally the default one, and is then
      serialised with that stream's eager work); otherwise a capture-private
      buffer is allocated whose zero-fill is a node of the captured graph (so
      it is zeroed on every replay, and no eager launch ever sees it).
      Graphs replayed concurrently with split-K GEMMs on other streams should
      pass their own buffer.
    Callers may also pass their own zeroed buffer (`workspace=` in linear.py).
    """

    _per_stream: dict = {}
    _retired: list = []
    _captured: list = []

    @classmethod
    def get(cls, nbytes: int):
        t = torch()
        dev = device()
        stream = t.cuda.current_stream(dev)
        key = (dev.index, stream.cuda_stream)
        cur = cls._per_stream.get(key)
        if cur is not None and cur.numel() >= nbytes:
            return cur
        if t.cuda.is_current_stream_capturing():
            # torch captures on a side stream but a graph replays on the stream
            # it is launched from — normally the default stream, whose eager
            # work it is then serialised with: adopt that stream's buffer
            dflt = cls._per_stream.get((dev.index, t.cuda.default_stream(dev).cuda_stream))
            if dflt is not None and dflt.numel() >= nbytes:
                return dflt
            buf = t.zeros(max(nbytes, 1 << 20), dtype=t.uint8, device=dev)   # memset captured in the graph
            cls._captured.append(buf)
            return buf
        if cur is not None:
            cls._retired.append(cur)
        size = max(nbytes, 1 << 20, 2 * cur.numel() if cur is not None else 0)
        cur = t.zeros(size, dtype=t.uint8, device=dev)
        cls._per_stream[key] = cur
        return cur


def launch_count() -> int:
    return int(load().lpqt_launch_count())
