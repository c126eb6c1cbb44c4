"""CPU-side checks of the C-ABI boundary (no GPU needed, no compute calls):
the in-tree liblpqt_b200.so loads, exports every function include/lpqt_b200.h
declares, the ctypes binding covers them, and the pure host queries (status
strings, plane lengths, tile bytes, launch plan) agree with the reference's
formulas (packing.py:28-36)."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lpqt_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lpqt_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2312_08583_b200 import _build, _lib
    if not os.path.exists(_lib.LIB_PATH):
        _build.build()
    return _lib.load()


def test_header_declares_the_path():
    names = declared_functions()
    for must in ("lpqt_fp6_quantize_pack", "lpqt_fp6_prepack", "lpqt_w6a16_linear", "lpqt_w6a16_linear_ex",
                 "lpqt_fp6_encode_rtn", "lpqt_fp6_pack", "lpqt_fp6_unpack", "lpqt_fp6_fold_scales"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2312_08583_b200 import _lib
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, f"declared in lpqt_b200.h but not exported: {missing}"
    unbound = [n for n in declared_functions() if n not in _lib.SIGNATURES]
    assert not unbound, f"declared but not bound in _lib.SIGNATURES: {unbound}"


def test_abi_version_and_status_strings(lib):
    assert lib.lpqt_abi_version() == 6
    from paper_2312_08583_b200 import _lib
    assert lib.lpqt_strerror(_lib.OK) == b"ok"
    assert b"ShapeError" in lib.lpqt_strerror(_lib.E_SHAPE)
    assert b"ScaleOverflow" in lib.lpqt_strerror(_lib.E_SCALE_OVERFLOW)
    assert b"InvalidInput" in lib.lpqt_strerror(_lib.E_INVALID_INPUT)


@pytest.mark.parametrize("n", [0, 1, 2, 3, 4, 5, 7, 8, 9, 1023, 1024, 1025, 16777216])
def test_plane_lengths_match_reference_formula(lib, n):
    # packing.py:28-36: align4(ceil(n/2)) and align4(ceil(n/4))
    align4 = lambda v: (v + 3) // 4 * 4
    assert lib.lpqt_fp6_seg4_length(n) == align4((n + 1) // 2)
    assert lib.lpqt_fp6_tail_length(n) == align4((n + 3) // 4)


@pytest.mark.parametrize("n,k", [(1, 1), (128, 128), (129, 130), (4096, 4096), (22016, 4096)])
def test_tile_bytes(lib, n, k):
    rt = (n + 127) // 128
    kt = (k + 127) // 128
    assert lib.lpqt_fp6_tiles_bytes(n, k) == rt * kt * 12288


def test_host_errors_without_launch(lib):
    """Argument errors are caught on the host before any launch."""
    from paper_2312_08583_b200 import _lib
    st = lib.lpqt_w6a16_linear(None, None, None, 7, 1, 128, 8, None, _lib.F32, _lib.Y_NM, 1, 0, None, 0, None)
    assert st == _lib.E_SHAPE          # ldx % 8 != 0
    st = lib.lpqt_w6a16_linear_ex(None, None, None, 8, 1, 128, 8, None, 9, _lib.Y_NM, 1, 0, None, 0, 0, None)
    assert st == _lib.E_UNSUPPORTED    # bad y dtype
    st = lib.lpqt_w6a16_linear_ex(None, None, None, 8, 1, 128, 8, None, _lib.F32, _lib.Y_NM, 1, 0, None, 0, 4096, None)
    assert st == _lib.E_INVALID_INPUT  # unknown flag
    st = lib.lpqt_w6a16_linear_ex(None, None, None, 8, 1, 128, 8, None, _lib.F32, _lib.Y_NM, 1, 0, None, 0, 32 | 64, None)
    assert st == _lib.E_INVALID_INPUT  # both ablation rebuilds
    st = lib.lpqt_w6a16_linear_ex(None, None, None, 8, 17, 128, 8, None, _lib.F32, _lib.Y_NM, 17, 0, None, 0, 64, None)
    assert st == _lib.E_UNSUPPORTED    # ablation rebuilds are decode-only (M <= 16)
    st = lib.lpqt_w6a16_linear_ex(None, None, None, 8, 1, 128, 8, None, _lib.F32, _lib.Y_NM, 1, 0, None, 0, 128 | 32, None)
    assert st == _lib.E_UNSUPPORTED    # native FP5 tiles run the hardware rebuild only
    assert lib.lpqt_w6a16_linear(None, None, None, 8, 0, 128, 8, None, _lib.F32, _lib.Y_NM, 1, 0, None, 0,
                                 None) == _lib.OK  # M == 0: nothing to do


def test_plan_is_host_only(lib):
    import ctypes
    vals = [ctypes.c_int(0) for _ in range(4)]
    assert lib.lpqt_w6a16_plan(16, 4096, 4096, 0, *[ctypes.addressof(v) for v in vals]) == 0
    block_n, splits, grid, stages = (v.value for v in vals)
    assert block_n == 16 and grid >= 1 and stages >= 2
    assert lib.lpqt_w6a16_workspace_bytes(16, 4096, 4096, 0) >= 0
