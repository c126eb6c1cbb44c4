"""Pin the CPU oracle (oracle/lpqt_oracle.py) to the reference.

Sources: golden.npz (outputs of the reference `lpqt` itself, made by
tests/golden/make_golden.py) and the reference tests' own known answers
(pkg/tests/test_codec.py, test_packing.py, test_dequant.py, test_quantizer.py).
"""

import hashlib

import numpy as np
import pytest

from oracle import lpqt_oracle as O
from tests.conftest import names


def test_value_table_and_compose_match_reference(golden):
    assert np.array_equal(O.value_table(), golden["value_table"])
    assert np.array_equal(O.compose_table_f16().view(np.uint16), golden["compose"])


def test_codec_kats():
    # pkg/tests/test_codec.py:47-62, :83-101
    assert O.decode(0b011111) == 28.0
    assert O.decode(0b000001) == 0.0625
    assert O.decode(0b001100) == 1.0
    assert np.signbit(O.decode(0b100000))
    enc = O.encode_rtn_array(np.array([28.0, 100.0, -100.0, 0.0, -0.0, 26.0, 0.03125, -0.01]))
    assert list(enc) == [0b011111, 0b011111, 0b111111, 0, 0, 0b011110, 0, 32]


def test_encode_matches_reference(golden):
    assert np.array_equal(O.encode_rtn_array(golden["enc/x"]), golden["enc/codes"])


def test_encode_rejects_non_finite():
    with pytest.raises(ValueError):
        O.encode_rtn_array(np.array([1.0, np.nan]))


def test_pack_kat():
    # pkg/tests/test_packing.py:36-42
    s4, s2 = O.pack(np.array([0b011111, 0b001100, 0, 0b100001]))
    assert list(s4) == [0x37, 0x80, 0, 0] and list(s2) == [0x43, 0, 0, 0]


def test_pack_unpack_match_reference(golden):
    for n in golden["p_lens"]:
        c = golden[f"p/{n}/codes"]
        s4, s2 = O.pack(c)
        assert np.array_equal(s4, golden[f"p/{n}/seg4"])
        assert np.array_equal(s2, golden[f"p/{n}/seg2"])
        assert np.array_equal(O.unpack(s4, s2, int(n)), c)


def test_fold_matches_reference(golden):
    s = golden["fold/scales"].view(np.float16)
    f = O.fold_scale_array(s)
    assert np.array_equal(f.view(np.uint16), golden["fold/folded"])
    with pytest.raises(ValueError):
        O.fold_scale_array(np.array([16.0], np.float16))


def test_exhaustive_bias_shift_sweep_hash(golden):
    # pkg/tests/test_acceptance.py:72-87 sweep, pinned by the reference's hash
    s = golden["fold/scales"].view(np.float16)
    f = O.fold_scale_array(s)
    sweep = O.dequant_bias_shift_array(np.arange(64, dtype=np.uint8)[:, None], f[None, :])
    naive = O.dequant_naive_array(np.arange(64, dtype=np.uint8)[:, None], s[None, :])
    assert np.array_equal(sweep.view(np.uint16), naive.view(np.uint16))
    h = hashlib.sha256(sweep.view(np.uint16).tobytes()).hexdigest()
    assert h == str(golden["fold/sweep_sha256"])


def test_quantize_matches_reference(golden):
    for name in names(golden, "q_names"):
        W = golden[f"q/{name}/W"]
        q = O.quantize_tensor(W, bias_shift=True)
        assert np.array_equal(q["scales"].view(np.uint16), golden[f"q/{name}/scales"]), name
        assert np.array_equal(q["folded"].view(np.uint16), golden[f"q/{name}/folded"]), name
        assert np.array_equal(q["seg4"], golden[f"q/{name}/seg4"]), name
        assert np.array_equal(q["seg2"], golden[f"q/{name}/seg2"]), name
        n, k = W.shape
        deq = O.dequantize_tensor(q["codes"], n, k, folded=q["folded"], path="bias_shift")
        assert np.array_equal(deq, golden[f"q/{name}/deq"]), name


def test_quantize_error_cases_match_reference(golden):
    for name in names(golden, "e_names"):
        W = golden[f"e/{name}/W"]
        bs = bool(golden[f"e/{name}/bias_shift"])
        want = str(golden[f"e/{name}/result"])
        try:
            O.quantize_tensor(W, bias_shift=bs)
            got = "ok"
        except ValueError as exc:
            got = {"invalid": "InvalidInput", "overflow": "ScaleOverflow"}[str(exc)]
        assert got == want, name


def test_gemm_matches_reference(golden):
    for name in names(golden, "g_names"):
        W, X = golden[f"g/{name}/W"], golden[f"g/{name}/X"]
        q = O.quantize_tensor(W, bias_shift=True)
        n, k = W.shape
        Y = O.gemm_quantized(q["codes"], q["scales"], n, k, X)
        # same algorithm, same order -> bit-identical to the reference
        assert np.array_equal(Y.view(np.uint32), golden[f"g/{name}/Y"].view(np.uint32)), name
