"""CLI parity (cli.py): same subcommands, flags, key=value stdout and
error lines.  Host-only commands are compared byte for byte with the
reference's output (tests/golden/container_golden.npz); the GPU commands
(quantize / dequantize / stats / gemm --check / bench) run on the B200."""

import os

import numpy as np
import pytest

from paper_2312_08583_b200 import cli
from tests.conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden", "container_golden.npz")


@pytest.fixture(scope="module")
def cg():
    return np.load(GOLD, allow_pickle=False)


def run(capsys, argv):
    rc = cli.main(argv)
    out = capsys.readouterr()
    return rc, out.out, out.err


def kv(text):
    return dict(line.split("=", 1) for line in text.strip().splitlines() if "=" in line and " " not in line)


def test_inspect_matches_reference(cg, tmp_path, capsys):
    path = tmp_path / "w.lpqt"
    path.write_bytes(cg["cli/inspect_input"].tobytes())
    rc, out, _ = run(capsys, ["inspect", "--input", str(path)])
    assert rc == int(cg["cli/inspect/rc"]) == 0
    assert out == str(cg["cli/inspect/stdout"])


@pytest.mark.parametrize("fmt", ["fp6", "fp5"])
def test_codebook_matches_reference(cg, capsys, fmt):
    rc, out, _ = run(capsys, ["codebook", "--format", fmt])
    assert rc == 0 and out == str(cg[f"cli/codebook_{fmt}/stdout"])


def test_errors(tmp_path, capsys):
    rc, _, err = run(capsys, ["inspect", "--input", str(tmp_path / "missing.lpqt")])
    assert rc == 1 and err.startswith("error=OSError msg=")
    bad = tmp_path / "bad.lpqt"
    bad.write_bytes(b"NOPE" + bytes(36))
    rc, _, err = run(capsys, ["inspect", "--input", str(bad)])
    assert rc == 1 and err.startswith("error=BadMagic ")
    rc, _, err = run(capsys, ["bench"])
    assert rc == 1 and err.startswith("error=LpqtError msg=bench needs --preset or --shape")
    rc, _, err = run(capsys, ["bench", "--preset", "nope"])
    assert rc == 1 and "unknown preset" in err
    assert cli.main(["codebook", "--format", "int4"]) == 2        # usage error (argparse)


def test_preset_table_is_the_papers():
    assert {k: (p.rows, p.cols, p.batch) for k, p in cli.BENCH_PRESETS.items()} == {"ffn1-1b": (5504, 2048, 8), "ffn2-1b": (2048, 5504, 8),
                                 "ffn1-13b": (13824, 5120, 8), "ffn2-13b": (5120, 13824, 8),
                                 "ffn1-65b": (22016, 8192, 8), "ffn2-65b": (8192, 22016, 8)}


# ---------------------------------------------------------------- GPU
@pytest.fixture
def weights_file(tmp_path):
    rng = np.random.default_rng(0)
    W = rng.standard_normal((64, 96)).astype("<f4")
    p = tmp_path / "w.f32"
    p.write_bytes(W.tobytes())
    return p, W


@pytest.mark.gpu
def test_quantize_inspect_dequantize_stats(tmp_path, weights_file, capsys):
    from oracle import lpqt_oracle as O
    p, W = weights_file
    out = tmp_path / "w.lpqt"
    rc, so, _ = run(capsys, ["quantize", "--input", str(p), "--shape", "64x96", "--format", "fp6", "--bias-shift",
                             "--output", str(out)])
    d = kv(so)
    assert rc == 0 and d["rows"] == "64" and d["cols"] == "96" and d["blocks"] == "64"
    assert int(d["payload_bytes"]) == 64 * 96 * 6 // 8 and int(d["container_bytes"]) == out.stat().st_size
    o = O.quantize_tensor(W.astype(np.float64), bias_shift=True)
    import paper_2312_08583_b200 as L
    q = L.read_lpqt(out.read_bytes())
    assert np.array_equal(q.payload.seg4, o["seg4"]) and np.array_equal(q.payload.seg_tail, o["seg2"])
    for path in ("naive", "bias-shift"):
        rc, so, _ = run(capsys, ["dequantize", "--input", str(out), "--output", str(tmp_path / f"{path}.f32"),
                                 "--path", path])
        assert rc == 0
    assert (tmp_path / "naive.f32").read_bytes() == (tmp_path / "bias-shift.f32").read_bytes()
    rc, so, _ = run(capsys, ["stats", "--input", str(out), "--reference", str(p), "--shape", "64x96"])
    d = kv(so)
    assert rc == 0 and float(d["sqnr_db"]) > 20.0
    rc, _, err = run(capsys, ["quantize", "--input", str(p), "--shape", "64x96", "--format", "int4", "--bias-shift",
                              "--output", str(out)])
    assert rc == 1 and err.startswith("error=InvalidScheme ")      # cli tests test_int4_with_bias_shift_rejected
    rc, so, _ = run(capsys, ["quantize", "--input", str(p), "--shape", "64x96", "--format", "int4", "--scheme", "fgq",
                             "--block-size", "32", "--output", str(out)])
    d = kv(so)
    assert rc == 0 and d["blocks"] == str(64 * 3) and int(d["payload_bytes"]) == 64 * 96 // 2


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "f16"])
def test_gemm_check_passes(tmp_path, weights_file, capsys, dtype):
    p, _ = weights_file
    w = tmp_path / "w.lpqt"
    assert cli.main(["quantize", "--input", str(p), "--shape", "64x96", "--format", "fp6", "--output", str(w)]) == 0
    X = np.random.default_rng(1).standard_normal((96, 5)).astype("<f4" if dtype == "f32" else "<f2")
    xp = tmp_path / "x.raw"
    xp.write_bytes(X.tobytes())
    capsys.readouterr()
    rc, so, _ = run(capsys, ["gemm", "--weights", str(w), "--activations", str(xp), "--m", "5", "--dtype", dtype,
                             "--check", "--output", str(tmp_path / "y.f32")])
    d = kv(so)
    assert rc == 0 and d["check"] == "pass" and d["rows"] == "64" and d["m"] == "5"
    assert (tmp_path / "y.f32").stat().st_size == 64 * 5 * 4


@pytest.mark.gpu
def test_bench_preset_smoke(capsys):
    rc, so, _ = run(capsys, ["bench", "--preset", "ffn1-1b", "--repeat", "3"])
    assert rc == 0
    lines = [ln for ln in so.splitlines() if ln.startswith("path=")]
    assert [ln.split()[0] for ln in lines] == ["path=fp16_dense", "path=fp6_naive", "path=fp6_bias_shift",
                                               "path=int4_fgq", "path=fp6_w6a16", "path=fp6_w6a16_naive",
                                               "path=fp6_w6a16_bias_shift"]
    assert "weight_bytes=8465152" in lines[1]   # 5504 x 2048 x 0.75 + 2 x 5504
