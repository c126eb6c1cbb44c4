"""Generate the `.lpqt` container fixtures from the REFERENCE itself.

Run here (the only place /root/reference exists):

    python tests/golden/make_container_golden.py

Imports the unmodified reference package `lpqt` (read-only, no bytecode) and
records, for seeded inputs, the bytes its `write_lpqt` produces
(container.py:50-77) for every scheme the format carries, the exception
class its `read_lpqt` raises (container.py:108-185) on corrupted streams,
the `read_raw` results (container.py:191-200) and the CLI's stdout for
`inspect` / `codebook` (cli.py:126-143, :220-228).  Output:
`container_golden.npz` next to this file.  Nothing on the GPU box reads
/root/reference.
"""

from __future__ import annotations

import contextlib
import io
import os
import struct
import sys
import tempfile

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import lpqt as ref  # noqa: E402  (the reference, read-only)
from lpqt import cli as ref_cli  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
G, F = ref.Granularity, ref.TensorFormat
SCHEMES = {
    "cgq_fp6": ref.QuantScheme(G.CGQ, F.FP6_E3M2),
    "cgq_fp5": ref.QuantScheme(G.CGQ, F.FP5_E3M1),
    "cgq_int4": ref.QuantScheme(G.CGQ, F.INT4_ASYM),
    "fgq_fp6_16": ref.QuantScheme(G.FGQ, F.FP6_E3M2, block_size=16),
    "fgq_fp5_7": ref.QuantScheme(G.FGQ, F.FP5_E3M1, block_size=7),
    "fgq_int4_32": ref.QuantScheme(G.FGQ, F.INT4_ASYM, block_size=32),
}


def u8(b: bytes) -> np.ndarray:
    return np.frombuffer(b, dtype=np.uint8).copy()


def main() -> None:
    out: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(2312)
    # ---- writer: every scheme, ragged shapes, with and without bias shift
    w_names = []
    for sname, scheme in SCHEMES.items():
        for shape in [(1, 4), (3, 5), (7, 33), (16, 64), (0, 5), (4, 0)]:
            for bias in (False, True):
                if bias and scheme.fmt is F.INT4_ASYM:
                    continue
                W = (rng.standard_normal(shape) * rng.choice([0.02, 1.0])).astype(np.float32)
                q = ref.quantize_tensor(W, scheme, bias_shift=bias)
                name = f"{sname}_{shape[0]}x{shape[1]}_b{int(bias)}"
                out[f"w/{name}/W"] = W
                out[f"w/{name}/bytes"] = u8(ref.write_lpqt(q))
                w_names.append(name)
    out["w_names"] = np.array(w_names)

    # ---- reader errors: corrupt one field of a valid FP6 stream
    base = bytearray(ref.write_lpqt(ref.quantize_tensor(
        rng.standard_normal((3, 10)).astype(np.float32), SCHEMES["cgq_fp6"], bias_shift=True)))
    int4 = bytearray(ref.write_lpqt(ref.quantize_tensor(
        rng.standard_normal((3, 10)).astype(np.float32), SCHEMES["cgq_int4"])))

    def patched(buf, off, fmt, val):
        b = bytearray(buf)
        struct.pack_into(fmt, b, off, val)
        return bytes(b)

    cases = {
        "ok": bytes(base),
        "bad_magic": b"LPQX" + bytes(base[4:]),
        "bad_version": patched(base, 4, "<H", 2),
        "unknown_format": patched(base, 6, "<B", 9),
        "unknown_granularity": patched(base, 7, "<B", 5),
        "cgq_block_size": patched(base, 8, "<I", 4),
        "bias_flag_2": patched(base, 28, "<B", 2),
        "reserved_nonzero": patched(base, 29, "<B", 1),
        "int4_bias_flag": patched(int4, 28, "<B", 1),
        "truncated_header": bytes(base[:20]),
        "truncated_payload": bytes(base[:-9]),
        "trailing_bytes": bytes(base) + b"\x00" * 8,
        "pad_nonzero": patched(base, 40 + 6, "<B", 1),   # scales section padding (3 scales -> 6 B + 2 pad)
        "zero_scale": patched(base, 40, "<H", 0),
        "neg_scale": patched(base, 40, "<H", 0xBC00),
        "inf_folded": patched(base, 48, "<H", 0x7C00),
        "seg4_len": patched(base, 56, "<Q", 99),
    }
    e_names = []
    for name, data in cases.items():
        try:
            ref.read_lpqt(data)
            res = "ok"
        except ref.LpqtError as exc:
            res = type(exc).__name__
        out[f"e/{name}/bytes"] = u8(data)
        out[f"e/{name}/result"] = np.array(res)
        e_names.append(name)
    out["e_names"] = np.array(e_names)

    # ---- read_raw
    raw = rng.standard_normal((3, 4)).astype("<f4")
    out["raw/f32"] = u8(raw.tobytes())
    out["raw/f32_val"] = ref.read_raw(raw.tobytes(), 3, 4, "f32le")
    out["raw/f16"] = u8(raw.astype("<f2").tobytes())
    out["raw/f16_val"] = ref.read_raw(raw.astype("<f2").tobytes(), 3, 4, "f16le")

    # ---- CLI stdout for the host-only subcommands
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "w.lpqt")
        with open(path, "wb") as fh:
            fh.write(bytes(base))
        for key, argv in {"inspect": ["inspect", "--input", path],
                          "codebook_fp6": ["codebook", "--format", "fp6"],
                          "codebook_fp5": ["codebook", "--format", "fp5"]}.items():
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                rc = ref_cli.main(argv)
            out[f"cli/{key}/stdout"] = np.array(buf.getvalue().replace(path, "<input>"))
            out[f"cli/{key}/rc"] = np.array(rc)
    out["cli/inspect_input"] = u8(bytes(base))

    np.savez_compressed(os.path.join(HERE, "container_golden.npz"), **out)
    print(f"wrote {len(w_names)} writer cases, {len(e_names)} reader cases")


if __name__ == "__main__":
    main()
