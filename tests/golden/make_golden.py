"""Generate the golden fixtures in this directory from the REFERENCE itself.

Run here (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package `lpqt` from
/root/reference/pkg/src (read-only; bytecode writing disabled) and records
its outputs for seeded inputs into `golden.npz`.  Nothing on the GPU box reads
/root/reference: the tests only read the committed `golden.npz`.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import lpqt as ref  # noqa: E402  (the reference, read-only)

HERE = os.path.dirname(os.path.abspath(__file__))
CGQ_FP6 = ref.QuantScheme(ref.Granularity.CGQ, ref.TensorFormat.FP6_E3M2)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round f32 values to the nearest bf16 (RNE) and return them as f32."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32)


def quant_cases():
    """(name, W with its storage dtype) pairs for quantize parity."""
    cases = []
    r = np.random.default_rng(0)
    cases.append(("f64_randn_16x32", r.standard_normal((16, 32))))
    r = np.random.default_rng(1)
    cases.append(("f32_ragged_37x53", r.standard_normal((37, 53)).astype(np.float32)))
    r = np.random.default_rng(2)
    cases.append(("f16_llama_64x128", (r.standard_normal((64, 128)) * 0.02).astype(np.float16)))
    r = np.random.default_rng(3)
    cases.append(("bf16_96x256", bf16_round(r.standard_normal((96, 256)).astype(np.float32) * 0.05)))
    r = np.random.default_rng(4)
    cases.append(("f32_odd_k_5x7", r.uniform(-3, 3, size=(5, 7)).astype(np.float32)))
    # special rows: zero row, peak 447 (largest foldable region), tiny
    # negatives, signed zeros, exact midpoints * S
    W = np.zeros((6, 16), dtype=np.float64)
    W[1, :4] = [-1e-6, 28.0, -0.0, 0.0]
    W[2, 0] = 447.0
    W[2, 1:] = np.linspace(-447.0, 446.0, 15)
    W[3, :] = -1e-30
    W[3, 0] = 1.0
    mids = (np.array([d for _, d in ref.codebook(ref.FP6_E3M2)][:32])[:-1]
            + np.array([d for _, d in ref.codebook(ref.FP6_E3M2)][1:32])) / 2
    W[4, :] = np.concatenate([mids[:15], [28.0]]) * (28.0 / 28.0)
    W[5, :] = -mids[15:]
    cases.append(("f64_specials_6x16", W))
    # every finite positive f16 value as a weight column of one row block
    f16_all = np.arange(0x0000, 0x7C00, dtype=np.uint16).view(np.float16)
    cols = 124
    n = f16_all.size // cols + 1
    Wf = np.zeros(n * cols, dtype=np.float16)
    Wf[: f16_all.size] = f16_all
    Wf = Wf.reshape(n, cols)
    Wf[1::2] *= np.float16(-1)
    # keep every row foldable (peak < 447.9): clamp huge rows to a copy scaled
    peak = np.abs(Wf.astype(np.float64)).max(axis=1)
    big = peak >= 447.0
    Wf[big] = (Wf[big].astype(np.float64) / 256.0).astype(np.float16)
    cases.append(("f16_all_values", Wf))
    return cases


def main():
    out = {}
    names = []
    for name, W in quant_cases():
        q = ref.quantize_tensor(np.asarray(W, dtype=np.float64), CGQ_FP6, bias_shift=True)
        names.append(name)
        out[f"q/{name}/W"] = W
        out[f"q/{name}/scales"] = q.scales.view(np.uint16)
        out[f"q/{name}/folded"] = q.folded_scales.view(np.uint16)
        out[f"q/{name}/seg4"] = q.payload.seg4
        out[f"q/{name}/seg2"] = q.payload.seg_tail
        out[f"q/{name}/codes"] = ref.unpack(ref.FP6_E3M2, q.payload)
        out[f"q/{name}/deq"] = ref.dequantize_tensor(q, "bias_shift")
    out["q_names"] = np.array(names)

    # error cases: (name, W, bias_shift, expected exception class name)
    errs = [("peak_447_9", np.array([[447.9, 1.0]]), True),
            ("peak_1e6_fold", np.array([[1e6, 1.0]]), True),
            ("peak_1e6_nofold", np.array([[1e6, 1.0]]), False),
            ("peak_3e6", np.array([[3e6, 1.0]]), False),
            ("nan", np.array([[np.nan, 1.0]]), True),
            ("inf", np.array([[1.0, -np.inf]]), True)]
    enames = []
    for name, W, bs in errs:
        try:
            q = ref.quantize_tensor(W, CGQ_FP6, bias_shift=bs)
            res = "ok"
            out[f"e/{name}/scales"] = q.scales.view(np.uint16)
        except ref.LpqtError as exc:
            res = type(exc).__name__
        enames.append(name)
        out[f"e/{name}/W"] = W
        out[f"e/{name}/bias_shift"] = np.array(bs)
        out[f"e/{name}/result"] = np.array(res)
    out["e_names"] = np.array(enames)

    # encode: every midpoint and its f64 neighbours, plus seeded uniforms
    mids = np.array([d for _, d in ref.codebook(ref.FP6_E3M2)][:32])
    mids = (mids[:-1] + mids[1:]) / 2
    xs = np.concatenate([mids, np.nextafter(mids, 0), np.nextafter(mids, 100),
                         -mids, [0.0, -0.0, 28.0, 100.0, -100.0, -1e-300, 1e-300],
                         np.random.default_rng(101).uniform(-30, 30, 4000)])
    out["enc/x"] = xs
    out["enc/codes"] = ref.encode_rtn_array(ref.FP6_E3M2, xs)

    # packing KAT + random lengths
    r = np.random.default_rng(12)
    plens = [0, 1, 2, 3, 4, 5, 7, 8, 9, 31, 32, 33, 255, 1024, 1025]
    for n in plens:
        c = r.integers(0, 64, size=n, dtype=np.uint8)
        seg = ref.pack(ref.FP6_E3M2, c)
        out[f"p/{n}/codes"] = c
        out[f"p/{n}/seg4"] = seg.seg4
        out[f"p/{n}/seg2"] = seg.seg_tail
    out["p_lens"] = np.array(plens)

    # fold: every in-range f16 scale, and the exhaustive bias-shift sweep hash
    scales = np.arange(0x0001, 0x4C00, dtype=np.uint16).view(np.float16)
    folded = ref.fold_scale_array(ref.FP6_E3M2, scales)
    out["fold/scales"] = scales.view(np.uint16)
    out["fold/folded"] = folded.view(np.uint16)
    codes = np.arange(64, dtype=np.uint8)
    sweep = ref.dequant_bias_shift_array(ref.FP6_E3M2, codes[:, None], folded[None, :])
    out["fold/sweep_sha256"] = np.array(hashlib.sha256(sweep.view(np.uint16).tobytes()).hexdigest())
    out["compose"] = ref.compose_table_f16(ref.FP6_E3M2).view(np.uint16)
    out["value_table"] = ref.value_table(ref.FP6_E3M2)

    # GEMM: reference gemm_quantized (f32) and the f64 oracle on the same inputs
    gcases = []
    r = np.random.default_rng(309)
    values = np.array([v for _, v in ref.codebook(ref.FP6_E3M2)])
    W = 0.25 * r.choice(values, size=(8, 8))
    W[:, 0] = 0.25 * 28.0
    gcases.append(("grid_exact_8x8x8", W, r.integers(-2, 3, size=(8, 8)).astype(np.float16)))
    r = np.random.default_rng(34)
    for i in range(4):
        n, k, m = (int(v) for v in r.integers(2, 65, size=3))
        gcases.append((f"rand{i}_{n}x{k}x{m}", r.standard_normal((n, k)),
                       r.standard_normal((k, m)).astype(np.float16)))
    r = np.random.default_rng(35)
    gcases.append(("llama_256x512x16", (r.standard_normal((256, 512)) * 0.02).astype(np.float16),
                   r.standard_normal((512, 16)).astype(np.float16)))
    gcases.append(("decode_384x1024x1", (r.standard_normal((384, 1024)) * 0.02).astype(np.float16),
                   r.standard_normal((1024, 1)).astype(np.float16)))
    gnames = []
    for name, W, X in gcases:
        q = ref.quantize_tensor(np.asarray(W, np.float64), CGQ_FP6, bias_shift=True)
        gnames.append(name)
        out[f"g/{name}/W"] = W
        out[f"g/{name}/X"] = X
        out[f"g/{name}/Y"] = ref.gemm_quantized(q, X)
        out[f"g/{name}/Yf64"] = ref.gemm_reference(ref.dequantize_tensor(q, "bias_shift"), X)
        out[f"g/{name}/tol"] = np.array(ref.gemm_tolerance(W.shape[1], ref.dequantize_tensor(q), X))
    out["g_names"] = np.array(gnames)

    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
