"""Static SASS instruction counts per 32 weights of each FP6 -> FP16 rebuild
(dev tool, runs here without a GPU): compiles tools/dq_bench.cu for sm_100a
and counts the instructions of each bench<MODE> kernel, normalised by the
number of 32-weight groups the compiler unrolled (F2FP / 16, or PRMT / 16 for
the converter-free rebuilds, 32 for the naive cast).  Counts include the loop's own ~7 IADD3 and the
6 IMAD that perturb the input words.

python tools/rebuild_ops.py > profiles/r02_rebuild_sass_ops.txt
"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
exe = os.path.join(ROOT, "build", "dq_bench")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                os.path.join(ROOT, "tools", "dq_bench.cu"), "-o", exe], check=True)
sass = subprocess.run(["cuobjdump", "-sass", exe], capture_output=True, text=True, check=True).stdout
names = {0: "bias-shift PRMT (byte-form layout)", 1: "cvt e3m2x2, masked containers", 2: "cvt e3m2x2, no mask",
         3: "GEMM tile layout + cvt (product)", 4: "canonical 4+2 planes + cvt", 5: "native FP5 tiles + cvt",
         6: "ablation: software bias-shift x S", 7: "ablation: naive two-step x S"}
funcs, cur = {}, None
for line in sass.split("\n"):
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    if cur:
        m = re.search(r"\*/\s+(@!?U?P\d\s+)?([A-Z0-9_]+)", line)
        if m:
            funcs[cur][m.group(2)] += 1
alu = ["LOP3", "SHF", "PRMT", "IADD3", "LEA", "SEL", "ISETP", "LOP"]
print(f"{'rebuild':36s} {'F2FP':>5s} {'ALU':>5s} {'HMUL2':>6s} {'IMAD':>5s}   (per 32 weights)")
for f, c in sorted(funcs.items()):
    m = re.search(r"benchILi(\d)", f)
    if not m:
        continue
    mode = int(m.group(1))
    # (16 F2FP per 32 weights; without the converter: 16 PRMT, the naive cast 32)
    groups = c["F2FP"] / 16 if c["F2FP"] else c["PRMT"] / (32 if mode == 7 else 16)
    groups = groups or 1
    print(f"{names[mode]:36s} {c['F2FP'] / groups:5.1f} {sum(c[k] for k in alu) / groups:5.1f} "
          f"{(c['HMUL2'] + c['HFMA2']) / groups:6.1f} {c['IMAD'] / groups:5.1f}")
