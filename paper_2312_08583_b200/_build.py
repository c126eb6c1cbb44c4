"""Build liblpqt_b200.so in-tree with nvcc for sm_100a (no JIT, no torch ext).

    python -m paper_2312_08583_b200._build          # incremental
    python -m paper_2312_08583_b200._build --force  # rebuild everything
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "lpqt")
LIB = os.path.join(PKG, "liblpqt_b200.so")
SOURCES = ["capi.cu", "quantize.cu", "prepack.cu", "gemm.cu", "exact.cu", "prefill2sm.cu"]
HEADERS = ["common.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines: list[str] | None = None,
          lib_path: str | None = None, build_dir: str | None = None,
          source_override: dict[str, str] | None = None) -> str:
    """Compile + link.  `defines`/`lib_path`/`build_dir` build experiment
    variants (e.g. -DLPQT_WAIT_MODE=1) next to the default library."""
    lib_out = lib_path or LIB
    bdir = build_dir or BUILD
    extra = [f"-D{d}" for d in (defines or [])]
    os.makedirs(bdir, exist_ok=True)
    nvcc = _nvcc()
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "lpqt_b200.h")]
    objs = []
    jobs = []
    for src in SOURCES:
        s = (source_override or {}).get(src) or os.path.join(CSRC, src)
        o = os.path.join(bdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([nvcc, *ARCH, *FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    with ThreadPoolExecutor(max_workers=4) as ex:
        for cmd, r in ex.map(run, jobs):
            log = (r.stdout or "") + (r.stderr or "")
            with open(os.path.join(bdir, os.path.basename(cmd[-1]) + ".log"), "w") as f:
                f.write(log)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {cmd[-3]}:\n{log}")
            if verbose:
                print(log)
    if force or jobs or _stale(lib_out, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", lib_out, *objs, "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    return lib_out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
