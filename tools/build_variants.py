"""Build liblpqt_b200 variants with -D overrides into build/variants/ (dev tool).

python tools/build_variants.py name:DEF1=v,DEF2=v name2:DEF=v ...
Object files go to build/obj/<name> (gpurun-ignored); the .so travels.
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_08583_b200 import _build  # noqa: E402


def one(spec):
    name, _, defs = spec.partition(":")
    d = [x for x in defs.split(",") if x]
    return _build.build(defines=d, lib_path=f"build/variants/lib_{name}.so", build_dir=f"build/obj/{name}")


if __name__ == "__main__":
    os.makedirs("build/variants", exist_ok=True)
    with ThreadPoolExecutor(max_workers=4) as ex:
        for out in ex.map(one, sys.argv[1:]):
            print(out)
