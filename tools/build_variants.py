"""Build decode-kernel variants (compile-time macros) into separate libraries for A/B timing.

    python tools/build_variants.py NAME=-DFOO=1,-DBAR=0 NAME2=...
Outputs paper_2604_19157_b200/_lib/variants/libkvrot_<NAME>.so; time them with
    KVR_LIB_PATH=<so> python tools/trace_decode.py ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_19157_b200 import build as B  # noqa: E402

out_dir = os.path.join(B.LIB_DIR, "variants")
os.makedirs(out_dir, exist_ok=True)
nvcc = B.nvcc_path()
common = B.ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                   "-I", os.path.join(ROOT, "include")]
for spec in sys.argv[1:]:
    name, _, flags = spec.partition("=")
    defs = [f for f in flags.split(",") if f]
    objs = []
    for src in B.SOURCES:
        obj = os.path.join(out_dir, f"{name}_{src.replace('.cu', '.o')}")
        subprocess.run([nvcc] + common + defs + ["-c", os.path.join(B.CSRC, src), "-o", obj], check=True)
        objs.append(obj)
    lib = os.path.join(out_dir, f"libkvrot_{name}.so")
    subprocess.run([nvcc] + B.ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs, check=True)
    for o in objs:
        os.remove(o)
    print(lib)
