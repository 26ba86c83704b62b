"""Build the C-ABI library of an older git revision for same-box A/B timing.

    python tools/build_rev.py REV NAME
Outputs paper_2604_19157_b200/_lib/variants/libkvrot_<NAME>.so (use with KVR_LIB_PATH)."""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_19157_b200 import build as B  # noqa: E402

rev, name = sys.argv[1], sys.argv[2]
out_dir = os.path.join(B.LIB_DIR, "variants")
os.makedirs(out_dir, exist_ok=True)
with tempfile.TemporaryDirectory() as tmp:
    tar = subprocess.run(["git", "-C", ROOT, "archive", rev, "paper_2604_19157_b200/csrc", "include"],
                         check=True, capture_output=True).stdout
    subprocess.run(["tar", "-x", "-C", tmp], input=tar, check=True)
    csrc = os.path.join(tmp, "paper_2604_19157_b200", "csrc")
    common = B.ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                       "-I", os.path.join(tmp, "include")]
    objs = []
    for src in sorted(f for f in os.listdir(csrc) if f.endswith(".cu")):
        obj = os.path.join(tmp, src.replace(".cu", ".o"))
        subprocess.run([B.nvcc_path()] + common + ["-c", os.path.join(csrc, src), "-o", obj], check=True)
        objs.append(obj)
    lib = os.path.join(out_dir, f"libkvrot_{name}.so")
    subprocess.run([B.nvcc_path()] + B.ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs, check=True)
print(lib)
