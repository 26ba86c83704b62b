"""Build the reference's own compiled CPU kernels into oracle/_ref/ (checker / CPU
baseline only; never shipped, never on the product path).

    python oracle/build_ref.py

Compiles /root/reference/pkg/src/kvrot/_kernels/_core.pyx (the reference's Cython
backend: fwht_rows, pack_rows, unpack_rows, quantize_rows, dequantize_rows --
bit-identical to its numpy backend, _core.pyx:1-8) from where it lies, with the
image's Cython + gcc, into oracle/_ref/kvrot_core.*.so.  The reference's own build
system is not used; outputs go only to oracle/_ref/ (git-ignored, travels to the
GPU box with the snapshot).  Skips quietly when /root/reference is absent.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
import sysconfig
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
SRC = "/root/reference/pkg/src/kvrot/_kernels/_core.pyx"


def build() -> str | None:
    if not os.path.exists(SRC):
        return None
    import numpy as np

    os.makedirs(OUT, exist_ok=True)
    suffix = sysconfig.get_config_var("EXT_SUFFIX")
    target = os.path.join(OUT, "kvrot_core" + suffix)
    if os.path.exists(target) and os.path.getmtime(target) >= os.path.getmtime(SRC):
        return target
    with tempfile.TemporaryDirectory() as tmp:
        pyx = os.path.join(tmp, "kvrot_core.pyx")  # module name kvrot_core; the source is read, not copied in-tree
        shutil.copyfile(SRC, pyx)
        csrc = os.path.join(tmp, "kvrot_core.c")
        subprocess.run([sys.executable, "-m", "cython", "-3", "-o", csrc, pyx], check=True, capture_output=True)
        cmd = ["gcc", "-O3", "-shared", "-fPIC", "-I", sysconfig.get_paths()["include"], "-I", np.get_include(),
               "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION", csrc, "-o", target]
        subprocess.run(cmd, check=True, capture_output=True)
    return target


def load():
    """The compiled reference kernels module, or None when not built."""
    import importlib.util

    for path in glob.glob(os.path.join(OUT, "kvrot_core*.so")):
        spec = importlib.util.spec_from_file_location("kvrot_core", path)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        return mod
    return None


if __name__ == "__main__":
    print(build())
