"""The C-ABI library builds for sm_100a, loads without a GPU and exports
every entry point include/kvrot_b200.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kvrot_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(kvr_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2604_19157_b200 import build

    return build.build()


def test_header_symbols_exported(libpath):
    lib = ctypes.CDLL(libpath)
    syms = declared_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
    from paper_2604_19157_b200 import _lib

    assert sorted(_lib.EXPORTED) == syms


def test_cubin_is_sm100a_with_tma_and_mma(libpath):
    out = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper()
    assert "UTMALDG" in out          # TMA tile loads in the write kernel
    assert "HMMA" in out             # tensor-core decode
    assert "FADD2" in out or "FFMA2" in out  # packed f32x2 butterfly / quantizer


def test_pool_init_layout(libpath):
    from paper_2604_19157_b200 import _lib

    lib = _lib.lib()
    pool = _lib.KvrPool()
    assert lib.kvr_pool_init(ctypes.byref(pool), None, 10, 16, 8, 128) == 0
    # B200 cell layout: 8 heads x one 16-token cell of 16*(128+10) = 2208 B per page
    # (same bytes as a .kvpg record: 17664 B, cache.py:56-68)
    assert pool.page_bytes == 17664
    assert (pool.cell_tokens, pool.cell_bytes) == (16, 2208)
    assert lib.kvr_pool_init(ctypes.byref(pool), None, 10, 4, 2, 32) == 0
    assert (pool.cell_tokens, pool.cell_bytes, pool.page_bytes) == (4, 176, 2 * 176)
    assert lib.kvr_abi_version() == 2
    assert lib.kvr_decode_workspace_bytes(1, 8, 32, 128, 4) > 0


def test_errors_without_device(libpath):
    from paper_2604_19157_b200 import _lib

    lib = _lib.lib()
    # argument validation happens before any CUDA call
    assert lib.kvr_fwht_rows_f64(None, 4, 24, 16, None) == 2  # InvalidOrder: 16 does not divide 24
    assert b"does not divide" in lib.kvr_last_error()
    assert lib.kvr_quantize_rows_f64(None, 4, 7, None, None, None, None) == 1


def test_split_count_model(libpath):
    """kvr_decode_pick_splits on the BASELINE configs (148-SM fallback without a GPU):
    one wave of CTAs, inline merge for C2 / C3 B = 1, the merge kernel's 16-multiples
    and the one-wave fill for C5, no split for the batched configs."""
    from paper_2604_19157_b200 import _lib

    pick = _lib.lib().kvr_decode_pick_splits
    assert pick(1, 8, 32768 + 1, 16) == 18       # C2: 8 x 18 = 144 CTAs, inline merge
    assert pick(1, 8, 8192 + 1, 16) == 16        # C3 B = 1
    assert pick(16, 8, 8192 + 1, 16) == 1        # C3 B = 16: 128 units already
    assert pick(16, 8, 16384 + 1, 16) == 1       # C4 per-GPU shard
    assert pick(1, 1, 131072 + 1, 16) == 128     # C5 128k: a multiple of 16 above 32
    assert pick(1, 1, 1048576 + 1, 16) == 148    # C5 1M: the one-wave fill
    for b, h, L in ((1, 8, 32769), (2, 8, 32768), (1, 1, 1 << 20), (4, 8, 4096)):
        s = pick(b, h, L, 16)
        assert 1 <= s <= 256 and (b * h * s <= 148 or s == 1)


def test_learned_entry_points_validate_without_device(libpath):
    """Row f3's entry points reject bad arguments before any CUDA call (reference-style
    exceptions through _lib.check), and the host image packer is a pure host function."""
    import numpy as np

    from paper_2604_19157_b200 import _lib

    lib = _lib.lib()
    pool = _lib.KvrPool()
    assert lib.kvr_pool_init(ctypes.byref(pool), ctypes.c_void_p(16), 4, 16, 8, 128) == 0
    dummy = ctypes.c_void_p(256)
    args = (dummy, dummy, _lib.KVR_BF16, 16, dummy, ctypes.byref(pool), 128, _lib.KVR_KEYS_AND_VALUES, 1, None)
    assert lib.kvr_rotate_quantize_store_learned(*args, None, dummy, None, None) == 5  # null t_img
    assert lib.kvr_rotate_quantize_store_learned(*args[:7], 7, *args[8:], dummy, dummy, None, None) == 5  # targets
    assert lib.kvr_rotate_quantize_store_learned(*args[:6], 48, *args[7:], dummy, dummy, None, None) == 2  # order
    bf = _lib.KvrPool()
    assert lib.kvr_pool_init_bf16(ctypes.byref(bf), ctypes.c_void_p(16), 4, 16, 8, 128) == 0
    a2 = list(args)
    a2[5] = ctypes.byref(bf)
    assert lib.kvr_rotate_quantize_store_learned(*a2, dummy, dummy, None, None) == 3  # BF16 pool
    # the fused learned decode: null / misaligned T, out_mode, order (mode 1), BF16 pool, G = 3
    dargs = (dummy, _lib.KVR_BF16, ctypes.byref(pool), dummy, 4, dummy, 1, 32, 64)
    tail = (128, None, dummy, dummy, 1 << 20, 0, None)
    assert lib.kvr_paged_decode_learned(*dargs, None, 2, *tail) == 5  # null T
    assert lib.kvr_paged_decode_learned(*dargs, ctypes.c_void_p(264), 2, *tail) == 5  # misaligned T
    assert lib.kvr_paged_decode_learned(*dargs, dummy, 3, *tail) == 5  # out_mode
    assert lib.kvr_paged_decode_learned(*dargs, dummy, 1, 48, *tail[1:]) == 2  # Hadamard order
    d_bf = list(dargs)
    d_bf[2] = ctypes.byref(bf)
    assert lib.kvr_paged_decode_learned(*d_bf, dummy, 2, *tail) == 3  # BF16 pool: the row-matmul route
    d_g3 = list(dargs)
    d_g3[7] = 24
    assert lib.kvr_paged_decode_learned(*d_g3, dummy, 2, *tail) == 3  # G = 3
    # rows_matmul: shape, size, aliasing and null checks
    assert lib.kvr_rows_matmul_f64(dummy, _lib.KVR_F64, dummy, dummy, _lib.KVR_F64, -1, 128, None) == 1
    assert lib.kvr_rows_matmul_f64(dummy, _lib.KVR_F64, dummy, ctypes.c_void_p(512), _lib.KVR_F64, 4, 1024,
                                   None) == 3
    assert lib.kvr_rows_matmul_f64(dummy, _lib.KVR_F64, dummy, dummy, _lib.KVR_F64, 4, 128, None) == 5
    assert lib.kvr_rows_matmul_f64(None, _lib.KVR_F64, dummy, ctypes.c_void_p(512), _lib.KVR_F64, 4, 128, None) == 5
    assert lib.kvr_rows_matmul_f64(dummy, _lib.KVR_F64, dummy, ctypes.c_void_p(512), _lib.KVR_F64, 0, 128, None) == 0
    # the T image: part p of element (n, k) sits at the SW128 K-major offset; hi + mid + lo == T to ~2^-24
    t = np.random.default_rng(0).standard_normal((128, 128)) * 0.1
    img = np.zeros(3 * 128 * 128, dtype=np.uint16)
    lib.kvr_learned_pack_image(t.ctypes.data, img.ctypes.data)

    def bf(u):
        return (u.astype(np.uint32) << 16).view(np.float32).astype(np.float64)

    for n, k in ((0, 0), (5, 70), (127, 127), (64, 3)):
        byte = (k & 63) * 2
        off = (k >> 6) * 16384 + (n >> 3) * 1024 + (n & 7) * 128 + (((byte >> 4) ^ (n & 7)) << 4) + (byte & 15)
        parts = [bf(img[(p * 32768 + off) // 2:(p * 32768 + off) // 2 + 1])[0] for p in range(3)]
        assert abs(sum(parts) - t[k, n]) <= 2.0 ** -24 * abs(t[k, n]) + 1e-30
