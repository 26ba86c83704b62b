"""ctypes binding of libkvrot_b200.so (the C ABI in include/kvrot_b200.h).

This is the only place the package touches native code.  Loading fails loudly
if the library is missing: there is no CPU fallback anywhere in the package.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KVR_LIB_PATH") or os.path.join(_HERE, "_lib", "libkvrot_b200.so")  # override: tools only

KVR_F64, KVR_F32, KVR_BF16, KVR_F16 = 0, 1, 2, 3
KVR_KEYS_ONLY, KVR_KEYS_AND_VALUES = 0, 1
KVR_FLAG_NONFINITE = 1
KVR_FLAG_LEN_OVERFLOW = 2
KVR_PREC_INT4, KVR_PREC_BF16 = 0, 1
KVR_ERR_UNSUPPORTED = 3

# every symbol include/kvrot_b200.h declares
EXPORTED = (
    "kvr_pool_init", "kvr_pool_init_bf16", "kvr_last_error", "kvr_abi_version", "kvr_device_sms",
    "kvr_fwht_rows_f64", "kvr_pack_rows", "kvr_unpack_rows", "kvr_quantize_rows_f64",
    "kvr_dequantize_rows_f64", "kvr_block_rotate", "kvr_rotate_quantize_store",
    "kvr_dequantize_pages", "kvr_decode_workspace_bytes", "kvr_decode_pick_splits",
    "kvr_paged_decode", "kvr_decode_step", "kvr_debug_decode_trace", "kvr_debug_set_k1_impl", "kvr_note_pool_write",
    "kvr_host_all_finite", "kvr_decode_flat_f64", "kvr_step_stage", "kvr_step_launch",
    "kvr_step_ring_create", "kvr_step_ring_set_slot", "kvr_step_ring_run", "kvr_step_ring_destroy",
    "kvr_step_ring_set_copy_stream", "kvr_step_ring_set_decode", "kvr_debug_step_ring_times",
    "kvr_rotate_quantize_store_learned", "kvr_learned_pack_image", "kvr_rows_matmul_f64",
    "kvr_paged_decode_learned",
)


class KvrPool(ctypes.Structure):
    _fields_ = [
        ("base", ctypes.c_void_p),
        ("num_pages", ctypes.c_int64),
        ("page_tokens", ctypes.c_int32),
        ("num_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("page_bytes", ctypes.c_int32),
        ("cell_tokens", ctypes.c_int32),
        ("cell_bytes", ctypes.c_int32),
        ("precision", ctypes.c_int32),
    ]


_lib = None

_P, _I32, _I64, _SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t


def _declare(lib):
    sig = {
        "kvr_pool_init": (_I32, [ctypes.POINTER(KvrPool), _P, _I64, _I32, _I32, _I32]),
        "kvr_pool_init_bf16": (_I32, [ctypes.POINTER(KvrPool), _P, _I64, _I32, _I32, _I32]),
        "kvr_last_error": (ctypes.c_char_p, []),
        "kvr_debug_decode_trace": (None, [_P]),
        "kvr_debug_set_k1_impl": (None, [_I32]),
        "kvr_note_pool_write": (None, [_P]),
        "kvr_host_all_finite": (_I32, [_P, _I32, _I64]),
        "kvr_step_stage": (_I32, [_P, _P, _P, _I64, _I64, _I32, _P, _I64, _P, _I64, _I64, _I32, _I32]),
        "kvr_step_launch": (_I32, [_P, _P, _I64, _P, _P, _P]),
        "kvr_step_ring_create": (_P, [_I32, _P, _I64, _I64, _I32, _P, _I64, _P, _I64, _I64, _I32, _I64, _I64, _I32, _P]),
        "kvr_step_ring_set_slot": (_I32, [_P, _I32, _P, _P, _P, _P]),
        "kvr_step_ring_run": (_I32, [_P, _I32, _P]),
        "kvr_step_ring_destroy": (None, [_P]),
        "kvr_step_ring_set_copy_stream": (_I32, [_P, _P]),
        "kvr_debug_step_ring_times": (None, [_P]),
        "kvr_step_ring_set_decode": (_I32, [_P, _I32, _I32, ctypes.POINTER(KvrPool), _P, _I32, _I32, _I32, _I32, _I32,
                                            _I32, _I32, _P, _P, _P, _SZ, _I32, _P, _I32]),
        "kvr_decode_flat_f64": (_I32, [_P, _P, _P, _I64, _I32, _I32, _I32, _P, _P]),
        "kvr_abi_version": (_I32, []),
        "kvr_device_sms": (_I32, []),
        "kvr_fwht_rows_f64": (_I32, [_P, _I64, _I32, _I32, _P]),
        "kvr_pack_rows": (_I32, [_P, _P, _I64, _I32, _P]),
        "kvr_unpack_rows": (_I32, [_P, _P, _I64, _I32, _P]),
        "kvr_quantize_rows_f64": (_I32, [_P, _I64, _I32, _P, _P, _P, _P]),
        "kvr_dequantize_rows_f64": (_I32, [_P, _P, _P, _I64, _I32, _P, _P]),
        "kvr_block_rotate": (_I32, [_P, _I32, _P, _I32, _I64, _I32, _I32, _P, _I32, _P]),
        "kvr_rotate_quantize_store": (_I32, [_P, _P, _I32, _I64, _P, ctypes.POINTER(KvrPool), _I32, _I32, _I32,
                                             _P, _I32, _P, _P]),
        "kvr_rotate_quantize_store_learned": (_I32, [_P, _P, _I32, _I64, _P, ctypes.POINTER(KvrPool), _I32, _I32,
                                                     _I32, _P, _P, _P, _P, _P]),
        "kvr_learned_pack_image": (None, [_P, _P]),
        "kvr_rows_matmul_f64": (_I32, [_P, _I32, _P, _P, _I32, _I64, _I32, _P]),
        "kvr_dequantize_pages": (_I32, [ctypes.POINTER(KvrPool), _P, _I32, _P, _I32, _I32, _P, _P, _I32, _P]),
        "kvr_decode_workspace_bytes": (_SZ, [_I32, _I32, _I32, _I32, _I32]),
        "kvr_decode_pick_splits": (_I32, [_I32, _I32, _I32, _I32]),
        "kvr_paged_decode": (_I32, [_P, _I32, ctypes.POINTER(KvrPool), _P, _I32, _P, _I32, _I32, _I32, _I32, _I32,
                                    _I32, _P, _P, _P, _SZ, _I32, _P]),
        "kvr_paged_decode_learned": (_I32, [_P, _I32, ctypes.POINTER(KvrPool), _P, _I32, _P, _I32, _I32, _I32, _P,
                                            _I32, _I32, _P, _P, _P, _SZ, _I32, _P]),
        "kvr_decode_step": (_I32, [_P, _I32, _P, _P, _I32, _P, ctypes.POINTER(KvrPool), _P, _I32, _P, _I32, _I32,
                                   _I32, _I32, _I32, _I32, _P, _P, _P, _SZ, _I32, _P, _P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """The loaded native library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise errors.BackendUnavailableError(
                f"native library missing: {LIB_PATH} (run `python -m paper_2604_19157_b200.build`)")
        handle = ctypes.CDLL(LIB_PATH)
        _declare(handle)
        _lib = handle
    return _lib


_STATUS = {
    1: errors.ShapeError,
    2: errors.InvalidOrderError,
    3: errors.UnsupportedConfigError,
    4: errors.DeviceError,
    5: errors.ShapeError,
    6: errors.NonFiniteInputError,
}


def check(rc: int) -> None:
    if rc:
        msg = lib().kvr_last_error().decode(errors="replace")
        raise _STATUS.get(rc, errors.DeviceError)(msg)


def sign_words(signs, head_dim: int):
    """(d,) +-1 vector -> ctypes uint32 array, bit i set <=> signs[i] == -1."""
    if signs is None:
        return None
    bits = np.zeros(((head_dim + 31) // 32) * 32, dtype=np.uint8)
    neg = np.asarray(signs) < 0
    bits[:neg.size] = neg
    w = np.packbits(bits.reshape(-1, 32), axis=1, bitorder="little").view("<u4").reshape(-1)
    return (ctypes.c_uint32 * w.size)(*w.tolist())
