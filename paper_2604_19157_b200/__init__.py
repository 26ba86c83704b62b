"""B200-native Hadamard-rotated INT4 KV cache: the serving hot path of arXiv 2604.19157.

Drop-in for the `kvrot` reference's hot-path API (rotate / quantize /
dequantize, paged-cache write, decode attention); every numeric path runs in
the sm_100a CUDA library `_lib/libkvrot_b200.so` through a C ABI
(include/kvrot_b200.h).  There is no CPU fallback.
"""

__version__ = "0.1.0"

from ._kernels import available_backends, get_backend
from .attention import DecodePlan, DecodeRequest, decode_batch, decode_step, decode_step_fp
from .cache import BF16, INT4, PageTable, bf16_bits_to_float, capacity_tokens, float_to_bf16_bits, token_bytes
from .errors import KvrotError
from .hadamard import HadamardMatrix, block_hadamard_matrix, fwht_blocks, make_hadamard
from .int4 import PackedNibbles, QuantParams, dequantize_head, pack, quantize_head, unpack
from .layout import HeadLayout
from .rotation import (RotationSpec, Targets, apply_block_rotation, apply_inverse_rotation, compose_transform,
                       make_signs, value_branch_spec)

__all__ = [
    "__version__", "available_backends", "get_backend",
    "DecodePlan", "DecodeRequest", "decode_batch", "decode_step", "decode_step_fp",
    "BF16", "INT4", "PageTable", "bf16_bits_to_float", "capacity_tokens", "float_to_bf16_bits", "token_bytes",
    "KvrotError",
    "HadamardMatrix", "block_hadamard_matrix", "fwht_blocks", "make_hadamard",
    "PackedNibbles", "QuantParams", "dequantize_head", "pack", "quantize_head", "unpack",
    "HeadLayout",
    "RotationSpec", "Targets", "apply_block_rotation", "apply_inverse_rotation", "compose_transform", "make_signs",
    "value_branch_spec",
]
