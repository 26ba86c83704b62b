"""Rotation specs and block-diagonal Hadamard rotation (mirrors kvrot.rotation, transform part).

Row convention as in the reference (rotation.py:118-159):
    forward  x -> x diag(s) H_blk R      inverse  x -> x R^T H_blk diag(s)
The block butterfly runs in the native library in f64 (bit-identical to the
reference).  The optional learned factor R (row f3; its Hessian calibration is out
of scope) is applied by the library's f64 row-matmul kernel (kvr_rows_matmul_f64),
composed with the butterfly into one dense T for decode queries and outputs, and
fused into the tcgen05 K1 for bf16 writes (kvr_rotate_quantize_store_learned).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np
import torch

from . import _kernels, _lib
from .errors import InvalidOrderError, ShapeError
from .hadamard import block_hadamard_matrix
from .layout import HeadLayout, is_power_of_two


class Targets(enum.Enum):
    KEYS_ONLY = "keys_only"
    KEYS_AND_VALUES = "keys_and_values"


@dataclass(frozen=True)
class RotationSpec:
    """Hadamard block order, optional +-1 signs, optional learned orthogonal R, targets."""

    order: int
    signs: Optional[np.ndarray] = None
    learned: Optional[np.ndarray] = None
    targets: Targets = Targets.KEYS_AND_VALUES
    learned_values: bool = False

    def __post_init__(self) -> None:
        if not is_power_of_two(self.order):
            raise InvalidOrderError(f"order={self.order} is not a power of two")
        if self.signs is not None:
            s = np.array(self.signs, dtype=np.float64, copy=True).reshape(np.shape(self.signs))
            if s.ndim != 1:
                raise ShapeError("signs must be a vector")
            if not np.all(np.abs(s) == 1.0):
                raise ShapeError("signs entries must be +-1")
            s.setflags(write=False)
            object.__setattr__(self, "signs", s)
        if self.learned is not None:
            r = np.array(self.learned, dtype=np.float64, copy=True)
            if r.ndim != 2 or r.shape[0] != r.shape[1]:
                raise ShapeError(f"learned rotation must be square, got {r.shape}")
            dev = np.abs(r.T @ r - np.eye(r.shape[0])).max()
            if dev > 1e-6:
                raise ShapeError(f"learned rotation not orthogonal (max dev {dev:.2e})")
            r.setflags(write=False)
            object.__setattr__(self, "learned", r)

    def sign_words(self, head_dim: int):
        """The signs as the C ABI's bitmask words (memoised: the spec is immutable)."""
        cache = self.__dict__.setdefault("_words", {})
        if head_dim not in cache:
            cache[head_dim] = _lib.sign_words(self.signs, head_dim)
        return cache[head_dim]


def make_signs(seed: int, layer: int, head_dim: int, order: int) -> np.ndarray:
    """Deterministic +-1 vector, one Philox stream per (seed, layer, block) (rotation.py:81-101).

    The sign vector is a parameter of the rotation (computed once per layer),
    so it is generated with numpy's Philox exactly as the reference does.
    """
    if not is_power_of_two(order) or head_dim % order:
        raise InvalidOrderError(f"order={order} does not divide head_dim={head_dim}")
    if not 0 <= layer < (1 << 24):
        raise ShapeError(f"layer={layer} outside supported range [0, 2^24)")
    blocks = []
    for blk in range(head_dim // order):
        key = np.array([seed & ((1 << 64) - 1), (0x5164 << 48) | (layer << 24) | blk], dtype=np.uint64)
        draws = np.random.Generator(np.random.Philox(key=key)).integers(0, 2, size=order)
        blocks.append(draws * 2.0 - 1.0)
    return np.concatenate(blocks).astype(np.float64)


def _check_spec_layout(spec: RotationSpec, layout: HeadLayout) -> None:
    d = layout.head_dim
    if spec.order != layout.rot_order:
        raise ShapeError(f"spec order {spec.order} != layout rot_order {layout.rot_order}")
    if d % spec.order:
        raise InvalidOrderError(f"order={spec.order} does not divide head_dim={d}")
    if spec.signs is not None and spec.signs.shape != (d,):
        raise ShapeError(f"signs length {spec.signs.shape} != head_dim {d}")
    if spec.learned is not None and spec.learned.shape != (d, d):
        raise ShapeError(f"learned shape {spec.learned.shape} != ({d}, {d})")


def _rotate(x, layout: HeadLayout, spec: RotationSpec, inverse: bool):
    is_np = not isinstance(x, torch.Tensor)
    t = _kernels.to_device(np.asarray(x, dtype=np.float64) if is_np else x, torch.float64)
    if t.ndim != 2 or t.shape[1] != layout.head_dim:
        raise ShapeError(f"expected (n, {layout.head_dim}) rows, got {tuple(t.shape)}")
    _check_spec_layout(spec, layout)
    n, d = t.shape
    if inverse and spec.learned is not None:
        t = rows_matmul(t, learned_on(spec, t.device, transpose=True))
    out = torch.empty_like(t)
    _lib.check(_lib.lib().kvr_block_rotate(_kernels.ptr(t), _lib.KVR_F64, _kernels.ptr(out), _lib.KVR_F64, n, d,
                                           spec.order, spec.sign_words(d), 1 if inverse else 0,
                                           _kernels.stream_ptr()))
    if not inverse and spec.learned is not None:
        out = rows_matmul(out, learned_on(spec, t.device))
    return out.cpu().numpy() if is_np else out


def rows_matmul(x: torch.Tensor, m: torch.Tensor, out: Optional[torch.Tensor] = None,
                out_dtype=torch.float64) -> torch.Tensor:
    """y = x @ m on the device in f64 arithmetic (kvr_rows_matmul_f64): the learned
    factor of row f3 (rotation.py:140-141, 154-155) and the composed transforms."""
    x = x.contiguous()
    n, d = x.shape[0], x.shape[-1]
    if out is None:
        out = torch.empty(x.shape, dtype=out_dtype, device=x.device)
    code = {torch.float64: _lib.KVR_F64, torch.float32: _lib.KVR_F32, torch.bfloat16: _lib.KVR_BF16,
            torch.float16: _lib.KVR_F16}
    _lib.check(_lib.lib().kvr_rows_matmul_f64(_kernels.ptr(x), code[x.dtype], _kernels.ptr(m), _kernels.ptr(out),
                                              code[out.dtype], x.numel() // d, d, _kernels.stream_ptr()))
    return out


def learned_on(spec: RotationSpec, device, transpose: bool = False) -> Optional[torch.Tensor]:
    """The learned factor (or its transpose) as a contiguous f64 device tensor (memoised
    per device, so graph capture and steady-state steps do no host->device copy)."""
    if spec.learned is None:
        return None
    cache = spec.__dict__.setdefault("_learned_dev", {})
    key = (str(torch.device(device)), transpose)
    if key not in cache:
        r = np.array(spec.learned, dtype=np.float64)
        cache[key] = torch.from_numpy(np.ascontiguousarray(r.T if transpose else r)).to(device)
    return cache[key]


def composed_on(spec: RotationSpec, layout: HeadLayout, device, transpose: bool = False,
                values: bool = False) -> Optional[torch.Tensor]:
    """The dense T = diag(s) H_blk R (compose_transform, rotation.py:171-184), or T^T,
    as a contiguous f64 device tensor (memoised on the spec per device and layout): one
    kvr_rows_matmul_f64 launch applies the whole transform to decode queries (T) or
    maps decode outputs back (T^T, T orthogonal).  values=True: the value branch's
    transform (value_branch_spec, rotation.py:162-168); None when values stay raw."""
    cache = spec.__dict__.setdefault("_composed_dev", {})
    key = (str(torch.device(device)), layout.head_dim, layout.rot_order, transpose, values)
    if key not in cache:
        sp = value_branch_spec(spec) if values else spec
        if sp is None:
            cache[key] = None
        else:
            t = compose_transform(sp, layout)
            cache[key] = torch.from_numpy(np.ascontiguousarray(t.T if transpose else t)).to(device)
    return cache[key]


def learned_store_operands(spec: RotationSpec, layout: HeadLayout, device):
    """Row f3, fused K1 operands (memoised per device and layout): the kernel's
    shared-memory image of the dense T = diag(s) H_blk R (compose_transform,
    rotation.py:171-184) as three bf16 parts, and R^T in f64 for the kernel's exact
    recomputation of codes near a rounding boundary."""
    cache = spec.__dict__.setdefault("_learned_store", {})
    key = (str(torch.device(device)), layout.head_dim, layout.rot_order)
    if key not in cache:
        t = np.ascontiguousarray(compose_transform(spec, layout), dtype=np.float64)
        img = np.zeros(3 * t.shape[0] * t.shape[1], dtype=np.uint16)
        _lib.lib().kvr_learned_pack_image(t.ctypes.data, img.ctypes.data)
        rt = np.ascontiguousarray(np.asarray(spec.learned, dtype=np.float64).T)
        cache[key] = (torch.from_numpy(img).to(device), torch.from_numpy(rt).to(device))
    return cache[key]


def learned_decode_operand(spec: RotationSpec, layout: HeadLayout, device):
    """Row f3, fused decode operand (memoised per device and layout): the composed key
    transform T = diag(s) H_blk R (compose_transform, rotation.py:171-184) as f32 with a row
    stride of 129 floats (kvr_paged_decode_learned), and the output mode of the value branch
    (value_branch_spec, rotation.py:162-168): 0 none, 1 the Hadamard part only, 2 T itself."""
    cache = spec.__dict__.setdefault("_learned_dec", {})
    key = (str(torch.device(device)), layout.head_dim, layout.rot_order)
    if key not in cache:
        t = compose_transform(spec, layout)
        pad = np.zeros((t.shape[0], t.shape[1] + 1), dtype=np.float32)
        pad[:, :t.shape[1]] = t
        vb = value_branch_spec(spec)
        mode = 0 if vb is None else (2 if vb.learned is not None else 1)
        cache[key] = (torch.from_numpy(pad).to(device), mode)
    return cache[key]


def rotate_kv_learned(k: torch.Tensor, v: torch.Tensor, layout: HeadLayout, spec: RotationSpec):
    """Row f3 (learned R composed after the Hadamard), unfused on the device: the
    K rows through the full transform, the V rows through value_branch_spec
    (rotation.py:118-142, 162-168).  Returns f64 tensors shaped like k / v."""
    d = layout.head_dim
    kr = rows_matmul(k.reshape(-1, d), composed_on(spec, layout, k.device)).reshape(k.shape)
    tv = composed_on(spec, layout, v.device, values=True)
    vr = v.to(torch.float64) if tv is None else rows_matmul(v.reshape(-1, d), tv).reshape(v.shape)
    return kr.contiguous(), vr.contiguous()


def apply_block_rotation(x, layout: HeadLayout, spec: RotationSpec):
    """Rotate rows: x diag(signs) H_blk learned (rotation.py:118-142)."""
    return _rotate(x, layout, spec, inverse=False)


def apply_inverse_rotation(x, layout: HeadLayout, spec: RotationSpec):
    """Map rotated rows back: x learned^T H_blk diag(signs) (rotation.py:145-159)."""
    return _rotate(x, layout, spec, inverse=True)


def value_branch_spec(spec: RotationSpec) -> Optional[RotationSpec]:
    """Value-side transform: None for KEYS_ONLY; learned part only if learned_values (rotation.py:162-168)."""
    if spec.targets is Targets.KEYS_ONLY:
        return None
    if spec.learned is not None and not spec.learned_values:
        return replace(spec, learned=None)
    return spec


def compose_transform(spec: RotationSpec, layout: HeadLayout) -> np.ndarray:
    """Dense T = diag(signs) H_blk learned (rotation.py:171-184)."""
    _check_spec_layout(spec, layout)
    t = block_hadamard_matrix(layout.head_dim, spec.order)
    if spec.signs is not None:
        t = spec.signs[:, None] * t
    if spec.learned is not None:
        t = t @ spec.learned
    return t
