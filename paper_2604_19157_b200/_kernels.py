"""Operator layer: the five kvrot._kernels entry points on the B200.

Drop-in for `kvrot._kernels` (pkg/src/kvrot/_kernels/__init__.py:35-39).  Each
function accepts numpy arrays (results come back as numpy, device round trip
included) or CUDA torch tensors (zero-copy, results stay on the device).  The
arithmetic is IEEE f64 in the reference's operation order, so results are
bit-identical to kvrot's numpy and Cython backends.  There is exactly one
backend; it is native CUDA (no CPU fallback).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import BackendUnavailableError, ShapeError

BACKEND = "cuda-sm100a"


def get_backend() -> str:
    return BACKEND


def available_backends() -> dict:
    import sys

    return {BACKEND: sys.modules[__name__]}


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise BackendUnavailableError("no CUDA device: this package has no CPU fallback")
    _lib.lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> ctypes.c_void_p:
    # the raw current stream of the current device (torch.cuda.current_stream() costs ~15 us)
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))


_CUDART = None


def _cudart():
    """The CUDA runtime torch already loaded (cudaEventRecord / Synchronize through
    ctypes cost ~0.3 us against ~5 / ~2.5 us for torch.cuda.Event's methods)."""
    global _CUDART
    if _CUDART is None:
        lib = ctypes.CDLL("libcudart.so.12")
        lib.cudaEventRecord.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        lib.cudaEventSynchronize.argtypes = [ctypes.c_void_p]
        lib.cudaGraphLaunch.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        lib.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                        ctypes.c_void_p]
        lib.cudaStreamWaitEvent.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint]
        _CUDART = lib
    return _CUDART


def host_event() -> torch.cuda.Event:
    """A timing-free event whose handle exists (torch creates it on first record)."""
    ev = torch.cuda.Event()
    ev.record()
    return ev


def event_record(ev: torch.cuda.Event, stream: int) -> None:
    if _cudart().cudaEventRecord(ev.cuda_event, stream):
        raise BackendUnavailableError("cudaEventRecord failed")


def event_sync(ev: torch.cuda.Event) -> None:
    if _cudart().cudaEventSynchronize(ev.cuda_event):
        raise BackendUnavailableError("cudaEventSynchronize failed")


def h2d_async(dst: int, src: int, nbytes: int, stream: int) -> None:
    if _cudart().cudaMemcpyAsync(dst, src, nbytes, 1, stream):  # cudaMemcpyHostToDevice
        raise BackendUnavailableError("cudaMemcpyAsync failed")



def stream_wait(stream: int, ev: torch.cuda.Event) -> None:
    if _cudart().cudaStreamWaitEvent(stream, ev.cuda_event, 0):
        raise BackendUnavailableError("cudaStreamWaitEvent failed")


def graph_launch(exec_handle: int, stream: int) -> None:
    """cudaGraphLaunch of an instantiated torch CUDA graph (raw_cuda_graph_exec()),
    ~1 us of host time against ~2.5 us for CUDAGraph.replay()."""
    if _cudart().cudaGraphLaunch(exec_handle, stream):
        raise BackendUnavailableError("cudaGraphLaunch failed")


def ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def to_device(a, dtype: torch.dtype) -> torch.Tensor:
    dev = device()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    arr = np.ascontiguousarray(a, dtype=torch.empty((), dtype=dtype).numpy().dtype)
    if not arr.flags.writeable:  # read-only inputs (e.g. frozen arrays): torch wants writable memory
        arr = arr.copy()
    return torch.from_numpy(arr).to(dev)


def _is_numpy(a) -> bool:
    return not isinstance(a, torch.Tensor)


def fwht_rows(x, order: int) -> None:
    """In place orthonormal block Walsh-Hadamard transform of f64 rows (_ref.py:22-40)."""
    if x.ndim != 2:
        raise ShapeError(f"expected 2-D rows, got ndim={x.ndim}")
    n, d = x.shape
    if isinstance(x, torch.Tensor):
        if x.dtype != torch.float64 or not x.is_cuda or not x.is_contiguous():
            raise ShapeError("fwht_rows needs a contiguous float64 CUDA tensor")
        _lib.check(_lib.lib().kvr_fwht_rows_f64(ptr(x), n, d, order, stream_ptr()))
        return
    t = to_device(x, torch.float64)
    _lib.check(_lib.lib().kvr_fwht_rows_f64(ptr(t), n, d, order, stream_ptr()))
    x[...] = t.cpu().numpy()


def pack_rows(nibbles):
    """u8 (n, d) -> u8 (n, d/2), element 2i in the low nibble (_ref.py:43-45)."""
    t = to_device(nibbles, torch.uint8)
    n, d = t.shape
    out = torch.empty((n, d // 2), dtype=torch.uint8, device=t.device)
    _lib.check(_lib.lib().kvr_pack_rows(ptr(t), ptr(out), n, d, stream_ptr()))
    return out.cpu().numpy() if _is_numpy(nibbles) else out


def unpack_rows(packed, logical_len: int):
    """Inverse of pack_rows (_ref.py:48-54)."""
    t = to_device(packed, torch.uint8)
    n = t.shape[0]
    out = torch.empty((n, logical_len), dtype=torch.uint8, device=t.device)
    _lib.check(_lib.lib().kvr_unpack_rows(ptr(t), ptr(out), n, logical_len, stream_ptr()))
    return out.cpu().numpy() if _is_numpy(packed) else out


def quantize_rows(x):
    """Token-wise asymmetric INT4 + nibble packing of f64 rows (_ref.py:57-80).

    Returns (packed u8 (n, d/2), scale f32 (n,), zp u8 (n,)); zp 0xFF marks a
    constant row whose scale slot holds the row offset.
    """
    t = to_device(x, torch.float64)
    if t.ndim != 2:
        raise ShapeError(f"expected (n, even d) rows, got {tuple(t.shape)}")
    n, d = t.shape
    packed = torch.empty((n, d // 2), dtype=torch.uint8, device=t.device)
    scale = torch.empty((n,), dtype=torch.float32, device=t.device)
    zp = torch.empty((n,), dtype=torch.uint8, device=t.device)
    _lib.check(_lib.lib().kvr_quantize_rows_f64(ptr(t), n, d, ptr(packed), ptr(scale), ptr(zp), stream_ptr()))
    if _is_numpy(x):
        return packed.cpu().numpy(), scale.cpu().numpy(), zp.cpu().numpy()
    return packed, scale, zp


def dequantize_rows(packed, scale, zp, logical_len: int):
    """f64 rows s * (q - z); sentinel rows return the offset (_ref.py:83-95)."""
    p = to_device(packed, torch.uint8)
    s = to_device(scale, torch.float32)
    z = to_device(zp, torch.uint8)
    n = p.shape[0]
    out = torch.empty((n, logical_len), dtype=torch.float64, device=p.device)
    _lib.check(_lib.lib().kvr_dequantize_rows_f64(ptr(p), ptr(s), ptr(z), n, logical_len, ptr(out), stream_ptr()))
    return out.cpu().numpy() if _is_numpy(packed) else out
