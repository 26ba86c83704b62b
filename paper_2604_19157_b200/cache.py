"""Paged INT4 KV cache in B200 HBM (mirrors kvrot.cache.PageTable, cache.py:122-450).

Device layout: one uint8 tensor [num_pages, page_bytes]; a page holds, per kv
head, P / 16 "cells" of 16 tokens with everything a decode tile needs contiguous
(k_scale | v_scale | K codes | V codes | k_zp | v_zp, include/kvrot_b200.h), so a
(page, head) tile is one bulk copy.  `dump` / `load` convert cells to and from
the reference `.kvpg` page records (cache.py:387-397) byte for byte.

Host side: the same lowest-id-first page heap and per-sequence page lists as
the reference (cache.py:150-151, 211-223), so page ids -- and therefore dump
bytes -- match it token for token.  All data movement and arithmetic (rotate,
quantize, store, dequantize) happens in the native library.
"""

from __future__ import annotations

import ctypes
import heapq
import json
import struct
from typing import Optional, Sequence

import numpy as np
import torch

from . import _kernels, _lib
from .errors import CapacityExceededError, ConfigError, NonFiniteInputError, SequenceNotFoundError, ShapeError
from .layout import HeadLayout
from .rotation import RotationSpec, Targets

BF16 = "bf16"
INT4 = "int4"

_DUMP_MAGIC = b"KVPG"
_DUMP_VERSION = 1

_TORCH_DTYPE_CODE = {torch.float64: _lib.KVR_F64, torch.float32: _lib.KVR_F32, torch.bfloat16: _lib.KVR_BF16,
                     torch.float16: _lib.KVR_F16}


def float_to_bf16_bits(x) -> np.ndarray:
    """RNE f32 -> bf16 storage bits (cache.py:43-47)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def bf16_bits_to_float(bits) -> np.ndarray:
    """bf16 storage bits -> f64 (cache.py:50-53)."""
    return (np.asarray(bits).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def token_bytes(layout: HeadLayout, precision: str, include_sidecar: bool = False) -> int:
    """Bytes of one token's K+V (cache.py:56-68)."""
    h, d = layout.num_kv_heads, layout.head_dim
    if precision == BF16:
        return 4 * h * d
    if precision == INT4:
        return h * d + (10 * h if include_sidecar else 0)
    raise ConfigError(f"unknown precision {precision!r}")


def capacity_tokens(budget_bytes: int, layout: HeadLayout, precision: str) -> int:
    """Token capacity at BF16-token granularity; INT4 holds exactly 4x (cache.py:71-86)."""
    if budget_bytes < 0:
        raise ConfigError(f"budget_bytes={budget_bytes} must be >= 0")
    base = budget_bytes // token_bytes(layout, BF16)
    if precision == BF16:
        return base
    if precision == INT4:
        return 4 * base
    raise ConfigError(f"unknown precision {precision!r}")


def cell_tokens(layout: HeadLayout) -> int:
    """Tokens per cell (include/kvrot_b200.h): 16 when page_tokens % 16 == 0, else page_tokens."""
    return 16 if layout.page_tokens % 16 == 0 else layout.page_tokens


def cell_bytes(layout: HeadLayout, precision: str = INT4) -> int:
    if precision == BF16:  # k_bits u16[T][d] | v_bits u16[T][d]
        return 4 * cell_tokens(layout) * layout.head_dim
    return (cell_tokens(layout) * (layout.head_dim + 10) + 15) & ~15


def page_bytes(layout: HeadLayout, precision: str = INT4) -> int:
    """Size of one device page blob: H x (P / T) cells."""
    return layout.num_kv_heads * (layout.page_tokens // cell_tokens(layout)) * cell_bytes(layout, precision)


def record_bytes(layout: HeadLayout, precision: str = INT4) -> int:
    """Size of one reference `.kvpg` page record (cache.py:387-397)."""
    if precision == BF16:  # k_payload u16[P][H][d] | v_payload
        return 4 * layout.page_tokens * layout.num_kv_heads * layout.head_dim
    return layout.page_tokens * layout.num_kv_heads * (layout.head_dim + 10)


def _bf16_cells_to_records(blobs: np.ndarray, layout: HeadLayout) -> np.ndarray:
    P, H, d = layout.page_tokens, layout.num_kv_heads, layout.head_dim
    T = cell_tokens(layout)
    n = blobs.shape[0]
    c = np.ascontiguousarray(blobs, dtype=np.uint8).reshape(n, H, P // T, 2, T, 2 * d)  # [.., side, t, row bytes]
    kv = np.ascontiguousarray(c.transpose(3, 0, 2, 4, 1, 5)).reshape(2, n, P * H * 2 * d)  # (side, n, P, H, row)
    return np.concatenate([kv[0], kv[1]], axis=1)


def _bf16_records_to_cells(records: np.ndarray, layout: HeadLayout) -> np.ndarray:
    P, H, d = layout.page_tokens, layout.num_kv_heads, layout.head_dim
    T = cell_tokens(layout)
    n = records.shape[0]
    r = np.ascontiguousarray(records, dtype=np.uint8).reshape(n, 2, P, H, 2 * d)
    r = np.moveaxis(r, 3, 2)  # (n, 2, H, P, 2d)
    r = r.reshape(n, 2, H, P // T, T, 2 * d)
    r = np.ascontiguousarray(np.moveaxis(r, 1, 3))  # (n, H, P/T, 2, T, 2d)
    return r.reshape(n, -1)


def cells_to_records(blobs: np.ndarray, layout: HeadLayout, precision: str = INT4) -> np.ndarray:
    """Device page blobs [n, page_bytes] -> reference page records [n, record_bytes]
    (INT4: k_payload [P][H][d/2] | v_payload | k_scale f32[P][H] | k_zp [P][H] | v_scale | v_zp;
    BF16: k_payload u16[P][H][d] | v_payload)."""
    if precision == BF16:
        return _bf16_cells_to_records(blobs, layout)
    P, H, d = layout.page_tokens, layout.num_kv_heads, layout.head_dim
    T, cb = cell_tokens(layout), cell_bytes(layout)
    n = blobs.shape[0]
    cells = np.ascontiguousarray(blobs, dtype=np.uint8).reshape(n, H, P // T, cb)
    o = 0

    def take(nbytes, dt, shape):
        nonlocal o
        a = cells[..., o:o + nbytes].copy().view(dt).reshape((n, H, P // T) + shape)
        o += nbytes
        return a

    ks = take(4 * T, np.float32, (T,))
    vs = take(4 * T, np.float32, (T,))
    kc = take(T * d // 2, np.uint8, (T, d // 2))
    vc = take(T * d // 2, np.uint8, (T, d // 2))
    kz = take(T, np.uint8, (T,))
    vz = take(T, np.uint8, (T,))

    def tok_major(a):  # (n, H, P/T, T, ...) -> (n, P, H, ...)
        a = a.reshape((n, H, P) + a.shape[4:])
        return np.ascontiguousarray(np.moveaxis(a, 1, 2))

    parts = [tok_major(kc), tok_major(vc), tok_major(ks), tok_major(kz), tok_major(vs), tok_major(vz)]
    return np.concatenate([p.reshape(n, -1).view(np.uint8) for p in parts], axis=1)


def records_to_cells(records: np.ndarray, layout: HeadLayout, precision: str = INT4) -> np.ndarray:
    """Inverse of cells_to_records (used by PageTable.load)."""
    if precision == BF16:
        return _bf16_records_to_cells(records, layout)
    P, H, d = layout.page_tokens, layout.num_kv_heads, layout.head_dim
    T, cb = cell_tokens(layout), cell_bytes(layout)
    n = records.shape[0]
    r = np.ascontiguousarray(records, dtype=np.uint8).reshape(n, -1)
    o = 0

    def take(nbytes, dt, shape):
        nonlocal o
        a = r[:, o:o + nbytes].copy().view(dt).reshape((n,) + shape)
        o += nbytes
        return a

    kc = take(P * H * d // 2, np.uint8, (P, H, d // 2))
    vc = take(P * H * d // 2, np.uint8, (P, H, d // 2))
    ks = take(4 * P * H, np.float32, (P, H))
    kz = take(P * H, np.uint8, (P, H))
    vs = take(4 * P * H, np.float32, (P, H))
    vz = take(P * H, np.uint8, (P, H))

    def cell_major(a):  # (n, P, H, ...) -> (n, H, P/T, T*...) bytes
        a = np.ascontiguousarray(np.moveaxis(a, 2, 1))  # (n, H, P, ...)
        return a.reshape(n, H, P // T, -1).view(np.uint8)

    out = np.zeros((n, H, P // T, cb), dtype=np.uint8)
    o2 = 0
    for a in (cell_major(ks), cell_major(vs), cell_major(kc), cell_major(vc), cell_major(kz), cell_major(vz)):
        out[..., o2:o2 + a.shape[-1]] = a
        o2 += a.shape[-1]
    return out.reshape(n, -1)


class PageAllocator:
    """Host-side page bookkeeping of a pool: lowest-id-first free heap and
    per-sequence page lists (cache.py:150-151, 157-186, 211-223).  Pure Python,
    no device state, so the allocation order is testable without a GPU."""

    def __init__(self, num_pages: int, page_tokens: int) -> None:
        self.num_pages = num_pages
        self.page_tokens = page_tokens
        self.free = list(range(num_pages))
        heapq.heapify(self.free)
        self.seq_pages: dict[int, list[int]] = {}
        self.seq_len: dict[int, int] = {}

    def require(self, seq: int) -> None:
        if seq not in self.seq_pages:
            raise SequenceNotFoundError(f"unknown sequence {seq}")

    def create(self, seq: int) -> None:
        if seq in self.seq_pages:
            raise ConfigError(f"sequence {seq} already exists")
        self.seq_pages[seq] = []
        self.seq_len[seq] = 0

    def reserve(self, seq: int, n: int) -> np.ndarray:
        """Bulk form of plan([seq] * n): slot ids of the next n tokens of `seq`,
        taking new pages lowest id first (O(pages), for prefill-sized appends)."""
        self.require(seq)
        P = self.page_tokens
        t0 = self.seq_len[seq]
        owned = self.seq_pages[seq]
        need = max(0, -(-(t0 + n) // P) - len(owned))
        if need > len(self.free):
            raise CapacityExceededError(f"page pool exhausted ({self.num_pages} pages)")
        owned.extend(heapq.heappop(self.free) for _ in range(need))
        pos = np.arange(t0, t0 + n, dtype=np.int64)
        slots = np.asarray(owned, dtype=np.int64)[pos // P] * P + pos % P
        self.seq_len[seq] = t0 + n
        return slots

    def release(self, seq: int) -> list[int]:
        """Drop `seq`; its pages go back to the free heap.  Returns them."""
        self.require(seq)
        pages = self.seq_pages.pop(seq)
        self.seq_len.pop(seq)
        for pid in pages:
            heapq.heappush(self.free, pid)
        return pages

    def unplan(self, seqs: Sequence[int], fresh: Sequence[int]) -> None:
        """Undo a plan(seqs) that returned `fresh` (or a reserve): lengths back,
        the fresh pages back on the free heap.  Used when a step fails after its
        slots were planned, so a rejected token never stays in a sequence."""
        counts: dict[int, int] = {}
        for seq in seqs:
            counts[seq] = counts.get(seq, 0) + 1
        taken = set(fresh)
        for seq, n in counts.items():
            self.seq_len[seq] -= n
            owned = self.seq_pages[seq]
            while owned and owned[-1] in taken:
                owned.pop()
        for pid in fresh:
            heapq.heappush(self.free, pid)

    def plan(self, seqs: Sequence[int]) -> tuple[np.ndarray, list[int]]:
        """Slot ids (page * P + slot) for appending one token per entry of `seqs`
        (in order), taking new pages lowest id first.  All-or-nothing: on
        exhaustion nothing is committed.  Returns (slots, freshly taken pages)."""
        P = self.page_tokens
        # pass 1: validate and count the pages needed (no state touched), so a
        # step costs O(len(seqs) log free) and never copies the free heap
        lens: dict[int, int] = {}
        need = 0
        for seq in seqs:
            self.require(seq)
            t = lens.get(seq, self.seq_len[seq])
            if t % P == 0 and t // P >= len(self.seq_pages[seq]):
                need += 1
            lens[seq] = t + 1
        if need > len(self.free):
            raise CapacityExceededError(f"page pool exhausted ({self.num_pages} pages)")
        # pass 2: commit
        slots = np.empty(len(seqs), dtype=np.int64)
        fresh = []
        for n, seq in enumerate(seqs):
            t = self.seq_len[seq]
            owned = self.seq_pages[seq]
            idx = t // P
            if idx >= len(owned):
                pid = heapq.heappop(self.free)
                owned.append(pid)
                fresh.append(pid)
            slots[n] = owned[idx] * P + t % P
            self.seq_len[seq] = t + 1
        return slots, fresh


class PageTable:
    """GPU page pool + per-sequence page lists (drop-in for kvrot.cache.PageTable)."""

    def __init__(self, layout: HeadLayout, precision: str = INT4, budget_bytes: Optional[int] = None,
                 num_pages: Optional[int] = None, device=None) -> None:
        if precision not in (INT4, BF16):
            raise ConfigError(f"unknown precision {precision!r}")
        if (budget_bytes is None) == (num_pages is None):
            raise ConfigError("specify exactly one of budget_bytes or num_pages")
        self.layout = layout
        self.precision = precision
        self.budget_bytes = budget_bytes
        if num_pages is None:
            num_pages = capacity_tokens(budget_bytes, layout, precision) // layout.page_tokens
        if num_pages < 0:
            raise ConfigError(f"num_pages={num_pages} must be >= 0")
        self.num_pages = num_pages
        self.device = torch.device(device) if device is not None else _kernels.device()
        self.page_bytes = page_bytes(layout, precision)
        self.pool = torch.zeros((max(num_pages, 1), self.page_bytes), dtype=torch.uint8, device=self.device)
        self.desc = _lib.KvrPool()
        init = _lib.lib().kvr_pool_init_bf16 if precision == BF16 else _lib.lib().kvr_pool_init
        _lib.check(init(ctypes.byref(self.desc), ctypes.c_void_p(self.pool.data_ptr()), num_pages,
                        layout.page_tokens, layout.num_kv_heads, layout.head_dim))
        assert self.desc.page_bytes == self.page_bytes
        self.flags = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.alloc = PageAllocator(num_pages, layout.page_tokens)
        self._ws = None
        self._ws_cnt = 0

    # reference-compatible views of the allocator state (cache.py:149-153)
    @property
    def _seq_pages(self) -> dict:
        return self.alloc.seq_pages

    @property
    def _seq_len(self) -> dict:
        return self.alloc.seq_len

    @property
    def _free(self) -> list:
        return self.alloc.free

    # -- sequence management (cache.py:157-186) --------------------------------
    def create_sequence(self, seq: int) -> None:
        self.alloc.create(seq)

    def has_sequence(self, seq: int) -> bool:
        return seq in self.alloc.seq_pages

    def sequence_length(self, seq: int) -> int:
        self._require(seq)
        return self.alloc.seq_len[seq]

    def sequence_ids(self) -> list[int]:
        return sorted(self.alloc.seq_pages)

    def sequence_pages(self, seq: int) -> list[int]:
        self._require(seq)
        return list(self.alloc.seq_pages[seq])

    def free_sequence(self, seq: int) -> int:
        pages = self.alloc.release(seq)
        # pages on the free heap hold zeros (the reference hands out freshly zeroed
        # pages, cache.py:103-119): zeroing at release keeps allocation -- every
        # 16th serving step -- free of device work
        self._zero_pages(pages)
        return len(pages)

    def _require(self, seq: int) -> None:
        self.alloc.require(seq)

    # -- capacity (cache.py:190-207) ----------------------------------------------
    def capacity_tokens(self, precision: Optional[str] = None) -> int:
        if self.budget_bytes is None:
            return self.num_pages * self.layout.page_tokens
        return capacity_tokens(self.budget_bytes, self.layout, precision or self.precision)

    @property
    def used_tokens(self) -> int:
        return sum(self._seq_len.values())

    @property
    def free_pages(self) -> int:
        return len(self._free)

    @property
    def allocated_pages(self) -> int:
        return self.num_pages - len(self._free)

    # -- slot allocation --------------------------------------------------------
    def _plan_slots(self, seqs: Sequence[int]) -> tuple[np.ndarray, list[int]]:
        return self.alloc.plan(seqs)

    def _zero_pages(self, pids) -> None:
        """Zero device pages (pool bytes written outside the library's store kernels:
        the next decode on this stream is told, see kvr_note_pool_write)."""
        if len(pids):
            idx = torch.tensor(list(pids), dtype=torch.long).to(self.device, non_blocking=True)
            self.pool.index_fill_(0, idx, 0)
            _lib.lib().kvr_note_pool_write(_kernels.stream_ptr())

    # -- writes -----------------------------------------------------------------
    def _store(self, k: torch.Tensor, v: torch.Tensor, slots: np.ndarray, spec: Optional[RotationSpec],
               exact: bool) -> None:
        if self.precision == BF16:
            spec = None  # BF16 pools store the raw vectors and ignore the spec (cache.py:243-246)
        n = k.shape[0]
        slot_t = torch.from_numpy(slots).to(self.device, non_blocking=True)
        rotate = spec is not None
        if rotate:
            if spec.order != self.layout.rot_order:
                raise ShapeError(f"spec order {spec.order} != layout rot_order {self.layout.rot_order}")
            if spec.learned is not None:  # row f3: learned R after H
                if not exact and self._store_learned(k, v, slot_t, spec):
                    return
                from .rotation import rotate_kv_learned  # unfused: f64 transform on the device, exact store

                k, v = rotate_kv_learned(k, v, self.layout, spec)
                spec, rotate, exact = None, False, True
        targets = _lib.KVR_KEYS_ONLY if (rotate and spec.targets is Targets.KEYS_ONLY) else _lib.KVR_KEYS_AND_VALUES
        words = spec.sign_words(self.layout.head_dim) if rotate else None
        _lib.check(_lib.lib().kvr_rotate_quantize_store(
            _kernels.ptr(k), _kernels.ptr(v), _TORCH_DTYPE_CODE[k.dtype], n, _kernels.ptr(slot_t),
            ctypes.byref(self.desc), spec.order if rotate else 1, 1 if rotate else 0, targets, words,
            1 if exact else 0, _kernels.ptr(self.flags), _kernels.stream_ptr()))

    def _store_learned(self, k: torch.Tensor, v: torch.Tensor, slot_t: torch.Tensor, spec: RotationSpec) -> bool:
        """Row f3 fused: the tcgen05 K1 with T = diag(s) H_blk R in shared memory (bf16 rows,
        head_dim 128).  False when the kernel does not cover the configuration (the caller
        takes the unfused path)."""
        if k.dtype != torch.bfloat16 or self.layout.head_dim != 128 or cell_tokens(self.layout) != 16:
            return False
        from .rotation import learned_store_operands

        img, rt = learned_store_operands(spec, self.layout, self.device)
        targets = _lib.KVR_KEYS_ONLY if spec.targets is Targets.KEYS_ONLY else _lib.KVR_KEYS_AND_VALUES
        rc = _lib.lib().kvr_rotate_quantize_store_learned(
            _kernels.ptr(k), _kernels.ptr(v), _TORCH_DTYPE_CODE[k.dtype], k.shape[0], _kernels.ptr(slot_t),
            ctypes.byref(self.desc), spec.order, targets, 1 if spec.learned_values else 0,
            spec.sign_words(self.layout.head_dim), _kernels.ptr(img), _kernels.ptr(rt), _kernels.ptr(self.flags),
            _kernels.stream_ptr())
        if rc == _lib.KVR_ERR_UNSUPPORTED:
            return False
        _lib.check(rc)
        return True

    def _check_kv_host(self, k, v, ndim: int):
        h, d = self.layout.num_kv_heads, self.layout.head_dim
        k = np.ascontiguousarray(k, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        shape = (h, d) if ndim == 2 else (None, h, d)
        if k.ndim != ndim or v.shape != k.shape or k.shape[-2:] != (h, d):
            raise ShapeError(f"expected {shape} k and v, got {k.shape}, {v.shape}")
        if not (np.isfinite(k).all() and np.isfinite(v).all()):
            raise NonFiniteInputError("k/v contain NaN or Inf")
        return k, v

    def append_token(self, seq: int, k, v, spec: Optional[RotationSpec] = None) -> int:
        """Fused rotate-quantize-write of one token; returns its index (cache.py:235-270).
        f64 inputs take the bit-exact f64 kernel path."""
        self._require(seq)
        k, v = self._check_kv_host(k, v, 2)
        first = self._seq_len[seq]
        slots, fresh = self._plan_slots([seq])
        kt = torch.from_numpy(k).to(self.device).reshape(1, *k.shape)
        vt = torch.from_numpy(v).to(self.device).reshape(1, *v.shape)
        self._store(kt, vt, slots, spec, exact=True)
        return first

    def append_tokens_two_pass(self, seq: int, ks, vs, spec: Optional[RotationSpec] = None) -> int:
        """Unfused route (cache.py:272-317): materialise the rotated stacks for all
        tokens, then quantize + write them.  Must equal the fused path bitwise."""
        self._require(seq)
        ks, vs = self._check_kv_host(ks, vs, 3)
        first = self._seq_len[seq]
        t = ks.shape[0]
        if t == 0:
            return first
        slots, fresh = self._plan_slots([seq] * t)
        h, d = self.layout.num_kv_heads, self.layout.head_dim
        kt = torch.from_numpy(ks).to(self.device)
        vt = torch.from_numpy(vs).to(self.device)
        if spec is not None and self.precision == INT4:
            from .rotation import apply_block_rotation, value_branch_spec

            kt = apply_block_rotation(kt.reshape(t * h, d), self.layout, spec).reshape(t, h, d)
            vspec = value_branch_spec(spec)
            if vspec is not None:
                vt = apply_block_rotation(vt.reshape(t * h, d), self.layout, vspec).reshape(t, h, d)
        self._store(kt.contiguous(), vt.contiguous(), slots, None, exact=True)
        return first

    def append_batch(self, seqs: Sequence[int], k, v, spec: Optional[RotationSpec] = None,
                     exact: Optional[bool] = None, check: bool = True) -> np.ndarray:
        """Serving write: token n of (k, v) [n, H, d] is appended to sequence seqs[n].
        bf16/fp16 CUDA tensors take the fast K1 kernel; f64 takes the exact one.
        Returns the slot ids.

        check=True (default) validates before anything is committed, like the
        reference (cache.py:225-233): a NaN/Inf anywhere raises NonFiniteInputError
        and no token is appended (the batch is atomic).  check=False skips that
        (no host synchronisation): rows with NaN/Inf are then not written, the
        device flag is set (check_flags) and the other rows are committed."""
        kt = k if isinstance(k, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(k))
        vt = v if isinstance(v, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(v))
        kt = kt.to(self.device, non_blocking=True).contiguous()
        vt = vt.to(self.device, non_blocking=True).contiguous()
        h, d = self.layout.num_kv_heads, self.layout.head_dim
        if kt.shape != vt.shape or kt.ndim != 3 or tuple(kt.shape[1:]) != (h, d) or kt.shape[0] != len(seqs):
            raise ShapeError(f"expected ({len(seqs)}, {h}, {d}) k and v, got {tuple(kt.shape)}, {tuple(vt.shape)}")
        if kt.dtype not in _TORCH_DTYPE_CODE or vt.dtype != kt.dtype:
            raise ShapeError(f"unsupported k/v dtype {kt.dtype}/{vt.dtype}")
        if exact is None:
            exact = kt.dtype == torch.float64
        if check and not bool(torch.isfinite(kt).all() & torch.isfinite(vt).all()):
            raise NonFiniteInputError("k/v contain NaN or Inf")
        slots, fresh = self._plan_slots(list(seqs))
        self._store(kt, vt, slots, spec, exact=exact)
        return slots

    def store_slots(self, k: torch.Tensor, v: torch.Tensor, slots: torch.Tensor, spec: Optional[RotationSpec] = None,
                    exact: bool = False) -> None:
        """Engine-level write (no host bookkeeping, no sync): token n of the CUDA
        tensors k, v [n, H, d] goes to the precomputed slot id slots[n]
        (page * P + slot, int64, negative = skip), like a serving engine's
        slot_mapping.  The caller owns the slot assignment."""
        if slots.dtype != torch.int64 or not slots.is_cuda:
            raise ShapeError("slots must be an int64 CUDA tensor")
        if self.precision == BF16:
            spec = None
        if spec is not None and spec.learned is not None:  # row f3 (see _store)
            if not exact and self._store_learned(k, v, slots, spec):
                return
            from .rotation import rotate_kv_learned

            k, v = rotate_kv_learned(k, v, self.layout, spec)
            spec, exact = None, True
        rotate = spec is not None
        targets = _lib.KVR_KEYS_ONLY if (rotate and spec.targets is Targets.KEYS_ONLY) else _lib.KVR_KEYS_AND_VALUES
        _lib.check(_lib.lib().kvr_rotate_quantize_store(
            _kernels.ptr(k), _kernels.ptr(v), _TORCH_DTYPE_CODE[k.dtype], k.shape[0], _kernels.ptr(slots),
            ctypes.byref(self.desc), spec.order if rotate else 1, 1 if rotate else 0, targets,
            spec.sign_words(self.layout.head_dim) if rotate else None, 1 if exact else 0, _kernels.ptr(self.flags),
            _kernels.stream_ptr()))

    def check_flags(self) -> None:
        """Raise if a launch since the last check flagged a problem (synchronises):
        NonFiniteInputError for NaN/Inf K/V rows (those tokens were not written),
        ShapeError for a decode length past the launch's max_seq_len."""
        f = int(self.flags.item())
        if f:
            self.flags.zero_()
        if f & _lib.KVR_FLAG_NONFINITE:
            raise NonFiniteInputError("k/v contained NaN or Inf (rows were not written)")
        if f & _lib.KVR_FLAG_LEN_OVERFLOW:
            raise ShapeError("a decode sequence length exceeded the launch's max_seq_len (tokens past it ignored)")

    # -- reads (cache.py:319-362) -------------------------------------------------
    def block_table(self, seqs: Sequence[int], width: int = 0) -> tuple[torch.Tensor, torch.Tensor, int]:
        """Device (int32 [B, max_pages] page ids, int32 [B] lengths, max length).
        `width` reserves room for pages a decode plan will append later."""
        rows = [self._seq_pages[s] for s in seqs]
        width = max(1, width, max((len(r) for r in rows), default=1))
        bt = np.zeros((len(seqs), width), dtype=np.int32)
        for i, r in enumerate(rows):
            bt[i, :len(r)] = r
        lens = np.array([self._seq_len[s] for s in seqs], dtype=np.int32)
        return (torch.from_numpy(bt).to(self.device), torch.from_numpy(lens).to(self.device),
                int(lens.max()) if len(lens) else 0)

    def read_sequence_device(self, seqs: Sequence[int], dtype: torch.dtype = torch.float64):
        """Flatten-dequant of several sequences -> (k, v) [B, max_len, H, d] on the device."""
        for s in seqs:
            self._require(s)
        bt, lens, max_len = self.block_table(seqs)
        h, d = self.layout.num_kv_heads, self.layout.head_dim
        k = torch.zeros((len(seqs), max_len, h, d), dtype=dtype, device=self.device)
        v = torch.zeros_like(k)
        code = {torch.float64: _lib.KVR_F64, torch.float32: _lib.KVR_F32, torch.bfloat16: _lib.KVR_BF16}[dtype]
        _lib.check(_lib.lib().kvr_dequantize_pages(ctypes.byref(self.desc), _kernels.ptr(bt), bt.shape[1],
                                                   _kernels.ptr(lens), len(seqs), max_len, _kernels.ptr(k),
                                                   _kernels.ptr(v), code, _kernels.stream_ptr()))
        return k, v

    def read_sequence(self, seq: int) -> tuple[np.ndarray, np.ndarray]:
        """Dequantized stored-space (t, H, d) f64 stacks (cache.py:337-362)."""
        k, v = self.read_sequence_device([seq], torch.float64)
        return k[0].cpu().numpy(), v[0].cpu().numpy()

    def read_token(self, seq: int, t: int) -> tuple[np.ndarray, np.ndarray]:
        self._require(seq)
        if not 0 <= t < self._seq_len[seq]:
            raise IndexError(f"token {t} out of range for sequence of {self._seq_len[seq]}")
        k, v = self.read_sequence(seq)
        return k[t], v[t]

    # -- serialization (cache.py:366-450) ------------------------------------------
    def _header(self) -> bytes:
        lay = self.layout
        header = {
            "version": _DUMP_VERSION,
            "precision": self.precision,
            "budget_bytes": self.budget_bytes,
            "num_pages": self.num_pages,
            "layout": {"num_q_heads": lay.num_q_heads, "num_kv_heads": lay.num_kv_heads, "head_dim": lay.head_dim,
                       "rot_order": lay.rot_order, "page_tokens": lay.page_tokens},
            "sequences": {str(s): {"pages": self._seq_pages[s], "length": self._seq_len[s]}
                          for s in sorted(self._seq_pages)},
        }
        return json.dumps(header, sort_keys=True, separators=(",", ":")).encode()

    def page_records(self, pids) -> np.ndarray:
        """Reference `.kvpg` page records [len(pids), record_bytes] of device pages."""
        if len(pids) == 0:
            return np.zeros((0, record_bytes(self.layout, self.precision)), dtype=np.uint8)
        idx = torch.tensor(list(pids), dtype=torch.long, device=self.device)
        return cells_to_records(self.pool.index_select(0, idx).cpu().numpy(), self.layout, self.precision)

    def dump_bytes(self) -> bytes:
        blob = self._header()
        pids = sorted(p for ps in self._seq_pages.values() for p in ps)
        pages = self.page_records(pids).tobytes() if pids else b""
        return _DUMP_MAGIC + struct.pack("<II", _DUMP_VERSION, len(blob)) + blob + pages

    def dump(self, path) -> None:
        with open(path, "wb") as f:
            f.write(self.dump_bytes())

    @classmethod
    def load(cls, path, device=None) -> "PageTable":
        with open(path, "rb") as f:
            raw = f.read()
        if raw[:4] != _DUMP_MAGIC:
            raise ConfigError(f"{path} is not a page dump")
        version, hlen = struct.unpack("<II", raw[4:12])
        if version != _DUMP_VERSION:
            raise ConfigError(f"unsupported dump version {version}")
        header = json.loads(raw[12:12 + hlen].decode())
        lay = header["layout"]
        layout = HeadLayout(num_q_heads=lay["num_q_heads"], num_kv_heads=lay["num_kv_heads"],
                            head_dim=lay["head_dim"], rot_order=lay["rot_order"], page_tokens=lay["page_tokens"])
        table = cls(layout, precision=header["precision"], num_pages=header["num_pages"], device=device)
        table.budget_bytes = header["budget_bytes"]
        allocated = sorted(p for s in header["sequences"].values() for p in s["pages"])
        body = np.frombuffer(raw, dtype=np.uint8, offset=12 + hlen)
        rb = record_bytes(layout, header["precision"])
        if body.size != len(allocated) * rb:
            raise ConfigError(f"{path}: page payload size mismatch")
        if allocated:
            cells = records_to_cells(body.reshape(len(allocated), rb), layout, header["precision"])
            blobs = torch.from_numpy(cells).to(table.device)
            table.pool.index_copy_(0, torch.tensor(allocated, dtype=torch.long, device=table.device), blobs)
            _lib.lib().kvr_note_pool_write(_kernels.stream_ptr())
        taken = set(allocated)
        table.alloc.free = [p for p in range(table.num_pages) if p not in taken]
        heapq.heapify(table.alloc.free)
        for seq_str, entry in sorted(header["sequences"].items(), key=lambda kv: int(kv[0])):
            table.alloc.seq_pages[int(seq_str)] = list(entry["pages"])
            table.alloc.seq_len[int(seq_str)] = entry["length"]
        return table

    # -- decode workspace --------------------------------------------------------------
    def workspace(self, batch: int, num_q_heads: int, splits: int) -> torch.Tensor:
        need = _lib.lib().kvr_decode_workspace_bytes(batch, self.layout.num_kv_heads, num_q_heads,
                                                     self.layout.head_dim, max(splits, 1))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
            self._ws_cnt = 0
        # the split counters sit at the start of the workspace and are left at
        # zero by every launch; bytes first used as counters are zeroed once here
        cnt = (batch * self.layout.num_kv_heads * 4 * 9 + 255) // 256 * 256  # counters + merge epochs
        if cnt > self._ws_cnt:
            self._ws[:cnt].zero_()
            self._ws_cnt = cnt
        return self._ws
