"""Decode attention over the paged INT4 cache (mirrors kvrot.attention, attention.py:24-115).

`decode_step` keeps the reference signature (one request, numpy in / numpy
out); `decode_batch` is the serving entry point (many sequences, CUDA tensors,
no host synchronisation).  Both run the split-K paged decode kernel, which
rotates the query into the stored-key frame in-kernel and inverse-rotates the
output when values were stored rotated.
"""

from __future__ import annotations

import ctypes
import os
import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _kernels, _lib
from .cache import INT4, PageTable
from .errors import EmptySequenceError, NonFiniteInputError, ShapeError
from .layout import HeadLayout
from .rotation import RotationSpec, Targets, composed_on, learned_decode_operand, rows_matmul

_Q_CODE = {torch.float32: _lib.KVR_F32, torch.bfloat16: _lib.KVR_BF16, torch.float16: _lib.KVR_F16}
_KV_CODE = {torch.float64: _lib.KVR_F64, **_Q_CODE}


def _all_finite(t: torch.Tensor) -> bool:
    """NaN/Inf check of a host tensor (native helper) or a CUDA tensor (synchronises)."""
    if t.is_cuda:
        return bool(torch.isfinite(t).all())
    t = t if t.is_contiguous() else t.contiguous()
    rc = _lib.lib().kvr_host_all_finite(ctypes.c_void_p(t.data_ptr()), _KV_CODE[t.dtype], t.numel())
    if rc < 0:
        raise ShapeError(f"unsupported dtype {t.dtype}")
    return rc == 1


def fused_step_supported(layout: HeadLayout, precision: str) -> bool:
    """Geometries with the one-launch append + decode kernel (kvr_decode_step);
    others run the store kernel, then the decode kernel."""
    P, G = layout.page_tokens, layout.group_size
    return (precision == INT4 and layout.head_dim == 128 and P % 16 == 0 and (P & (P - 1)) == 0
            and G in (1, 2, 4, 8))


@dataclass(frozen=True)
class DecodeRequest:
    q: np.ndarray  # (num_q_heads, head_dim)
    seq: int


def _check_query(q, layout: HeadLayout) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.float64)
    if q.shape != (layout.num_q_heads, layout.head_dim):
        raise ShapeError(f"expected ({layout.num_q_heads}, {layout.head_dim}) query, got {q.shape}")
    if not np.isfinite(q).all():
        raise NonFiniteInputError("query contains NaN or Inf")
    return q


class DecodePlan:
    """Device-resident decode arguments for a fixed batch of sequences
    (block table, lengths, split count, workspace) so repeated steps issue one
    kernel launch and no host<->device traffic."""

    _RING = 4  # pinned staging buffers in flight (step() inputs + metadata)

    def __init__(self, table: PageTable, seqs: Sequence[int], num_splits: int = 0, extra_tokens: int = 0):
        self.table = table
        self.seqs = list(seqs)
        if len(set(self.seqs)) != len(self.seqs):
            raise ShapeError("a DecodePlan's sequences must be distinct")
        lay = table.layout
        self.fused_ok = fused_step_supported(lay, table.precision)
        for s in self.seqs:
            if table.sequence_length(s) == 0 and extra_tokens == 0:
                raise EmptySequenceError(f"sequence {s} has no tokens")
        B, P = len(self.seqs), lay.page_tokens
        cur = max(table.sequence_length(s) for s in self.seqs)
        self.max_len = cur + extra_tokens
        # the block table reserves the pages of `extra_tokens` future steps, so
        # step() only patches new entries and never reallocates
        self.bt, lens, _ = table.block_table(self.seqs, width=-(-self.max_len // P))
        self._known_pages = [len(table._seq_pages[s]) for s in self.seqs]
        # pinned host mirror of the block table: pages gained by step() reach the
        # device with an async copy of just the new entry (no host synchronisation)
        self._bt_host = self.bt.cpu().pin_memory()
        # step metadata lives in one device block: slots int64[B] | lens int32[B];
        # step() refreshes it (plus the step's q/k/v when given on the host)
        # with a single pinned host->device copy
        self._meta_bytes = (12 * B + 255) // 256 * 256
        self._dev = torch.zeros(self._meta_bytes, dtype=torch.uint8, device=table.device)
        self.slots = self._dev[:8 * B].view(torch.int64)
        self.lens = self._dev[8 * B:12 * B].view(torch.int32)
        self.lens.copy_(lens)
        self._copy_stream = None
        self.side_copy = False  # True: staged inputs go over on a side stream (measured slower end to end)
        self.fast_copy_stream = os.environ.get("KVR_STEP_SIDE_COPY", "0") == "1"  # the native ring's copies (A/B)
        # the native ring launches the fused step itself on pinned inputs (no graph, no copy); A/B switch
        self.fast_direct = int(os.environ.get("KVR_STEP_DIRECT", "2"))  # 0 graph replay, 1 in place, 2 copy kernel
        self._lens_stale = False  # step() passes its own device copy of the lengths
        self._layouts = {}
        self._fast = None  # native step ring bound to the last graph step's host tensors
        if num_splits <= 0:
            num_splits = _lib.lib().kvr_decode_pick_splits(B, lay.num_kv_heads, self.max_len, P)
        self.splits = num_splits
        self.ws = table.workspace(B, lay.num_q_heads, num_splits)

    def _patch_pages(self, stream: Optional[int] = None) -> None:
        """Write block-table entries of pages the sequences gained since the last call
        (async copies of the new entries from the pinned mirror, on `stream`)."""
        P = self.table.layout.page_tokens
        W = self.bt.shape[1]
        if stream is None:
            stream = torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
        hb = self._bt_host.numpy()
        for i, s in enumerate(self.seqs):
            pages = self.table._seq_pages[s]
            k0 = self._known_pages[i]
            if len(pages) > k0:
                if len(pages) > W:
                    raise ShapeError(f"sequence {s} grew to {len(pages) * P} tokens, beyond the plan's "
                                     f"{W * P}-token block table; build a new DecodePlan "
                                     f"(or pass extra_tokens)")
                hb[i, k0:len(pages)] = pages[k0:]
                off = (i * W + k0) * 4
                _kernels.h2d_async(self.bt.data_ptr() + off, self._bt_host.data_ptr() + off, 4 * (len(pages) - k0),
                                   stream)
                self._known_pages[i] = len(pages)

    def refresh(self) -> None:
        """Re-read block table and lengths after appends (small host->device copies)."""
        self._patch_pages()
        lens = [self.table.sequence_length(s) for s in self.seqs]
        self.lens.copy_(torch.tensor(lens, dtype=torch.int32))
        self._lens_stale = False
        self.max_len = max(self.max_len, max(lens))

    def run(self, q: torch.Tensor, spec: Optional[RotationSpec], out: Optional[torch.Tensor] = None,
            lens: Optional[torch.Tensor] = None) -> torch.Tensor:
        table, lay = self.table, self.table.layout
        if lens is None:
            if self._lens_stale:
                self.refresh()
            lens = self.lens
        if q.dtype not in _Q_CODE:
            q = q.float()
        q = q.contiguous()
        if tuple(q.shape) != (len(self.seqs), lay.num_q_heads, lay.head_dim):
            raise ShapeError(f"expected ({len(self.seqs)}, {lay.num_q_heads}, {lay.head_dim}) queries, "
                             f"got {tuple(q.shape)}")
        if out is None:
            out = torch.empty(q.shape, dtype=torch.float32, device=table.device)
        if table.precision != INT4:
            spec = None  # BF16 pools hold raw vectors: the query is used as-is (attention.py:67-71)
        rotate = spec is not None
        if rotate:
            if spec.order != lay.rot_order:
                raise ShapeError(f"spec order {spec.order} != layout rot_order {lay.rot_order}")
            if spec.learned is not None:
                return self._run_learned(q, spec, out, lens)
        targets = _lib.KVR_KEYS_ONLY if (rotate and spec.targets is Targets.KEYS_ONLY) else _lib.KVR_KEYS_AND_VALUES
        _lib.check(_lib.lib().kvr_paged_decode(
            _kernels.ptr(q), _Q_CODE[q.dtype], ctypes.byref(table.desc), _kernels.ptr(self.bt), self.bt.shape[1],
            _kernels.ptr(lens), len(self.seqs), lay.num_q_heads, self.max_len, spec.order if rotate else 1,
            1 if rotate else 0, targets, spec.sign_words(lay.head_dim) if rotate else None, _kernels.ptr(out),
            _kernels.ptr(self.ws), self.ws.numel(), self.splits, _kernels.stream_ptr()))
        return out


    def _run_learned(self, q: torch.Tensor, spec: RotationSpec, out: torch.Tensor,
                     lens: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Row f3 (attention.py:63-85 on a learned spec): one kvr_paged_decode_learned launch -- the
        query through the composed T = diag(s) H_blk R in the kernel's prologue, the value branch's
        inverse before the store.  Geometries that kernel does not take: the query through T (one
        f64 row-matmul launch, f32 out), the INT4 decode on the pre-rotated query, then the value
        branch's T^T on the output (one launch)."""
        lay = self.table.layout
        dev = self.table.device
        if (self.table.precision == INT4 and lay.head_dim == 128 and os.environ.get("KVR_LEARNED_DECODE", "fused")
                == "fused"):
            # one launch: q T in the kernel's prologue, the value branch's inverse before the store
            t_pad, mode = learned_decode_operand(spec, lay, dev)
            if not q.is_contiguous():
                q = q.contiguous()
            rc = _lib.lib().kvr_paged_decode_learned(
                _kernels.ptr(q), _Q_CODE[q.dtype], ctypes.byref(self.table.desc), _kernels.ptr(self.bt),
                self.bt.shape[1], _kernels.ptr(lens), len(self.seqs), lay.num_q_heads, self.max_len,
                _kernels.ptr(t_pad), mode, spec.order, spec.sign_words(lay.head_dim), _kernels.ptr(out),
                _kernels.ptr(self.ws), self.ws.numel(), self.splits, _kernels.stream_ptr())
            if rc != _lib.KVR_ERR_UNSUPPORTED:
                _lib.check(rc)
                return out
        qr = getattr(self, "_lq", None)
        if qr is None or qr.shape != q.shape:
            qr = self._lq = torch.empty(q.shape, dtype=torch.float32, device=dev)
            self._lo = torch.empty(q.shape, dtype=torch.float32, device=dev)
        rows_matmul(q, composed_on(spec, lay, dev), out=qr)
        tv = composed_on(spec, lay, dev, transpose=True, values=True)
        # the caller's lengths go through (a serving step's staged ones: nothing host-side may run
        # inside a captured step graph)
        if tv is None:
            return self.run(qr, None, out, lens=lens)
        self.run(qr, None, self._lo, lens=lens)
        rows_matmul(self._lo, tv, out=out)
        return out

    def run_step(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor, slots: torch.Tensor,
                 spec: Optional[RotationSpec], out: Optional[torch.Tensor] = None,
                 lens: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Fused serving step (no host bookkeeping): write token b's K/V rows (B, H, d)
        into slot slots[b] (rotated + INT4-quantized bit-exactly in f64) and decode
        over the lengths (default: the plan's), which must already include it.  The
        buffers may be device memory or pinned host memory (read / written by the
        kernel in place)."""
        table, lay = self.table, self.table.layout
        if lens is None:
            if self._lens_stale:
                self.refresh()
            lens = self.lens
        if not q.is_contiguous():
            q = q.contiguous()
        if not (k_new.is_contiguous() and v_new.is_contiguous()):
            k_new, v_new = k_new.contiguous(), v_new.contiguous()
        if out is None:
            out = torch.empty(q.shape, dtype=torch.float32, device=table.device)
        if table.precision != INT4:
            spec = None
        rotate = spec is not None
        if (rotate and spec.learned is not None) or not self.fused_ok:
            # row f3 (learned R) and geometries without the one-launch kernel: the store kernel,
            # then the decode.  Hadamard / plain rows: exact f64 arithmetic, as the fused writer.
            # Learned rows: the fused learned K1 where it applies (bf16, d = 128) -- the same
            # one-step-at-a-boundary bar as the exact route, whose dense f64 product also sums in
            # its own order (rotation.py:140-141 leaves that order to the BLAS)
            dev = table.device
            learned = rotate and spec.learned is not None
            table.store_slots(k_new.to(dev), v_new.to(dev), slots.to(dev), spec, exact=not learned)
            res = self.run(q.to(dev), spec, out if out.is_cuda else None, lens=lens.to(dev))
            if res is not out:
                out.copy_(res, non_blocking=True)
            return out
        # the argument list is rebuilt only when a buffer, the spec or the stream changes
        stream = torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
        key = (q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), slots.data_ptr(), out.data_ptr(), q.dtype,
               k_new.dtype, id(spec), stream, self.bt.data_ptr(), lens.data_ptr(), self.ws.data_ptr())
        cached = getattr(self, "_step_args", None)
        if cached is None or cached[0] != key:
            targets = _lib.KVR_KEYS_ONLY if (rotate and spec.targets is Targets.KEYS_ONLY) else _lib.KVR_KEYS_AND_VALUES
            head = (_kernels.ptr(q), _Q_CODE[q.dtype], _kernels.ptr(k_new), _kernels.ptr(v_new), _KV_CODE[k_new.dtype],
                    _kernels.ptr(slots), ctypes.byref(table.desc), _kernels.ptr(self.bt), self.bt.shape[1],
                    _kernels.ptr(lens), len(self.seqs), lay.num_q_heads)
            tail = (spec.order if rotate else 1, 1 if rotate else 0, targets,
                    spec.sign_words(lay.head_dim) if rotate else None, _kernels.ptr(out), _kernels.ptr(self.ws),
                    self.ws.numel(), self.splits, _kernels.ptr(table.flags), ctypes.c_void_p(stream))
            cached = self._step_args = (key, head, tail)
        _lib.check(_lib.lib().kvr_decode_step(*cached[1], self.max_len, *cached[2]))
        return out


    def _step_layout(self, host_in) -> dict:
        """Staging layout for a given set of host inputs (cached per shapes/dtypes): a
        ring of pinned host buffers, each with its device twin (slot ids | lengths |
        the host inputs) and the views the kernel reads."""
        key = tuple((tuple(t.shape), t.dtype) for t in host_in)
        lay = self._layouts.get(key)
        if lay is not None:
            return lay
        B = len(self.seqs)
        sizes = [t.numel() * t.element_size() for t in host_in]
        offs, o = [], self._meta_bytes
        for n in sizes:
            offs.append(o)
            o += (n + 255) // 256 * 256
        ring = []
        for _ in range(self._RING):
            buf = torch.empty(o, dtype=torch.uint8).pin_memory()
            dbuf = torch.zeros(o, dtype=torch.uint8, device=self.table.device)
            views = {"slots": dbuf[:8 * B].view(torch.int64), "lens": dbuf[8 * B:12 * B].view(torch.int32),
                     "inputs": [dbuf[off:off + n].view(t.dtype).view(t.shape) for t, off, n in zip(host_in, offs, sizes)]}
            ring.append((buf, buf.numpy(), buf.data_ptr(), _kernels.host_event(), dbuf.data_ptr(), views,
                         _kernels.host_event()))
            views["dbuf"] = dbuf  # keeps the device twin alive
        lay = {"bytes": o, "offs": offs, "sizes": sizes, "ring": ring, "i": 0}
        self._layouts[key] = lay
        return lay

    def step(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor, spec: Optional[RotationSpec],
             out: Optional[torch.Tensor] = None, graph: bool = False, check: bool = True) -> torch.Tensor:
        """One serving decode step (see _step_general for the contract).  Repeated graph
        steps with the same host tensors take a native fast path: the slot ids and
        lengths are planned here (no new page: every page_tokens-th step takes the
        general path, which allocates it) and one kvr_step_ring_run call stages,
        checks and copies the inputs and replays the step's CUDA graph."""
        fr = self._fast
        if (graph and fr is not None and fr["q"] is q and fr["k"] is k_new and fr["v"] is v_new and fr["out"] is out
                and fr["spec"] is spec and fr["check"] == check):
            r = self._fast_step(fr)
            if r is not None:
                return r
        return self._step_general(q, k_new, v_new, spec, out, graph, check)

    def _fast_step(self, fr: dict) -> Optional[torch.Tensor]:
        if (fr["max_len"] != self.max_len or fr["q"].data_ptr() != fr["qp"] or fr["k"].data_ptr() != fr["kp"]
                or fr["v"].data_ptr() != fr["vp"]
                or torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()) != fr["stream"]):
            self._drop_fast()
            return None
        alloc = self.table.alloc
        P = alloc.page_tokens
        seq_len, seq_pages = alloc.seq_len, alloc.seq_pages
        slots, lens, known = fr["slots"], fr["lens"], self._known_pages
        for n, s in enumerate(self.seqs):
            t = seq_len[s]
            # a new page, the capacity error, pages the block table has not seen: the general path
            if t % P == 0 or t + 1 > self.max_len or len(seq_pages[s]) != known[n]:
                return None
            slots[n] = seq_pages[s][t // P] * P + t % P
            lens[n] = t + 1
        for n, s in enumerate(self.seqs):
            seq_len[s] = int(lens[n])
        sl = fr["layout"]
        i = sl["i"]
        sl["i"] = (i + 1) % self._RING
        rc = _lib.lib().kvr_step_ring_run(fr["handle"], i, fr["meta_ptr"])
        if rc:
            for n, s in enumerate(self.seqs):
                seq_len[s] = int(lens[n]) - 1  # nothing of a rejected step stays behind
            _lib.check(rc)
        self._lens_stale = True
        return fr["out"]

    def _drop_fast(self) -> None:
        if self._fast is not None:
            _lib.lib().kvr_step_ring_destroy(self._fast["handle"])
            self._fast = None

    def __del__(self):
        try:
            self._drop_fast()
        except Exception:
            pass

    def _arm_fast(self, q, k_new, v_new, spec, out, check, lay, stream) -> None:
        """After a general graph step: when every staging slot has its graph, bind a native
        step ring to these host tensors (kvr_step_ring_create)."""
        B = len(self.seqs)
        if not (q.is_contiguous() and k_new.is_contiguous() and v_new.is_contiguous()):
            return
        execs = []
        for i, ring in enumerate(lay["ring"]):
            dq, dk, dv = ring[5]["inputs"]
            g = lay.get("graphs", {}).get((i, out.data_ptr(), id(spec), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                                           self.max_len, self.splits))
            if g is None or g[1] is None:
                return
            execs.append(g[1])
        self._drop_fast()
        meta = np.zeros(12 * B, dtype=np.uint8)
        h = _lib.lib().kvr_step_ring_create(
            self._RING, q.data_ptr(), lay["offs"][0], q.numel() * q.element_size(), _KV_CODE[q.dtype],
            k_new.data_ptr(), lay["offs"][1], v_new.data_ptr(), lay["offs"][2], k_new.numel() * k_new.element_size(),
            _KV_CODE[k_new.dtype], 12 * B, lay["bytes"], 1 if check else 0, stream)
        if not h:
            return
        for i, ring in enumerate(lay["ring"]):
            _lib.check(_lib.lib().kvr_step_ring_set_slot(h, i, ring[2], ring[4], execs[i], ring[3].cuda_event))
        if self.fast_direct and lay["bytes"] <= 65536 and fused_step_supported(self.table.layout, self.table.precision) and not (
                spec is not None and spec.learned is not None):
            # direct mode: the kernel reads q / k / v / slot ids / lengths from the pinned slot
            rotate = spec is not None and self.table.precision == INT4
            lay_ = self.table.layout
            targets = _lib.KVR_KEYS_ONLY if (rotate and spec.targets is Targets.KEYS_ONLY) else _lib.KVR_KEYS_AND_VALUES
            _lib.check(_lib.lib().kvr_step_ring_set_decode(
                h, _Q_CODE[q.dtype], _KV_CODE[k_new.dtype], ctypes.byref(self.table.desc), self.bt.data_ptr(),
                self.bt.shape[1], B, lay_.num_q_heads, self.max_len, spec.order if rotate else 1, 1 if rotate else 0,
                targets, spec.sign_words(lay_.head_dim) if rotate else None, out.data_ptr(), self.ws.data_ptr(),
                self.ws.numel(), self.splits, self.table.flags.data_ptr(), self.fast_direct))
        elif self.fast_copy_stream:  # stage-in copies on a side stream (they may overlap the previous step)
            if self._copy_stream is None:
                self._copy_stream = torch.cuda.Stream(device=self.table.device)
            _lib.check(_lib.lib().kvr_step_ring_set_copy_stream(h, self._copy_stream.cuda_stream))
        self._fast = {"q": q, "k": k_new, "v": v_new, "out": out, "spec": spec, "check": check,
                      "qp": q.data_ptr(), "kp": k_new.data_ptr(), "vp": v_new.data_ptr(), "stream": stream,
                      "max_len": self.max_len, "layout": lay, "handle": h, "meta": meta,
                      "meta_ptr": meta.ctypes.data, "slots": meta[:8 * B].view(np.int64),
                      "lens": meta[8 * B:].view(np.int32)}

    def _step_general(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor, spec: Optional[RotationSpec],
                      out: Optional[torch.Tensor] = None, graph: bool = False, check: bool = True) -> torch.Tensor:
        """One serving decode step for every sequence of the plan: allocate the new
        token's slot (reference page order), then one fused append + decode launch.
        q (B, nq, d) and k_new/v_new (B, H, d) may be host tensors: they are staged
        with the step metadata (slot ids, lengths) in a ring of pinned buffers, each
        going to its device twin in one copy ahead of the kernel (every CTA of a head
        re-reads q, so reading the staged bytes over the bus in place was measured
        slower (tools/e2e_probe.py); `side_copy` moves the copy to a side stream).  `out` may be
        a pinned host tensor: the kernel then writes the result there directly
        (valid once the step has completed, e.g. after torch.cuda.synchronize()).

        graph=True launches the kernel from a CUDA graph captured on first use per
        ring slot; the block table keeps its address and the plan's max_len (its
        capacity) is fixed, so only the host bookkeeping runs per step.

        Every check runs before any allocator state is committed, so a failing
        step leaves the sequences as they were (the reference validates before it
        mutates, cache.py:225-233): shapes, the block-table and graph capacity, and
        with check=True (default) NaN/Inf in q / k_new / v_new (host tensors by a
        native scan; CUDA tensors by a synchronising device reduction -- pass
        check=False to skip it: a non-finite token is then neither written nor
        attended, and table.check_flags() reports it)."""
        table = self.table
        lay = table.layout
        B = len(self.seqs)
        stream = torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
        kv_shape = (B, lay.num_kv_heads, lay.head_dim)
        if q.shape != (B, lay.num_q_heads, lay.head_dim) or k_new.shape != kv_shape or v_new.shape != kv_shape:
            raise ShapeError(f"expected q ({B}, {lay.num_q_heads}, {lay.head_dim}) and k/v ({B}, {lay.num_kv_heads}, "
                             f"{lay.head_dim}), got {tuple(q.shape)}, {tuple(k_new.shape)}, {tuple(v_new.shape)}")
        if k_new.dtype != v_new.dtype:
            raise ShapeError(f"k_new and v_new dtypes differ ({k_new.dtype}, {v_new.dtype})")
        if out is not None and not out.is_cuda and not out.is_pinned():
            raise ShapeError("out must be a CUDA tensor or a pinned host tensor")
        host = [not t.is_cuda for t in (q, k_new, v_new)]
        if check and not all(_all_finite(t) for t, h in zip((q, k_new, v_new), host) if not h):
            raise NonFiniteInputError("q / k_new / v_new contain NaN or Inf")
        cur = [table.sequence_length(s) for s in self.seqs]
        mx = max(cur) + 1
        W = self.bt.shape[1] * lay.page_tokens
        if mx > W:
            raise ShapeError(f"a sequence would grow to {mx} tokens, beyond the plan's {W}-token block table; "
                             f"build a new DecodePlan (extra_tokens)")
        if mx > self.max_len and graph:
            raise ShapeError(f"sequence length {mx} passed the plan's capacity {self.max_len}; "
                             f"build a new DecodePlan (extra_tokens)")
        # stage the host inputs into the next pinned ring slot (once its last reader has run)
        # and scan them for NaN/Inf -- one native call, before any allocator state changes
        host_in = [t if t.is_contiguous() else t.contiguous() for t, h in zip((q, k_new, v_new), host) if h]
        lkey = tuple((t.shape, t.dtype) for t in host_in)
        sl = self._layouts.get(lkey) or self._step_layout(host_in)
        slot_i = sl["i"]
        ring = sl["ring"][slot_i]
        sl["i"] = (slot_i + 1) % self._RING
        ptrs, offs = [None, None, None], [0, 0, 0]
        j = 0
        for r in range(3):
            if host[r]:
                ptrs[r], offs[r] = host_in[j].data_ptr(), sl["offs"][j]
                j += 1
        rc = _lib.lib().kvr_step_stage(ring[3].cuda_event, ring[2], ptrs[0], offs[0],
                                       q.numel() * q.element_size(), _KV_CODE.get(q.dtype, -1), ptrs[1], offs[1],
                                       ptrs[2], offs[2], k_new.numel() * k_new.element_size(),
                                       _KV_CODE.get(k_new.dtype, -1), 1 if check else 0)
        if rc == 0:
            raise NonFiniteInputError("q / k_new / v_new contain NaN or Inf")
        _lib.check(rc if rc < 0 else 0)
        slots, fresh = table.alloc.plan(self.seqs)  # commit (pages on the free heap are zero)
        known = list(self._known_pages)
        try:
            res = self._step_committed(q, k_new, v_new, spec, out, graph, slots, fresh, cur, mx, stream, sl, slot_i)
        except BaseException:
            table.alloc.unplan(self.seqs, fresh)  # nothing of a failed step stays behind
            self._known_pages = known
            raise
        if graph and out is not None and all(host) and not self.side_copy and (
                self._fast is None or self._fast["q"] is not q or self._fast["out"] is not out):
            self._arm_fast(q, k_new, v_new, spec, out, check, sl, stream)
        return res

    def _step_committed(self, q, k_new, v_new, spec, out, graph, slots, fresh, cur, mx, stream, lay, slot_i):
        table = self.table
        B = len(self.seqs)
        if fresh:
            self._patch_pages(stream)
        if mx > self.max_len:
            self.max_len = mx
        buf, buf_np, buf_ptr, ev, dptr, dviews, cev = lay["ring"][slot_i]
        buf_np[:8 * B] = slots.view(np.uint8)
        lens = buf_np[8 * B:12 * B].view(np.int32)
        for i, c in enumerate(cur):
            lens[i] = c + 1
        self._lens_stale = True  # the plan's own device lengths are refreshed on demand
        staged = iter(dviews["inputs"])
        q, k_new, v_new = (t if t.is_cuda else next(staged) for t in (q, k_new, v_new))
        if out is None:
            out = torch.empty(q.shape, dtype=torch.float32, device=table.device)
        side = self.side_copy
        if graph and not side:
            gkey = (slot_i, out.data_ptr(), id(spec), q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(),
                    self.max_len, self.splits)
            g = lay.setdefault("graphs", {}).get(gkey)
            if g is not None and g[1] is not None:  # the common path: copy + graph + event in one native call
                _lib.check(_lib.lib().kvr_step_launch(dptr, buf_ptr, lay["bytes"], g[1], ev.cuda_event, stream))
                return out
        if side:  # the staged bytes go over on the side stream; the compute stream waits for them
            if self._copy_stream is None:
                self._copy_stream = torch.cuda.Stream(device=table.device)
            cs = self._copy_stream.cuda_stream
            _kernels.h2d_async(dptr, buf_ptr, lay["bytes"], cs)
            _kernels.event_record(cev, cs)
            _kernels.stream_wait(stream, cev)
        else:  # the staged bytes go over on the compute stream, ahead of the kernel
            _kernels.h2d_async(dptr, buf_ptr, lay["bytes"], stream)

        def device_part():
            self.run_step(q, k_new, v_new, dviews["slots"], spec, out, lens=dviews["lens"])

        if not graph:
            device_part()
        else:
            graphs = lay.setdefault("graphs", {})
            gkey = (slot_i, out.data_ptr(), id(spec), q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(),
                    self.max_len, self.splits)
            if side:
                gkey = gkey + ("side",)
            g = graphs.get(gkey)
            if g is not None:
                if g[1] is not None:
                    _kernels.graph_launch(g[1], stream)
                else:
                    g[0].replay()
            else:
                device_part()  # eager first run (also warms the launch path)
                g = torch.cuda.CUDAGraph()
                cap = torch.cuda.Stream()
                cap.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(cap), torch.cuda.graph(g, stream=cap):
                    device_part()
                torch.cuda.current_stream().wait_stream(cap)
                ex = g.raw_cuda_graph_exec()
                graphs[gkey] = (g, ex if isinstance(ex, int) and ex else None)
        _kernels.event_record(ev, stream)
        return out


def decode_batch(q: torch.Tensor, table: PageTable, seqs: Sequence[int], spec: Optional[RotationSpec] = None,
                 num_splits: int = 0) -> torch.Tensor:
    """Serving decode: q (B, num_q_heads, d) CUDA tensor -> f32 (B, num_q_heads, d)."""
    plan = DecodePlan(table, seqs, num_splits)
    return plan.run(q.to(table.device), spec)


def decode_step(req: DecodeRequest, table: PageTable, spec: Optional[RotationSpec] = None) -> np.ndarray:
    """One query token over one cached sequence; returns (num_q_heads, d) f64 (attention.py:50-87)."""
    layout = table.layout
    q = _check_query(req.q, layout)
    if table.sequence_length(req.seq) == 0:
        raise EmptySequenceError(f"sequence {req.seq} has no tokens")
    qt = torch.from_numpy(q).to(table.device, dtype=torch.float32).reshape(1, *q.shape)
    out = DecodePlan(table, [req.seq]).run(qt, spec)
    return out[0].double().cpu().numpy()


def decode_step_fp(q, flat_k, flat_v, layout: HeadLayout) -> np.ndarray:
    """Full-precision decode over flat (t, kv_heads, d) arrays (attention.py:90-115): the
    f64 flat-decode kernel (kvr_decode_flat_f64)."""
    q = _check_query(q, layout)
    k = np.asarray(flat_k, dtype=np.float64)
    v = np.asarray(flat_v, dtype=np.float64)
    if k.ndim != 3 or k.shape[1:] != (layout.num_kv_heads, layout.head_dim):
        raise ShapeError(f"expected (t, kv_heads, dim) keys, got {k.shape}")
    if k.shape != v.shape:
        raise ShapeError(f"key/value shape mismatch: {k.shape} vs {v.shape}")
    if k.shape[0] == 0:
        raise EmptySequenceError("no cached tokens")
    if layout.head_dim > 256:
        raise ShapeError(f"head_dim {layout.head_dim} > 256")
    dev = _kernels.device()
    qt = torch.from_numpy(q).to(dev)
    kt = torch.from_numpy(np.ascontiguousarray(k)).to(dev)
    vt = torch.from_numpy(np.ascontiguousarray(v)).to(dev)
    out = torch.empty_like(qt)
    _lib.check(_lib.lib().kvr_decode_flat_f64(_kernels.ptr(qt), _kernels.ptr(kt), _kernels.ptr(vt), k.shape[0],
                                              layout.num_q_heads, layout.num_kv_heads, layout.head_dim,
                                              _kernels.ptr(out), _kernels.stream_ptr()))
    return out.cpu().numpy()
