"""CPU oracle for the Hadamard-INT4 KV hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference `kvrot` package
(/root/reference/pkg/src/kvrot, the arithmetic spec of arXiv 2604.19157's
desk-scale reproduction).  It exists so that tests, `__graft_entry__.smoke()`
and the `cpu_baseline` / `--impl reference` legs of `bench.py` can check and
time the CUDA product path.  Nothing in `paper_2604_19157_b200/` imports it;
the product fails loudly when its CUDA library is missing.

Parity of this restatement is PINNED against golden vectors produced by the
real reference in the build container (tests/golden/make_golden.py ->
tests/golden/golden_v1.npz, *.kvpg) -- see tests/test_oracle_golden.py.

Every function cites the reference file:line whose floating-point operation
order it reproduces.  Operation order matters: the product's f64 paths are
required to be bit-identical to these functions.
"""

from __future__ import annotations

import heapq
import json
import math
import struct
from typing import Optional

import numpy as np

# ---------------------------------------------------------------- constants --

CONST_SENTINEL = 0xFF            # int4.py:33
KVPG_MAGIC = b"KVPG"             # cache.py:39
KVPG_VERSION = 1                 # cache.py:40
KEYS_ONLY = "keys_only"          # rotation.py:35
KEYS_AND_VALUES = "keys_and_values"  # rotation.py:36


# ------------------------------------------------------------ L0 kernels ----

def round_half_away(t):
    """copysign(floor(|t| + 0.5), t) in f64 -- _ref.py:16-19 / _core.pyx:18-19.

    Note the f64 corner: |t| = 0.5 - 2**-54 rounds |t| + 0.5 up to 1.0.
    """
    return np.copysign(np.floor(np.abs(t) + 0.5), t)


def fwht_rows(x: np.ndarray, order: int) -> None:
    """In-place orthonormal block Walsh-Hadamard transform (_ref.py:22-40).

    Stage schedule half = 1, 2, ..., order/2; every stage maps the pair
    (j, j+half) inside each block to (a+b, a-b); afterwards every element is
    multiplied by fl(1/fl(sqrt(order))) (_core.pyx:30, 46-47).
    """
    n, d = x.shape
    if order == 1:
        return
    nb = d // order
    half = 1
    while half < order:
        view = x.reshape(n, nb, order // (2 * half), 2, half)
        top = np.array(view[:, :, :, 0, :])
        bot = np.array(view[:, :, :, 1, :])
        np.add(top, bot, out=view[:, :, :, 0, :])
        np.subtract(top, bot, out=view[:, :, :, 1, :])
        half <<= 1
    x *= 1.0 / math.sqrt(order)


def pack_rows(nibbles: np.ndarray) -> np.ndarray:
    """u8 (n, d) -> u8 (n, d/2); element 2i in the low nibble (_ref.py:43-45)."""
    lo = nibbles[:, 0::2].astype(np.uint8)
    hi = nibbles[:, 1::2].astype(np.uint8)
    return (lo | (hi << np.uint8(4))).astype(np.uint8)


def unpack_rows(packed: np.ndarray, logical_len: int) -> np.ndarray:
    """Inverse of pack_rows (_ref.py:48-54)."""
    out = np.empty((packed.shape[0], logical_len), dtype=np.uint8)
    out[:, 0::2] = packed & np.uint8(0x0F)
    out[:, 1::2] = packed >> np.uint8(4)
    return out


def quantize_rows(x: np.ndarray):
    """Token-wise asymmetric INT4 with nibble packing (_ref.py:57-80).

    scale32 = f32((max - min) / 15); s64 = f64(scale32);
    z = clip(round_half_away(-min / s64), 0, 15);
    q = clip(round_half_away(x / s64) + z, 0, 15).
    Rows whose f32 scale is zero store zp = 0xFF and the row offset f32(min)
    in the scale slot, with all-zero nibbles (_ref.py:68-79).
    """
    x = np.ascontiguousarray(x, dtype=np.float64)
    lo = x.min(axis=1)
    hi = x.max(axis=1)
    scale = ((hi - lo) / 15.0).astype(np.float32)
    flat = scale == np.float32(0.0)
    step = scale.astype(np.float64)
    step[flat] = 1.0
    zero = np.clip(round_half_away(-lo / step), 0.0, 15.0)
    codes = np.clip(round_half_away(x / step[:, None]) + zero[:, None], 0.0, 15.0)
    codes = codes.astype(np.uint8)
    zp = zero.astype(np.uint8)
    if flat.any():
        codes[flat] = 0
        zp[flat] = CONST_SENTINEL
        scale[flat] = lo[flat].astype(np.float32)
    return pack_rows(codes), scale, zp


def dequantize_rows(packed, scale, zp, logical_len: int) -> np.ndarray:
    """x_hat = f64(scale) * (q - z); sentinel rows give the offset (_ref.py:83-95)."""
    q = unpack_rows(np.ascontiguousarray(packed, dtype=np.uint8), logical_len).astype(np.float64)
    zp = np.asarray(zp, dtype=np.uint8)
    flat = zp == CONST_SENTINEL
    step = np.asarray(scale, dtype=np.float32).astype(np.float64)
    zf = zp.astype(np.float64)
    zf[flat] = 0.0
    out = step[:, None] * (q - zf[:, None])
    if flat.any():
        out[flat] = step[flat, None]
    return out


# --------------------------------------------------------- L1 / L2 method ----

def use_reference_kernels(mod) -> None:
    """Route this module's L0 kernels through the reference's own compiled ones
    (oracle/_ref, built by oracle/build_ref.py from _core.pyx, bit-identical to
    _ref.py per _core.pyx:1-8); used by the CPU-baseline legs of bench.py."""
    g = globals()
    for name in ("fwht_rows", "pack_rows", "unpack_rows", "quantize_rows", "dequantize_rows"):
        g[name] = getattr(mod, name)


def make_hadamard(order: int) -> np.ndarray:
    """Orthonormal Sylvester matrix (hadamard.py:33-52): kron-doubling then * 1/sqrt(order)."""
    h = np.ones((1, 1))
    while h.shape[0] < order:
        h = np.kron(h, np.array([[1.0, 1.0], [1.0, -1.0]]))
    return h * (1.0 / math.sqrt(order))


def block_hadamard_matrix(dim: int, order: int) -> np.ndarray:
    """diag(H, ..., H) -- hadamard.py:55-67."""
    out = np.zeros((dim, dim))
    h = make_hadamard(order)
    for b in range(0, dim, order):
        out[b:b + order, b:b + order] = h
    return out


def make_signs(seed: int, layer: int, head_dim: int, order: int) -> np.ndarray:
    """+-1 vector; one Philox stream per (seed, layer, block) -- rotation.py:81-101.

    Key word layout: (0x5164 << 48) | (layer << 24) | block.
    """
    out = np.empty(head_dim)
    for blk in range(head_dim // order):
        word = (0x5164 << 48) | (layer << 24) | blk
        key = np.array([seed & (2**64 - 1), word], dtype=np.uint64)
        bits = np.random.Generator(np.random.Philox(key=key)).integers(0, 2, size=order)
        out[blk * order:(blk + 1) * order] = 2.0 * bits - 1.0
    return out


def signs_to_bits(signs: Optional[np.ndarray], head_dim: int) -> np.ndarray:
    """Bit i set <=> signs[i] == -1 (the GPU encoding of a sign vector)."""
    bits = np.zeros(head_dim, dtype=np.uint8)
    if signs is not None:
        bits = (np.asarray(signs) < 0).astype(np.uint8)
    return bits


def rotate_rows(x: np.ndarray, order: int, signs: Optional[np.ndarray]) -> np.ndarray:
    """x @ diag(signs) @ H_blk (rotation.py:118-142 without the learned factor)."""
    out = np.array(x, dtype=np.float64, order="C", copy=True)
    if signs is not None:
        out *= signs
    fwht_rows(out, order)
    return out


def unrotate_rows(x: np.ndarray, order: int, signs: Optional[np.ndarray]) -> np.ndarray:
    """x @ H_blk @ diag(signs) (rotation.py:145-159 without the learned factor)."""
    out = np.array(x, dtype=np.float64, order="C", copy=True)
    fwht_rows(out, order)
    if signs is not None:
        out *= signs
    return out


def compose_transform(order: int, signs: Optional[np.ndarray], dim: int) -> np.ndarray:
    """Dense T = diag(signs) @ H_blk (rotation.py:171-184)."""
    t = block_hadamard_matrix(dim, order)
    if signs is not None:
        t = signs[:, None] * t
    return t


# ------------------------------------------------------------ L3 storage ----

def bf16_bits(x) -> np.ndarray:
    """RNE f32 -> bf16 bits (cache.py:43-47)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return ((u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)).astype(np.uint16)


def bf16_to_f64(bits) -> np.ndarray:
    """bf16 bits -> f64 (cache.py:50-53)."""
    return (np.asarray(bits).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def token_bytes(num_kv_heads: int, head_dim: int, sidecar: bool = False) -> int:
    """INT4 K+V bytes per token (cache.py:56-68)."""
    return 2 * num_kv_heads * (head_dim // 2) + (2 * num_kv_heads * 5 if sidecar else 0)


class OraclePages:
    """Host-only paged INT4 pool mirroring kvrot.cache.PageTable (cache.py:122-450).

    Pages: k_payload u8[P,H,d/2], v_payload, k_scale f32[P,H], k_zp u8[P,H],
    v_scale, v_zp (cache.py:103-114).  Pages are handed out lowest id first
    from a min-heap (cache.py:150-151, 211-223).
    """

    def __init__(self, num_q_heads, num_kv_heads, head_dim, rot_order, page_tokens, num_pages):
        self.q_heads, self.h, self.d = num_q_heads, num_kv_heads, head_dim
        self.order, self.p, self.num_pages = rot_order, page_tokens, num_pages
        self.pages = {}
        self.free = list(range(num_pages))
        heapq.heapify(self.free)
        self.seq_pages = {}
        self.seq_len = {}

    def _blank(self):
        p, h, d = self.p, self.h, self.d
        return {
            "k_payload": np.zeros((p, h, d // 2), np.uint8),
            "v_payload": np.zeros((p, h, d // 2), np.uint8),
            "k_scale": np.zeros((p, h), np.float32),
            "k_zp": np.zeros((p, h), np.uint8),
            "v_scale": np.zeros((p, h), np.float32),
            "v_zp": np.zeros((p, h), np.uint8),
        }

    def create_sequence(self, seq):
        self.seq_pages[seq] = []
        self.seq_len[seq] = 0

    def _slot(self, seq):
        t = self.seq_len[seq]
        if t % self.p == 0:
            if not self.free:
                raise RuntimeError("oracle pool exhausted")
            pid = heapq.heappop(self.free)
            self.pages[pid] = self._blank()
            self.seq_pages[seq].append(pid)
        return self.pages[self.seq_pages[seq][-1]], t % self.p

    def _store_side(self, k_store, v_store):
        return quantize_rows(k_store), quantize_rows(v_store)

    def append_token(self, seq, k, v, signs=None, targets=KEYS_AND_VALUES, rotate=True):
        """Fused append (cache.py:235-270, _rotate_token :453-462)."""
        k = np.asarray(k, np.float64)
        v = np.asarray(v, np.float64)
        page, slot = self._slot(seq)
        ks = rotate_rows(k, self.order, signs) if rotate else k
        vs = rotate_rows(v, self.order, signs) if (rotate and targets == KEYS_AND_VALUES) else v
        (kp, kscale, kz), (vp, vscale, vz) = self._store_side(ks, vs)
        page["k_payload"][slot], page["k_scale"][slot], page["k_zp"][slot] = kp, kscale, kz
        page["v_payload"][slot], page["v_scale"][slot], page["v_zp"][slot] = vp, vscale, vz
        self.seq_len[seq] += 1

    def append_tokens(self, seq, ks, vs, signs=None, targets=KEYS_AND_VALUES, rotate=True):
        for i in range(ks.shape[0]):
            self.append_token(seq, ks[i], vs[i], signs, targets, rotate)

    def read_sequence(self, seq):
        """Flatten-dequant of a sequence (cache.py:337-362)."""
        n = self.seq_len[seq]
        ko = np.empty((n, self.h, self.d))
        vo = np.empty((n, self.h, self.d))
        for i, pid in enumerate(self.seq_pages[seq]):
            pg = self.pages[pid]
            a, b = i * self.p, min(n, (i + 1) * self.p)
            u = b - a
            for side, dst in (("k", ko), ("v", vo)):
                rows = pg[f"{side}_payload"][:u].reshape(u * self.h, self.d // 2)
                dst[a:b] = dequantize_rows(rows, pg[f"{side}_scale"][:u].reshape(-1),
                                           pg[f"{side}_zp"][:u].reshape(-1), self.d).reshape(u, self.h, self.d)
        return ko, vo

    def dump_bytes(self, budget_bytes=None) -> bytes:
        """`.kvpg` image (cache.py:366-399): magic, <II (version, hlen), canonical JSON, page blobs."""
        header = {
            "budget_bytes": budget_bytes,
            "layout": {"head_dim": self.d, "num_kv_heads": self.h, "num_q_heads": self.q_heads,
                       "page_tokens": self.p, "rot_order": self.order},
            "num_pages": self.num_pages,
            "precision": "int4",
            "sequences": {str(s): {"length": self.seq_len[s], "pages": self.seq_pages[s]}
                          for s in sorted(self.seq_pages)},
            "version": KVPG_VERSION,
        }
        blob = json.dumps(header, sort_keys=True, separators=(",", ":")).encode()
        out = [KVPG_MAGIC, struct.pack("<II", KVPG_VERSION, len(blob)), blob]
        for pid in sorted(p for ps in self.seq_pages.values() for p in ps):
            pg = self.pages[pid]
            for name in ("k_payload", "v_payload", "k_scale", "k_zp", "v_scale", "v_zp"):
                out.append(pg[name].tobytes())
        return b"".join(out)


# --------------------------------------------------------- L3 attention -----

def softmax_rows(logits: np.ndarray) -> np.ndarray:
    """Max-subtracted softmax (attention.py:32-36)."""
    e = np.exp(logits - logits.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def decode_flat(q, k_hat, v_hat, group: int) -> np.ndarray:
    """Per q head: softmax(K q / sqrt(d)) V (attention.py:76-80 / 90-115)."""
    q = np.asarray(q, np.float64)
    d = q.shape[1]
    scale = 1.0 / math.sqrt(d)
    out = np.empty_like(q)
    for qh in range(q.shape[0]):
        kv = qh // group
        w = softmax_rows((k_hat[:, kv, :] @ q[qh] * scale)[None, :])[0]
        out[qh] = w @ v_hat[:, kv, :]
    return out


def decode_step(pages: OraclePages, seq, q, signs=None, targets=KEYS_AND_VALUES, rotate=True):
    """Rotated-frame decode (attention.py:50-87): rotate q, attend over the
    dequantized (stored-space) sequence, un-rotate the output when V was rotated."""
    k_hat, v_hat = pages.read_sequence(seq)
    group = pages.q_heads // pages.h
    q = np.asarray(q, np.float64)
    qf = rotate_rows(q, pages.order, signs) if rotate else q
    out = decode_flat(qf, k_hat, v_hat, group)
    if rotate and targets == KEYS_AND_VALUES:
        out = out @ compose_transform(pages.order, signs, pages.d).T
    return out
