"""Shared helpers for the test-suite (imported as a top-level module)."""
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def golden_bytes(name: str) -> bytes:
    with open(os.path.join(GOLDEN_DIR, name), "rb") as f:
        return f.read()


def bf16_round(a) -> np.ndarray:
    """Round to the nearest bf16 (RNE through f32), returned as f64."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    r = ((u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)) << np.uint32(16)
    return r.astype(np.uint32).view(np.float32).astype(np.float64).reshape(np.shape(a))


def page_fields(blob: np.ndarray, P: int, H: int, d: int) -> dict:
    """Split page blobs [n, page_bytes] (u8) into the .kvpg record fields."""
    blob = np.ascontiguousarray(blob, dtype=np.uint8).reshape(-1, P * H * (d + 10))
    n = blob.shape[0]
    cells = P * H
    off = 0
    out = {}
    for name, nbytes, dt, shape in (("k_payload", cells * d // 2, np.uint8, (P, H, d // 2)),
                                    ("v_payload", cells * d // 2, np.uint8, (P, H, d // 2)),
                                    ("k_scale", cells * 4, np.float32, (P, H)),
                                    ("k_zp", cells, np.uint8, (P, H)),
                                    ("v_scale", cells * 4, np.float32, (P, H)),
                                    ("v_zp", cells, np.uint8, (P, H))):
        out[name] = blob[:, off:off + nbytes].copy().view(dt).reshape((n,) + shape)
        off += nbytes
    return out


def kvpg_pages(raw: bytes):
    """(header dict, page blob array) of a .kvpg image."""
    import json
    import struct

    _, hlen = struct.unpack("<II", raw[4:12])
    header = json.loads(raw[12:12 + hlen])
    body = np.frombuffer(raw, dtype=np.uint8, offset=12 + hlen)
    return header, body


def nibble_mismatches(a_packed: np.ndarray, b_packed: np.ndarray) -> int:
    a = np.asarray(a_packed, dtype=np.uint8).ravel()
    b = np.asarray(b_packed, dtype=np.uint8).ravel()
    x = a ^ b
    return int(np.count_nonzero(x & 0x0F) + np.count_nonzero(x & 0xF0))


def ulp_distance_f32(a, b) -> np.ndarray:
    ai = np.asarray(a, dtype=np.float32).view(np.int32).astype(np.int64)
    bi = np.asarray(b, dtype=np.float32).view(np.int32).astype(np.int64)
    ai = np.where(ai < 0, -(ai & 0x7FFFFFFF), ai)
    bi = np.where(bi < 0, -(bi & 0x7FFFFFFF), bi)
    return np.abs(ai - bi)


def gen_rows(kind: str, n: int, d: int, seed: int) -> np.ndarray:
    """bf16-exact synthetic K/V rows (f64).  Kinds follow the reference's harness
    profiles (harness.py:82-176): gaussian, outlier (Rademacher bulk + one fixed
    +-27 hot channel), correlated (Student-t, dense rank-4 mixing, x100 hot
    channels), plus adversarial rows."""
    rng = np.random.default_rng(seed)
    if kind == "gaussian":
        x = rng.standard_normal((n, d))
    elif kind == "outlier":
        x = np.where(rng.random((n, d)) < 0.5, -1.0, 1.0)
        ch = rng.integers(0, d)
        x[:, ch] = np.sign(rng.standard_normal(n)) * 27.0
    elif kind == "correlated":
        x = rng.standard_t(4.0, size=(n, d)) / np.sqrt(2.0)
        a = rng.standard_normal((d, 4))
        b = rng.standard_normal((4, d))
        mix = np.eye(d) + (0.75 / np.sqrt(4 * d)) * (a @ b)
        x = x @ mix.T
        ch = rng.choice(d, size=2, replace=False)
        x[:, ch] *= 100.0
    elif kind == "adversarial":
        x = rng.standard_normal((n, d)) * rng.uniform(0.01, 300, size=(n, 1))
        m = n // 8
        x[0:m] = 0.0
        x[m:2 * m] = np.arange(d) % 16
        x[2 * m:3 * m] = np.abs(x[2 * m:3 * m]) + 1.0
        x[3 * m:4 * m] = -np.abs(x[3 * m:4 * m]) - 1.0
        x[4 * m:5 * m] = np.linspace(-7.5, 7.5, d)
        x[5 * m:5 * m + 1] = 3.25
    else:
        raise ValueError(kind)
    return bf16_round(x)
