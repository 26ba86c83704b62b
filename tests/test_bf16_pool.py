"""BF16 pools (cache.py:115-118, 264-266, 355-361; attention.py:67-71) against the
reference's own outputs (tests/golden/make_golden_bf16.py).

CPU: the `.kvpg` record <-> device cell conversion round-trips the reference dumps.
GPU: appends (per token and two-pass, f64 inputs incl. RNE ties and f32
subnormals) reproduce the reference dumps byte for byte, read_sequence is exact,
decode matches within the decode tolerance and ignores the rotation spec."""

import json
import struct

import numpy as np
import pytest
import torch

from kvtest_util import golden_bytes
from paper_2604_19157_b200.cache import BF16, capacity_tokens, cells_to_records, page_bytes, record_bytes, \
    records_to_cells, token_bytes
from paper_2604_19157_b200.layout import HeadLayout

LAYOUTS = {"bf_small": (8, 2, 32, 32, 4), "bf_big": (32, 8, 128, 128, 16)}
LENS = (5, 17, 1)


def _layout(tag):
    nq, nkv, d, order, P = LAYOUTS[tag]
    return HeadLayout(num_q_heads=nq, num_kv_heads=nkv, head_dim=d, rot_order=order, page_tokens=P)


@pytest.mark.parametrize("tag", list(LAYOUTS))
def test_bf16_record_cell_round_trip(tag):
    lay = _layout(tag)
    raw = golden_bytes(f"{tag}.kvpg")
    _, hlen = struct.unpack("<II", raw[4:12])
    header = json.loads(raw[12:12 + hlen])
    assert header["precision"] == BF16
    body = np.frombuffer(raw, np.uint8, offset=12 + hlen).reshape(-1, record_bytes(lay, BF16))
    cells = records_to_cells(body, lay, BF16)
    assert cells.shape[1] == page_bytes(lay, BF16)
    assert np.array_equal(cells_to_records(cells, lay, BF16), body)


def test_bf16_accounting():
    lay = _layout("bf_big")
    assert token_bytes(lay, BF16) == 4096 and record_bytes(lay, BF16) == 16 * 4096
    assert capacity_tokens(1 << 30, lay, "int4") == 4 * capacity_tokens(1 << 30, lay, BF16)


def _filled(tag, golden_bf16):
    from paper_2604_19157_b200 import PageTable, RotationSpec, make_signs

    lay = _layout(tag)
    spec = RotationSpec(order=lay.rot_order, signs=make_signs(3, 0, lay.head_dim, lay.rot_order))
    t = PageTable(lay, precision=BF16, num_pages=16)
    for s, n in enumerate(LENS):
        t.create_sequence(s)
        k, v = golden_bf16[f"{tag}_k_{s}"], golden_bf16[f"{tag}_v_{s}"]
        if s == 1:
            t.append_tokens_two_pass(s, k, v, spec=spec)
        else:
            for i in range(n):
                t.append_token(s, k[i], v[i], spec=spec)
    return t, spec


@pytest.mark.gpu
@pytest.mark.parametrize("tag", list(LAYOUTS))
def test_bf16_dump_read_decode_match_reference(tag, golden_bf16):
    from paper_2604_19157_b200 import DecodeRequest, decode_step

    t, spec = _filled(tag, golden_bf16)
    assert t.dump_bytes() == golden_bytes(f"{tag}.kvpg")
    for s in range(len(LENS)):
        kh, vh = t.read_sequence(s)
        np.testing.assert_array_equal(kh, golden_bf16[f"{tag}_read_k_{s}"])
        np.testing.assert_array_equal(vh, golden_bf16[f"{tag}_read_v_{s}"])
        q = golden_bf16[f"{tag}_q_{s}"]
        want = golden_bf16[f"{tag}_dec_{s}"]
        np.testing.assert_array_equal(want, golden_bf16[f"{tag}_dec_nospec_{s}"])  # the spec is ignored
        for sp in (spec, None):
            out = decode_step(DecodeRequest(q=q, seq=s), t, spec=sp)
            assert np.abs(out - want).max() <= 1e-3 * np.abs(want).max()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float16])
def test_bf16_batch_write_and_load(tmp_path, dtype, golden_bf16):
    """Serving-path writes (append_batch, CUDA tensors of any dtype) round to the same
    bf16 bits as the reference rule; a dump reloads to the same pool."""
    from paper_2604_19157_b200 import PageTable
    from paper_2604_19157_b200.cache import float_to_bf16_bits

    lay = _layout("bf_big")
    t = PageTable(lay, precision=BF16, num_pages=8)
    t.create_sequence(0)
    x = torch.tensor(np.random.default_rng(5).standard_normal((40, 8, 128)) * 7, dtype=dtype)
    t.append_batch([0] * 40, x.cuda(), (-x).cuda())
    kh, vh = t.read_sequence(0)
    want = float_to_bf16_bits(x.double().numpy())
    assert np.array_equal(kh.astype(np.float32).view(np.uint32) >> 16, want.astype(np.uint32))
    assert np.array_equal(vh, -kh)
    path = tmp_path / "p.kvpg"
    t.dump(path)
    t2 = PageTable.load(path)
    assert t2.precision == BF16 and t2.dump_bytes() == path.read_bytes()
    np.testing.assert_array_equal(t2.read_sequence(0)[0], kh)


@pytest.mark.gpu
@pytest.mark.parametrize("L,G,splits", [(37, 4, 1), (300, 4, 0), (4096, 4, 0), (4096, 8, 0), (32768, 4, 0), (1000, 1, 3)])
def test_bf16_tuned_decode_vs_f64(L, G, splits):
    """The tensor-core BF16-pool decode (d = 128, 16-token cells) against an f64 decode of
    the same raw bf16 rows, any split count; the ragged last cell holds stale NaN rows."""
    from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable
    from paper_2604_19157_b200.cache import BF16

    H, d = 2, 128
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=16)
    t = PageTable(layout, precision=BF16, num_pages=(L + 15) // 16 + 1)
    t.pool.fill_(0xFF)  # unwritten slots: NaN bit patterns
    t.create_sequence(0)
    g = torch.Generator(device="cuda").manual_seed(L + G)
    k = torch.randn((L, H, d), generator=g, device="cuda").bfloat16()
    v = torch.randn((L, H, d), generator=g, device="cuda").bfloat16()
    t.store_slots(k, v, torch.from_numpy(t.alloc.reserve(0, L)).cuda(), None)
    q = torch.randn((1, G * H, d), generator=g, device="cuda").bfloat16()
    out = DecodePlan(t, [0], num_splits=splits).run(q, None)
    torch.cuda.synchronize()
    kk, vv, qq = k.double().cpu(), v.double().cpu(), q[0].double().cpu()
    ref = torch.empty((G * H, d), dtype=torch.float64)
    for qh in range(G * H):
        s = kk[:, qh // G] @ qq[qh] / np.sqrt(d)
        w = torch.softmax(s, 0)
        ref[qh] = w @ vv[:, qh // G]
    got = out[0].double().cpu()
    err = float((got - ref).abs().max() / ref.abs().max())
    print(f"L={L} G={G} splits={splits}: rel err {err:.2e}")
    assert torch.isfinite(got).all() and err <= 1e-4
