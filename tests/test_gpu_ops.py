"""Operator layer on the B200 vs golden vectors of the reference (bit-exact).

Ports of the reference's kernel / int4 / hadamard / rotation unit tests
(test_kernels.py, test_int4.py, test_hadamard.py, test_rotation.py) run
against the CUDA library.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

kv = pytest.importorskip("paper_2604_19157_b200")
from paper_2604_19157_b200 import _kernels as K  # noqa: E402
from paper_2604_19157_b200 import errors as E  # noqa: E402
from paper_2604_19157_b200.hadamard import block_hadamard_matrix, fwht_blocks, make_hadamard  # noqa: E402
from paper_2604_19157_b200.int4 import (CONST_SENTINEL, dequantize_head, dequantize_rows, pack, quantize_head,  # noqa: E402
                                        quantize_rows, unpack)
from paper_2604_19157_b200.layout import HeadLayout  # noqa: E402
from paper_2604_19157_b200.rotation import (RotationSpec, apply_block_rotation, apply_inverse_rotation,  # noqa: E402
                                            compose_transform, make_signs)

from oracle import kvrot_oracle as O  # noqa: E402


@pytest.fixture
def small_layout():
    return HeadLayout(num_q_heads=4, num_kv_heads=2, head_dim=32, rot_order=16, page_tokens=4)


def test_backend_is_native():
    assert K.get_backend() == "cuda-sm100a"
    import os
    from paper_2604_19157_b200 import _lib
    assert os.path.exists(_lib.LIB_PATH)


def test_fwht_rows_bit_exact(golden):
    x = golden["fwht_in"]
    for order in (1, 2, 4, 16, 32, 64, 128):
        y = x.copy()
        K.fwht_rows(y, order)
        np.testing.assert_array_equal(y, golden[f"fwht_out_{order}"])
    y = golden["fwht_adv_in"].copy()
    K.fwht_rows(y, 64)
    np.testing.assert_array_equal(y, golden["fwht_adv_out_64"])


@pytest.mark.parametrize("fam", ["gauss_bf16", "outlier", "correlated", "adversarial"])
def test_quantize_dequantize_bit_exact(golden, fam):
    rows = golden[f"q_{fam}_in"]
    p, s, z = K.quantize_rows(rows)
    np.testing.assert_array_equal(p, golden[f"q_{fam}_packed"])
    np.testing.assert_array_equal(z, golden[f"q_{fam}_zp"])
    # sentinel offsets by value (numpy's min of +-0 is order dependent)
    np.testing.assert_array_equal(s.astype(np.float64), golden[f"q_{fam}_scale"].astype(np.float64))
    d = K.dequantize_rows(p, s, z, rows.shape[1])
    np.testing.assert_array_equal(d, golden[f"q_{fam}_deq"])


def test_quantize_matches_oracle_large(rng):
    x = rng.standard_normal((20000, 128)) * rng.uniform(0.01, 300, size=(20000, 1))
    x[::97] = 1.5
    p, s, z = K.quantize_rows(x)
    po, so, zo = O.quantize_rows(x)
    np.testing.assert_array_equal(p, po)
    np.testing.assert_array_equal(s, so)
    np.testing.assert_array_equal(z, zo)


def test_pack_unpack(rng):
    nib = rng.integers(0, 16, size=(23, 64), dtype=np.uint8)
    p = K.pack_rows(nib)
    np.testing.assert_array_equal(p, O.pack_rows(nib))
    np.testing.assert_array_equal(K.unpack_rows(p, 64), nib)
    assert pack(np.array([0x3, 0xA], dtype=np.uint8)).data == bytes([0xA3])
    for n in range(1, 20):
        seq = rng.integers(0, 16, size=n, dtype=np.uint8)
        np.testing.assert_array_equal(unpack(pack(seq)), seq)
    with pytest.raises(E.NibbleRangeError):
        pack(np.array([16, 0]))


def test_int4_frozen_and_sentinel():
    packed, params = quantize_head(np.array([1.0, 1.0, 1.0, 100.0]))
    assert params.scale == 6.599999904632568 and params.zero_point == 0
    np.testing.assert_array_equal(unpack(packed), [0, 0, 0, 15])
    np.testing.assert_allclose(dequantize_head(packed, params), [0, 0, 0, 98.99999856948853], atol=0)
    packed, params = quantize_head(np.full(8, 5.0))
    assert params.scale == 0.0 and params.offset == 5.0
    np.testing.assert_array_equal(dequantize_head(packed, params), np.full(8, 5.0))
    p, s, z = quantize_rows(np.array([[5.0, 5.0, 5.0, 5.0]]))
    assert z.tolist() == [CONST_SENTINEL] and s.tolist() == [5.0]


def test_int4_bounds_and_clipping(rng):
    for _ in range(50):
        d = int(rng.integers(2, 65)) * 2
        x = rng.standard_normal(d) * float(rng.uniform(0.01, 100))
        x -= x.mean()
        packed, params = quantize_head(x)
        xhat = dequantize_head(packed, params)
        assert np.max(np.abs(x - xhat)) <= params.scale / 2 + 1e-9
    x = rng.uniform(1.0, 3.0, size=32)
    packed, params = quantize_head(x)
    assert params.zero_point == 0
    packed, params = quantize_head(-x)
    assert params.zero_point == 15


def test_int4_validation():
    with pytest.raises(E.ShapeError):
        quantize_head(np.ones(5))
    with pytest.raises(E.NonFiniteInputError):
        quantize_head(np.array([1.0, np.nan, 0.0, 0.0]))
    with pytest.raises(E.NonFiniteInputError):
        quantize_rows(np.array([[1.0, np.inf]]))


def test_rows_match_per_head(rng):
    x = rng.standard_normal((25, 32)) * 7
    x[7] = 2.5
    packed, scale, zp = quantize_rows(x)
    xhat = dequantize_rows(packed, scale, zp, 32)
    for i in range(25):
        p_i, prm = quantize_head(x[i])
        np.testing.assert_array_equal(packed[i], np.frombuffer(p_i.data, dtype=np.uint8))
        np.testing.assert_array_equal(xhat[i], dequantize_head(p_i, prm))


def test_hadamard_dense_and_fwht(rng):
    for order in (1, 2, 4, 8, 16, 32, 64, 128):
        h = make_hadamard(order).entries
        np.testing.assert_array_equal(h, O.make_hadamard(order))
    out = fwht_blocks(np.arange(8, dtype=np.float64).reshape(1, 8), 4)
    np.testing.assert_allclose(out, [[3.0, -1.0, -2.0, 0.0, 11.0, -1.0, -2.0, 0.0]], atol=1e-12)
    for dim, order in ((32, 4), (32, 16), (128, 128), (64, 8)):
        x = rng.standard_normal((20, dim))
        np.testing.assert_allclose(fwht_blocks(x, order), x @ block_hadamard_matrix(dim, order).T, atol=1e-12)
    x = rng.standard_normal((5, 16))
    keep = x.copy()
    fwht_blocks(x, 16)
    np.testing.assert_array_equal(x, keep)
    with pytest.raises(E.InvalidOrderError):
        fwht_blocks(rng.standard_normal((4, 24)), 16)


def test_rotation_bit_exact(golden):
    lay = HeadLayout(num_q_heads=32, num_kv_heads=8, head_dim=128, rot_order=128)
    spec = RotationSpec(order=128, signs=golden["signs_0_0_128_128"])
    np.testing.assert_array_equal(apply_block_rotation(golden["rot_in"], lay, spec), golden["rot_fwd"])
    np.testing.assert_array_equal(apply_inverse_rotation(golden["rot_in"], lay, spec), golden["rot_inv"])


def test_signs_pinned(golden):
    for key in [k for k in golden if k.startswith("signs_")]:
        _, seed, layer, d, order = key.split("_")
        np.testing.assert_array_equal(make_signs(int(seed), int(layer), int(d), int(order)), golden[key])


def test_rotation_round_trip_and_dense(rng, small_layout):
    d = small_layout.head_dim
    q, r = np.linalg.qr(rng.standard_normal((d, d)))
    learned = q * np.sign(np.diag(r))
    spec = RotationSpec(order=small_layout.rot_order, signs=make_signs(3, 0, d, small_layout.rot_order),
                        learned=learned)
    x = rng.standard_normal((40, d)) * 9
    back = apply_inverse_rotation(apply_block_rotation(x, small_layout, spec), small_layout, spec)
    np.testing.assert_allclose(back, x, atol=1e-12)
    t = compose_transform(spec, small_layout)
    np.testing.assert_allclose(apply_block_rotation(x, small_layout, spec), x @ t, atol=1e-12)


def test_rotation_preserves_logits():
    # acceptance c01 (test_acceptance.py:45-70)
    rng = np.random.default_rng(20260816)
    q = rng.standard_normal((10_000, 128))
    k = rng.standard_normal((10_000, 128))
    base = np.einsum("td,td->t", q, k)
    worst = 0.0
    for order in (16, 32, 64, 128):
        lay = HeadLayout(num_q_heads=1, num_kv_heads=1, head_dim=128, rot_order=order)
        spec = RotationSpec(order=order, signs=make_signs(7, 0, 128, order))
        qr = apply_block_rotation(q, lay, spec)
        kr = apply_block_rotation(k, lay, spec)
        worst = max(worst, float((np.abs(np.einsum("td,td->t", qr, kr) - base) / np.abs(base)).max()))
    assert worst <= 1e-4
