"""Row f3: a learned orthogonal R composed after the block Hadamard
(rotation.py:118-168): writes, decode and the serving step on the device,
against the oracle with the reference's composition order.

The dense x @ R product goes through a BLAS on both sides (numpy/OpenBLAS in the
reference, cuBLAS DGEMM here) with unspecified summation order, so stored codes
may differ by one step where the rotated value sits on a rounding boundary:
the test bounds that count; decode outputs stay within the 1e-3 tolerance.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from kvtest_util import bf16_round, gen_rows, page_fields  # noqa: E402
from oracle import kvrot_oracle as O  # noqa: E402
from paper_2604_19157_b200.attention import DecodePlan, decode_batch  # noqa: E402
from paper_2604_19157_b200.cache import PageTable  # noqa: E402
from paper_2604_19157_b200.layout import HeadLayout  # noqa: E402
from paper_2604_19157_b200.rotation import RotationSpec, Targets, make_signs  # noqa: E402

TOL = 1e-3


def _orth(d, seed):
    q, r = np.linalg.qr(np.random.default_rng(seed).standard_normal((d, d)))
    return q * np.sign(np.diag(r))


def _ref_rotate(x, spec, values):
    """Reference transform of rows: signs, FWHT, then R (values: R only if learned_values)."""
    if values and spec.targets is Targets.KEYS_ONLY:
        return x
    y = O.rotate_rows(x, spec.order, spec.signs)
    if not values or spec.learned_values:
        y = y @ spec.learned
    return y


@pytest.mark.parametrize("targets,learned_values", [(Targets.KEYS_AND_VALUES, False), (Targets.KEYS_AND_VALUES, True),
                                                    (Targets.KEYS_ONLY, False)])
def test_learned_write_and_decode(targets, learned_values):
    H, G, d, P = 2, 4, 128, 16
    lens = [7, 40, 300]
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=P)
    t = PageTable(layout, num_pages=sum((L + P - 1) // P for L in lens) + 2)
    spec = RotationSpec(order=128, signs=make_signs(4, 0, d, 128), learned=_orth(d, 11), targets=targets,
                        learned_values=learned_values)
    seqs, ks, vs = [], [], []
    for s, L in enumerate(lens):
        t.create_sequence(s)
        seqs += [s] * L
        ks.append(gen_rows("gaussian", L * H, d, 100 + s).reshape(L, H, d))
        vs.append(gen_rows("outlier", L * H, d, 200 + s).reshape(L, H, d))
    k, v = np.concatenate(ks), np.concatenate(vs)
    t.append_batch(seqs, torch.tensor(k), torch.tensor(v), spec=spec)
    # 1) stored bytes vs the reference composition (codes: at most a few boundary steps)
    kr = _ref_rotate(k.reshape(-1, d), spec, values=False)
    vr = _ref_rotate(v.reshape(-1, d), spec, values=True)
    mism = total = 0
    row = 0
    for s, L in enumerate(lens):
        f = page_fields(t.page_records(t.sequence_pages(s)), P, H, d)
        for side, ref in (("k", kr), ("v", vr)):
            pk, sk, zk = O.quantize_rows(ref[row * H:(row + L) * H])
            got = f[f"{side}_payload"].reshape(-1, H, d // 2)[:L].reshape(-1, d // 2)
            gl, gh = got & 15, got >> 4
            rl, rh = pk & 15, pk >> 4
            dl = np.abs(gl.astype(int) - rl) + np.abs(gh.astype(int) - rh)
            assert dl.max() <= 1
            mism += int((dl > 0).sum())
            total += dl.size * 2
            np.testing.assert_allclose(f[f"{side}_scale"].reshape(-1, H)[:L].reshape(-1), sk, rtol=1e-6)
        row += L
    print("learned: nibble mismatches", mism, "of", total)
    assert mism <= total * 1e-3
    # 2) decode: q through the full transform, the value branch undone on the output
    q = np.random.default_rng(9).standard_normal((len(lens), G * H, d))
    out = decode_batch(torch.tensor(q, dtype=torch.float32).cuda(), t, list(range(len(lens))), spec=spec)
    kd, vd = t.read_sequence_device(list(range(len(lens))), torch.float64)
    for b, L in enumerate(lens):
        qf = _ref_rotate(q[b], spec, values=False)
        o = O.decode_flat(qf, kd[b, :L].cpu().numpy(), vd[b, :L].cpu().numpy(), G)
        if targets is Targets.KEYS_AND_VALUES:
            if learned_values:
                o = o @ spec.learned.T
            o = O.unrotate_rows(o, spec.order, spec.signs)
        err = np.abs(out[b].double().cpu().numpy() - o).max() / np.abs(o).max()
        print("learned decode", b, err)
        assert err <= TOL


def test_learned_serving_step():
    """DecodePlan.step with a learned spec: unfused write of the new token, then decode."""
    H, G, d = 2, 4, 128
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=16)
    t = PageTable(layout, num_pages=16)
    spec = RotationSpec(order=128, signs=make_signs(4, 0, d, 128), learned=_orth(d, 12), learned_values=True)
    for s in range(2):
        t.create_sequence(s)
    k0 = gen_rows("gaussian", 2 * 50 * H, d, 5).reshape(100, H, d)
    v0 = gen_rows("gaussian", 2 * 50 * H, d, 6).reshape(100, H, d)
    t.append_batch([0] * 50 + [1] * 50, torch.tensor(k0), torch.tensor(v0), spec=spec)
    plan = DecodePlan(t, [0, 1], extra_tokens=4)
    rng = np.random.default_rng(3)
    for _ in range(3):
        q = rng.standard_normal((2, G * H, d))
        kn = torch.tensor(rng.standard_normal((2, H, d)), dtype=torch.bfloat16)
        vn = torch.tensor(rng.standard_normal((2, H, d)), dtype=torch.bfloat16)
        out = plan.step(torch.tensor(q, dtype=torch.float32), kn, vn, spec).cpu().numpy()
        kd, vd = t.read_sequence_device([0, 1], torch.float64)
        for b in range(2):
            L = t.sequence_length(b)
            o = O.decode_flat(_ref_rotate(q[b], spec, False), kd[b, :L].cpu().numpy(), vd[b, :L].cpu().numpy(), G)
            o = O.unrotate_rows(o @ spec.learned.T, spec.order, spec.signs)
            assert np.abs(out[b] - o).max() / np.abs(o).max() <= TOL


def _bf16(a):
    return torch.tensor(bf16_round(a), dtype=torch.float64).to(torch.bfloat16)


@pytest.mark.parametrize("fast", [False, True])
@pytest.mark.parametrize("order", [128, 32])
@pytest.mark.parametrize("targets,learned_values", [(Targets.KEYS_AND_VALUES, False), (Targets.KEYS_AND_VALUES, True),
                                                    (Targets.KEYS_ONLY, False)])
def test_learned_fused_store_bf16(monkeypatch, order, targets, learned_values, fast):
    """Row f3 fused: bf16 rows through the tcgen05 K1 with T = diag(s) H_blk R in shared memory,
    against the reference composition (f64 FWHT then R).  Default (exact rows): codes and zero
    points identical (a row with a code near a boundary is redone whole under the reference's
    (s, z)).  Fast mode (KVR_K1L_FAST=1): codes at most one step off, in <= 1e-5 of the
    nibbles.  Scales within rtol 1e-5 either way (f32 accumulation of the dense product for the
    rows not redone; the stated tolerance is 1e-3)."""
    import paper_2604_19157_b200.rotation as rotmod

    if fast:
        monkeypatch.setenv("KVR_K1L_FAST", "1")

    def _no_unfused(*a, **kw):
        raise AssertionError("the fused learned K1 must take bf16 rows")

    monkeypatch.setattr(rotmod, "rotate_kv_learned", _no_unfused)
    H, G, d, P = 8, 4, 128, 16
    lens = [7, 40, 1500, 2049]
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=order, page_tokens=P)
    t = PageTable(layout, num_pages=sum((L + P - 1) // P for L in lens) + 2)
    spec = RotationSpec(order=order, signs=make_signs(4, 0, d, order), learned=_orth(d, 21), targets=targets,
                        learned_values=learned_values)
    kinds = ["gaussian", "outlier", "correlated", "gaussian"]
    seqs, ks, vs = [], [], []
    for s, L in enumerate(lens):
        t.create_sequence(s)
        seqs += [s] * L
        ks.append(bf16_round(gen_rows(kinds[s], L * H, d, 300 + s)).reshape(L, H, d))
        vs.append(bf16_round(gen_rows(kinds[3 - s], L * H, d, 400 + s)).reshape(L, H, d))
    k, v = np.concatenate(ks), np.concatenate(vs)
    t.append_batch(seqs, _bf16(k), _bf16(v), spec=spec)
    t.check_flags()
    kr = _ref_rotate(k.reshape(-1, d), spec, values=False)
    vr = _ref_rotate(v.reshape(-1, d), spec, values=True)
    mism = total = zmis = rows = 0
    worst = 0.0
    row = 0
    for s, L in enumerate(lens):
        f = page_fields(t.page_records(t.sequence_pages(s)), P, H, d)
        for side, ref in (("k", kr), ("v", vr)):
            pk_, sk, zk = O.quantize_rows(ref[row * H:(row + L) * H])
            got = f[f"{side}_payload"].reshape(-1, H, d // 2)[:L].reshape(-1, d // 2)
            dl = np.abs((got & 15).astype(int) - (pk_ & 15)) + np.abs((got >> 4).astype(int) - (pk_ >> 4))
            assert dl.max() <= 1
            mism += int((dl > 0).sum())
            total += dl.size * 2
            gz = f[f"{side}_zp"].reshape(-1, H)[:L].reshape(-1).astype(int)
            assert np.abs(gz - zk.astype(int)).max() <= 1
            zmis += int((gz != zk).sum())
            rows += gz.size
            gs = f[f"{side}_scale"].reshape(-1, H)[:L].reshape(-1).astype(np.float64)
            worst = max(worst, float(np.max(np.abs(gs - sk) / np.abs(sk))))
        row += L
    print(f"learned fused (order {order}, {targets.name}, lv={learned_values}, fast={fast}): nibble mismatches "
          f"{mism} of {total}, zp {zmis} of {rows}, scale max rel {worst:.2e}")
    if fast:
        assert mism <= total * 1e-5 and zmis <= rows * 1e-4
    else:
        assert mism == 0 and zmis == 0
    assert worst <= 1e-5


def test_learned_fused_nonfinite_and_skip():
    """A NaN row is not written and raises the flag; negative slots are skipped; the other
    rows are stored."""
    H, d, P = 2, 128, 16
    layout = HeadLayout(num_q_heads=4 * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=P)
    t = PageTable(layout, num_pages=4)
    spec = RotationSpec(order=128, signs=make_signs(4, 0, d, 128), learned=_orth(d, 5), learned_values=True)
    t.create_sequence(0)
    k = bf16_round(gen_rows("gaussian", 3 * H, d, 1)).reshape(3, H, d)
    v = bf16_round(gen_rows("gaussian", 3 * H, d, 2)).reshape(3, H, d)
    k[1, 0, 17] = np.nan
    t.append_batch([0, 0, 0], _bf16(k), _bf16(v), spec=spec, check=False)
    with pytest.raises(Exception):
        t.check_flags()
    f = page_fields(t.page_records(t.sequence_pages(0)), P, H, d)
    kr = _ref_rotate(k.reshape(-1, d), spec, values=False)
    pk_, sk, zk = O.quantize_rows(np.nan_to_num(kr))
    got = f["k_payload"].reshape(-1, H, d // 2)[:3].reshape(-1, d // 2)
    for r in (0, 1, 3, 4, 5):  # row 2 = token 1, head 0: the NaN row
        dl = np.abs((got[r] & 15).astype(int) - (pk_[r] & 15)) + np.abs((got[r] >> 4).astype(int) - (pk_[r] >> 4))
        assert dl.max() <= 1
    assert not got[2].any()
    # skipped slots: nothing written
    slots = torch.full((2,), -1, dtype=torch.int64, device="cuda")
    before = t.page_records(t.sequence_pages(0)).copy()
    t.store_slots(_bf16(k[:2]).cuda(), _bf16(v[:2]).cuda(), slots, spec=spec)
    torch.cuda.synchronize()
    assert np.array_equal(before, t.page_records(t.sequence_pages(0)))


@pytest.mark.parametrize("n,d,dt", [(1, 128, torch.float64), (37, 128, torch.float32), (300, 64, torch.bfloat16),
                                    (9, 256, torch.float16)])
def test_rows_matmul_f64(n, d, dt):
    """kvr_rows_matmul_f64 (the learned factor and the composed transforms) vs numpy f64."""
    from paper_2604_19157_b200.rotation import rows_matmul

    rng = np.random.default_rng(n + d)
    x = torch.tensor(rng.standard_normal((n, d))).to(dt).cuda()
    m = torch.tensor(_orth(d, 3)).cuda()
    y = rows_matmul(x, m).cpu().numpy()
    ref = x.double().cpu().numpy() @ m.cpu().numpy()
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
    y32 = rows_matmul(x, m, out_dtype=torch.float32).cpu().numpy()
    assert np.abs(y32 - ref).max() <= 1e-6 * np.abs(ref).max()


def test_learned_composed_matches_reference_order():
    """The composed T (one launch) agrees with the reference's FWHT-then-R order to f64 rounding."""
    from paper_2604_19157_b200.rotation import composed_on, rows_matmul

    d = 128
    layout = HeadLayout(num_q_heads=8, num_kv_heads=2, head_dim=d, rot_order=64, page_tokens=16)
    spec = RotationSpec(order=64, signs=make_signs(2, 1, d, 64), learned=_orth(d, 8), learned_values=True)
    x = np.random.default_rng(1).standard_normal((50, d))
    got = rows_matmul(torch.tensor(x).cuda(), composed_on(spec, layout, "cuda")).cpu().numpy()
    ref = _ref_rotate(x, spec, values=False)
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    back = rows_matmul(torch.tensor(got).cuda(), composed_on(spec, layout, "cuda", transpose=True)).cpu().numpy()
    assert np.abs(back - x).max() <= 1e-13 * np.abs(x).max()


@pytest.mark.parametrize("P,H,dt", [(64, 8, torch.bfloat16), (16, 2, torch.float16), (32, 4, torch.bfloat16)])
def test_learned_store_geometries_and_dtypes(P, H, dt):
    """The fused learned K1 at other page sizes / head counts (bf16), and fp16 rows through the
    unfused route (the fused kernel takes bf16 only): the same bars as the bf16 fused test."""
    d = 128
    L = 700
    layout = HeadLayout(num_q_heads=4 * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=P)
    t = PageTable(layout, num_pages=L // P + 2)
    spec = RotationSpec(order=128, signs=make_signs(9, 2, d, 128), learned=_orth(d, 31), learned_values=True)
    t.create_sequence(0)
    rnd = bf16_round if dt == torch.bfloat16 else (lambda a: np.asarray(a, dtype=np.float16).astype(np.float64))
    k = rnd(gen_rows("gaussian", L * H, d, 41)).reshape(L, H, d)
    v = rnd(gen_rows("outlier", L * H, d, 42)).reshape(L, H, d)
    t.append_batch([0] * L, torch.tensor(k).to(dt), torch.tensor(v).to(dt), spec=spec)
    t.check_flags()
    f = page_fields(t.page_records(t.sequence_pages(0)), P, H, d)
    mism = total = 0
    for side, x in (("k", k), ("v", v)):
        ref = _ref_rotate(x.reshape(-1, d), spec, values=side == "v")
        pk_, sk, zk = O.quantize_rows(ref)
        got = f[f"{side}_payload"].reshape(-1, H, d // 2)[:L].reshape(-1, d // 2)
        dl = np.abs((got & 15).astype(int) - (pk_ & 15)) + np.abs((got >> 4).astype(int) - (pk_ >> 4))
        assert dl.max() <= 1
        mism += int((dl > 0).sum())
        total += dl.size * 2
        gz = f[f"{side}_zp"].reshape(-1, H)[:L].reshape(-1).astype(int)
        assert np.abs(gz - zk.astype(int)).max() <= 1
        gs = f[f"{side}_scale"].reshape(-1, H)[:L].reshape(-1).astype(np.float64)
        assert np.max(np.abs(gs - sk) / np.abs(sk)) <= 1e-5
    print(f"learned P={P} H={H} {dt}: nibble mismatches {mism} of {total}")
    assert mism <= total * 1e-4


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("targets,learned_values", [(Targets.KEYS_AND_VALUES, False), (Targets.KEYS_AND_VALUES, True),
                                                    (Targets.KEYS_ONLY, False)])
def test_learned_fused_decode_matches_unfused(monkeypatch, G, targets, learned_values):
    """kvr_paged_decode_learned (q T in the kernel's prologue, the value branch's inverse before
    the store) == the unfused route (f64 row-matmul launches around the plain decode) for every
    merge path: one split, a cluster, the flag-in-data merge, and a split count above 32 (clamped)."""
    H, d, P = 2, 128, 16
    lens = [37, 2000, 700]
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=64, page_tokens=P)
    t = PageTable(layout, num_pages=sum((L + P - 1) // P for L in lens) + 2)
    spec = RotationSpec(order=64, signs=make_signs(5, 0, d, 64), learned=_orth(d, 13), targets=targets,
                        learned_values=learned_values)
    rng = np.random.default_rng(G)
    for s, L in enumerate(lens):
        t.create_sequence(s)
        t.append_batch([s] * L, torch.tensor(rng.standard_normal((L, H, d))), torch.tensor(rng.standard_normal((L, H, d))),
                       spec=spec, check=False)
    q = torch.tensor(rng.standard_normal((len(lens), G * H, d)), dtype=torch.float32).cuda()
    for splits in (1, 4, 16, 64):
        plan = DecodePlan(t, list(range(len(lens))), num_splits=splits)
        monkeypatch.setenv("KVR_LEARNED_DECODE", "fused")
        fused = plan.run(q, spec).clone()
        monkeypatch.setenv("KVR_LEARNED_DECODE", "unfused")
        ref = plan.run(q, spec).clone()
        err = float((fused - ref).abs().max() / ref.abs().max())
        assert err < 2e-5, (splits, err)
