"""K2/K3 paged INT4 decode on the B200 vs the oracle / reference goldens.

Tolerance (BASELINE.json north_star): fp32 decode outputs within
1e-3 * max|ref| of the f64 oracle (measured error is ~1e-6).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from kvtest_util import gen_rows  # noqa: E402
from oracle import kvrot_oracle as O  # noqa: E402
from paper_2604_19157_b200 import errors as E  # noqa: E402
from paper_2604_19157_b200.attention import DecodePlan, DecodeRequest, decode_batch, decode_step, decode_step_fp  # noqa: E402
from paper_2604_19157_b200.cache import PageTable  # noqa: E402
from paper_2604_19157_b200.layout import HeadLayout  # noqa: E402
from paper_2604_19157_b200.rotation import RotationSpec, Targets, make_signs  # noqa: E402

TOL = 1e-3

GOLD = {
    "small_kv": ((4, 2, 32, 16, 4), 8, (11, 3, 32, 16), Targets.KEYS_AND_VALUES),
    "big_kv": ((32, 8, 128, 128, 16), 4, (0, 0, 128, 128), Targets.KEYS_AND_VALUES),
    "big_konly": ((32, 8, 128, 128, 16), 4, (0, 1, 128, 128), Targets.KEYS_ONLY),
    "big_plain": ((32, 8, 128, 128, 16), 4, None, Targets.KEYS_AND_VALUES),
    "o64_kv": ((4, 1, 128, 64, 16), 3, (0, 0, 128, 64), Targets.KEYS_AND_VALUES),
}


def rel_err(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-30))


@pytest.mark.parametrize("tag", list(GOLD))
def test_decode_step_matches_reference(golden, tag):
    lay, npages, sargs, targets = GOLD[tag]
    layout = HeadLayout(num_q_heads=lay[0], num_kv_heads=lay[1], head_dim=lay[2], rot_order=lay[3], page_tokens=lay[4])
    spec = None if sargs is None else RotationSpec(order=lay[3], signs=make_signs(*sargs), targets=targets)
    t = PageTable(layout, num_pages=npages)
    t.create_sequence(0)
    t.append_tokens_two_pass(0, golden[f"tab_{tag}_k_0"], golden[f"tab_{tag}_v_0"], spec=spec)
    out = decode_step(DecodeRequest(q=golden[f"dec_{tag}_q"], seq=0), t, spec=spec)
    err = rel_err(out, golden[f"dec_{tag}_out"])
    print(tag, "rel err", err)
    assert err <= TOL


def _build(n_seq, lens, H, G, d, order, P, kind, targets, rotate, seed, dtype=torch.bfloat16, extra_pages=0):
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=order, page_tokens=P)
    npages = sum((L + P - 1) // P for L in lens) + extra_pages
    t = PageTable(layout, num_pages=npages)
    signs = make_signs(seed, 0, d, order) if rotate else None
    spec = RotationSpec(order=order, signs=signs, targets=targets) if rotate else None
    seqs, ks, vs = [], [], []
    for s, L in enumerate(lens):
        t.create_sequence(s)
        seqs += [s] * L
        ks.append(gen_rows(kind, L * H, d, seed + 2 * s).reshape(L, H, d))
        vs.append(gen_rows(kind, L * H, d, seed + 2 * s + 1).reshape(L, H, d))
    k = np.concatenate(ks)
    v = np.concatenate(vs)
    t.append_batch(seqs, torch.tensor(k, dtype=dtype).cuda(), torch.tensor(v, dtype=dtype).cuda(), spec=spec)
    return t, spec, layout


def _oracle_decode(t, layout, spec, q, seqs):
    kd, vd = t.read_sequence_device(seqs, torch.float64)  # bit-exact dequant (K4) of what the kernel reads
    outs = []
    for b, s in enumerate(seqs):
        L = t.sequence_length(s)
        kh, vh = kd[b, :L].cpu().numpy(), vd[b, :L].cpu().numpy()
        signs = None if spec is None else spec.signs
        qf = O.rotate_rows(q[b], layout.rot_order, signs) if spec is not None else q[b]
        o = O.decode_flat(qf, kh, vh, layout.group_size)
        if spec is not None and spec.targets is Targets.KEYS_AND_VALUES:
            o = O.unrotate_rows(o, layout.rot_order, signs)
        outs.append(o)
    return np.stack(outs)


@pytest.mark.parametrize("rotate,targets", [(True, Targets.KEYS_AND_VALUES), (True, Targets.KEYS_ONLY),
                                            (False, Targets.KEYS_AND_VALUES)])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_decode_mma_vs_oracle(rotate, targets, G):
    lens = [1, 15, 16, 17, 333, 1000]
    t, spec, layout = _build(len(lens), lens, 2, G, 128, 128, 16, "gaussian", targets, rotate, seed=3)
    rng = np.random.default_rng(5)
    q = rng.standard_normal((len(lens), G * 2, 128))
    out = decode_batch(torch.tensor(q, dtype=torch.float32).cuda(), t, list(range(len(lens))), spec=spec)
    ref = _oracle_decode(t, layout, spec, q, list(range(len(lens))))
    err = rel_err(out.double().cpu().numpy(), ref)
    print("G", G, rotate, targets, "rel err", err)
    assert err <= TOL


@pytest.mark.parametrize("splits", [1, 2, 7, 64])
def test_decode_split_counts(splits):
    lens = [2000, 513]
    t, spec, layout = _build(2, lens, 8, 4, 128, 128, 16, "outlier", Targets.KEYS_AND_VALUES, True, seed=9)
    q = np.random.default_rng(1).standard_normal((2, 32, 128))
    plan = DecodePlan(t, [0, 1], num_splits=splits)
    out = plan.run(torch.tensor(q, dtype=torch.float32).cuda(), spec)
    ref = _oracle_decode(t, layout, spec, q, [0, 1])
    err = rel_err(out.double().cpu().numpy(), ref)
    print("splits", splits, err)
    assert err <= TOL
    # the workspace counters re-arm: a second launch gives the same answer
    out2 = plan.run(torch.tensor(q, dtype=torch.float32).cuda(), spec)
    assert torch.equal(out, out2)


@pytest.mark.parametrize("P", [4, 8, 32])
def test_decode_page_sizes(P):
    lens = [100, 37]
    t, spec, layout = _build(2, lens, 2, 4, 128, 64, P, "correlated", Targets.KEYS_AND_VALUES, True, seed=4)
    q = np.random.default_rng(2).standard_normal((2, 8, 128))
    out = decode_batch(torch.tensor(q, dtype=torch.float32).cuda(), t, [0, 1], spec=spec)
    ref = _oracle_decode(t, layout, spec, q, [0, 1])
    assert rel_err(out.double().cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("d,order", [(32, 16), (64, 64), (256, 128)])
def test_decode_generic_dims(d, order):
    lens = [50, 9]
    t, spec, layout = _build(2, lens, 2, 2, d, order, 8, "gaussian", Targets.KEYS_AND_VALUES, True, seed=6,
                             dtype=torch.float64)
    q = np.random.default_rng(3).standard_normal((2, 4, d))
    out = decode_batch(torch.tensor(q, dtype=torch.float32).cuda(), t, [0, 1], spec=spec)
    ref = _oracle_decode(t, layout, spec, q, [0, 1])
    assert rel_err(out.double().cpu().numpy(), ref) <= TOL


def test_decode_c2_shape():
    # configs[1]: batch 1, 32k context, GQA 32q/8kv, rotated Q and inverse-rotated V
    t, spec, layout = _build(1, [32768], 8, 4, 128, 128, 16, "gaussian", Targets.KEYS_AND_VALUES, True, seed=12)
    q = np.random.default_rng(4).standard_normal((1, 32, 128))
    out = decode_batch(torch.tensor(q, dtype=torch.bfloat16).cuda(), t, [0], spec=spec)
    qb = torch.tensor(q, dtype=torch.bfloat16).double().numpy()
    ref = _oracle_decode(t, layout, spec, qb, [0])
    err = rel_err(out.double().cpu().numpy(), ref)
    print("C2 rel err", err)
    assert err <= TOL


def test_decode_sentinel_and_shift():
    layout = HeadLayout(num_q_heads=8, num_kv_heads=2, head_dim=128, rot_order=128)
    t = PageTable(layout, num_pages=4)
    t.create_sequence(0)
    rng = np.random.default_rng(8)
    k = rng.standard_normal((20, 2, 128))
    v = rng.standard_normal((20, 2, 128))
    k[3] = 2.5      # constant rows -> sentinel pages
    v[4] = -1.25
    k[5] = 0.0
    t.append_tokens_two_pass(0, k, v)
    q = rng.standard_normal((1, 8, 128)) * 30  # large logits
    out = decode_batch(torch.tensor(q, dtype=torch.float32).cuda(), t, [0])
    ref = _oracle_decode(t, layout, None, q, [0])
    assert rel_err(out.double().cpu().numpy(), ref) <= TOL


def test_decode_validation(rng):
    layout = HeadLayout(num_q_heads=4, num_kv_heads=2, head_dim=32, rot_order=16, page_tokens=4)
    t = PageTable(layout, num_pages=2)
    t.create_sequence(0)
    q = rng.standard_normal((4, 32))
    with pytest.raises(E.EmptySequenceError):
        decode_step(DecodeRequest(q=q, seq=0), t)
    t.append_token(0, rng.standard_normal((2, 32)), rng.standard_normal((2, 32)))
    with pytest.raises(E.ShapeError):
        decode_step(DecodeRequest(q=np.zeros((1, 32)), seq=0), t)
    bad = np.zeros((4, 32))
    bad[0, 0] = np.inf
    with pytest.raises(E.NonFiniteInputError):
        decode_step(DecodeRequest(q=bad, seq=0), t)


def test_decode_step_fp_gqa():
    layout = HeadLayout(num_q_heads=4, num_kv_heads=2, head_dim=32, rot_order=16, page_tokens=4)
    k = np.zeros((5, 2, 32))
    v = np.zeros((5, 2, 32))
    v[:, 0, :] = 1.0
    v[:, 1, :] = 2.0
    out = decode_step_fp(np.zeros((4, 32)), k, v, layout)
    np.testing.assert_allclose(out[:2], 1.0)
    np.testing.assert_allclose(out[2:], 2.0)


@pytest.mark.parametrize("targets", [Targets.KEYS_AND_VALUES, Targets.KEYS_ONLY, None])
@pytest.mark.parametrize("G", [4, 8])
def test_fused_decode_step(targets, G):
    """One serving step = append the new token (bit-exact f64 rotate + INT4 into its
    slot) + decode over it, in one launch (kvr_decode_step)."""
    H, d = 2, 128
    lens = [15, 16, 300, 1025]
    rotate = targets is not None
    t, spec, layout = _build(len(lens), lens, H, G, d, 128, 16, "gaussian",
                             targets or Targets.KEYS_AND_VALUES, rotate, seed=31, extra_pages=len(lens))
    seqs = list(range(len(lens)))
    rng = np.random.default_rng(77)
    k_new = rng.standard_normal((len(lens), H, d))
    v_new = rng.standard_normal((len(lens), H, d))
    q = rng.standard_normal((len(lens), G * H, d))
    plan = DecodePlan(t, seqs, extra_tokens=1)
    kb = torch.tensor(k_new, dtype=torch.bfloat16)
    vb = torch.tensor(v_new, dtype=torch.bfloat16)
    out = plan.step(torch.tensor(q, dtype=torch.float32).cuda(), kb.cuda(), vb.cuda(), spec)
    # 1) the appended slots are bit-identical to the reference append of the same bf16 values
    signs = None if spec is None else spec.signs
    for b, s in enumerate(seqs):
        L = t.sequence_length(s) - 1
        page = t.sequence_pages(s)[L // 16]
        blob = t.page_records([page])
        from kvtest_util import page_fields
        f = page_fields(blob, 16, H, d)
        kk = O.rotate_rows(kb[b].double().numpy(), 128, signs) if rotate else kb[b].double().numpy()
        vrot = rotate and targets is Targets.KEYS_AND_VALUES
        vv = O.rotate_rows(vb[b].double().numpy(), 128, signs) if vrot else vb[b].double().numpy()
        for side, x in (("k", kk), ("v", vv)):
            pk, sk, zk = O.quantize_rows(x)
            np.testing.assert_array_equal(f[f"{side}_payload"][0, L % 16], pk)
            np.testing.assert_array_equal(f[f"{side}_scale"][0, L % 16], sk)
            np.testing.assert_array_equal(f[f"{side}_zp"][0, L % 16], zk)
    # 2) the decode saw the new token
    refo = _oracle_decode(t, layout, spec, q, seqs)
    err = rel_err(out.double().cpu().numpy(), refo)
    print("fused step", G, targets, err)
    assert err <= TOL


def test_step_graph_replay_matches_eager():
    """DecodePlan.step(graph=True) (CUDA-graph replay of the H2D + decode kernels)
    gives the same outputs and page bytes as the eager path, across page
    boundaries (fresh pages every 16 steps) and pinned-ring wraparound."""
    H, G, d = 2, 4, 128
    lens = [30, 77]
    outs = {}
    dumps = {}
    for mode in (False, True):
        t, spec, layout = _build(len(lens), lens, H, G, d, 128, 16, "gaussian", Targets.KEYS_AND_VALUES, True,
                                 seed=5, extra_pages=8)
        plan = DecodePlan(t, [0, 1], extra_tokens=40)
        rng = np.random.default_rng(123)
        res = []
        od = torch.empty((2, G * H, d), dtype=torch.float32, device="cuda")
        for _ in range(37):
            q = torch.tensor(rng.standard_normal((2, G * H, d)), dtype=torch.bfloat16).pin_memory()
            k = torch.tensor(rng.standard_normal((2, H, d)), dtype=torch.bfloat16).pin_memory()
            v = torch.tensor(rng.standard_normal((2, H, d)), dtype=torch.bfloat16).pin_memory()
            res.append(plan.step(q, k, v, spec, out=od, graph=mode).cpu().clone())
        torch.cuda.synchronize()
        outs[mode] = torch.stack(res)
        dumps[mode] = t.dump_bytes()
    assert torch.equal(outs[False], outs[True])
    assert dumps[False] == dumps[True]


@pytest.mark.parametrize("kind", ["gaussian", "outlier", "correlated", "adversarial"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
def test_fused_append_bit_exact_many_rows(kind, dtype):
    """The fused step's writer warp (f64 rotate + quantize, reciprocal-based
    correctly rounded divisions) stores exactly the reference's bytes for 256
    sequences x 8 heads of each row family, in bf16 / f32 / f64 inputs."""
    B, H, G, d = 256, 8, 1, 128
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=16)
    t = PageTable(layout, num_pages=B)
    spec = RotationSpec(order=128, signs=make_signs(9, 0, d, 128), targets=Targets.KEYS_AND_VALUES)
    for s in range(B):
        t.create_sequence(s)
    rows = gen_rows(kind, 2 * B * H, d, 1234)
    if dtype is not torch.bfloat16:  # full-mantissa inputs: dense rounding-boundary coverage
        rng = np.random.default_rng(5)
        rows = rows * (1.0 + rng.standard_normal(rows.shape) * 1e-3)
        if dtype is torch.float32:
            rows = rows.astype(np.float32).astype(np.float64)
    k_new = rows[: B * H].reshape(B, H, d)
    v_new = rows[B * H:].reshape(B, H, d)
    plan = DecodePlan(t, list(range(B)), extra_tokens=1)
    q = torch.zeros((B, G * H, d), dtype=torch.float32, device="cuda")
    plan.step(q, torch.tensor(k_new, dtype=dtype).cuda(), torch.tensor(v_new, dtype=dtype).cuda(), spec)
    torch.cuda.synchronize()
    from kvtest_util import page_fields
    for b in range(B):
        f = page_fields(t.page_records([t.sequence_pages(b)[0]]), 16, H, d)
        for side, x in (("k", k_new[b]), ("v", v_new[b])):
            pk, sk, zk = O.quantize_rows(O.rotate_rows(np.array(x, dtype=np.float64), 128, spec.signs))
            np.testing.assert_array_equal(f[f"{side}_payload"][0, 0], pk)
            np.testing.assert_array_equal(f[f"{side}_scale"][0, 0], sk)
            np.testing.assert_array_equal(f[f"{side}_zp"][0, 0], zk)


@pytest.mark.parametrize("graph", [False, True])
def test_step_pinned_host_out_matches_device_out(graph):
    """DecodePlan.step with a pinned host `out` (the kernel writes the result over the
    bus) gives the same bytes as with a device `out`, step after step."""
    H, G, d = 2, 4, 128
    lens = [33, 70]
    res = {}
    for host_out in (False, True):
        t, spec, layout = _build(len(lens), lens, H, G, d, 128, 16, "gaussian", Targets.KEYS_AND_VALUES, True,
                                 seed=8, extra_pages=4)
        plan = DecodePlan(t, [0, 1], extra_tokens=12)
        rng = np.random.default_rng(99)
        od = (torch.empty((2, G * H, d), dtype=torch.float32).pin_memory() if host_out
              else torch.empty((2, G * H, d), dtype=torch.float32, device="cuda"))
        outs = []
        for _ in range(9):
            q = torch.tensor(rng.standard_normal((2, G * H, d)), dtype=torch.bfloat16).pin_memory()
            k = torch.tensor(rng.standard_normal((2, H, d)), dtype=torch.bfloat16).pin_memory()
            v = torch.tensor(rng.standard_normal((2, H, d)), dtype=torch.bfloat16).pin_memory()
            o = plan.step(q, k, v, spec, out=od, graph=graph)
            torch.cuda.synchronize()
            outs.append(o.cpu().clone())
        res[host_out] = torch.stack(outs)
        # the plan's own lengths follow the steps (refreshed on demand)
        assert plan.run(torch.zeros((2, G * H, d), device="cuda"), spec).shape == (2, G * H, d)
        assert [int(x) for x in plan.lens.cpu()] == [lens[0] + 9, lens[1] + 9]
    assert torch.equal(res[False], res[True])


@pytest.mark.parametrize("fused", [False, True])
def test_decode_full_size_c5_uniform_keys(fused):
    """C5 at full size (1 kv head, 4 q heads, 1,048,576 cached tokens: 148 splits and
    the split-merge kernel) through a size-independent property: with every key row
    identical the softmax is uniform, so the output is the mean of the stored
    values, undone by the inverse rotation -- computed exactly from the dequantized
    pool in f64."""
    H, G, d, L = 1, 4, 128, 1 << 20
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=16)
    t = PageTable(layout, num_pages=L // 16 + 2)
    spec = RotationSpec(order=128, signs=make_signs(2, 0, d, 128), targets=Targets.KEYS_AND_VALUES)
    t.create_sequence(0)
    gen = torch.Generator(device="cuda").manual_seed(3)
    krow = torch.randn((1, H, d), generator=gen, device="cuda").bfloat16()
    n0 = L - 1 if fused else L
    slots = torch.from_numpy(t.alloc.reserve(0, n0)).cuda()
    for c0 in range(0, n0, 1 << 16):
        n = min(1 << 16, n0 - c0)
        v = torch.randn((n, H, d), generator=gen, device="cuda").bfloat16()
        t.store_slots(krow.expand(n, H, d).contiguous(), v, slots[c0:c0 + n], spec)
    q = torch.randn((1, G * H, d), generator=gen, device="cuda").bfloat16()
    if fused:  # the step's token is written (same key row) and attended in one launch
        plan = DecodePlan(t, [0], extra_tokens=1)
        vnew = torch.randn((1, H, d), generator=gen, device="cuda").bfloat16()
        out = plan.step(q, krow, vnew, spec)
    else:
        plan = DecodePlan(t, [0])
        out = plan.run(q, spec)
    torch.cuda.synchronize()
    assert plan.splits > 32  # the split-merge kernel path
    kd, vd = t.read_sequence_device([0], torch.float64)
    assert t.sequence_length(0) == L
    assert torch.equal(kd[0, 0], kd[0, L - 1])  # identical stored keys
    mean_v = vd[0, :L, 0].mean(dim=0, keepdim=True).cpu().numpy()
    ref = O.unrotate_rows(mean_v, 128, spec.signs)[0]
    got = out[0].double().cpu().numpy()
    err = np.abs(got - ref[None, :]).max() / np.abs(ref).max()
    print("C5 full size uniform-key rel err", err)
    assert err <= TOL


def test_decode_unaligned_query_view():
    """A query that is a contiguous view at a 2-byte offset (not 8-B aligned) decodes
    the same as an aligned copy (the kernel falls back to element loads)."""
    H, G, d = 2, 4, 128
    lens = [40, 90]
    t, spec, layout = _build(len(lens), lens, H, G, d, 128, 16, "gaussian", Targets.KEYS_AND_VALUES, True, seed=6)
    base = torch.randn(2 * G * H * d + 1, device="cuda").bfloat16()
    q_view = base[1:].view(2, G * H, d)  # storage offset of one element
    assert q_view.data_ptr() % 8 != 0 and q_view.is_contiguous()
    a = decode_batch(q_view, t, [0, 1], spec=spec)
    b = decode_batch(q_view.clone(), t, [0, 1], spec=spec)
    assert torch.equal(a, b)


@pytest.mark.parametrize("G", [4, 8])
def test_decode_ignores_nan_in_unwritten_slots(G):
    """Slots past a sequence's length (the rest of its last page, whole pages a split
    range covers but the sequence does not) may hold anything -- here NaN scale and
    code bytes -- and must not reach the output (the reference never reads them);
    plain decode over several split paths and the fused serving step."""
    H, d, P = 2, 128, 16
    lens = [21, 70]  # partial last pages
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=P)
    spec = RotationSpec(order=128, signs=make_signs(3, 0, d, 128), targets=Targets.KEYS_AND_VALUES)
    ref = {}
    for poison in (False, True):
        t = PageTable(layout, num_pages=16)
        if poison:  # every byte 0xFF: NaN scales, 0xFF zero points
            t.pool.fill_(0xFF)
        slots = []
        for s, L in enumerate(lens):
            t.create_sequence(s)
            slots.append(torch.from_numpy(t.alloc.reserve(s, L)).cuda())
        gen = torch.Generator(device="cuda").manual_seed(5)
        for s, L in enumerate(lens):
            t.store_slots(torch.randn(L, H, d, generator=gen, device="cuda").bfloat16(),
                          torch.randn(L, H, d, generator=gen, device="cuda").bfloat16(), slots[s], spec)
        q = torch.randn((2, G * H, d), generator=gen, device="cuda").bfloat16()
        outs = [decode_batch(q, t, [0, 1], spec=spec, num_splits=n) for n in (1, 3, 12, 40)]
        plan = DecodePlan(t, [0, 1], extra_tokens=2)
        kn = torch.randn((2, H, d), generator=gen, device="cuda").bfloat16()
        vn = torch.randn((2, H, d), generator=gen, device="cuda").bfloat16()
        outs.append(plan.step(q, kn, vn, spec).clone())
        torch.cuda.synchronize()
        for o in outs:
            assert torch.isfinite(o).all()
        ref[poison] = outs
    for a, b in zip(ref[False], ref[True]):
        assert torch.equal(a, b)
