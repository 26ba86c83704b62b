"""Full-size parity on every BASELINE config, against ORACLE-quantised pages.

Unlike tests/test_gpu_decode.py (which dequantises the GPU's own pages), here the
oracle quantises the same bf16 K/V itself -- rotate (f64 FWHT, _ref.py:22-40) ->
quantize (_ref.py:57-80) -> dequantize (_ref.py:83-95) -> decode (attention.py:50-87)
-- so the GPU write path (K1 or the fused step's writer) and the decode kernel are
checked end to end against the reference arithmetic, at the configs' real sizes
(sampled sequences / heads where the oracle would be slow).

Two bars per config:
* end to end against the oracle-quantised pages: 1e-3 * max|ref| (BASELINE.json
  north_star).  At long contexts the output is small (a mean over ~L/e tokens), so a
  single code that the fast K1 rounds differently (its scale may differ from the
  reference's by 1 ulp in ~0.5 % of rotated rows) moves it by
  ~1e-4 of max|ref|;
* the decode kernel alone, against an f64 decode of the pages it actually read:
  1e-5 (measured ~1.2e-6: exact integer QK, signed (c - z) PV operands).
"""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import kvrot_oracle as O  # noqa: E402
from paper_2604_19157_b200 import _kernels, _lib  # noqa: E402
from paper_2604_19157_b200 import errors as E  # noqa: E402
from paper_2604_19157_b200.attention import DecodePlan, DecodeRequest, decode_batch, decode_step  # noqa: E402
from paper_2604_19157_b200.cache import BF16, INT4, PageTable  # noqa: E402
from paper_2604_19157_b200.layout import HeadLayout  # noqa: E402
from paper_2604_19157_b200.rotation import RotationSpec, Targets, make_signs  # noqa: E402

TOL = 1e-3


def rel_err(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-30))


def _kv(seed, n, H, d, dev="cuda"):
    """bf16 K/V rows of one sequence from a per-sequence generator (reproducible on demand)."""
    g = torch.Generator(device=dev).manual_seed(seed)
    k = torch.randn((n, H, d), generator=g, device=dev).to(torch.bfloat16)
    v = torch.randn((n, H, d), generator=g, device=dev).to(torch.bfloat16)
    return k, v


def oracle_decode(k, v, q, order, signs, targets, group):
    """The reference pipeline on (L, H, d) bf16-exact f64 K/V and (nq, d) f64 q."""
    L, H, d = k.shape
    rot_v = signs is not None and targets is Targets.KEYS_AND_VALUES

    def store(x, rot):
        rows = x.reshape(-1, d)
        if rot:
            rows = O.rotate_rows(rows, order, signs)
        p, s, z = O.quantize_rows(rows)
        return O.dequantize_rows(p, s, z, d).reshape(L, H, d)

    kh = store(k, signs is not None)
    vh = store(v, rot_v)
    qf = O.rotate_rows(q, order, signs) if signs is not None else q
    out = O.decode_flat(qf, kh, vh, group)
    if rot_v:
        out = O.unrotate_rows(out, order, signs)
    return out


def own_pages_decode(table, seqs, q, spec, G):
    """f64 decode over the GPU's own dequantised pages (isolates the decode kernel)."""
    lay = table.layout
    kd, vd = table.read_sequence_device(seqs, torch.float64)
    outs = []
    for b, s in enumerate(seqs):
        L = table.sequence_length(s)
        kh, vh = kd[b, :L].cpu().numpy(), vd[b, :L].cpu().numpy()
        qn = np.asarray(q[b], dtype=np.float64)
        qf = O.rotate_rows(qn, lay.rot_order, spec.signs) if spec is not None else qn
        o = O.decode_flat(qf, kh, vh, G)
        if spec is not None and spec.targets is Targets.KEYS_AND_VALUES:
            o = O.unrotate_rows(o, lay.rot_order, spec.signs)
        outs.append(o)
    del kd, vd
    return np.stack(outs)


def _fill(table, seq, seed, L, chunk=1 << 16, spec=None):
    H, d = table.layout.num_kv_heads, table.layout.head_dim
    slots = torch.from_numpy(table.alloc.reserve(seq, L)).cuda()
    k, v = _kv(seed, L, H, d)
    for c0 in range(0, L, chunk):
        table.store_slots(k[c0:c0 + chunk], v[c0:c0 + chunk], slots[c0:c0 + chunk], spec)
    return k, v


def test_c2_full_size_random_keys():
    """configs[1]: batch 1, 32k context, GQA 32/8, K & V rotated; the fused serving
    step (append of token 32,768 + decode over 32,769)."""
    H, G, d, L = 8, 4, 128, 32768
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=16)
    spec = RotationSpec(order=128, signs=make_signs(0, 0, d, 128), targets=Targets.KEYS_AND_VALUES)
    t = PageTable(layout, num_pages=L // 16 + 2)
    t.create_sequence(0)
    k, v = _fill(t, 0, 11, L, spec=spec)
    plan = DecodePlan(t, [0], extra_tokens=1)
    g = torch.Generator(device="cuda").manual_seed(12)
    kn = torch.randn((1, H, d), generator=g, device="cuda").bfloat16()
    vn = torch.randn((1, H, d), generator=g, device="cuda").bfloat16()
    q = torch.randn((1, G * H, d), generator=g, device="cuda").bfloat16()
    out = plan.step(q, kn, vn, spec)
    torch.cuda.synchronize()
    kk = torch.cat([k, kn]).double().cpu().numpy()
    vv = torch.cat([v, vn]).double().cpu().numpy()
    ref = oracle_decode(kk, vv, q[0].double().cpu().numpy(), 128, spec.signs, spec.targets, G)
    got = out[0].double().cpu().numpy()
    err = rel_err(got, ref)
    kern = rel_err(got, own_pages_decode(t, [0], q.double().cpu().numpy(), spec, G)[0])
    print("C2 full size rel err: vs oracle-quantised", err, "| decode kernel vs f64 of its pages", kern)
    assert err <= TOL and kern <= 1e-5


def test_c3_b256_8k_sampled():
    """configs[2] at B = 256 x 8k (one split per unit): every sequence decoded,
    8 sampled sequences checked against the oracle."""
    H, G, d, L, B = 8, 4, 128, 8192, 256
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=16)
    spec = RotationSpec(order=128, signs=make_signs(0, 0, d, 128), targets=Targets.KEYS_AND_VALUES)
    t = PageTable(layout, num_pages=B * L // 16)
    for s in range(B):
        t.create_sequence(s)
        _fill(t, s, 1000 + s, L, spec=spec)
    q = torch.randn((B, G * H, d), generator=torch.Generator(device="cuda").manual_seed(5), device="cuda").bfloat16()
    out = decode_batch(q, t, list(range(B)), spec=spec).double().cpu().numpy()
    worst = kern = 0.0
    for s in (0, 1, 77, 128, 200, 253, 254, 255):
        k, v = _kv(1000 + s, L, H, d)
        ref = oracle_decode(k.double().cpu().numpy(), v.double().cpu().numpy(), q[s].double().cpu().numpy(), 128,
                            spec.signs, spec.targets, G)
        worst = max(worst, rel_err(out[s], ref))
        own = own_pages_decode(t, [s], q[s:s + 1].double().cpu().numpy(), spec, G)[0]
        kern = max(kern, rel_err(out[s], own))
    print("C3 B=256 x 8k sampled rel err: vs oracle-quantised", worst, "| decode kernel", kern)
    assert worst <= TOL and kern <= 1e-5


def test_c4_g8_16x16k_fused_layer():
    """configs[3] (Llama-3-70B KV geometry, G = 8) at the 8-GPU shard: 16 sequences x
    16k, one layer's fused append + decode step; 4 sampled sequences."""
    H, G, d, L, B = 8, 8, 128, 16384, 16
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=16)
    spec = RotationSpec(order=128, signs=make_signs(1, 3, d, 128), targets=Targets.KEYS_AND_VALUES)
    t = PageTable(layout, num_pages=B * (L // 16 + 1))
    for s in range(B):
        t.create_sequence(s)
        _fill(t, s, 2000 + s, L, spec=spec)
    plan = DecodePlan(t, list(range(B)), extra_tokens=1)
    g = torch.Generator(device="cuda").manual_seed(7)
    kn = torch.randn((B, H, d), generator=g, device="cuda").bfloat16()
    vn = torch.randn((B, H, d), generator=g, device="cuda").bfloat16()
    q = torch.randn((B, G * H, d), generator=g, device="cuda").bfloat16()
    out = plan.step(q, kn, vn, spec).double().cpu().numpy()
    worst = kern = 0.0
    for s in (0, 5, 10, 15):
        k, v = _kv(2000 + s, L, H, d)
        kk = torch.cat([k, kn[s:s + 1]]).double().cpu().numpy()
        vv = torch.cat([v, vn[s:s + 1]]).double().cpu().numpy()
        ref = oracle_decode(kk, vv, q[s].double().cpu().numpy(), 128, spec.signs, spec.targets, G)
        worst = max(worst, rel_err(out[s], ref))
        own = own_pages_decode(t, [s], q[s:s + 1].double().cpu().numpy(), spec, G)[0]
        kern = max(kern, rel_err(out[s], own))
    print("C4 G=8 16 x 16k fused layer, sampled rel err: vs oracle-quantised", worst, "| decode kernel", kern)
    assert worst <= TOL and kern <= 1e-5


@pytest.mark.parametrize("L,order,fused", [(131072, 128, False), (131072, 64, True), (1 << 20, 128, True)])
def test_c5_long_context_random_keys(L, order, fused):
    """configs[4]: one request, 1 kv head + its 4 q heads per GPU (the 8-way KV-head
    shard), random keys, split-K over 128-148 splits with the split-merge kernel."""
    H, G, d = 1, 4, 128
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=order, page_tokens=16)
    spec = RotationSpec(order=order, signs=make_signs(4, 0, d, order), targets=Targets.KEYS_AND_VALUES)
    t = PageTable(layout, num_pages=L // 16 + 2)
    t.create_sequence(0)
    n0 = L - 1 if fused else L
    k, v = _fill(t, 0, 31, n0, spec=spec)
    g = torch.Generator(device="cuda").manual_seed(32)
    q = torch.randn((1, G * H, d), generator=g, device="cuda").bfloat16()
    if fused:
        kn = torch.randn((1, H, d), generator=g, device="cuda").bfloat16()
        vn = torch.randn((1, H, d), generator=g, device="cuda").bfloat16()
        plan = DecodePlan(t, [0], extra_tokens=1)
        out = plan.step(q, kn, vn, spec)
        k, v = torch.cat([k, kn]), torch.cat([v, vn])
    else:
        plan = DecodePlan(t, [0])
        out = plan.run(q, spec)
    torch.cuda.synchronize()
    assert plan.splits > 32
    ref = oracle_decode(k.double().cpu().numpy(), v.double().cpu().numpy(), q[0].double().cpu().numpy(), order,
                        spec.signs, spec.targets, G)
    got = out[0].double().cpu().numpy()
    err = rel_err(got, ref)
    kern = rel_err(got, own_pages_decode(t, [0], q.double().cpu().numpy(), spec, G)[0])
    print(f"C5 L={L} order={order} fused={fused} rel err: vs oracle-quantised {err} | decode kernel {kern}")
    assert err <= TOL and kern <= 1e-5


def test_store_then_decode_back_to_back():
    """K1 over 4,096 tokens immediately followed by a C-ABI decode on the same stream
    (no op in between), 50 times with alternating data: every output equals the one
    of a run with a device synchronisation between the write and the decode (the
    decode must not read cells before the write's grid has finished)."""
    H, G, d, L = 8, 4, 128, 4096
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=16)
    spec = RotationSpec(order=128, signs=make_signs(0, 0, d, 128), targets=Targets.KEYS_AND_VALUES)
    t = PageTable(layout, num_pages=L // 16)
    t.create_sequence(0)
    slots = torch.from_numpy(t.alloc.reserve(0, L)).cuda()
    data = [_kv(s, L, H, d) for s in (1, 2)]
    q = torch.randn((1, G * H, d), device="cuda").bfloat16()
    plan = DecodePlan(t, [0])
    words = spec.sign_words(d)
    out = torch.empty((1, G * H, d), dtype=torch.float32, device="cuda")

    def write(i):
        k, v = data[i % 2]
        _lib.check(_lib.lib().kvr_rotate_quantize_store(
            _kernels.ptr(k), _kernels.ptr(v), _lib.KVR_BF16, L, _kernels.ptr(slots), ctypes.byref(t.desc), 128, 1,
            _lib.KVR_KEYS_AND_VALUES, words, 0, _kernels.ptr(t.flags), _kernels.stream_ptr()))

    def decode():
        _lib.check(_lib.lib().kvr_paged_decode(
            _kernels.ptr(q), _lib.KVR_BF16, ctypes.byref(t.desc), _kernels.ptr(plan.bt), plan.bt.shape[1],
            _kernels.ptr(plan.lens), 1, G * H, L, 128, 1, _lib.KVR_KEYS_AND_VALUES, words, _kernels.ptr(out),
            _kernels.ptr(plan.ws), plan.ws.numel(), plan.splits, _kernels.stream_ptr()))

    want = []
    for i in range(2):
        write(i)
        torch.cuda.synchronize()
        decode()
        torch.cuda.synchronize()
        want.append(out.clone())
    assert not torch.equal(want[0], want[1])
    got = []
    for i in range(50):
        write(i)
        decode()
        got.append(out.clone())
    torch.cuda.synchronize()
    for i, o in enumerate(got):
        assert torch.equal(o, want[i % 2]), f"repetition {i} read stale cells"


def test_append_batch_nonfinite_is_atomic():
    """A NaN anywhere in a batch raises before anything is committed (cache.py:225-233):
    lengths, pages and the dump are unchanged."""
    layout = HeadLayout(num_q_heads=32, num_kv_heads=8, head_dim=128, rot_order=128)
    spec = RotationSpec(order=128, signs=make_signs(0, 0, 128, 128))
    t = PageTable(layout, num_pages=8)
    t.create_sequence(0)
    k, v = _kv(3, 20, 8, 128)
    t.append_batch([0] * 20, k, v, spec=spec)
    before = (t.dump_bytes(), t.free_pages, t.sequence_length(0))
    k2, v2 = _kv(4, 10, 8, 128)
    v2[7, 3, 100] = float("nan")
    with pytest.raises(E.NonFiniteInputError):
        t.append_batch([0] * 10, k2, v2, spec=spec)
    assert (t.dump_bytes(), t.free_pages, t.sequence_length(0)) == before


@pytest.mark.parametrize("host", [True, False])
def test_step_nonfinite_rejected_before_commit(host):
    """DecodePlan.step rejects NaN/Inf inputs before it plans the slot: the sequence,
    the pool and the next step are as if the bad step never happened."""
    H, G, d = 2, 4, 128
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=16)
    spec = RotationSpec(order=128, signs=make_signs(0, 0, d, 128))
    t = PageTable(layout, num_pages=8)
    for s in (0, 1):
        t.create_sequence(s)
    k, v = _kv(5, 32, H, d)
    t.append_batch([0] * 16 + [1] * 16, k, v, spec=spec)  # both sequences end on a page boundary
    plan = DecodePlan(t, [0, 1], extra_tokens=8)
    before = (t.dump_bytes(), t.free_pages, [t.sequence_length(s) for s in (0, 1)])
    q = torch.randn((2, G * H, d)).bfloat16()
    kn = torch.randn((2, H, d)).bfloat16()
    vn = torch.randn((2, H, d)).bfloat16()
    kn[1, 0, 3] = float("inf")
    if not host:
        q, kn, vn = q.cuda(), kn.cuda(), vn.cuda()
    with pytest.raises(E.NonFiniteInputError):
        plan.step(q, kn, vn, spec)
    assert (t.dump_bytes(), t.free_pages, [t.sequence_length(s) for s in (0, 1)]) == before
    kn[1, 0, 3] = 0.5
    out = plan.step(q, kn, vn, spec)
    assert torch.isfinite(out).all() and [t.sequence_length(s) for s in (0, 1)] == [17, 17]


def test_fused_step_unchecked_nonfinite_token_not_attended():
    """check=False: the fused kernel writes no row of a NaN token and does not attend
    it (no phantom zero key / value); the device flag reports it."""
    H, G, d = 2, 4, 128
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=16)
    spec = RotationSpec(order=128, signs=make_signs(0, 0, d, 128))
    t = PageTable(layout, num_pages=8)
    t.create_sequence(0)
    k, v = _kv(6, 40, H, d)
    t.append_batch([0] * 40, k, v, spec=spec)
    q = torch.randn((1, G * H, d), device="cuda").bfloat16()
    base = DecodePlan(t, [0]).run(q, spec).clone()
    plan = DecodePlan(t, [0], extra_tokens=1)
    kn = torch.randn((1, H, d), device="cuda").bfloat16()
    vn = torch.randn((1, H, d), device="cuda").bfloat16()
    vn[0, 1, 7] = float("nan")
    out = plan.step(q, kn, vn, spec, check=False)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    torch.testing.assert_close(out, base, rtol=1e-5, atol=1e-6)
    with pytest.raises(E.NonFiniteInputError):
        t.check_flags()


def test_step_capacity_error_leaves_state():
    """A step that would outgrow the plan's block table raises before committing."""
    H, G, d = 2, 4, 128
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=16)
    t = PageTable(layout, num_pages=8)
    t.create_sequence(0)
    k, v = _kv(7, 32, H, d)
    t.append_batch([0] * 32, k, v)
    plan = DecodePlan(t, [0])  # block table exactly 2 pages wide
    before = (t.free_pages, t.sequence_length(0))
    with pytest.raises(E.ShapeError):
        plan.step(torch.randn((1, G * H, d)), torch.randn((1, H, d)), torch.randn((1, H, d)), None)
    assert (t.free_pages, t.sequence_length(0)) == before


@pytest.mark.parametrize("P,d,order", [(12, 16, 16), (12, 128, 64), (4, 16, 8), (24, 32, 16)])
def test_generic_geometries_decode_and_step(P, d, order):
    """Page sizes that are not powers of two and head dims below 32 (the reference's
    own test layouts use d = 16): decode parity, and DecodePlan.step falls back to the
    store kernel + decode kernel (no fused kernel for these)."""
    H, G = 2, 2
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=order, page_tokens=P)
    spec = RotationSpec(order=order, signs=make_signs(2, 0, d, order), targets=Targets.KEYS_AND_VALUES)
    t = PageTable(layout, num_pages=40)
    rng = np.random.default_rng(P * d)
    lens = [50, 7]
    kvs = []
    for s, L in enumerate(lens):
        t.create_sequence(s)
        k = rng.standard_normal((L, H, d))
        v = rng.standard_normal((L, H, d))
        t.append_tokens_two_pass(s, k, v, spec=spec)
        kvs.append((k, v))
    q = rng.standard_normal((2, G * H, d))
    out = decode_batch(torch.tensor(q, dtype=torch.float32).cuda(), t, [0, 1], spec=spec).double().cpu().numpy()
    for s in range(2):
        ref = oracle_decode(kvs[s][0], kvs[s][1], q[s], order, spec.signs, spec.targets, G)
        assert rel_err(out[s], ref) <= 1e-5
    plan = DecodePlan(t, [0, 1], extra_tokens=2)
    assert not plan.fused_ok
    kn = rng.standard_normal((2, H, d))
    vn = rng.standard_normal((2, H, d))
    o2 = plan.step(torch.tensor(q, dtype=torch.float32), torch.tensor(kn), torch.tensor(vn), spec)
    torch.cuda.synchronize()
    for s in range(2):
        k = np.concatenate([kvs[s][0], kn[s:s + 1]])
        v = np.concatenate([kvs[s][1], vn[s:s + 1]])
        ref = oracle_decode(k, v, q[s], order, spec.signs, spec.targets, G)
        assert rel_err(o2[s].double().cpu().numpy(), ref) <= 1e-5


# ---------------------------------------------------------------- reference KATs

def test_c03_thousand_fused_appends_equal_two_pass(tmp_path):
    """test_acceptance.py:100-133: 1,000 fused appends == the two-pass write, dump bytes."""
    layout = HeadLayout(num_q_heads=4, num_kv_heads=2, head_dim=64, rot_order=64, page_tokens=16)
    spec = RotationSpec(order=64, signs=make_signs(3, 0, 64, 64), targets=Targets.KEYS_AND_VALUES)
    rng = np.random.default_rng(99)
    ks = rng.standard_normal((1000, 2, 64))
    vs = rng.standard_normal((1000, 2, 64))
    fused = PageTable(layout, precision=INT4, num_pages=63)
    fused.create_sequence(0)
    for i in range(1000):
        fused.append_token(0, ks[i], vs[i], spec=spec)
    two = PageTable(layout, precision=INT4, num_pages=63)
    two.create_sequence(0)
    two.append_tokens_two_pass(0, ks, vs, spec=spec)
    assert fused.dump_bytes() == two.dump_bytes()
    ref = O.OraclePages(4, 2, 64, 64, 16, 63)
    ref.create_sequence(0)
    ref.append_tokens(0, ks, vs, signs=spec.signs)
    assert fused.dump_bytes() == ref.dump_bytes()


def test_c04_paged_matches_flat_100_layouts(golden_reads):
    """test_acceptance.py:136-172: 100 random small layouts (d 16-128, 1-4 kv heads,
    pages of 4-16 tokens, every third pool BF16), paged decode vs the flat decode,
    both against the reference's own outputs (golden_reads.npz)."""
    from paper_2604_19157_b200.attention import decode_step_fp

    rng = np.random.default_rng(2718)
    worst_paged = worst_flat = 0.0
    for i in range(100):
        d = int(rng.choice([16, 32, 64, 128]))
        kv_heads = int(rng.choice([1, 2, 4]))
        group = int(rng.choice([1, 2]))
        page_tokens = int(rng.choice([4, 8, 16]))
        s = int(rng.integers(1, 257))
        layout = HeadLayout(num_q_heads=kv_heads * group, num_kv_heads=kv_heads, head_dim=d, rot_order=16,
                            page_tokens=page_tokens)
        precision = BF16 if i % 3 == 0 else INT4
        np.testing.assert_array_equal(golden_reads[f"c04_{i}_geom"],
                                      [d, kv_heads, group, page_tokens, s, int(precision == BF16)])
        table = PageTable(layout, precision=precision, num_pages=-(-s // page_tokens))
        table.create_sequence(0)
        k = rng.standard_normal((s, kv_heads, d))
        v = rng.standard_normal((s, kv_heads, d))
        table.append_tokens_two_pass(0, k, v)
        q = rng.standard_normal((layout.num_q_heads, d))
        np.testing.assert_array_equal(golden_reads[f"c04_{i}_sums"], [k.sum(), v.sum(), q.sum()])
        paged = decode_step(DecodeRequest(q=q, seq=0), table)
        fk, fv = table.read_sequence(0)
        flat = decode_step_fp(q, fk, fv, layout)
        worst_paged = max(worst_paged, rel_err(paged, golden_reads[f"c04_{i}_paged"]))
        worst_flat = max(worst_flat, float(np.abs(flat - golden_reads[f"c04_{i}_flat"]).max()))
        assert rel_err(paged, flat) <= 1e-5
    print("c04 worst rel err paged (fp32 kernel) vs reference", worst_paged, "flat f64 abs", worst_flat)
    assert worst_paged <= 1e-5 and worst_flat <= 1e-12


def test_softmax_shift_invariance_plus_5000():
    """test_attention.py:146-160: +5000 on every key along the query direction leaves
    the flat decode unchanged and finite (max-subtracted softmax)."""
    from paper_2604_19157_b200.attention import decode_step_fp

    layout = HeadLayout(num_q_heads=4, num_kv_heads=2, head_dim=32, rot_order=16, page_tokens=4)
    rng = np.random.default_rng(1234)
    q = np.zeros((4, 32))
    q[:, 0] = 1.0
    k = rng.standard_normal((7, 2, 32))
    v = rng.standard_normal((7, 2, 32))
    base = decode_step_fp(q, k, v, layout)
    kh = k.copy()
    kh[:, :, 0] += 5000.0
    shifted = decode_step_fp(q, kh, v, layout)
    np.testing.assert_allclose(shifted, base, atol=1e-9)
    assert np.isfinite(shifted).all()
    # and the paged INT4 kernel: a key table shifted the same way (huge logits) stays finite
    t = PageTable(layout, num_pages=4)
    t.create_sequence(0)
    t.append_tokens_two_pass(0, kh, v)
    out = decode_step(DecodeRequest(q=q, seq=0), t)
    fk, fv = t.read_sequence(0)
    # logits of ~880 in fp32 carry ~5e-5 absolute rounding: 1e-4 here (f64 reference: exact)
    assert np.isfinite(out).all() and rel_err(out, decode_step_fp(q, fk, fv, layout)) <= 1e-4


def test_decode_step_fp_matches_reference_goldens(golden):
    """The flat full-precision decode (f64 kernel) on the reference's own dequantised
    reads equals decode_step_fp's golden outputs (attention.py:90-115) to 1e-12."""
    from paper_2604_19157_b200.attention import decode_step_fp

    lays = {"small_kv": (4, 2, 32, 16, 4), "big_kv": (32, 8, 128, 128, 16), "big_konly": (32, 8, 128, 128, 16),
            "big_plain": (32, 8, 128, 128, 16), "o64_kv": (4, 1, 128, 64, 16)}
    for tag, lay in lays.items():
        layout = HeadLayout(num_q_heads=lay[0], num_kv_heads=lay[1], head_dim=lay[2], rot_order=lay[3],
                            page_tokens=lay[4])
        from kvtest_util import golden_bytes
        import tempfile, os
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "t.kvpg")
            with open(path, "wb") as f:
                f.write(golden_bytes(f"{tag}.kvpg"))
            t = PageTable.load(path)
        fk, fv = t.read_sequence(0)
        got = decode_step_fp(golden[f"dec_{tag}_q"], fk, fv, layout)
        err = float(np.abs(got - golden[f"dec_{tag}_fp"]).max())
        print(tag, "decode_step_fp abs err", err)
        assert err <= 1e-12


def test_read_sequence_full_arrays_match_reference(golden_reads):
    """read_sequence (K4, f64 out) of the reference's dumps loaded into the device pool
    equals the reference's own read_sequence arrays element for element (INT4 and BF16)."""
    from kvtest_util import golden_bytes
    import tempfile, os

    for tag in ("small_kv", "big_kv", "o64_kv", "bf_small"):
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "t.kvpg")
            with open(path, "wb") as f:
                f.write(golden_bytes(f"{tag}.kvpg"))
            t = PageTable.load(path)
        for s in t.sequence_ids():
            k, v = t.read_sequence(s)
            np.testing.assert_array_equal(k, golden_reads[f"read_{tag}_{s}_k"])
            np.testing.assert_array_equal(v, golden_reads[f"read_{tag}_{s}_v"])


def test_c2_full_size_learned_step():
    """configs[1] with a learned R (row f3, learned_values): the serving step -- the new token
    through the fused learned K1, the decode with q T and o T^T inside the kernel -- against the
    reference composition (FWHT then R, rotation.py:118-168) on oracle-quantised pages, and the
    decode kernel against an f64 decode of its own pages."""
    H, G, d, L = 8, 4, 128, 32768
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=16)
    qm, rm = np.linalg.qr(np.random.default_rng(21).standard_normal((d, d)))
    R = qm * np.sign(np.diag(rm))
    spec = RotationSpec(order=128, signs=make_signs(0, 0, d, 128), learned=R, learned_values=True)
    t = PageTable(layout, num_pages=L // 16 + 2)
    t.create_sequence(0)
    k, v = _fill(t, 0, 31, L, spec=spec)
    plan = DecodePlan(t, [0], extra_tokens=1)
    g = torch.Generator(device="cuda").manual_seed(32)
    kn = torch.randn((1, H, d), generator=g, device="cuda").bfloat16()
    vn = torch.randn((1, H, d), generator=g, device="cuda").bfloat16()
    q = torch.randn((1, G * H, d), generator=g, device="cuda").bfloat16()
    out = plan.step(q, kn, vn, spec)
    torch.cuda.synchronize()
    kk = torch.cat([k, kn]).double().cpu().numpy().reshape(-1, d)
    vv = torch.cat([v, vn]).double().cpu().numpy().reshape(-1, d)

    def store(x):
        p_, s_, z_ = O.quantize_rows(O.rotate_rows(x, 128, spec.signs) @ R)
        return O.dequantize_rows(p_, s_, z_, d).reshape(L + 1, H, d)

    qf = O.rotate_rows(q[0].double().cpu().numpy(), 128, spec.signs) @ R
    ref = O.unrotate_rows(O.decode_flat(qf, store(kk), store(vv), G) @ R.T, 128, spec.signs)
    got = out[0].double().cpu().numpy()
    err = rel_err(got, ref)
    kd, vd = t.read_sequence_device([0], torch.float64)
    own = O.unrotate_rows(O.decode_flat(qf, kd[0, :L + 1].cpu().numpy(), vd[0, :L + 1].cpu().numpy(), G) @ R.T, 128,
                          spec.signs)
    kern = rel_err(got, own)
    print("C2 learned step rel err: vs oracle-quantised", err, "| decode kernel vs f64 of its pages", kern)
    assert err <= TOL and kern <= 1e-5
